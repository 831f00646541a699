"""GPU: the row-partitioned multi-GPU engine (csrc/rows.cu) with G virtual
ranks on one B200 — fused mode (one cooperative launch, CTA range per rank, frontier
stores into the sibling ranks' buffers + the cross-rank arrival barrier) and stepped mode
(one launch per level, the all-gather a device concatenation). Levels bit-exact against
the oracle's reference_bfs; each rank's BVSS equals the oracle's BVSS of the row-filtered
graph; the slice-balanced partition matches a host count."""
import ctypes as C
import os
import sys

import numpy as np
import pytest

import paper_2512_21967_b200 as B
from paper_2512_21967_b200 import _lib as L
from paper_2512_21967_b200.multigpu import (RowsEngine, assemble, group_bfs, partition_rows, rows_of,
                                             run_stepped_local, set_local_peers)

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def graphs():
    yield "rmat", B.Graph.generate_rmat(13, 16, 6)
    yield "grid", B.apply_permutation(B.Graph.generate_grid(61, 67), B.relabel_permutation(61 * 67, 2))
    # directed: BFS follows out-edges, rows are destinations (SURVEY §8(a) pitfall 1)
    rng = np.random.default_rng(3)
    n = 3000
    s = rng.integers(0, n, 9000).astype(np.uint32)
    d = rng.integers(0, n, 9000).astype(np.uint32)
    yield "directed", B.Graph.from_edges(n, (s, d), directed=True)


def slices_per_row(csr):
    """(column slice set, row) pairs per row: the host count the partition balances."""
    src = np.repeat(np.arange(csr.n, dtype=np.int64), np.diff(csr.offsets).astype(np.int64))
    key = np.unique((src >> 3) * (1 << 32) + csr.targets.astype(np.int64))
    return np.bincount(key & 0xFFFFFFFF, minlength=csr.n)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_balances_slices(oracle, world):
    for kind, g in graphs():
        n = g.num_vertices()
        off, tgt = g.csr()
        per_row = slices_per_row(oracle.Csr(n, off, tgt))
        bounds, slices = partition_rows(g, world)
        words = (n + 31) // 32
        assert bounds[0] == 0 and bounds[-1] == words and all(a <= b for a, b in zip(bounds, bounds[1:]))
        pref = np.concatenate([[0], np.cumsum(np.pad(per_row, (0, 32 * words - n)).reshape(words, 32).sum(1))])
        assert slices == [int(pref[b] - pref[a]) for a, b in zip(bounds, bounds[1:])], kind
        total = int(pref[-1])
        for r in range(1, world):  # each cut is the first word reaching r/world of the slices
            assert pref[bounds[r]] >= (total * r + world - 1) // world
            assert bounds[r] == 0 or pref[bounds[r] - 1] < (total * r + world - 1) // world


def test_rows_bvss_matches_oracle(oracle):
    sys.path.insert(0, HERE)
    from partition_cpu import rows_graph
    s, d = oracle.gen_rmat(11, 8, 4)
    g = B.Graph.from_edges(1 << 11, (s, d), directed=False)
    off, tgt = g.csr()
    csr = oracle.Csr(1 << 11, off, tgt)
    bounds, _ = partition_rows(g, 3)
    for r in range(3):
        lo, hi = rows_of(bounds, r, g.num_vertices())
        h = C.c_void_p()
        L.check(L.lib().blest_bvss_build_rows(g.handle, lo, hi, C.byref(h)))
        b = B.Bvss(h.value)
        want = oracle.build_bvss(rows_graph(csr, lo, hi))
        rp, v2r, rows, masks = b.arrays()
        assert np.array_equal(rp, want.real_ptrs) and np.array_equal(rows, want.row_ids)
        assert np.array_equal(masks, want.masks) and b.m == want.m


def engines_for(g, world):
    bounds, _ = partition_rows(g, world)
    engs = [RowsEngine(g, r, world, bounds) for r in range(world)]
    set_local_peers(engs)
    return engs


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_virtual_ranks_fused(oracle, world):
    import torch
    for kind, g in graphs():
        n = g.num_vertices()
        off, tgt = g.csr()
        csr = oracle.Csr(n, off, tgt)
        engs = engines_for(g, world)
        for src in list(g.pick_sources(3, 9)) + [0, n - 1]:
            group_bfs(engs, int(src))
            res = [e.finish() for e in engs]
            want, _, _ = oracle.reference_bfs(csr, int(src))
            assert np.array_equal(assemble(res, n), want), (kind, world, int(src))
            assert len({r.iterations for r in res}) == 1
            reached = int(np.count_nonzero(want != 0xFFFFFFFF))
            assert sum(r.discovered for r in res) == reached - 1
        torch.cuda.synchronize()


@pytest.mark.parametrize("world", [1, 2, 5])
def test_virtual_ranks_stepped(oracle, world):
    for kind, g in graphs():
        n = g.num_vertices()
        off, tgt = g.csr()
        csr = oracle.Csr(n, off, tgt)
        bounds, _ = partition_rows(g, world)
        engs = [RowsEngine(g, r, world, bounds) for r in range(world)]
        for src in list(g.pick_sources(3, 4)) + [n // 2]:
            res = run_stepped_local(engs, int(src))
            want = oracle.reference_bfs(csr, int(src))[0]
            assert np.array_equal(assemble(res, n), want), (kind, world, int(src))


def test_fused_matches_single_gpu_lazy_counters(oracle):
    """One rank = the whole graph: iterations and discoveries equal the lazy engine's."""
    g = B.Graph.generate_rmat(14, 16, 2)
    b = B.build_bvss(g)
    engs = engines_for(g, 1)
    for src in g.pick_sources(4, 1):
        group_bfs(engs, int(src))
        r = engs[0].finish()
        res, cnt = B.run_lazy(b, int(src), B.EngineConfig())
        assert np.array_equal(r.levels, res.levels)
        assert r.iterations == len(cnt.trace)
        assert r.queue == cnt.vss_dequeues


@pytest.mark.parametrize("kind", ["urand", "grid"])
def test_rows_exhaustion_exit(oracle, monkeypatch, kind):
    """Connected graphs: every rank stops pulling at the same barren last level (exhaustion
    exit), levels stay bit-exact, the iteration count equals the single-GPU lazy engine's,
    and one rank's queue / unpulled equal the lazy engine's dequeues / unpulled VSSs; fused
    (1, 3, 8 virtual ranks) and stepped (2 ranks), exit armed and off."""
    if kind == "urand":
        g = B.Graph.generate_urand(1 << 13, 16 << 13, 7)
    else:
        g = B.apply_permutation(B.Graph.generate_grid(40, 52), B.relabel_permutation(40 * 52, 3))
    n = g.num_vertices()
    off, tgt = g.csr()
    csr = oracle.Csr(n, off, tgt)
    b = B.build_bvss(g)
    for ex in ("1", "0"):
        monkeypatch.setenv("BLEST_EXHAUST", ex)
        for src in g.pick_sources(2, 5):
            src = int(src)
            want = oracle.reference_bfs(csr, src)[0]
            res1, cnt1 = B.run_lazy(b, src, B.EngineConfig())
            unp1 = C.c_uint64(0)
            L.check(L.lib().blest_bfs_last_unpulled(b.handle, C.byref(unp1)))
            assert (unp1.value > 0) == (ex == "1")
            for world in (1, 3, 8):
                engs = engines_for(g, world)
                group_bfs(engs, src)
                res = [e.finish() for e in engs]
                assert np.array_equal(assemble(res, n), want), (kind, world, src, ex)
                assert {r.iterations for r in res} == {len(cnt1.trace)}
                assert (sum(r.unpulled for r in res) > 0) == (ex == "1")
                if world == 1:
                    assert res[0].queue == cnt1.vss_dequeues and res[0].unpulled == unp1.value
            bounds, _ = partition_rows(g, 2)
            engs = [RowsEngine(g, r, 2, bounds) for r in range(2)]
            res = run_stepped_local(engs, src)
            assert np.array_equal(assemble(res, n), want), (kind, "stepped", src, ex)
            assert {r.iterations for r in res} == {len(cnt1.trace)}


def test_errors():
    g = B.Graph.generate_rmat(8, 8, 1)
    bounds, _ = partition_rows(g, 2)
    with pytest.raises(ValueError):
        RowsEngine(g, 2, 2, bounds)
    with pytest.raises(ValueError):
        RowsEngine(g, 0, 2, [0, 1, 2])
    e = RowsEngine(g, 0, 1, [0, (g.num_vertices() + 31) // 32])
    with pytest.raises(ValueError):
        e.bfs(g.num_vertices())
    with pytest.raises(ValueError):
        e.step(2, 0, None)


def _gloo_worker(rank, world, port, out_dir):
    import socket  # noqa: F401
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2512_21967_b200 as Bw
    from paper_2512_21967_b200 import _lib as Lw
    from paper_2512_21967_b200.multigpu import RowsEngine as RE, SteppedBfs, partition_rows as pr, torch_allgather
    Lw.check(Lw.lib().blest_set_stream(C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    g = Bw.Graph.generate_rmat(12, 16, 5)
    n = g.num_vertices()
    bounds, _ = pr(g, world)
    eng = RE(g, rank, world, bounds)
    bfs = SteppedBfs(eng, torch_allgather(), ahead=2)
    for k, src in enumerate(g.pick_sources(3, 2)):
        r = bfs.run(int(src))
        mine = torch.full((32 * eng.per,), -1, dtype=torch.int64)
        mine[: r.row_hi - r.row_lo] = torch.from_numpy(r.levels.astype(np.int64))
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        cnt = torch.tensor([r.collectives, r.iterations])
        cnts = [torch.empty_like(cnt) for _ in range(world)]
        dist.all_gather(cnts, cnt)
        if rank == 0:
            got = np.concatenate([p.numpy()[: min(32 * bounds[i + 1], n) - min(32 * bounds[i], n)]
                                  for i, p in enumerate(parts)])
            off, tgt = g.csr()
            np.savez(os.path.join(out_dir, f"s{k}.npz"), got=got, src=int(src), off=off, tgt=tgt,
                     cnt=torch.stack(cnts).numpy())
    dist.destroy_process_group()


def test_gloo_world2_drives_gpu_engines(oracle, tmp_path):
    """Two processes (ranks) sharing this GPU, each with its own stepped rows engine; the
    frontier all-gather goes through torch.distributed (gloo here, NCCL on a multi-GPU
    node): the same host protocol (SteppedBfs) as bench.py --gpus N."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_gloo_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    files = sorted(os.listdir(tmp_path))
    assert len(files) == 3
    for f in files:
        z = np.load(os.path.join(tmp_path, f))
        got = z["got"].astype(np.int64)
        off, tgt = z["off"], z["tgt"]
        want = oracle.reference_bfs(oracle.Csr(len(off) - 1, off, tgt), int(z["src"]))[0].astype(np.int64)
        got[got == 0xFFFFFFFF] = -1
        want[want == 0xFFFFFFFF] = -1
        assert np.array_equal(got, want), f
        cnt = z["cnt"]
        assert (cnt[:, 0] == cnt[0, 0]).all() and cnt[0, 0] == cnt[0, 1] + 1 + 2


def _ipc_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2512_21967_b200 as Bw
    from paper_2512_21967_b200 import _lib as Lw
    from paper_2512_21967_b200.multigpu import RowsEngine as RE, exchange_ipc_handles, partition_rows as pr
    Lw.check(Lw.lib().blest_set_stream(C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    g = Bw.Graph.generate_rmat(10, 8, 3)
    n = g.num_vertices()
    bounds, _ = pr(g, world)
    eng = RE(g, rank, world, bounds)
    exchange_ipc_handles(eng)  # CUDA IPC mappings of the peers' frontier buffers
    for k, src in enumerate(g.pick_sources(2, 5)):
        dist.barrier()
        eng.bfs(int(src))  # fused: peer stores + in-kernel cross-rank barrier (system scope)
        r = eng.finish()
        mine = torch.full((32 * eng.per,), -1, dtype=torch.int64)
        mine[: r.row_hi - r.row_lo] = torch.from_numpy(r.levels.astype(np.int64))
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        if rank == 0:
            got = np.concatenate([p.numpy()[: min(32 * bounds[i + 1], n) - min(32 * bounds[i], n)]
                                  for i, p in enumerate(parts)])
            off, tgt = g.csr()
            np.savez(os.path.join(out_dir, f"s{k}.npz"), got=got, src=int(src), off=off, tgt=tgt)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(os.environ.get("BLEST_TEST_IPC") != "1",
                    reason="opt-in (BLEST_TEST_IPC=1): two processes time-share one GPU, each fused "
                           "kernel waiting for the other at every level")
def test_ipc_fused_two_processes(oracle, tmp_path):
    """The fused P2P mode across two real processes: CUDA IPC handles exchanged over
    torch.distributed, frontier words stored into the peer's buffer, system-scope arrival
    barrier. On one GPU the two cooperative kernels time-slice, so each level waits for a
    context switch — a functional test of the multi-GPU plumbing, not a timing."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_ipc_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    files = sorted(os.listdir(tmp_path))
    assert len(files) == 2
    for f in files:
        z = np.load(os.path.join(tmp_path, f))
        got = z["got"].astype(np.int64)
        off, tgt = z["off"], z["tgt"]
        want = oracle.reference_bfs(oracle.Csr(len(off) - 1, off, tgt), int(z["src"]))[0].astype(np.int64)
        got[got == 0xFFFFFFFF] = -1
        want[want == 0xFFFFFFFF] = -1
        assert np.array_equal(got, want), f
