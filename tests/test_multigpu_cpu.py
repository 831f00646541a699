"""CPU (gloo, world_size 2 and 3): the row-partitioned multi-GPU protocol — partition,
per-level frontier all-gather, termination — gives the reference's levels. The per-rank
level steps come from an oracle-backed numpy backend (tests/partition_cpu.py); the GPU
kernels of the same steps are checked in tests/test_gpu_multigpu.py."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def gloo_allgather(local):
    world = dist.get_world_size()
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    return torch.cat(parts)


def worker(rank, world, port, out_dir, kind, ahead):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
    sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from partition_cpu import NumpyRows
    from paper_2512_21967_b200.multigpu import SteppedBfs, partition_rows_even
    if kind == "rmat":
        s, d = O.gen_rmat(10, 8, 3)
        g = O.from_edges(1 << 10, s, d, directed=False)
    else:
        s, d = O.gen_grid(23, 29)
        g = O.from_edges(23 * 29, s, d, directed=False)
    bounds = partition_rows_even(g.n, world)
    eng = NumpyRows(g, rank, bounds)
    bfs = SteppedBfs(eng, gloo_allgather, ahead=ahead)
    srcs = O.pick_sources(g, 3, 5)
    for k, src in enumerate(srcs):
        r = bfs.run(int(src))
        per_rows = 32 * eng.per
        mine = torch.full((per_rows,), -1, dtype=torch.int64)
        mine[: r.row_hi - r.row_lo] = torch.from_numpy(r.levels.astype(np.int64))
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        cnt = torch.tensor([r.collectives, r.iterations])
        cnts = [torch.empty_like(cnt) for _ in range(world)]
        dist.all_gather(cnts, cnt)
        if rank == 0:
            got = np.concatenate([p.numpy()[: min(32 * bounds[i + 1], g.n) - min(32 * bounds[i], g.n)]
                                  for i, p in enumerate(parts)])
            want = O.reference_bfs(g, int(src))[0].astype(np.int64)
            want[want == 0xFFFFFFFF] = -1
            got[got == 0xFFFFFFFF] = -1
            np.save(os.path.join(out_dir, f"{kind}_{k}.npy"), np.stack([got, want]))
            np.save(os.path.join(out_dir, f"cnt_{kind}_{k}.npy"), torch.stack(cnts).numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,ahead", [(2, "rmat", 2), (3, "grid", 0), (2, "grid", 1)])
def test_row_partitioned_protocol_gloo(tmp_path, world, kind, ahead):
    """SteppedBfs (the host protocol the GPU ranks run) over gloo: levels equal the
    reference's, and every rank issued the same number of collectives
    (iterations + 1 + ahead), so NCCL collectives would match up."""
    mp.spawn(worker, args=(world, free_port(), str(tmp_path), kind, ahead), nprocs=world, join=True)
    files = sorted(f for f in os.listdir(tmp_path) if not f.startswith("cnt_"))
    assert len(files) == 3
    for f in files:
        got, want = np.load(os.path.join(tmp_path, f))
        assert np.array_equal(got, want), f
        cnt = np.load(os.path.join(tmp_path, "cnt_" + f))
        assert (cnt[:, 0] == cnt[0, 0]).all() and (cnt[:, 1] == cnt[0, 1]).all()
        assert cnt[0, 0] == cnt[0, 1] + 1 + ahead


def test_partition_rows_are_aligned_and_cover():
    from paper_2512_21967_b200.multigpu import partition_rows_even
    for n in (1, 31, 32, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            b = partition_rows_even(n, world)
            assert len(b) == world + 1 and b[0] == 0 and b[-1] == (n + 31) // 32
            assert all(x <= y for x, y in zip(b, b[1:]))
