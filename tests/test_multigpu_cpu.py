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


def worker(rank, world, port, out_dir, kind):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
    sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from partition_cpu import NumpyPartition
    from paper_2512_21967_b200.multigpu import RowPartitionedBfs, partition_rows, words_per_rank
    if kind == "rmat":
        s, d = O.gen_rmat(10, 8, 3)
        g = O.from_edges(1 << 10, s, d, directed=False)
    else:
        s, d = O.gen_grid(23, 29)
        g = O.from_edges(23 * 29, s, d, directed=False)
    lo, hi = partition_rows(g.n, world)[rank]
    per = words_per_rank(g.n, world)
    bfs = RowPartitionedBfs(NumpyPartition(g, lo, hi, per), g.n, gloo_allgather)
    srcs = O.pick_sources(g, 3, 5)
    for k, src in enumerate(srcs):
        r = bfs.run(int(src))
        full = torch.zeros(world * per * 32, dtype=torch.int64)
        mine = torch.full((per * 32,), -1, dtype=torch.int64)
        mine[: hi - lo] = torch.from_numpy(r.levels.astype(np.int64))
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        if rank == 0:
            got = torch.cat([p[: min(per * 32, g.n - i * per * 32)] for i, p in enumerate(parts)]).numpy()
            want = O.reference_bfs(g, int(src))[0].astype(np.int64)
            want[want == 0xFFFFFFFF] = -1
            got[got == 0xFFFFFFFF] = -1
            np.save(os.path.join(out_dir, f"{kind}_{k}.npy"), np.stack([got, want]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "rmat"), (3, "grid")])
def test_row_partitioned_protocol_gloo(tmp_path, world, kind):
    mp.spawn(worker, args=(world, free_port(), str(tmp_path), kind), nprocs=world, join=True)
    files = sorted(os.listdir(tmp_path))
    assert len(files) == 3
    for f in files:
        got, want = np.load(os.path.join(tmp_path, f))
        assert np.array_equal(got, want), f


def test_partition_rows_are_aligned_and_cover():
    from paper_2512_21967_b200.multigpu import partition_rows
    for n in (1, 31, 32, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            parts = partition_rows(n, world)
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            assert all(lo % 32 == 0 for lo, hi in parts if hi > lo)
