"""GPU: the row-partitioned kernels (blest_bvss_build_rows / blest_part_*) with G virtual
ranks on one B200 (shard the BVSS G-way, the all-gather becomes a device
concatenation). Levels bit-exact against the oracle; each rank's BVSS equals the oracle's
BVSS of the row-filtered graph."""
import hashlib

import numpy as np
import pytest

import paper_2512_21967_b200 as B
from paper_2512_21967_b200.multigpu import GpuPartition, partition_rows, run_lockstep, words_per_rank

pytestmark = pytest.mark.gpu


def test_rows_bvss_matches_oracle(oracle):
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from partition_cpu import rows_graph
    s, d = oracle.gen_rmat(11, 8, 4)
    g = B.Graph.from_edges(1 << 11, (s, d), directed=False)
    off, tgt = g.csr()
    csr = oracle.Csr(1 << 11, off, tgt)
    for lo, hi in partition_rows(1 << 11, 3):
        import ctypes as C
        from paper_2512_21967_b200 import _lib as L
        h = C.c_void_p()
        L.check(L.lib().blest_bvss_build_rows(g.handle, lo, hi, C.byref(h)))
        b = B.Bvss(h.value)
        want = oracle.build_bvss(rows_graph(csr, lo, hi))
        rp, v2r, rows, masks = b.arrays()
        assert np.array_equal(rp, want.real_ptrs) and np.array_equal(rows, want.row_ids)
        assert np.array_equal(masks, want.masks) and b.m == want.m


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_virtual_ranks_levels(oracle, world):
    for kind in ("rmat", "grid"):
        if kind == "rmat":
            g = B.Graph.generate_rmat(13, 16, 6)
        else:
            g = B.apply_permutation(B.Graph.generate_grid(61, 67), B.relabel_permutation(61 * 67, 2))
        n = g.num_vertices()
        off, tgt = g.csr()
        csr = oracle.Csr(n, off, tgt)
        per = words_per_rank(n, world)
        backends = [GpuPartition(g, lo, hi, per) for lo, hi in partition_rows(n, world)]
        for src in g.pick_sources(3, 9):
            got, iters = run_lockstep(backends, n, int(src))
            want = oracle.reference_bfs(csr, int(src))[0]
            assert np.array_equal(got, want), (kind, world, int(src))
