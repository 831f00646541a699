"""CPU: the full-scale half of the oracle (oracle/blest_oracle_scale.c) is pinned to the
single-threaded restatement and to the UNMODIFIED reference (oracle/_ref) before the
bench and the GPU tests trust it at scale 20-27."""
import numpy as np
import pytest


def same_csr(a, b):
    return np.array_equal(a.offsets, b.offsets) and np.array_equal(a.targets, b.targets)


@pytest.mark.parametrize("kind", ["rmat", "urand", "grid"])
def test_gen_csr_equals_from_edges(oracle, kind):
    """orc_gen_csr == from_edges(generator lists) (R:src/graph.cpp:33-55), with and without the
    relabel, for any thread count; the multi-threaded relabel equals the serial one."""
    if kind == "rmat":
        n, spec = 1 << 12, ("rmat", 12, 0, 16 << 12, 5)
        s, d = oracle.gen_rmat(12, 16, 5)
    elif kind == "urand":
        n, spec = 5000, ("urand", 5000, 0, 80000, 3)
        s, d = oracle.gen_urand(5000, 80000, 3)
    else:
        n, spec = 37 * 53, ("grid", 37, 53, 0, 0)
        s, d = oracle.gen_grid(37, 53)
    fw = oracle.random_relabel(n, 9)
    assert np.array_equal(fw, oracle.random_relabel_mt(n, 9, 4))
    for f in (None, fw):
        want = oracle.from_edges(n, s if f is None else f[s], d if f is None else f[d], directed=False)
        for t in (1, 3, 8):
            assert same_csr(oracle.gen_csr(*spec, forward=f, threads=t), want), (kind, t)


def test_permute_and_bvss_mt(oracle):
    s, d = oracle.gen_rmat(13, 16, 2)
    g = oracle.from_edges(1 << 13, s, d, directed=False)
    f = oracle.random_relabel(g.n, 4)
    assert same_csr(oracle.permute_csr(g, f, 3), oracle.apply_permutation(g, f))
    a, b = oracle.build_bvss(g), oracle.build_bvss_mt(g, 5)
    for k in ("real_ptrs", "virtual_to_real", "row_ids", "masks"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.num_unpadded_slices == b.num_unpadded_slices
    rb = oracle.ref_from_csr(g).build_bvss().arrays(g.n)  # and the reference's build_bvss
    assert np.array_equal(rb.row_ids, b.row_ids) and np.array_equal(rb.masks, b.masks)


def test_orderings_and_classifier_match_reference_on_corpus(oracle):
    """jaccard_with_windows (several w), rcm and classify_social_like restatements equal the
    reference's on the 12-graph acceptance corpus (one of them directed)."""
    for name, rg in oracle.synthetic_corpus():
        g = rg.csr()
        gi = rg.csr(incoming=True)
        g.directed = not same_csr(g, gi)
        for w in (8, 32, 256):
            assert np.array_equal(rg.jaccard_windows(w), oracle.jaccard_windows(g, w, threads=4)), (name, w)
        assert np.array_equal(rg.rcm(), oracle.rcm(g)), name
        assert rg.classify() == oracle.classify(g), name


def test_orderings_match_reference_rmat_urand(oracle):
    for scale in (12, 14):
        n = 1 << scale
        s, d = oracle.gen_rmat(scale, 16, 1)
        g = oracle.from_edges(n, s, d, directed=False)
        rg = oracle.ref_from_csr(g)
        assert rg.classify() == oracle.classify(g)
        for w in (64, 1024):
            assert np.array_equal(rg.jaccard_windows(w), oracle.jaccard_windows(g, w)), (scale, w)
        s, d = oracle.gen_urand(n, 16 * n, 3)
        g = oracle.from_edges(n, s, d, directed=False)
        rg = oracle.ref_from_csr(g)
        assert rg.classify() == oracle.classify(g)
        assert np.array_equal(rg.rcm(), oracle.rcm(g)), scale


def test_traversed_edges(oracle):
    s, d = oracle.gen_rmat(10, 16, 1)
    g = oracle.from_edges(1 << 10, s, d, directed=False)
    lv = oracle.reference_bfs(g, int(oracle.pick_sources(g, 1, 1)[0]))[0]
    deg = np.diff(g.offsets.astype(np.int64))
    assert oracle.traversed_edges(g, lv) == int(deg[lv != 0xFFFFFFFF].sum()) // 2
