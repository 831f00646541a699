"""GPU: orderings and classifier against the reference's permutations (golden fixtures made
from the reference; the corpus graphs are rebuilt with the reference's own generators)."""
import numpy as np
import pytest

import paper_2512_21967_b200 as B

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def corpus(oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    out = []
    for name, rg in oracle.synthetic_corpus():
        c = rg.csr()
        out.append((name, rg, B.Graph.from_csr(c.n, c.offsets, c.targets, directed=True)))
    return out


def test_rcm_matches_reference(corpus, golden):
    """rcm (R:src/ordering.cpp:246-266), identical permutation."""
    acc = golden("corpus.npz")
    for name, rg, g in corpus:
        assert np.array_equal(B.rcm(g).forward_map(), acc[name + "/rcm"]), name


def test_jaccard_windows_matches_reference(corpus, golden):
    """jaccard_with_windows (R:src/ordering.cpp:139-166), w = 256, identical permutation."""
    acc = golden("corpus.npz")
    for name, rg, g in corpus:
        key = name + "/jaccard_w256"
        if key in acc.files:
            got = B.jaccard_with_windows(g, 8, 256).forward_map()
            assert np.array_equal(got, acc[key]), name


def test_jaccard_windows_various_w(corpus, oracle):
    """Against the reference directly for more window sizes and the naive oracle
    (R:tests/ordering_test.cpp:62-73)."""
    for name, rg, g in corpus[:7]:
        for w in (8, 64, 1024):
            assert np.array_equal(B.jaccard_with_windows(g, 8, w).forward_map(),
                                  rg.jaccard_windows(w)), (name, w)
    name, rg, g = corpus[6]
    assert np.array_equal(B.jaccard_with_windows(g, 8, 32).forward_map(), rg.naive_window_order(32))


def test_classifier_matches_reference(corpus, golden):
    """classify_social_like (R:src/ordering.cpp:346-387), bit-exact shares/slope/r2."""
    acc = golden("corpus.npz")
    for name, rg, g in corpus:
        r = B.classify_social_like(g)
        want = acc[name + "/classify"]
        assert [r.top1_share, r.top10_share, r.power_law_slope, r.power_law_fit_r2] == list(want), name
        assert r.is_social_like == bool(acc[name + "/social"][0])


def test_random_order_matches_reference(oracle):
    """random_order (R:src/ordering.cpp:268-275) with the reference Rng."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    for n, seed in ((1, 0), (1000, 99), (4097, 12345)):
        assert np.array_equal(B.random_order(n, seed).forward_map(), oracle.ref_random_order(n, seed))


def test_rcm_reduces_divergence():
    """R:tests/bvss_test.cpp:202-208 on a scrambled mesh."""
    g = B.Graph.generate_grid(40, 40)
    g = B.apply_permutation(g, B.relabel_permutation(1600, 12))
    before = B.build_bvss(g).update_divergence()
    after = B.build_bvss(B.apply_permutation(g, B.rcm(g))).update_divergence()
    assert after < before


def test_auto_routing():
    """R:tests/bfs_engine_test.cpp:317-345: meshes -> RCM + eager; star -> windows + eager."""
    g = B.apply_permutation(B.Graph.generate_grid(22, 22), B.relabel_permutation(484, 57))
    a = B.run_auto(g, 7)
    assert a.plan.strategy == B.OrderingStrategy.Rcm and a.chosen_mode == B.EngineMode.Eager
    assert not a.plan.classification.is_social_like
    n = 900
    star = B.Graph.from_edges(n, np.stack([np.zeros(n - 1), np.arange(1, n)], 1), directed=False)
    cfg = B.AutoConfig(ordering=B.SelectDefaults(window_size=1 << 10))
    a = B.run_auto(star, 3, cfg)
    assert a.plan.strategy == B.OrderingStrategy.JaccardWindows
    assert a.plan.classification.is_social_like and a.chosen_mode == B.EngineMode.Eager
    assert a.bfs.levels[3] == 0 and a.bfs.levels[0] == 1 and a.bfs.visited_count == n


@pytest.mark.parametrize("kind", ["urand20", "grid1024", "rmat14_directed", "components"])
def test_gpu_rcm_at_scale_matches_reference(oracle, kind):
    """The GPU RCM (csrc/rcm.cu: cooperative plain BFSs for pseudo_peripheral, Cuthill-McKee
    order level by level with radix sorts) gives the reference's permutation
    (R:src/ordering.cpp:171-266) at scale: urand-20, a 1024 x 1024 grid (1 K levels), a
    directed RMAT (symmetrised adjacency) and a graph of many small components."""
    import time
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    if kind == "urand20":
        s, d = oracle.gen_urand(1 << 20, 16 << 20, 3)
        n, directed = 1 << 20, False
    elif kind == "grid1024":
        s, d = oracle.gen_grid(1024, 1024)
        n, directed = 1024 * 1024, False
        f = oracle.random_relabel(n, 5)
        s, d = f[s], f[d]
    elif kind == "rmat14_directed":
        s, d = oracle.gen_rmat(14, 8, 2)
        n, directed = 1 << 14, True
    else:  # paths of 1..9 vertices plus isolated vertices, shuffled ids
        n, src, dst, v = 20000, [], [], 0
        rng = np.random.default_rng(1)
        while v < n - 10:
            k = int(rng.integers(1, 10))
            src += list(range(v, v + k - 1))
            dst += list(range(v + 1, v + k))
            v += k + int(rng.integers(0, 3))
        f = rng.permutation(n).astype(np.uint32)
        s, d = f[np.array(src, np.uint32)], f[np.array(dst, np.uint32)]
        directed = False
    rg = oracle.ref_from_edges(n, s, d, directed=directed)
    c = rg.csr()
    g = B.Graph.from_csr(n, c.offsets, c.targets, directed=directed)
    t0 = time.perf_counter()
    got = B.rcm(g).forward_map()
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    want = rg.rcm()
    t_ref = time.perf_counter() - t0
    assert np.array_equal(got, want), kind
    print(f"{kind}: GPU rcm {t_gpu:.3f} s, reference {t_ref:.3f} s")
