"""GPU parity beyond the small cases: the reference's acceptance oracle pass on the 12-graph
corpus, the b1 tile known answers through the real instruction, and graphs large enough
to take the code paths the BASELINE configs take (C2: Jaccard w = 2^16 and the lazy
hot-row view with K < n on dense levels; C3: urand + RCM on the lazy engine; C4: a
scrambled grid + RCM on the eager engine, thousands of levels). Levels are compared with
the CPU reference BFS on an independently host-built original graph, in original ids."""
import hashlib

import numpy as np
import pytest

import paper_2512_21967_b200 as B

pytestmark = pytest.mark.gpu
INF = 0xFFFFFFFF


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest()


# ---------------------------------------------------------------------------------------
# tile (R:tests/tc_emu_test.cpp:186-241) through mma.sync.m8n8k128.b1.and.popc on the B200
# ---------------------------------------------------------------------------------------
def test_tile_kats_on_device(golden):
    t = golden("tile.npz")
    assert np.array_equal(B.tile_pull(t["masks"], t["alpha"]), t["counts"])  # 64 random tiles x 2 rounds
    m = np.zeros((1, 32), np.uint32)
    m[0, 0] = 0x4A  # worked example: mask 0x4A vs alpha 0x03 -> (1, 0) (:186-201)
    got = B.tile_pull(m, [0x03])[0, 0]
    assert np.array_equal(got, t["worked"]) and got[0] == 1 and got[1] == 0


def test_tile_lane_locality_on_device():
    """Lane t's FragC pair is its own two column popcounts (:203-223, 500 trials); padded
    lanes (mask 0) give 0 (:225-241)."""
    rng = np.random.default_rng(11)
    T = 500
    masks = rng.integers(0, 2**32, size=(T, 32), dtype=np.uint64).astype(np.uint32)
    masks[:, 20:] = 0  # padded lanes
    alpha = rng.integers(0, 256, size=T).astype(np.uint8)
    c = B.tile_pull(masks, alpha)
    lanes = np.arange(32)
    for r in (0, 1):
        for h in (0, 1):
            byte = (masks >> np.uint32(16 * r + 8 * h)) & np.uint32(0xFF)
            want = np.vectorize(lambda x: bin(x).count("1"))(byte & alpha[:, None].astype(np.uint32))
            got = c[:, r, 8 * (lanes // 4) + 2 * (lanes % 4) + h]
            assert np.array_equal(got, want), (r, h)
    assert not c[:, :, 8 * (20 // 4):].any()


# ---------------------------------------------------------------------------------------
# acceptance oracle pass (R:tests/acceptance_main.cpp:140-274)
# ---------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def acceptance(oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    out = []
    for i, (name, rg) in enumerate(oracle.synthetic_corpus()):
        c = rg.csr()
        g = B.Graph.from_csr(c.n, c.offsets, c.targets, directed=True)
        cfg = B.AutoConfig(seed=40000 + i)
        routed, plan = B.prepare(g, cfg)
        srcs = oracle.ref_rng_next_below(0xACCE5500 + i, c.n, 16).astype(np.uint32)
        want = [rg.reference_bfs(int(s))[0] for s in srcs]
        out.append((name, rg, c, g, B.build_bvss(g), routed, plan, cfg, srcs, want))
    return out


def test_acceptance_oracle_pass(acceptance, oracle):
    """12 graphs x 16 seeded sources x {eager, lazy on the identity BVSS, auto on the routed
    BVSS}: levels equal reference_bfs; eager and lazy deterministic counters (dequeues,
    pushes, per-level queue sizes / discoveries / pushes) equal the reference engines' (4
    simulated warps, as the acceptance binary runs them)."""
    runs = 0
    for name, rg, c, g, ident, routed, plan, cfg, srcs, want in acceptance:
        rb = rg.build_bvss()
        for k, s in enumerate(srcs):
            s = int(s)
            for mode, fn in (("eager", B.run_eager), ("lazy", B.run_lazy)):
                res, cnt = fn(ident, s)
                assert np.array_equal(res.levels, want[k]), (name, s, mode)
                ref = rb.run(s, mode == "lazy", warps=4, want_levels=False, n=c.n)
                assert cnt.vss_dequeues == ref.counters["vss_dequeues"], (name, s, mode)
                assert cnt.queue_pushes == ref.counters["queue_pushes"], (name, s, mode)
                tr = np.array([[t.queue_size, t.discovered, t.queue_pushes] for t in cnt.trace], np.uint64)
                assert np.array_equal(tr.reshape(-1, 3), ref.trace[:, [1, 3, 7]]), (name, s, mode)
            ar = B.run_auto_prebuilt(routed, plan, s, cfg)
            assert np.array_equal(ar.bfs.levels, want[k]), (name, s, "auto")
            runs += 3
    assert runs == 12 * 16 * 3


def test_acceptance_levels_golden(acceptance, golden):
    """The committed reference level digests (corpus.npz, 4 sources per graph)."""
    acc = golden("corpus.npz")
    for name, rg, c, g, ident, routed, plan, cfg, srcs, want in acceptance:
        for k, s in enumerate(acc[name + "/sources"]):
            for fn in (B.run_eager, B.run_lazy):
                res, _ = fn(ident, int(s))
                assert sha(res.levels) == bytes(acc[name + "/levels_sha"][k]), (name, int(s))


# ---------------------------------------------------------------------------------------
# the BASELINE configs' code paths at scale 20
# ---------------------------------------------------------------------------------------
def levels_in_original_ids(b, perm, src_orig, mode):
    src = int(perm.forward(src_orig)) if not perm.is_identity() else int(src_orig)
    res, cnt = (B.run_lazy if mode == "lazy" else B.run_eager)(b, src)
    lv = res.levels if perm.is_identity() else res.levels[perm.forward_map()]
    return lv, cnt


def test_c2_path_rmat20_jaccard_w16_hot_view(oracle, monkeypatch):
    """C2's path at scale 20: GAP-style relabel, Jaccard windows at the C2 window w = 2^16
    (GPU permutation identical to the CPU restatement, which is pinned to the reference's
    jaccard_with_windows), lazy engine with the hot-row view — at the default K (= n here)
    and at K = 2^16 < n (most rows outside the hot prefix, as at C2) — and the dense-level
    tail hand-out. 8 sources, levels in original ids vs the CPU reference BFS on the
    host-built original graph; dequeues vs the reference engine."""
    scale, n = 20, 1 << 20
    g = B.apply_permutation(B.Graph.generate_rmat(scale, 16, 1), B.relabel_permutation(n, 2))
    gc = oracle.gen_csr("rmat", scale, 0, 16 << scale, 1, forward=oracle.random_relabel_mt(n, 2))
    off, tgt = g.csr()
    assert np.array_equal(off, gc.offsets) and np.array_equal(tgt, gc.targets)  # GPU vs CPU builder
    plan = B.select_plan(g, 8, B.SelectDefaults(window_size=1 << 16))
    assert plan.strategy == B.OrderingStrategy.JaccardWindows
    perm = B.make_permutation(g, plan, 8)
    assert np.array_equal(perm.forward_map(), oracle.jaccard_windows(gc, 1 << 16))
    gp = B.apply_permutation(g, perm)
    srcs = oracle.pick_sources(gc, 8, 3)
    want, _ = oracle.reference_bfs_many(gc, srcs)
    ob = oracle.build_bvss_mt(oracle.permute_csr(gc, perm.forward_map()))
    rb = oracle.ref_bvss_from_arrays(ob)
    for hot in (None, str(1 << 16)):
        if hot:
            monkeypatch.setenv("BLEST_HOT", hot)
        b = B.build_bvss(gp)
        for k, s in enumerate(srcs):
            lv, cnt = levels_in_original_ids(b, perm, int(s), "lazy")
            assert np.array_equal(lv, want[k]), (hot, int(s))
            if k < 2:
                ref = rb.run(int(perm.forward(int(s))), True, warps=512, workers=8, want_levels=False, n=n)
                assert cnt.vss_dequeues == ref.counters["vss_dequeues"]
        assert max(t.queue_size for t in cnt.trace) >= 148 * 2 * 16 * 8  # a dense level ran


def test_c3_path_urand20_rcm_lazy(oracle):
    """C3's kind at scale 20: urand is not social-like, so the classifier routes it to RCM
    (permutation identical to the CPU restatement of R:src/ordering.cpp:246-266); the b200
    policy runs it on the lazy engine. Levels of 8 sources vs the CPU reference BFS."""
    n = 1 << 20
    g = B.Graph.generate_urand(n, 16 * n, 3)
    gc = oracle.gen_csr("urand", n, 0, 16 * n, 3)
    plan = B.select_plan(g, 8)
    assert plan.strategy == B.OrderingStrategy.Rcm
    perm = B.make_permutation(g, plan, 8)
    assert np.array_equal(perm.forward_map(), oracle.rcm(gc))
    b = B.build_bvss(B.apply_permutation(g, perm))
    srcs = oracle.pick_sources(gc, 8, 5)
    want, _ = oracle.reference_bfs_many(gc, srcs)
    for k, s in enumerate(srcs):
        for mode in ("lazy", "eager"):
            lv, _ = levels_in_original_ids(b, perm, int(s), mode)
            assert np.array_equal(lv, want[k]), (mode, int(s))


def test_c4_path_grid1024_rcm_eager(oracle):
    """C4's kind: a scrambled 1024x1024 grid reordered by RCM, eager engine (~2000 levels,
    the persistent kernel's level loop and grid barrier thousands of times). 4 sources."""
    rows = cols = 1024
    n = rows * cols
    g = B.apply_permutation(B.Graph.generate_grid(rows, cols), B.relabel_permutation(n, 4))
    gc = oracle.gen_csr("grid", rows, cols, forward=oracle.random_relabel_mt(n, 4))
    plan = B.select_plan(g, 8, B.SelectDefaults(force=B.OrderingStrategy.Rcm))
    perm = B.make_permutation(g, plan, 8)
    assert np.array_equal(perm.forward_map(), oracle.rcm(gc))
    b = B.build_bvss(B.apply_permutation(g, perm))
    srcs = oracle.pick_sources(gc, 4, 7)
    want, _ = oracle.reference_bfs_many(gc, srcs)
    for k, s in enumerate(srcs):
        lv, cnt = levels_in_original_ids(b, perm, int(s), "eager")
        assert np.array_equal(lv, want[k]), int(s)
        assert len(cnt.trace) > 1000


def test_jaccard_w16_rmat16_vs_reference(oracle):
    """GPU Jaccard windows at the C2 window size (one 2^16 window) against the reference's
    own jaccard_with_windows (R:src/ordering.cpp:139-166) on RMAT-16."""
    g = B.Graph.generate_rmat(16, 16, 1)
    off, tgt = g.csr()
    rg = oracle.ref_from_csr(oracle.Csr(g.num_vertices(), off, tgt))
    got = B.jaccard_with_windows(g, 8, 1 << 16).forward_map()
    assert np.array_equal(got, rg.jaccard_windows(1 << 16, 8, 8))
