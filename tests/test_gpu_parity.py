"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the golden fixtures.
Bit-exact throughout: graph CSR, BVSS arrays, level arrays, per-level queue sizes /
discoveries / pushes (deterministic per SPEC.md:456)."""
import hashlib

import numpy as np
import pytest

import paper_2512_21967_b200 as B

pytestmark = pytest.mark.gpu
INF = 0xFFFFFFFF
VARIANTS = [("eager", "popc"), ("eager", "mma"), ("lazy", "popc"), ("lazy", "mma")]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.digest()


def run(b, src, mode, pull, **kw):
    cfg = B.EngineConfig(pull=pull, **kw)
    return (B.run_lazy if mode == "lazy" else B.run_eager)(b, src, cfg)


def trace_cols(cnt):
    return np.array([[t.level, t.queue_size, t.frontier_population, t.discovered, t.queue_pushes]
                     for t in cnt.trace], np.uint64).reshape(-1, 5)


def check_identities(res, cnt, n):
    """R:tests/bfs_engine_test.cpp:27-48."""
    assert cnt.mma_calls == 2 * cnt.vss_dequeues
    assert cnt.brs_baseline_mma_calls == 16 * cnt.vss_dequeues
    assert sum(t.queue_pushes for t in cnt.trace) == cnt.queue_pushes
    assert sum(t.queue_size for t in cnt.trace) == cnt.vss_dequeues
    assert sum(t.discovered for t in cnt.trace) + 1 == res.visited_count
    assert res.num_levels == cnt.levels_processed + 1
    assert len(res.levels) == n


def test_device_is_b200():
    info = B.device_info()
    assert info["cc"].startswith("10."), info


def test_graph_from_edges_matches_oracle(oracle, golden):
    f = golden("engine_families.npz")
    for name in f["names"]:
        name = str(name)
        n = int(f[name + "/n"][0])
        off, tgt = f[name + "/offsets"], f[name + "/targets"]
        src = np.repeat(np.arange(n, dtype=np.uint32), np.diff(off).astype(np.int64))
        g = B.Graph.from_edges(n, (src, tgt), directed=True)
        o, t = g.csr()
        assert np.array_equal(o, off) and np.array_equal(t, tgt), name
        g2 = B.Graph.from_csr(n, off, tgt)
        assert np.array_equal(g2.csr()[1], tgt)
    # undirected mirroring, self-loops and duplicates (R:src/graph.cpp:35-46)
    e = np.array([[0, 1], [1, 0], [2, 2], [1, 3], [1, 3]], np.uint32)
    g = B.Graph.from_edges(4, e, directed=False)
    o, t = g.csr()
    want = oracle.from_edges(4, e[:, 0], e[:, 1], directed=False)
    assert np.array_equal(o, want.offsets) and np.array_equal(t, want.targets)
    with pytest.raises(ValueError):
        B.Graph.from_edges(3, np.array([[0, 5]]))


def test_generators_match_oracle(oracle, golden):
    gz = golden("generators.npz")
    for scale in (8, 10, 12):
        g = B.Graph.generate_rmat(scale, 16, 1)
        o, t = g.csr()
        assert sha(o, t) == bytes(gz[f"rmat{scale}/graph_sha"]), scale
    s, d = oracle.gen_urand(1000, 16000, 3)
    g = B.Graph.generate_urand(1000, 16000, 3)
    want = oracle.from_edges(1000, s, d, directed=False)
    o, t = g.csr()
    assert np.array_equal(o, want.offsets) and np.array_equal(t, want.targets)
    s, d = oracle.gen_grid(37, 53)
    g = B.Graph.generate_grid(37, 53)
    want = oracle.from_edges(37 * 53, s, d, directed=False)
    assert np.array_equal(g.csr()[1], want.targets)
    assert np.array_equal(B.relabel_permutation(1000, 7).forward_map(), gz["relabel1000"])


def test_apply_permutation_matches_oracle(oracle):
    s, d = oracle.gen_rmat(11, 8, 9)
    g = B.Graph.from_edges(1 << 11, (s, d), directed=False)
    f = oracle.random_relabel(1 << 11, 3)
    h = B.apply_permutation(g, B.Permutation(f))
    o, t = g.csr()
    want = oracle.apply_permutation(oracle.Csr(1 << 11, o, t), f)
    ho, ht = h.csr()
    assert np.array_equal(ho, want.offsets) and np.array_equal(ht, want.targets)


def test_bvss_kats(golden):
    """R:tests/bvss_test.cpp:39-109: byte-identical arrays from the GPU builder."""
    k = golden("bvss_kats.npz")
    for name in sorted({key.split("/")[0] for key in k.files}):
        n = int(k[name + "/n"][0])
        e = k[name + "/edges"]
        g = B.Graph.from_edges(n, e, directed=True)
        b = B.build_bvss(g)
        rp, v2r, rows, masks = b.arrays()
        assert np.array_equal(rp, k[name + "/real_ptrs"]), name
        assert np.array_equal(v2r, k[name + "/v2r"]), name
        assert np.array_equal(rows, k[name + "/row_ids"]), name
        assert np.array_equal(masks, k[name + "/masks"]), name


@pytest.mark.parametrize("mode,pull", VARIANTS)
def test_engine_families(golden, mode, pull):
    """R:tests/bfs_engine_test.cpp:163-203: levels equal the reference; per-level queue sizes,
    discoveries and pushes equal the reference engines' traces."""
    f = golden("engine_families.npz")
    for name in f["names"]:
        name = str(name)
        n = int(f[name + "/n"][0])
        off, tgt = f[name + "/offsets"], f[name + "/targets"]
        g = B.Graph.from_csr(n, off, tgt, directed=True)
        b = B.build_bvss(g)
        rp, v2r, rows, masks = b.arrays()
        assert sha(rp, v2r, rows, masks) == bytes(f[name + "/bvss_sha"]), name
        assert B.compression_ratio(b) == f[name + "/compression"][0]
        assert b.update_divergence() == f[name + "/divergence"][0]
        for i, s in enumerate(f[name + "/sources"]):
            res, cnt = run(b, int(s), mode, pull)
            assert np.array_equal(res.levels, f[f"{name}/levels{i}"]), (name, i)
            ref = f[f"{name}/trace{i}_{1 if mode == 'lazy' else 0}"]
            assert np.array_equal(trace_cols(cnt), ref[:, [0, 1, 2, 3, 7]]), (name, i)
            check_identities(res, cnt, n)


def test_init_state_and_worked_pull():
    """R:tests/bfs_engine_test.cpp:69-97 and :116-144."""
    e = [(17, 3), (19, 3), (22, 3)] + [(0, r) for r in range(64, 322)]
    g = B.Graph.from_edges(384, np.array(e), directed=True)
    b = B.build_bvss(g)
    st = B.init_state(b, 17, B.EngineMode.Eager)
    assert st.levels[17] == 0 and (st.levels == INF).sum() == 383
    for mode, pull in VARIANTS:
        res, cnt = run(b, 17, mode, pull)
        assert res.levels[17] == 0 and res.levels[3] == 1 and res.visited_count == 2
        assert len(cnt.trace) == 2
        assert cnt.trace[0].queue_size == 1 and cnt.trace[0].queue_pushes == 3
        assert cnt.trace[0].frontier_population == 1
        assert cnt.trace[1].queue_size == 3 and cnt.trace[1].discovered == 0
        assert cnt.mma_calls == 8 and cnt.vss_dequeues == 4 and cnt.brs_baseline_mma_calls == 64
        assert cnt.levels_processed == 1


def test_chain_diamond_and_empty_start():
    """R:tests/bfs_engine_test.cpp:99-114, :146-161; empty start (SURVEY §8(a) pitfall 5)."""
    g = B.Graph.from_edges(3, np.array([[0, 1], [1, 2]]), directed=True)
    b = B.build_bvss(g)
    g5 = B.Graph.from_edges(5, np.array([[0, 1], [0, 2], [1, 3], [2, 3], [3, 4]]), directed=True)
    b5 = B.build_bvss(g5)
    for mode, pull in VARIANTS:
        res, cnt = run(b, 0, mode, pull)
        assert list(res.levels) == [0, 1, 2] and res.num_levels == 3
        assert cnt.levels_processed == 2 and len(cnt.trace) == 3 and cnt.trace[-1].discovered == 0
        res, cnt = run(b5, 0, mode, pull, num_warps=4)
        assert list(res.levels) == [0, 1, 1, 2, 3]
        assert [t.queue_pushes for t in cnt.trace] == [1, 1, 1, 0]
        # vertex 2 has no out-edges into any slice: src 2's set (set 0) has VSSs, but
        # a sink-only graph gives an empty start
    g = B.Graph.from_edges(16, np.array([[0, 1]]), directed=True)
    b = B.build_bvss(g)
    res, cnt = B.run_eager(b, 9)
    assert res.visited_count == 1 and len(cnt.trace) == 0 and res.levels[9] == 0


def test_errors_and_level_cap():
    """R:tests/bfs_engine_test.cpp:308-315 and bfs source range (R:src/bfs_engine.cpp:31)."""
    s = np.arange(15, dtype=np.uint32)
    g = B.Graph.from_edges(16, (s, s + 1), directed=False)
    b = B.build_bvss(g)
    for mode, pull in VARIANTS:
        with pytest.raises(RuntimeError):
            run(b, 0, mode, pull, max_levels=2)
    with pytest.raises(ValueError):
        B.run_eager(b, 16)
    # the engine still works after an error
    res, _ = B.run_lazy(b, 0)
    assert list(res.levels) == list(range(16))


@pytest.mark.parametrize("warps", [1, 7, 32, 128, 0])
def test_warp_count_invariance(warps):
    """R:tests/bfs_engine_test.cpp:246-289: results invariant across warp counts."""
    g = B.Graph.generate_rmat(12, 8, 4)
    b = B.build_bvss(g)
    base, bc = B.run_eager(b, 5, B.EngineConfig(num_warps=1))
    for mode, pull in VARIANTS:
        res, cnt = run(b, 5, mode, pull, num_warps=warps)
        assert np.array_equal(res.levels, base.levels)
        assert cnt.vss_dequeues == bc.vss_dequeues and cnt.queue_pushes == bc.queue_pushes


def test_c1_rmat16_sixteen_sources(oracle):
    """BASELINE config 1: RMAT scale 16, edgefactor 16, 16 sources, levels bit-exact against the
    reference BFS (oracle restatement; compiled reference too when present), identity order,
    both engines and both pull variants; counters equal the reference engine's."""
    g = B.Graph.generate_rmat(16, 16, 1)
    off, tgt = g.csr()
    csr = oracle.Csr(g.num_vertices(), off, tgt)
    srcs = g.pick_sources(16, 1)
    want, _ = oracle.reference_bfs_many(csr, srcs)
    b = B.build_bvss(g)
    ob = oracle.build_bvss(csr)
    rp, v2r, rows, masks = b.arrays()
    assert np.array_equal(rows, ob.row_ids) and np.array_equal(masks, ob.masks)
    for k, s in enumerate(srcs):
        o_eng = oracle.run_engine(ob, int(s), False)
        for mode, pull in VARIANTS:
            res, cnt = run(b, int(s), mode, pull)
            assert np.array_equal(res.levels, want[k]), (int(s), mode, pull)
            assert cnt.vss_dequeues == o_eng.counters["vss_dequeues"]
            assert cnt.queue_pushes == o_eng.counters["queue_pushes"]
            assert np.array_equal(trace_cols(cnt)[:, [1, 3, 4]], o_eng.trace[:, [1, 3, 7]])
    if oracle.ref_available():
        s, d = oracle.gen_rmat(16, 16, 1)
        rg = oracle.ref_from_edges(1 << 16, s, d, directed=False)
        for k, src in enumerate(srcs[:4]):
            assert np.array_equal(rg.reference_bfs(int(src))[0], want[k])


def test_auto_pipeline_maps_levels_back(oracle):
    """R:tests/bfs_engine_test.cpp:205-222: run_auto levels (original ids) equal the reference
    for random, RCM and Jaccard-window orderings."""
    g = B.Graph.generate_rmat(13, 16, 2)
    off, tgt = g.csr()
    csr = oracle.Csr(g.num_vertices(), off, tgt)
    for strat in (B.OrderingStrategy.JaccardWindows, B.OrderingStrategy.Rcm,
                  B.OrderingStrategy.Random, B.OrderingStrategy.Identity):
        cfg = B.AutoConfig(ordering=B.SelectDefaults(window_size=1 << 10, force=strat), seed=3)
        b, plan = B.prepare(g, cfg)
        for src in g.pick_sources(3, 11):
            r = B.run_auto_prebuilt(b, plan, int(src), cfg)
            assert np.array_equal(r.bfs.levels, oracle.reference_bfs(csr, int(src))[0]), strat
            assert r.bfs.source == int(src)


@pytest.mark.parametrize("env", [
    {},
    {"BLEST_SIGMA": "0"},                  # lazy: visited bitmaps by plain row id (no σ view)
    {"BLEST_LAZY_RECHECK": "1"},           # lazy: test V_curr, re-check V_next at L2
    {"BLEST_DENSE_MIN": "1"},              # eager: F_next re-check on every level; lazy: queue + barrier on every level
    {"BLEST_DENSE_MIN": "1000000000"},     # eager: never (straight to the atomic); lazy: every level expanded inside stage 1
    {"BLEST_DENSE_MIN": "1", "BLEST_TAIL_DIV": "2"},  # lazy: dense levels, last half handed out dynamically
    {"BLEST_DENSE_MIN": "1", "BLEST_TAIL_DIV": "0"},  # lazy: dense levels, static round-robin only
    {"BLEST_LAZY_VARIANT": "tma"},         # lazy: TMA producer/consumer stage 1 (ablation)
    {"BLEST_SMALL_S2": "0"},               # lazy: every stage 2 sweeps all words (no dirty-word log)
    {"BLEST_SMALL_S2": "48"},              # lazy: tiny log — small stage 2 only where it fits, sweep elsewhere
    {"BLEST_DENSE_MIN": "1000000000", "BLEST_SMALL_S2": "100000000"},  # lazy: every level sparse, log as large as Q0
])
def test_engine_phase_variants(oracle, monkeypatch, env):
    """The batch-wide visited-test phases, the lazy σ view and their switches change only how
    the tests are answered: levels and every deterministic counter equal the reference
    engine's, for both engines and pulls, on undirected and directed graphs, including the
    most connected (first in σ) vertex as source."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for directed in (False, True):
        s, d = oracle.gen_rmat(14, 16, 5)
        n = 1 << 14
        csr = oracle.from_edges(n, s, d, directed=directed)
        g = B.Graph.from_csr(n, csr.offsets, csr.targets, directed=directed)
        b = B.build_bvss(g)
        ob = oracle.build_bvss(csr)
        deg = np.diff(csr.offsets.astype(np.int64))
        hub_src = int(np.argmax(deg))
        srcs = [hub_src] + [int(x) for x in oracle.pick_sources(csr, 3, 9)]
        for src in srcs:
            want = oracle.reference_bfs(csr, src)[0]
            for mode in ("eager", "lazy"):
                o_eng = oracle.run_engine(ob, src, mode == "lazy")
                for pull in ("popc", "mma"):
                    res, cnt = run(b, src, mode, pull)
                    assert np.array_equal(res.levels, want), (env, directed, src, mode, pull)
                    assert cnt.vss_dequeues == o_eng.counters["vss_dequeues"]
                    assert cnt.queue_pushes == o_eng.counters["queue_pushes"]
                    assert np.array_equal(trace_cols(cnt)[:, [1, 3, 4]], o_eng.trace[:, [1, 3, 7]])


def test_run_batch_pipelined(oracle):
    """blest_bfs_batch (pipelined level copies) equals per-source blest_bfs: levels bit-exact
    with the oracle and every counter equal, both engines; a bad source fails before any work."""
    g = B.Graph.generate_rmat(15, 16, 3)
    off, tgt = g.csr()
    csr = oracle.Csr(g.num_vertices(), off, tgt)
    b = B.build_bvss(g)
    srcs = g.pick_sources(5, 4)
    want, _ = oracle.reference_bfs_many(csr, srcs)
    for mode, fn in ((B.EngineMode.Eager, B.run_eager), (B.EngineMode.Lazy, B.run_lazy)):
        lv, cnts = B.run_batch(b, srcs, mode)
        assert np.array_equal(lv, want)
        for k, s in enumerate(srcs):
            _, c1 = fn(b, int(s))
            assert (cnts[k].vss_dequeues, cnts[k].queue_pushes, cnts[k].levels_processed) == \
                (c1.vss_dequeues, c1.queue_pushes, c1.levels_processed)
    with pytest.raises(ValueError):
        B.run_batch(b, [0, g.num_vertices()], B.EngineMode.Lazy)


@pytest.mark.parametrize("mode", ["lazy", "eager"])
@pytest.mark.parametrize("kind", ["urand", "grid", "rmat"])
def test_exhaustion_exit(oracle, monkeypatch, kind, mode):
    """The engines' exhaustion exit (bfs_lazy.cu, bfs_eager.cu): on a connected graph the
    barren last level is accounted without a pull (blest_bfs_last_unpulled = its queue), and
    levels,
    counters and the whole per-level trace still equal the reference engine's, with the exit
    armed (BLEST_EXHAUST=1, default) and off; on RMAT it fires only if the source's component
    holds every vertex with an edge."""
    import ctypes as C
    from paper_2512_21967_b200 import _lib as L
    if kind == "urand":
        g = B.Graph.generate_urand(1 << 14, 16 << 14, 5)
    elif kind == "grid":
        g = B.Graph.generate_grid(64, 96)
    else:
        g = B.Graph.generate_rmat(14, 16, 5)
    off, tgt = g.csr()
    csr = oracle.Csr(g.num_vertices(), off, tgt)
    b = B.build_bvss(g)
    ob = oracle.build_bvss(csr)
    if mode == "eager":  # the eager count is exact only after a dense level: make them all dense
        monkeypatch.setenv("BLEST_DENSE_MIN", "1")
    for src in g.pick_sources(3, 11):
        src = int(src)
        want = oracle.reference_bfs(csr, src)[0]
        o_eng = oracle.run_engine(ob, src, mode == "lazy")
        got = {}
        for ex in ("1", "0"):
            monkeypatch.setenv("BLEST_EXHAUST", ex)
            res, cnt = run(b, src, mode, "popc")
            unp = C.c_uint64(7)
            L.check(L.lib().blest_bfs_last_unpulled(b.handle, C.byref(unp)))
            assert np.array_equal(res.levels, want), (kind, src, ex)
            assert cnt.vss_dequeues == o_eng.counters["vss_dequeues"]
            assert np.array_equal(trace_cols(cnt)[:, [1, 3, 4]], o_eng.trace[:, [1, 3, 7]])
            got[ex] = (int(unp.value), int(cnt.trace[-1].queue_size), int(cnt.trace[-1].discovered))
        assert got["0"][0] == 0
        assert got["1"][0] in (0, got["1"][1]) and (got["1"][0] == 0 or got["1"][2] == 0), got
        if kind != "rmat":  # connected: the last level is barren and was not pulled
            assert got["1"][0] > 0, got


def test_run_batch_narrow_transfers(oracle, monkeypatch):
    """blest_bfs_batch's narrow level transfers (xfer.cuh): u8 while the deepest level fits,
    u16 after a source overflows it, plain u32 after that — every source's u32 array equal to
    the oracle's and to the plain-copy path (BLEST_D2H_PACK=0), unreached vertices included."""
    g = B.Graph.generate_rmat(15, 16, 5)
    off, tgt = g.csr()
    csr = oracle.Csr(g.num_vertices(), off, tgt)
    b = B.build_bvss(g)
    srcs = g.pick_sources(7, 9)
    want, _ = oracle.reference_bfs_many(csr, srcs)
    assert (want == INF).any()  # RMAT leaves vertices unreached: the 0 -> kInf mapping is hit
    lv, _ = B.run_batch(b, srcs, B.EngineMode.Lazy)
    assert np.array_equal(lv, want)
    # a path of 70 000 vertices (levels past 255 and past 65535) plus a separate triangle
    n_path = 70_000
    e = [(i, i + 1) for i in range(n_path - 1)] + [(n_path, n_path + 1), (n_path + 1, n_path + 2), (n_path + 2, n_path)]
    n = n_path + 3 + 30  # + isolated vertices; odd n (the second pack buffer's alignment)
    g2 = B.Graph.from_edges(n, e, directed=False)
    off2, tgt2 = g2.csr()
    csr2 = oracle.Csr(n, off2, tgt2)
    b2 = B.build_bvss(g2)
    # mid: u8 overflows (-> u16); mid again: u16; 0: u16 overflows (-> u32); triangle: u32 path
    srcs2 = np.array([n_path // 2, n_path // 2 + 7, 0, n_path + 1, 5], np.uint32)
    want2, _ = oracle.reference_bfs_many(csr2, srcs2)
    for pack in ("1", "0"):
        monkeypatch.setenv("BLEST_D2H_PACK", pack)
        lv2, cnts = B.run_batch(b2, srcs2, B.EngineMode.Eager)
        assert np.array_equal(lv2, want2), pack
        assert [c.levels_processed for c in cnts] == [int(w[w != INF].max()) for w in want2]
    monkeypatch.setenv("BLEST_D2H_PACK", "1")
    lv3, _ = B.run_batch(b2, srcs2[3:], B.EngineMode.Eager)  # triangle first: u8 all the way
    assert np.array_equal(lv3, want2[3:])


@pytest.mark.parametrize("kind", ["urand", "grid"])
def test_auto_pipeline_non_social(oracle, kind):
    """C3 / C4 graph kinds at small scale through the whole pipeline (GPU generator →
    classifier → RCM → BVSS → auto engine = eager for non-social graphs): levels in original
    ids equal the reference BFS for several sources, and batch runs agree."""
    if kind == "urand":
        n = 1 << 14
        g = B.Graph.generate_urand(n, 16 * n, 3)
    else:
        g = B.Graph.generate_grid(96, 160)
    off, tgt = g.csr()
    csr = oracle.Csr(g.num_vertices(), off, tgt)
    cfg = B.AutoConfig(seed=3)
    b, plan = B.prepare(g, cfg)
    srcs = g.pick_sources(4, 7)
    for src in srcs:
        r = B.run_auto_prebuilt(b, plan, int(src), cfg)
        assert np.array_equal(r.bfs.levels, oracle.reference_bfs(csr, int(src))[0]), (kind, int(src))
        if not plan.classification.is_social_like:  # the reference's auto rule (R:src/bfs_engine.cpp:358-362)
            assert r.chosen_mode == B.EngineMode.Eager


def test_lazy_dense_levels_rmat18(oracle, monkeypatch):
    """A graph big enough for dense levels (queue ≥ 8 VSSs per warp): the lazy engine's
    dynamic tail hand-out and the hot-row view run unforced; levels and counters equal the
    oracle's, and a hot-prefix cap of 4096 rows (most hubs outside the prefix) agrees too."""
    g = B.Graph.generate_rmat(18, 16, 2)
    off, tgt = g.csr()
    csr = oracle.Csr(g.num_vertices(), off, tgt)
    srcs = g.pick_sources(2, 5)
    want, _ = oracle.reference_bfs_many(csr, srcs)
    ob = oracle.build_bvss(csr)
    for hot in (None, "4096"):
        if hot:
            monkeypatch.setenv("BLEST_HOT", hot)
        b = B.build_bvss(g)  # a fresh structure builds its hot view under the current cap
        for k, s in enumerate(srcs):
            res, cnt = B.run_lazy(b, int(s))
            assert np.array_equal(res.levels, want[k]), (hot, int(s))
            o_eng = oracle.run_engine(ob, int(s), True)
            assert cnt.vss_dequeues == o_eng.counters["vss_dequeues"]
            assert max(t.queue_size for t in cnt.trace) >= 296 * 16 * 8  # a dense level ran (dense_min)
