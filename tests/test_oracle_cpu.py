"""CPU: pin the oracle restatement (oracle/blest_oracle.c) against the committed golden
fixtures made from the reference, and — where the compiled reference (oracle/_ref) is
present — against the reference itself on the full acceptance corpus."""
import numpy as np
import pytest

INF = 0xFFFFFFFF


def test_tile_worked_example(oracle, golden):
    """R:tests/tc_emu_test.cpp:186-201: mask 0x4A vs alpha 0x03 -> (1, 0) on lane 0 only."""
    t = golden("tile.npz")
    masks = np.zeros(32, np.uint32)
    masks[0] = 0x4A
    c = oracle.tile_pull(masks, 0x03, 0)
    assert np.array_equal(c, t["worked"])
    assert c[0] == 1 and c[1] == 0 and c.sum() == 1


def test_tile_random_and_lane_locality(oracle, golden):
    """R:tests/tc_emu_test.cpp:203-223: each lane's two outputs are its own mask popcounts."""
    t = golden("tile.npz")
    for i in range(len(t["alpha"])):
        m, a = t["masks"][i], int(t["alpha"][i])
        for r in (0, 1):
            c = oracle.tile_pull(m, a, r)
            assert np.array_equal(c, t["counts"][i, r])
            for lane in range(32):
                i8, j = lane // 4, 2 * (lane % 4)
                even = bin(int((m[lane] >> (16 * r)) & 0xFF) & a).count("1")
                odd = bin(int((m[lane] >> (16 * r + 8)) & 0xFF) & a).count("1")
                assert c[8 * i8 + j] == even and c[8 * i8 + j + 1] == odd


def test_bvss_kats(oracle, golden):
    """R:tests/bvss_test.cpp:39-109 known answers, re-derived by the oracle builder."""
    k = golden("bvss_kats.npz")
    names = sorted({key.split("/")[0] for key in k.files})
    for name in names:
        n = int(k[name + "/n"][0])
        e = k[name + "/edges"]
        g = oracle.from_edges(n, e[:, 0], e[:, 1], directed=True)
        b = oracle.build_bvss(g)
        assert np.array_equal(b.real_ptrs, k[name + "/real_ptrs"]), name
        assert np.array_equal(b.virtual_to_real, k[name + "/v2r"]), name
        assert np.array_equal(b.row_ids, k[name + "/row_ids"]), name
        assert np.array_equal(b.masks, k[name + "/masks"]), name
    # worked example: mask 0x4A in slice set 2, real_ptrs {0,0,0,1}
    assert list(k["worked-0x4A/real_ptrs"]) == [0, 0, 0, 1]
    assert (k["worked-0x4A/masks"][0] & 0xFF) == 0x4A


def _sha(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.digest()


def test_engine_families(oracle, golden):
    """R:tests/bfs_engine_test.cpp:163-203: levels + per-level traces of both engines."""
    f = golden("engine_families.npz")
    for name in f["names"]:
        name = str(name)
        g = oracle.Csr(int(f[name + "/n"][0]), f[name + "/offsets"], f[name + "/targets"])
        b = oracle.build_bvss(g)
        assert _sha(b.real_ptrs, b.virtual_to_real, b.row_ids, b.masks) == bytes(f[name + "/bvss_sha"])
        assert oracle.compression_ratio(b) == f[name + "/compression"][0]
        assert oracle.update_divergence(b) == f[name + "/divergence"][0]
        for i, s in enumerate(f[name + "/sources"]):
            lv, vis, nl = oracle.reference_bfs(g, int(s))
            assert np.array_equal(lv, f[f"{name}/levels{i}"]), name
            assert oracle.validate_levels(g, int(s), lv) == 0
            for lazy in (0, 1):
                r = oracle.run_engine(b, int(s), bool(lazy), num_warps=4)
                assert np.array_equal(r.levels, lv)
                assert np.array_equal(r.trace, f[f"{name}/trace{i}_{lazy}"]), (name, i, lazy)


def test_generators_pinned(oracle, golden):
    """Harness RMAT/urand/relabel definitions and the reference BFS on them."""
    gz = golden("generators.npz")
    for scale in (8, 10, 12):
        s, d = oracle.gen_rmat(scale, 16, 1)
        assert _sha(s, d) == bytes(gz[f"rmat{scale}/edges_sha"])
        g = oracle.from_edges(1 << scale, s, d, directed=False)
        assert _sha(g.offsets, g.targets) == bytes(gz[f"rmat{scale}/graph_sha"])
        for x, want in zip(gz[f"rmat{scale}/sources"], gz[f"rmat{scale}/levels"]):
            assert np.array_equal(oracle.reference_bfs(g, int(x))[0], want)
    s, d = oracle.gen_urand(1000, 16000, 3)
    assert _sha(s, d) == bytes(gz["urand1000/edges_sha"])
    assert np.array_equal(oracle.random_relabel(1000, 7), gz["relabel1000"])


def test_validate_levels_catches_faults(oracle):
    s, d = oracle.gen_rmat(10, 16, 5)
    g = oracle.from_edges(1024, s, d, directed=False)
    src = int(np.argmax(np.diff(g.offsets)))
    lv = oracle.reference_bfs(g, src)[0]
    assert oracle.validate_levels(g, src, lv) == 0
    bad = lv.copy()
    v = int(np.flatnonzero((lv != INF) & (lv > 1))[0])
    bad[v] += 1
    assert oracle.validate_levels(g, src, bad) != 0
    bad = lv.copy()
    bad[v] = INF
    assert oracle.validate_levels(g, src, bad) != 0


def test_oracle_engine_level_cap(oracle):
    """R:tests/bfs_engine_test.cpp:308-315: the level safety cap stops a run."""
    s = np.arange(15, dtype=np.uint32)
    g = oracle.from_edges(16, s, s + 1, directed=False)
    b = oracle.build_bvss(g)
    with pytest.raises(oracle.OracleError):
        oracle.run_engine(b, 0, False, max_levels=2)
    with pytest.raises(oracle.OracleError):
        oracle.run_engine(b, 0, True, max_levels=2)


@pytest.mark.skipif(not __import__("oracle").ref_available() and
                    not __import__("os").path.isdir("/root/reference/proj"),
                    reason="compiled reference not present")
def test_oracle_matches_reference_on_corpus(oracle, golden):
    """Acceptance corpus (R:tests/support/generators.cpp:164-179): the restatement equals the
    reference for BVSS arrays, stats, levels and full engine traces."""
    acc = golden("corpus.npz")
    for name, rg in oracle.synthetic_corpus():
        g = rg.csr()
        assert _sha(g.offsets, g.targets) == bytes(acc[name + "/graph_sha"])
        rb = rg.build_bvss()
        ref = rb.arrays(g.n)
        b = oracle.build_bvss(g)
        for fld in ("real_ptrs", "virtual_to_real", "row_ids", "masks"):
            assert np.array_equal(getattr(b, fld), getattr(ref, fld)), (name, fld)
        assert oracle.compression_ratio(b) == rb.compression_ratio()
        assert oracle.update_divergence(b) == rb.update_divergence()
        for src in acc[name + "/sources"][:2]:
            lv = rg.reference_bfs(int(src))[0]
            assert np.array_equal(oracle.reference_bfs(g, int(src))[0], lv)
            for lazy in (False, True):
                r = rb.run(int(src), lazy, warps=4, n=g.n)
                o = oracle.run_engine(b, int(src), lazy, num_warps=4)
                assert np.array_equal(r.levels, lv) and np.array_equal(o.levels, lv)
                assert np.array_equal(r.trace, o.trace), (name, lazy)
