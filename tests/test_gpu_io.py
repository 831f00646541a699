"""GPU: the boundary's file formats and checkers against the UNMODIFIED reference —
BVSS binary cache files and permutation files interchangeable both ways
(R:src/bvss.cpp:218-295, R:src/graph.cpp:396-417), load_graph (R:src/graph.cpp:233-394)
with the reference's parse errors, Graph::digest / in-views, reference_bfs on the device,
and validate_roundtrip with the reference's fault injections (R:tests/bvss_test.cpp:218-239)."""
import os

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
        out.append((name, rg, c, B.Graph.from_csr(c.n, c.offsets, c.targets, directed=True)))
    return out


def test_bvss_files_interchangeable(corpus, oracle, tmp_path):
    """Our save_bvss loads in the reference's load_bvss (same arrays) and the reference's file
    loads in ours; BFS over the loaded structure equals the reference BFS."""
    for name, rg, c, g in corpus:
        b = B.build_bvss(g)
        ours = str(tmp_path / f"{name}.ours.bvss")
        B.save_bvss(b, ours)
        rb = oracle.ref_load_bvss(ours)
        ra = rb.arrays(c.n)
        rp, v2r, rows, masks = b.arrays()
        assert np.array_equal(ra.real_ptrs, rp) and np.array_equal(ra.virtual_to_real, v2r)
        assert np.array_equal(ra.row_ids, rows) and np.array_equal(ra.masks, masks), name
        assert ra.num_unpadded_slices == b.num_unpadded_slices and ra.m == b.m
        theirs = str(tmp_path / f"{name}.ref.bvss")
        oracle.ref_save_bvss(rg.build_bvss(), theirs)
        with open(ours, "rb") as f1, open(theirs, "rb") as f2:
            assert f1.read() == f2.read(), name  # byte-identical files
        lb = B.load_bvss(theirs)
        assert (lb.n, lb.m, lb.num_vss, lb.num_unpadded_slices) == (b.n, b.m, b.num_vss, b.num_unpadded_slices)
        src = int(oracle.ref_rng_next_below(5, c.n, 1)[0])
        for fn in (B.run_eager, B.run_lazy):
            assert np.array_equal(fn(lb, src)[0].levels, rg.reference_bfs(src)[0]), name


def test_bvss_file_errors(corpus, tmp_path):
    """The reference's error classes: cannot open / bad magic / truncated / corrupt realPtrs
    -> RuntimeError (std::runtime_error)."""
    name, rg, c, g = corpus[4]
    path = str(tmp_path / "g.bvss")
    B.save_bvss(B.build_bvss(g), path)
    raw = open(path, "rb").read()
    with pytest.raises(RuntimeError, match="cannot open"):
        B.load_bvss(str(tmp_path / "absent.bvss"))
    bad = tmp_path / "bad.bvss"
    bad.write_bytes(b"XVSS" + raw[4:])
    with pytest.raises(RuntimeError, match="bad magic"):
        B.load_bvss(str(bad))
    bad.write_bytes(raw[: len(raw) - 8])
    with pytest.raises(RuntimeError, match="truncated"):
        B.load_bvss(str(bad))
    words = np.frombuffer(raw, np.uint32).copy()
    sets = (c.n + 7) // 8
    words[8 + sets] += 1  # realPtrs.back() != numVSS
    bad.write_bytes(words.tobytes())
    with pytest.raises(RuntimeError, match="corrupt realPtrs"):
        B.load_bvss(str(bad))


def test_permutation_files_interchangeable(oracle, tmp_path):
    for n, seed in ((1, 1), (1000, 3), (65536, 7)):
        f = oracle.ref_random_order(n, seed)
        p = str(tmp_path / f"{n}.perm")
        B.save_permutation(B.Permutation(f), p)
        assert np.array_equal(oracle.ref_load_permutation(p), f)
        q = str(tmp_path / f"{n}.ref.perm")
        oracle.ref_save_permutation(f, q)
        assert open(p).read() == open(q).read()
        assert np.array_equal(B.load_permutation(q).forward_map(), f)
    bad = tmp_path / "neg.perm"
    bad.write_text("0\n-1\n")
    with pytest.raises(B.ParseError) as e:
        B.load_permutation(str(bad))
    assert e.value.line == 2
    bad.write_text("0\n0\n")
    with pytest.raises(ValueError):
        B.load_permutation(str(bad))


def test_load_graph_matches_reference(oracle, tmp_path):
    cases = {
        "sym.mtx": "%%MatrixMarket matrix coordinate pattern symmetric\n% c\n5 5 4\n1 2\n2 3\n3 3\n5 1\n",
        "gen.mtx": "%%MatrixMarket matrix coordinate real general\n4 4 3\n1 2 0.5\n2 1 -1e3\n4 3 2\n",
        "int.mtx": "%%MatrixMarket matrix coordinate integer general\n3 3 2\n1 3 7\n\n3 1 -2\n",
        "snap.txt": "# Directed graph\n# Nodes: 10 Edges: 3\n0 1\n1 2\n\n9 0\n",
        "plain.txt": "0 5\n5 3\n3 3\n",
    }
    for fname, text in cases.items():
        path = tmp_path / fname
        path.write_text(text)
        g = B.load_graph(str(path))
        rg = oracle.ref_load_graph(str(path))
        rc = rg.csr()
        off, tgt = g.csr()
        assert g.num_vertices() == rg.n and np.array_equal(off, rc.offsets) and np.array_equal(tgt, rc.targets), fname
        assert g.digest() == rg.digest(), fname
    errors = {
        "banner.mtx": ("%%NotMarket matrix coordinate pattern general\n1 1 0\n", 1),
        "array.mtx": ("%%MatrixMarket matrix array real general\n1 1\n", 1),
        "nonsq.mtx": ("%%MatrixMarket matrix coordinate pattern general\n2 3 1\n1 1\n", 2),
        "oob.mtx": ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n3 1\n", 3),
        "trunc.mtx": ("%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n", 3),
        "extra.mtx": ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 2\n2 1\n", 4),
        "real.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 abc\n", 3),
        "tokens.txt": ("0 1 2\n", 1),
        "int.txt": ("0 x\n", 1),
        "declared.txt": ("# Nodes: 2\n0 5\n", 0),
    }
    for fname, (text, line) in errors.items():
        path = tmp_path / fname
        path.write_text(text)
        with pytest.raises(B.ParseError) as e:
            B.load_graph(str(path))
        with pytest.raises(oracle.RefError):
            oracle.ref_load_graph(str(path))
        assert e.value.line == line, (fname, str(e.value))
    neg = tmp_path / "neg.txt"
    neg.write_text("0 -1\n")
    with pytest.raises(ValueError):  # std::invalid_argument
        B.load_graph(str(neg))
    with pytest.raises(RuntimeError, match="cannot open"):
        B.load_graph(str(tmp_path / "absent.mtx"))


def test_digest_in_views_has_edge(corpus):
    for name, rg, c, g in corpus:
        assert g.digest() == rg.digest(), name
        ic = rg.csr(incoming=True)
        assert np.array_equal(g.in_offsets(), ic.offsets) and np.array_equal(g.in_sources(), ic.targets), name
        u = int(np.argmax(np.diff(c.offsets.astype(np.int64))))
        assert g.in_degree(u) == int(ic.offsets[u + 1] - ic.offsets[u])
        nb = g.out_neighbors(u)
        assert all(g.has_edge(u, int(v)) for v in nb)
        assert not g.has_edge(u, u)  # no self-loops


def test_reference_bfs_on_device(corpus, oracle):
    """reference_bfs (R:src/graph.cpp:144-167) straight over the CSR on the device."""
    for name, rg, c, g in corpus:
        for s in oracle.ref_rng_next_below(0xBF5, c.n, 4):
            r = B.reference_bfs(g, int(s))
            lv, vis, nl = rg.reference_bfs(int(s))
            assert np.array_equal(r.levels, lv) and r.visited_count == vis and r.num_levels == nl, name
    g = B.Graph.generate_rmat(18, 16, 4)
    off, tgt = g.csr()
    cs = oracle.Csr(g.num_vertices(), off, tgt)
    for s in g.pick_sources(3, 2):
        assert np.array_equal(B.reference_bfs(g, int(s)).levels, oracle.reference_bfs(cs, int(s))[0])
    with pytest.raises(ValueError):
        B.reference_bfs(g, g.num_vertices())


def test_validate_roundtrip_and_fault_injection(corpus, oracle, tmp_path):
    """ok on every corpus structure with the reference's checked-slice count; a flipped mask
    bit and corrupted padding are reported (R:tests/bvss_test.cpp:218-239)."""
    for name, rg, c, g in corpus:
        b = B.build_bvss(g)
        rep = B.validate_roundtrip(b, g)
        nd, checked = oracle.ref_validate_roundtrip(rg.build_bvss(), rg)
        assert rep.ok() and nd == 0 and rep.checked_slices == checked, (name, rep.discrepancies)
    name, rg, c, g = corpus[9]  # pa-10000
    b = B.build_bvss(g)
    rp, v2r, rows, masks = b.arrays()

    def loaded(m_words, tag):  # through a file: load_bvss checks only the header invariants
        path = str(tmp_path / f"{tag}.bvss")
        hdr = np.array([0x53535642, 1, 8, 128, c.n, c.m & 0xFFFFFFFF, c.m >> 32, len(v2r)], np.uint32)
        with open(path, "wb") as f:
            for a in (hdr, rp, v2r, rows, m_words):
                f.write(np.ascontiguousarray(a, np.uint32).tobytes())
        return B.load_bvss(path)

    assert B.validate_roundtrip(loaded(masks, "clean"), g).ok()
    m2 = masks.copy()
    m2[0] ^= 0x1  # flipped mask bit: row lists differ
    rep = B.validate_roundtrip(loaded(m2, "flip"), g)
    assert not rep.ok() and any("incoming list mismatch" in d for d in rep.discrepancies)
    k = int(np.flatnonzero(rows == c.n)[0])  # corrupted padding: a padded slot with a nonzero mask
    m3 = masks.copy()
    m3[k // 4] |= np.uint32(1 << (8 * (k % 4)))
    rep = B.validate_roundtrip(loaded(m3, "pad"), g)
    assert any("padded slot with nonzero mask" in d for d in rep.discrepancies)
