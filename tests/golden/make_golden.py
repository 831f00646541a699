"""Generate the committed golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/*.npz. Every expected value comes from a reference call; the cited
reference test is the one whose known answer the fixture re-expresses.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def engine_graphs():
    """R:tests/bfs_engine_test.cpp:163-175 (the 9-family equivalence list)."""
    g = O.ref_generate
    return [
        ("path-300", g("path", 300)),
        ("star-257", g("star", 257)),
        ("tree-511", g("tree", 511)),
        ("grid-18x20-scrambled-40", g("grid", 18, 20).scrambled(40)),
        ("gnp-400-directed", g("gnp", 400, 1, p=0.008, seed=41)),
        ("gnp-300", g("gnp", 300, 0, p=0.02, seed=42)),
        ("two-components-43", g("two_components", seed=43)),
        ("pa-1000", g("pa", 1000, 3, seed=44)),
        ("planted-2048", g("planted", 2048, 32, 16, 2, seed=45)),
    ]


def main():
    O.build()
    # ---- tile KATs (R:tests/tc_emu_test.cpp:186-241) ----
    masks = np.zeros(32, np.uint32)
    masks[0] = 0x4A
    worked = O.ref_tile_pull(masks, 0x03, 0)
    rng = np.random.default_rng(6)
    rnd_masks = rng.integers(0, 2**32, size=(64, 32), dtype=np.uint64).astype(np.uint32)
    rnd_alpha = rng.integers(0, 256, size=64).astype(np.uint8)
    rnd_c = np.stack([np.stack([O.ref_tile_pull(rnd_masks[i], int(rnd_alpha[i]), r) for r in (0, 1)])
                      for i in range(64)])
    np.savez_compressed(os.path.join(OUT, "tile.npz"), worked=worked, masks=rnd_masks,
                        alpha=rnd_alpha, counts=rnd_c)

    # ---- BVSS KATs (R:tests/bvss_test.cpp:39-93) ----
    kats = {}
    cases = {
        "worked-0x4A": (24, [(17, 3), (19, 3), (22, 3)]),
        "97-slices": (105, [(0, r) for r in range(8, 105)]),
        "130-slices": (140, [(0, r) for r in range(8, 138)]),
        "300-slice-set": (400, [(0, r) for r in range(8, 308)]),
        "worked-pull-384": (384, [(17, 3), (19, 3), (22, 3)] + [(0, r) for r in range(64, 322)]),
        "diamond": (5, [(0, 1), (0, 2), (1, 3), (2, 3), (3, 4)]),
        "chain-3": (3, [(0, 1), (1, 2)]),
        "edgeless-20": (20, []),
    }
    for name, (n, edges) in cases.items():
        e = np.array(edges, np.uint32).reshape(-1, 2)
        rg = O.ref_from_edges(n, e[:, 0], e[:, 1], directed=True)
        b = rg.build_bvss().arrays(n)
        kats[name + "/n"] = np.array([n], np.uint32)
        kats[name + "/edges"] = e
        kats[name + "/real_ptrs"] = b.real_ptrs
        kats[name + "/v2r"] = b.virtual_to_real
        kats[name + "/row_ids"] = b.row_ids
        kats[name + "/masks"] = b.masks
    np.savez_compressed(os.path.join(OUT, "bvss_kats.npz"), **kats)

    # ---- engine families (R:tests/bfs_engine_test.cpp:163-203) ----
    fam = {}
    names = []
    draw = O.ref_rng_next_below  # Rng(46) draws, as the test does per graph
    rng46_seq = []
    for name, rg in engine_graphs():
        names.append(name)
        g = rg.csr()
        rb = rg.build_bvss()
        b = rb.arrays(g.n)
        fam[name + "/n"] = np.array([g.n], np.uint32)
        fam[name + "/offsets"] = g.offsets
        fam[name + "/targets"] = g.targets
        fam[name + "/bvss_sha"] = np.frombuffer(
            bytes.fromhex(sha(b.real_ptrs, b.virtual_to_real, b.row_ids, b.masks)), np.uint8)
        fam[name + "/compression"] = np.array([rb.compression_ratio()])
        fam[name + "/divergence"] = np.array([rb.update_divergence()])
        srcs = [0, g.n - 1]
        srcs.append(int(draw(46, g.n, 1)[0]))  # first draw of a fresh Rng(46) for this size
        fam[name + "/sources"] = np.array(srcs, np.uint32)
        for i, s in enumerate(srcs):
            lv, vis, nl = rg.reference_bfs(s)
            fam[f"{name}/levels{i}"] = lv
            for lazy in (0, 1):
                r = rb.run(s, bool(lazy), warps=4, n=g.n)
                assert np.array_equal(r.levels, lv)
                fam[f"{name}/trace{i}_{lazy}"] = r.trace
    fam["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "engine_families.npz"), **fam)

    # ---- acceptance corpus digests + levels (R:tests/acceptance_main.cpp:140-274) ----
    acc = {}
    for name, rg in O.synthetic_corpus():
        g = rg.csr()
        acc[name + "/digest"] = np.array([rg.digest()], np.uint64)
        acc[name + "/graph_sha"] = np.frombuffer(bytes.fromhex(sha(g.offsets, g.targets)), np.uint8)
        rb = rg.build_bvss()
        b = rb.arrays(g.n)
        acc[name + "/bvss_sha"] = np.frombuffer(
            bytes.fromhex(sha(b.real_ptrs, b.virtual_to_real, b.row_ids, b.masks)), np.uint8)
        srcs = O.ref_rng_next_below(0xACCE5500, g.n, 4).astype(np.uint32)
        acc[name + "/sources"] = srcs
        acc[name + "/levels_sha"] = np.stack([
            np.frombuffer(bytes.fromhex(sha(rg.reference_bfs(int(s))[0])), np.uint8) for s in srcs])
        acc[name + "/classify"] = np.array(list(rg.classify().values())[:4])
        acc[name + "/social"] = np.array([rg.classify()["is_social_like"]])
        acc[name + "/rcm"] = rg.rcm()
        if g.n <= 12000:
            acc[name + "/jaccard_w256"] = rg.jaccard_windows(256)
    np.savez_compressed(os.path.join(OUT, "corpus.npz"), **acc)

    # ---- harness generators pinned through the reference (C1 shape at small scale) ----
    gen = {}
    for scale in (8, 10, 12):
        s, d = O.gen_rmat(scale, 16, 1)
        rg = O.ref_from_edges(1 << scale, s, d, directed=False)
        g = rg.csr()
        gen[f"rmat{scale}/edges_sha"] = np.frombuffer(bytes.fromhex(sha(s, d)), np.uint8)
        gen[f"rmat{scale}/graph_sha"] = np.frombuffer(bytes.fromhex(sha(g.offsets, g.targets)), np.uint8)
        gen[f"rmat{scale}/m"] = np.array([g.m], np.uint64)
        srcs = O.pick_sources(g, 4, 1)
        gen[f"rmat{scale}/sources"] = srcs
        gen[f"rmat{scale}/levels"] = np.stack([rg.reference_bfs(int(x))[0] for x in srcs])
    s, d = O.gen_urand(1000, 16000, 3)
    gen["urand1000/edges_sha"] = np.frombuffer(bytes.fromhex(sha(s, d)), np.uint8)
    gen["relabel1000"] = O.random_relabel(1000, 7)
    np.savez_compressed(os.path.join(OUT, "generators.npz"), **gen)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
