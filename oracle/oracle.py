"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle.

Two libraries, both checkers, never product code:

* ``oracle/_build/libblest_oracle.so`` — our plain-C restatement (blest_oracle.c), each
  function citing the reference file:line it follows.
* ``oracle/_ref/libblest_ref.so`` — the UNMODIFIED reference (/root/reference/proj)
  compiled from its own sources plus a C forwarder (ref_shim.cpp). Built here by
  ``make -C oracle ref``; travels to the GPU box as a prebuilt .so.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libblest_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libblest_ref.so")
INF = 0xFFFFFFFF

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_orc = None
_ref = None


def build(ref: bool = True) -> None:
    """Compile the oracle (and the reference when its sources are present)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        L.orc_hash64.restype = C.c_uint64
        L.orc_hash64.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_gen_rmat.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                   C.c_uint32, _u32p, _u32p]
        L.orc_gen_urand.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, _u32p, _u32p]
        L.orc_gen_grid.restype = C.c_uint64
        L.orc_gen_grid.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
        L.orc_random_relabel.argtypes = [C.c_uint32, C.c_uint64, _u32p]
        L.orc_from_edges.restype = C.c_uint64
        L.orc_from_edges.argtypes = [C.c_uint32, _u32p, _u32p, C.c_uint64, C.c_int, _u64p, _u32p]
        L.orc_apply_permutation.restype = C.c_uint64
        L.orc_apply_permutation.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, _u64p, _u32p]
        L.orc_reference_bfs.restype = C.c_uint32
        L.orc_reference_bfs.argtypes = [C.c_uint32, _u64p, _u32p, C.c_uint32, _u32p,
                                        C.POINTER(C.c_uint32)]
        L.orc_reference_bfs_many.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, C.c_uint32, _u32p,
                                             _u32p, C.c_int]
        L.orc_validate_levels.restype = C.c_uint64
        L.orc_validate_levels.argtypes = [C.c_uint32, _u64p, _u32p, C.c_uint32, _u32p]
        L.orc_bvss_count.restype = C.c_uint64
        L.orc_bvss_count.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, C.POINTER(C.c_uint64)]
        L.orc_bvss_fill.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, C.c_uint64, _u32p, _u32p,
                                    _u32p]
        L.orc_compression_ratio.restype = C.c_double
        L.orc_compression_ratio.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_update_divergence.restype = C.c_double
        L.orc_update_divergence.argtypes = [C.c_uint32, C.c_uint64, _u32p]
        L.orc_run_engine.restype = C.c_int64
        L.orc_run_engine.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _u32p, _u32p,
                                     C.c_uint32, C.c_int, C.c_uint32, C.c_uint32, _u32p, _u64p,
                                     C.c_uint64]
        L.orc_tile_pull.argtypes = [_u32p, C.c_uint8, C.c_uint, _u32p]
        vp = C.c_void_p
        L.orc_free.argtypes = [vp]
        L.orc_gen_csr.restype = C.c_uint64
        L.orc_gen_csr.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32,
                                  C.c_uint32, C.c_uint32, vp, C.c_int, C.POINTER(vp), C.POINTER(vp)]
        L.orc_random_relabel_mt.argtypes = [C.c_uint32, C.c_uint64, C.c_int, _u32p]
        L.orc_permute_csr.restype = C.c_uint64
        L.orc_permute_csr.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, C.c_int, _u64p, _u32p]
        L.orc_transpose_csr.restype = C.c_uint64
        L.orc_transpose_csr.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, _u32p]
        L.orc_symmetrise_csr.restype = C.c_uint64
        L.orc_symmetrise_csr.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, _u32p, _u64p, vp]
        L.orc_jaccard_windows.restype = C.c_int
        L.orc_jaccard_windows.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, _u32p, C.c_uint32,
                                          C.c_uint32, C.c_int, _u32p]
        L.orc_rcm.argtypes = [C.c_uint32, _u64p, _u32p, _u32p]
        L.orc_bvss_count_mt.restype = C.c_uint64
        L.orc_bvss_count_mt.argtypes = [C.c_uint32, _u64p, _u32p, C.c_int, _u32p, C.POINTER(C.c_uint64)]
        L.orc_bvss_fill_mt.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, C.c_int, _u32p, _u32p, _u32p]
        L.orc_traversed_edges.restype = C.c_uint64
        L.orc_traversed_edges.argtypes = [C.c_uint32, _u64p, _u32p]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build(ref=True)
        L = C.CDLL(REF_SO)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_graph_free.argtypes = [vp]
        L.ref_graph_from_edges.argtypes = [C.c_uint32, _u32p, _u32p, C.c_uint64, C.c_int,
                                           C.POINTER(vp)]
        L.ref_graph_from_csr.argtypes = [C.c_uint32, _u64p, _u32p, C.c_int, C.POINTER(vp)]
        L.ref_graph_n.restype = C.c_uint32
        L.ref_graph_n.argtypes = [vp]
        L.ref_graph_m.restype = C.c_uint64
        L.ref_graph_m.argtypes = [vp]
        L.ref_graph_digest.restype = C.c_uint64
        L.ref_graph_digest.argtypes = [vp]
        L.ref_graph_csr.argtypes = [vp, C.c_int, _u64p, _u32p]
        L.ref_reference_bfs.argtypes = [vp, C.c_uint32, _u32p, C.POINTER(C.c_uint32),
                                        C.POINTER(C.c_uint32)]
        L.ref_matrix_bfs.argtypes = [vp, C.c_uint32, _u32p]
        L.ref_apply_permutation.argtypes = [vp, _u32p, C.POINTER(vp)]
        L.ref_generate.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_double, C.c_uint64, C.POINTER(vp)]
        L.ref_scrambled.argtypes = [vp, C.c_uint64, C.POINTER(vp)]
        L.ref_rcm.argtypes = [vp, _u32p]
        L.ref_jaccard_windows.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint, _u32p]
        L.ref_naive_window_order.argtypes = [vp, C.c_uint32, C.c_uint32, _u32p]
        L.ref_random_order.argtypes = [C.c_uint32, C.c_uint64, _u32p]
        L.ref_bfs_locality_prepass.argtypes = [vp, _u32p]
        L.ref_is_cuthill_mckee_order.argtypes = [vp, _u32p, C.c_uint32]
        L.ref_classify.argtypes = [vp, _f64p, C.POINTER(C.c_int)]
        L.ref_bvss_free.argtypes = [vp]
        L.ref_build_bvss.argtypes = [vp, C.c_uint, C.POINTER(vp)]
        L.ref_bvss_from_arrays.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, _u32p, _u32p,
                                           _u32p, _u32p, C.POINTER(vp)]
        L.ref_bvss_sizes.argtypes = [vp, _u64p]
        L.ref_bvss_arrays.argtypes = [vp, _u32p, _u32p, _u32p, _u32p]
        L.ref_compression_ratio.restype = C.c_double
        L.ref_compression_ratio.argtypes = [vp]
        L.ref_update_divergence.restype = C.c_double
        L.ref_update_divergence.argtypes = [vp]
        L.ref_check_bvss_invariants.argtypes = [vp, vp]
        L.ref_run_engine.argtypes = [vp, C.c_uint32, C.c_int, C.c_uint, C.c_uint, C.c_uint32,
                                     C.c_void_p, _u64p, C.c_void_p, C.c_uint64,
                                     C.POINTER(C.c_uint64)]
        L.ref_init_state_queue.argtypes = [vp, C.c_uint32, _u32p, C.c_uint32,
                                           C.POINTER(C.c_uint32)]
        L.ref_tile_pull.argtypes = [_u32p, C.c_uint8, C.c_uint, _u32p]
        L.ref_rng_next_below.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.ref_save_bvss.argtypes = [vp, C.c_char_p]
        L.ref_load_bvss.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.ref_save_permutation.argtypes = [_u32p, C.c_uint32, C.c_char_p]
        L.ref_load_permutation.argtypes = [C.c_char_p, _u32p, C.c_uint32, C.POINTER(C.c_uint32)]
        L.ref_load_graph.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.ref_validate_roundtrip.argtypes = [vp, vp, C.POINTER(C.c_uint64)]
        _ref = L
    return _ref


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _chk(rc: int) -> None:
    if rc != 0:
        raise RefError(rc, ref().ref_last_error().decode())


# ----------------------------------------------------------------------------------
# Plain CSR graph container shared by tests (numpy arrays).
# ----------------------------------------------------------------------------------
@dataclass
class Csr:
    n: int
    offsets: np.ndarray  # uint64[n+1]
    targets: np.ndarray  # uint32[m]
    directed: bool = False

    @property
    def m(self) -> int:
        return int(self.offsets[-1]) if len(self.offsets) else 0

    def out_degree(self) -> np.ndarray:
        return np.diff(self.offsets).astype(np.uint64)


class RefGraph:
    """Handle on a reference blest::Graph (R:include/blest/graph.hpp:38-79)."""

    def __init__(self, ptr: int):
        self.ptr = C.c_void_p(ptr)

    def __del__(self):
        if _ref is not None and self.ptr:
            _ref.ref_graph_free(self.ptr)
            self.ptr = C.c_void_p(0)

    @property
    def n(self) -> int:
        return ref().ref_graph_n(self.ptr)

    @property
    def m(self) -> int:
        return ref().ref_graph_m(self.ptr)

    def digest(self) -> int:
        return ref().ref_graph_digest(self.ptr)

    def csr(self, incoming: bool = False) -> Csr:
        n, m = self.n, self.m
        off = np.zeros(n + 1, np.uint64)
        tgt = np.zeros(max(m, 1), np.uint32)
        ref().ref_graph_csr(self.ptr, 1 if incoming else 0, off, tgt)
        return Csr(n, off, tgt[:m].copy())

    # reference_bfs (R:src/graph.cpp:144-167)
    def reference_bfs(self, src: int):
        lv = np.zeros(self.n, np.uint32)
        vis, nl = C.c_uint32(), C.c_uint32()
        _chk(ref().ref_reference_bfs(self.ptr, src, lv, C.byref(vis), C.byref(nl)))
        return lv, vis.value, nl.value

    def matrix_bfs(self, src: int) -> np.ndarray:
        lv = np.zeros(self.n, np.uint32)
        _chk(ref().ref_matrix_bfs(self.ptr, src, lv))
        return lv

    def permuted(self, forward: np.ndarray) -> "RefGraph":
        out = C.c_void_p()
        _chk(ref().ref_apply_permutation(self.ptr, np.ascontiguousarray(forward, np.uint32),
                                         C.byref(out)))
        return RefGraph(out.value)

    def scrambled(self, seed: int) -> "RefGraph":
        out = C.c_void_p()
        _chk(ref().ref_scrambled(self.ptr, seed, C.byref(out)))
        return RefGraph(out.value)

    def rcm(self) -> np.ndarray:
        f = np.zeros(self.n, np.uint32)
        _chk(ref().ref_rcm(self.ptr, f))
        return f

    def jaccard_windows(self, w: int, sigma: int = 8, workers: int = 1) -> np.ndarray:
        f = np.zeros(self.n, np.uint32)
        _chk(ref().ref_jaccard_windows(self.ptr, sigma, w, workers, f))
        return f

    def naive_window_order(self, w: int, sigma: int = 8) -> np.ndarray:
        f = np.zeros(self.n, np.uint32)
        _chk(ref().ref_naive_window_order(self.ptr, sigma, w, f))
        return f

    def classify(self):
        out = np.zeros(4, np.float64)
        soc = C.c_int()
        _chk(ref().ref_classify(self.ptr, out, C.byref(soc)))
        return dict(top1_share=out[0], top10_share=out[1], power_law_slope=out[2],
                    power_law_fit_r2=out[3], is_social_like=bool(soc.value))

    def build_bvss(self, workers: int = 1) -> "RefBvss":
        out = C.c_void_p()
        _chk(ref().ref_build_bvss(self.ptr, workers, C.byref(out)))
        return RefBvss(out.value)


def ref_from_edges(n: int, src, dst, directed: bool = True) -> RefGraph:
    s = np.ascontiguousarray(src, np.uint32)
    d = np.ascontiguousarray(dst, np.uint32)
    out = C.c_void_p()
    _chk(ref().ref_graph_from_edges(n, s, d, len(s), 1 if directed else 0, C.byref(out)))
    return RefGraph(out.value)


def ref_from_csr(g: Csr) -> RefGraph:
    out = C.c_void_p()
    _chk(ref().ref_graph_from_csr(g.n, np.ascontiguousarray(g.offsets, np.uint64),
                                  np.ascontiguousarray(g.targets if g.m else np.zeros(1, np.uint32),
                                                       np.uint32),
                                  1, C.byref(out)))
    return RefGraph(out.value)


GEN_KINDS = {"path": 0, "ring": 1, "star": 2, "tree": 3, "grid": 4, "gnp": 5, "pa": 6,
             "rgg": 7, "planted": 8, "two_components": 9}


def ref_generate(kind: str, a: int = 0, b: int = 0, c: int = 0, d: int = 0, p: float = 0.0,
                 seed: int = 0) -> RefGraph:
    """The reference test corpus generators (R:tests/support/generators.cpp)."""
    out = C.c_void_p()
    _chk(ref().ref_generate(GEN_KINDS[kind], a, b, c, d, p, seed, C.byref(out)))
    return RefGraph(out.value)


def synthetic_corpus():
    """R:tests/support/generators.cpp:164-179 (the 12-graph acceptance corpus)."""
    return [
        ("path-1000", ref_generate("path", 1000)),
        ("ring-1024", ref_generate("ring", 1024)),
        ("star-1000", ref_generate("star", 1000)),
        ("tree-2047", ref_generate("tree", 2047)),
        ("grid-64x64", ref_generate("grid", 64, 64)),
        ("grid-100x100-scrambled", ref_generate("grid", 100, 100).scrambled(99)),
        ("gnp-1000", ref_generate("gnp", 1000, 0, p=0.004, seed=7)),
        ("gnp-dense-256", ref_generate("gnp", 256, 0, p=0.2, seed=11)),
        ("two-components-1500", ref_generate("two_components", seed=13)),
        ("pa-10000", ref_generate("pa", 10000, 3, seed=17)),
        ("rgg-10000", ref_generate("rgg", 10000, p=0.016, seed=19)),
        ("planted-32768", ref_generate("planted", 1 << 15, 128, 64, 2, seed=23)),
    ]


@dataclass
class BvssArrays:
    n: int
    m: int
    num_slice_sets: int
    num_vss: int
    num_unpadded_slices: int
    real_ptrs: np.ndarray
    virtual_to_real: np.ndarray
    row_ids: np.ndarray
    masks: np.ndarray


class RefBvss:
    """Handle on a reference blest::Bvss (R:include/blest/bvss.hpp:34-63)."""

    def __init__(self, ptr: int):
        self.ptr = C.c_void_p(ptr)

    def __del__(self):
        if _ref is not None and self.ptr:
            _ref.ref_bvss_free(self.ptr)
            self.ptr = C.c_void_p(0)

    def arrays(self, n: int) -> BvssArrays:
        sz = np.zeros(4, np.uint64)
        ref().ref_bvss_sizes(self.ptr, sz)
        sets, nv, unp, m = (int(x) for x in sz)
        rp = np.zeros(sets + 1, np.uint32)
        v2r = np.zeros(max(nv, 1), np.uint32)
        rows = np.zeros(max(nv * 128, 1), np.uint32)
        masks = np.zeros(max(nv * 32, 1), np.uint32)
        ref().ref_bvss_arrays(self.ptr, rp, v2r, rows, masks)
        return BvssArrays(n, m, sets, nv, unp, rp, v2r[:nv], rows[: nv * 128], masks[: nv * 32])

    def compression_ratio(self) -> float:
        return ref().ref_compression_ratio(self.ptr)

    def update_divergence(self) -> float:
        return ref().ref_update_divergence(self.ptr)

    def check_invariants(self, g: RefGraph) -> int:
        return ref().ref_check_bvss_invariants(self.ptr, g.ptr)

    def run(self, src: int, lazy: bool, warps: int = 4, workers: int = 1, max_levels: int = 0,
            want_levels: bool = True, n: int | None = None, trace_cap: int = 1 << 20):
        """run_eager / run_lazy (R:src/bfs_engine.cpp:155-350)."""
        ctr = np.zeros(10, np.uint64)
        lv = np.zeros(n, np.uint32) if (want_levels and n is not None) else None
        trace = np.zeros(8 * trace_cap, np.uint64)
        spread = C.c_uint64()
        _chk(ref().ref_run_engine(self.ptr, src, 1 if lazy else 0, warps, workers, max_levels,
                                  lv.ctypes.data if lv is not None else None, ctr,
                                  trace.ctypes.data, trace_cap, C.byref(spread)))
        tl = int(ctr[9])
        return EngineResult(levels=lv, counters=dict(
            mma_calls=int(ctr[0]), full_atomics=int(ctr[1]), relaxed_atomics=int(ctr[2]),
            queue_pushes=int(ctr[3]), vss_dequeues=int(ctr[4]),
            brs_baseline_mma_calls=int(ctr[5]), levels_processed=int(ctr[6]),
            visited_count=int(ctr[7]), num_levels=int(ctr[8])),
            trace=trace[: 8 * min(tl, trace_cap)].reshape(-1, 8).copy(),
            per_warp_spread=spread.value)


def ref_bvss_from_arrays(b: BvssArrays) -> RefBvss:
    out = C.c_void_p()

    def nz(a):
        a = np.ascontiguousarray(a, np.uint32)
        return a if len(a) else np.zeros(1, np.uint32)

    _chk(ref().ref_bvss_from_arrays(b.n, b.m, b.num_vss, nz(b.real_ptrs), nz(b.virtual_to_real),
                                    nz(b.row_ids), nz(b.masks), C.byref(out)))
    return RefBvss(out.value)


@dataclass
class EngineResult:
    levels: np.ndarray | None
    counters: dict
    trace: np.ndarray  # rows: level, queue_size, frontier_pop, discovered, full, stage1_full,
    #                        relaxed, pushes
    per_warp_spread: int = 0
    extra: dict = field(default_factory=dict)


def ref_rng_next_below(seed: int, bound: int, count: int) -> np.ndarray:
    out = np.zeros(count, np.uint64)
    ref().ref_rng_next_below(seed, bound, count, out)
    return out


def ref_random_order(n: int, seed: int) -> np.ndarray:
    f = np.zeros(n, np.uint32)
    _chk(ref().ref_random_order(n, seed, f))
    return f


def ref_tile_pull(mask_words, alpha: int, rnd: int) -> np.ndarray:
    c = np.zeros(64, np.uint32)
    _chk(ref().ref_tile_pull(np.ascontiguousarray(mask_words, np.uint32), alpha, rnd, c))
    return c


# ----------------------------------------------------------------------------------
# Our C restatement.
# ----------------------------------------------------------------------------------
RMAT_ABC = (2448131113, 816043786, 816043786)  # round(2^32 * .57/.19/.19); D = remainder


def gen_rmat(scale: int, edgefactor: int, seed: int, abc=RMAT_ABC):
    k = edgefactor << scale
    s = np.zeros(k, np.uint32)
    d = np.zeros(k, np.uint32)
    orc().orc_gen_rmat(scale, k, seed, abc[0], abc[1], abc[2], s, d)
    return s, d


def gen_urand(n: int, num_edges: int, seed: int):
    s = np.zeros(num_edges, np.uint32)
    d = np.zeros(num_edges, np.uint32)
    orc().orc_gen_urand(n, num_edges, seed, s, d)
    return s, d


def gen_grid(rows: int, cols: int):
    k = orc().orc_gen_grid(rows, cols, None, None)
    s = np.zeros(max(k, 1), np.uint32)
    d = np.zeros(max(k, 1), np.uint32)
    orc().orc_gen_grid(rows, cols, s.ctypes.data, d.ctypes.data)
    return s[:k], d[:k]


def random_relabel(n: int, seed: int) -> np.ndarray:
    f = np.zeros(n, np.uint32)
    orc().orc_random_relabel(n, seed, f)
    return f


def from_edges(n: int, src, dst, directed: bool = True) -> Csr:
    s = np.ascontiguousarray(src, np.uint32)
    d = np.ascontiguousarray(dst, np.uint32)
    off = np.zeros(n + 1, np.uint64)
    tgt = np.zeros(max((1 if directed else 2) * len(s), 1), np.uint32)
    m = orc().orc_from_edges(n, s, d, len(s), 1 if directed else 0, off, tgt)
    if m == 0xFFFFFFFFFFFFFFFF:
        raise ValueError("edge endpoint out of range")
    return Csr(n, off, tgt[:m].copy(), directed)


def apply_permutation(g: Csr, forward: np.ndarray) -> Csr:
    off = np.zeros(g.n + 1, np.uint64)
    tgt = np.zeros(max(g.m, 1), np.uint32)
    orc().orc_apply_permutation(g.n, g.offsets, _nz(g.targets), np.ascontiguousarray(forward, np.uint32),
                                off, tgt)
    return Csr(g.n, off, tgt[: g.m].copy(), g.directed)


def _nz(a):
    a = np.ascontiguousarray(a)
    return a if len(a) else np.zeros(1, a.dtype)


def reference_bfs(g: Csr, src: int):
    lv = np.zeros(g.n, np.uint32)
    nl = C.c_uint32()
    vis = orc().orc_reference_bfs(g.n, g.offsets, _nz(g.targets), src, lv, C.byref(nl))
    return lv, vis, nl.value


def reference_bfs_many(g: Csr, srcs, threads: int | None = None):
    srcs = np.ascontiguousarray(srcs, np.uint32)
    lv = np.zeros(len(srcs) * g.n, np.uint32)
    vis = np.zeros(len(srcs), np.uint32)
    orc().orc_reference_bfs_many(g.n, g.offsets, _nz(g.targets), srcs, len(srcs), lv, vis,
                                 threads or os.cpu_count() or 1)
    return lv.reshape(len(srcs), g.n), vis


def validate_levels(g: Csr, src: int, levels: np.ndarray) -> int:
    return int(orc().orc_validate_levels(g.n, g.offsets, _nz(g.targets), src,
                                         np.ascontiguousarray(levels, np.uint32)))


def build_bvss(g: Csr) -> BvssArrays:
    sets = (g.n + 7) // 8
    rp = np.zeros(sets + 1, np.uint32)
    unp = C.c_uint64()
    nv = orc().orc_bvss_count(g.n, g.offsets, _nz(g.targets), rp, C.byref(unp))
    v2r = np.zeros(max(nv, 1), np.uint32)
    rows = np.zeros(max(nv * 128, 1), np.uint32)
    masks = np.zeros(max(nv * 32, 1), np.uint32)
    orc().orc_bvss_fill(g.n, g.offsets, _nz(g.targets), rp, nv, v2r, rows, masks)
    return BvssArrays(g.n, g.m, sets, int(nv), unp.value, rp, v2r[:nv], rows[: nv * 128],
                      masks[: nv * 32])


def compression_ratio(b: BvssArrays) -> float:
    return orc().orc_compression_ratio(b.m, b.num_unpadded_slices)


def update_divergence(b: BvssArrays) -> float:
    return orc().orc_update_divergence(b.n, b.num_vss, _nz(b.row_ids))


class OracleError(Exception):
    pass


def run_engine(b: BvssArrays, src: int, lazy: bool, num_warps: int = 4, max_levels: int = 0,
               trace_cap: int = 1 << 20) -> EngineResult:
    lv = np.zeros(b.n, np.uint32)
    trace = np.zeros(8 * trace_cap, np.uint64)
    r = orc().orc_run_engine(b.n, b.real_ptrs, b.num_vss, _nz(b.virtual_to_real), _nz(b.row_ids),
                             _nz(b.masks), src, 1 if lazy else 0, num_warps, max_levels, lv,
                             trace, trace_cap)
    if r == -1:
        raise OracleError("BFS ran past the level safety cap")
    if r < 0:
        raise OracleError(f"oracle engine status {r}")
    tr = trace[: 8 * r].reshape(-1, 8).copy()
    d = int(tr[:, 1].sum()) if r else 0
    reached = lv != INF
    ml = int(lv[reached].max()) if reached.any() else 0
    return EngineResult(levels=lv, counters=dict(
        mma_calls=2 * d, vss_dequeues=d, brs_baseline_mma_calls=16 * d,
        queue_pushes=int(tr[:, 7].sum()) if r else 0, full_atomics=int(tr[:, 4].sum()) if r else 0,
        relaxed_atomics=int(tr[:, 6].sum()) if r else 0, levels_processed=ml,
        visited_count=int(reached.sum()), num_levels=ml + 1), trace=tr)


def tile_pull(mask_words, alpha: int, rnd: int) -> np.ndarray:
    c = np.zeros(64, np.uint32)
    orc().orc_tile_pull(np.ascontiguousarray(mask_words, np.uint32), alpha, rnd, c)
    return c


def pick_sources(g: Csr, count: int, seed: int) -> np.ndarray:
    """Seeded sources as the CLI draws them (Rng(seed).next_below(n), R:tools/blest.cpp:201-203),
    rejecting zero-out-degree vertices (Graph500 rule). Uses the reference
    mt19937_64 stream when available, else a splitmix stream (documented in DESIGN.md)."""
    deg = np.diff(g.offsets)
    out = []
    if ref_available():
        draws = ref_rng_next_below(seed, g.n, max(64, count * 64))
        for x in draws:
            if deg[int(x)] > 0:
                out.append(int(x))
                if len(out) == count:
                    break
    i = 0
    while len(out) < count:
        x = orc().orc_hash64(seed, i) % g.n
        i += 1
        if deg[x] > 0:
            out.append(int(x))
    return np.array(out, np.uint32)


# ----------------------------------------------------------------------------------
# Full scale (blest_oracle_scale.c): multi-threaded builders and orderings, same results.
# ----------------------------------------------------------------------------------
def _threads(threads):
    return int(threads or os.cpu_count() or 1)


class _COwned:
    """Keeps a malloc'd C buffer alive for the numpy view built on it."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr and _orc is not None:
            _orc.orc_free(self.ptr)
            self.ptr = None


def _adopt(ptr, count: int, ctype, dtype) -> np.ndarray:
    if count == 0:
        orc().orc_free(ptr)
        return np.zeros(0, dtype)
    arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(count,)).view(dtype)
    return _OwnedArray(arr, _COwned(ptr))  # views of it keep it (and the C buffer) alive


class _OwnedArray(np.ndarray):
    def __new__(cls, a, holder):
        obj = np.asarray(a).view(cls)
        obj._holder = holder
        return obj

    def __array_finalize__(self, obj):
        if obj is not None:
            self._holder = getattr(obj, "_holder", None)


GEN_CSR_KINDS = {"rmat": 0, "urand": 1, "grid": 2}


def gen_csr(kind: str, a: int, b: int = 0, k: int = 0, seed: int = 0, forward=None, abc=RMAT_ABC,
            threads: int | None = None) -> Csr:
    """Generator twin -> optional relabel (forward map) -> Graph::from_edges(undirected), built
    without the mirrored arc list: kind rmat (a = scale, k edges), urand (a = n, k edges),
    grid (a = rows, b = cols). Equal to from_edges(n, *gen_*(...)) permuted by `forward`."""
    n = (1 << a) if kind == "rmat" else (a if kind == "urand" else a * b)
    offp, tgtp = C.c_void_p(), C.c_void_p()
    fw = None if forward is None else np.ascontiguousarray(forward, np.uint32)
    m = orc().orc_gen_csr(GEN_CSR_KINDS[kind], a, b, k, seed, abc[0], abc[1], abc[2],
                          fw.ctypes.data if fw is not None else None, _threads(threads),
                          C.byref(offp), C.byref(tgtp))
    off = _adopt(offp.value, n + 1, C.c_uint64, np.uint64)
    tgt = _adopt(tgtp.value, m, C.c_uint32, np.uint32)
    return Csr(n, off, tgt, False)


def random_relabel_mt(n: int, seed: int, threads: int | None = None) -> np.ndarray:
    f = np.zeros(n, np.uint32)
    orc().orc_random_relabel_mt(n, seed, _threads(threads), f)
    return f


def permute_csr(g: Csr, forward, threads: int | None = None) -> Csr:
    """apply_permutation (R:src/graph.cpp:126-134), multi-threaded."""
    off = np.zeros(g.n + 1, np.uint64)
    tgt = np.zeros(max(g.m, 1), np.uint32)
    orc().orc_permute_csr(g.n, g.offsets, _nz(g.targets), np.ascontiguousarray(forward, np.uint32),
                          _threads(threads), off, tgt)
    return Csr(g.n, off, tgt[: g.m], g.directed)


def transpose_csr(g: Csr) -> Csr:
    off = np.zeros(g.n + 1, np.uint64)
    src = np.zeros(max(g.m, 1), np.uint32)
    orc().orc_transpose_csr(g.n, g.offsets, _nz(g.targets), off, src)
    return Csr(g.n, off, src[: g.m], g.directed)


def in_view(g: Csr) -> Csr:
    """The in-view: the graph itself when undirected (its arc set is symmetric)."""
    return g if not g.directed else transpose_csr(g)


def jaccard_windows(g: Csr, w: int, sigma: int = 8, threads: int | None = None) -> np.ndarray:
    """jaccard_with_windows (R:src/ordering.cpp:139-166), windows over host threads."""
    gi = in_view(g)
    f = np.zeros(max(g.n, 1), np.uint32)
    rc = orc().orc_jaccard_windows(g.n, g.offsets, _nz(g.targets), gi.offsets, _nz(gi.targets), sigma, w,
                                   _threads(threads), f)
    if rc != 0:
        raise ValueError("window size must be a positive multiple of sigma (sigma <= 8)")
    return f[: g.n]


def symmetrised(g: Csr) -> Csr:
    """symmetrised_adjacency (R:src/ordering.cpp:171-182) as a CSR."""
    if not g.directed:
        return g
    gi = transpose_csr(g)
    off = np.zeros(g.n + 1, np.uint64)
    m = orc().orc_symmetrise_csr(g.n, g.offsets, _nz(g.targets), gi.offsets, _nz(gi.targets), off, None)
    tgt = np.zeros(max(m, 1), np.uint32)
    orc().orc_symmetrise_csr(g.n, g.offsets, _nz(g.targets), gi.offsets, _nz(gi.targets), off, tgt.ctypes.data)
    return Csr(g.n, off, tgt[:m], False)


def rcm(g: Csr) -> np.ndarray:
    """rcm (R:src/ordering.cpp:246-266): forward map."""
    a = symmetrised(g)
    f = np.zeros(max(g.n, 1), np.uint32)
    orc().orc_rcm(g.n, a.offsets, _nz(a.targets), f)
    return f[: g.n]


def build_bvss_mt(g: Csr, threads: int | None = None) -> BvssArrays:
    """build_bvss (R:src/bvss.cpp:19-101) with slice sets over host threads."""
    t = _threads(threads)
    sets = (g.n + 7) // 8
    rp = np.zeros(sets + 1, np.uint32)
    unp = C.c_uint64()
    nv = orc().orc_bvss_count_mt(g.n, g.offsets, _nz(g.targets), t, rp, C.byref(unp))
    v2r = np.empty(max(nv, 1), np.uint32)
    rows = np.empty(max(nv * 128, 1), np.uint32)
    masks = np.empty(max(nv * 32, 1), np.uint32)
    orc().orc_bvss_fill_mt(g.n, g.offsets, _nz(g.targets), rp, t, v2r, rows, masks)
    return BvssArrays(g.n, g.m, sets, int(nv), unp.value, rp, v2r[:nv], rows[: nv * 128], masks[: nv * 32])


def traversed_edges(g: Csr, levels: np.ndarray) -> int:
    """1/2 * sum of the reached vertices' out-degrees."""
    return int(orc().orc_traversed_edges(g.n, g.offsets, np.ascontiguousarray(levels, np.uint32)))


def classify(g: Csr) -> dict:
    """classify_social_like(g, DegreeSide::Out) (R:src/ordering.cpp:346-387) with its log-log
    fit (fit_log_log :315-342): same operation order, so the doubles are bit-identical."""
    import math
    n = g.n
    deg = np.diff(g.offsets.astype(np.int64))
    total = int(deg.sum())
    rep = dict(top1_share=0.0, top10_share=0.0, power_law_slope=0.0, power_law_fit_r2=0.0,
               is_social_like=False)
    if n == 0 or total == 0:
        return rep
    srt = np.sort(deg)[::-1]
    pref = np.cumsum(srt)

    def share(percent):
        count = int(math.floor(n * percent / 100.0 + 1e-9))
        count = min(max(count, 1), n)
        return float(int(pref[count - 1])) / float(total)

    rep["top1_share"] = share(1.0)
    rep["top10_share"] = share(10.0)
    heavy = rep["top1_share"] > 0.05 and rep["top10_share"] > 0.40
    values, counts = np.unique(deg, return_counts=True)  # std::map order: ascending degree
    pts = [(math.log2(float(d)), math.log2(float(f))) for d, f in zip(values.tolist(), counts.tolist())
           if d >= 2 and f >= 1]
    slope = r2 = 0.0
    if len(pts) >= 3:
        sx = sy = 0.0
        for x, y in pts:
            sx += x
            sy += y
        mx, my = sx / len(pts), sy / len(pts)
        sxx = sxy = syy = 0.0
        for x, y in pts:
            sxx += (x - mx) * (x - mx)
            sxy += (x - mx) * (y - my)
            syy += (y - my) * (y - my)
        if sxx != 0:
            slope = sxy / sxx
            ss_res = syy - slope * sxy
            r2 = (1.0 if abs(ss_res) < 1e-12 else 0.0) if syy == 0 else min(max(1.0 - ss_res / syy, 0.0), 1.0)
    rep["power_law_slope"], rep["power_law_fit_r2"] = slope, r2
    power = len(pts) >= 3 and -3.5 <= slope <= -1.5 and r2 >= 0.8
    rep["is_social_like"] = bool(heavy or power)
    return rep


# ---- the reference's file formats (R:src/bvss.cpp:218-295, R:src/graph.cpp:233-417) ----
def ref_save_bvss(b: "RefBvss", path: str) -> None:
    _chk(ref().ref_save_bvss(b.ptr, os.fsencode(path)))


def ref_load_bvss(path: str) -> "RefBvss":
    out = C.c_void_p()
    _chk(ref().ref_load_bvss(os.fsencode(path), C.byref(out)))
    return RefBvss(out.value)


def ref_save_permutation(forward, path: str) -> None:
    f = np.ascontiguousarray(forward, np.uint32)
    _chk(ref().ref_save_permutation(f if len(f) else np.zeros(1, np.uint32), len(f), os.fsencode(path)))


def ref_load_permutation(path: str, cap: int = 1 << 24) -> np.ndarray:
    f = np.zeros(cap, np.uint32)
    n = C.c_uint32()
    _chk(ref().ref_load_permutation(os.fsencode(path), f, cap, C.byref(n)))
    return f[: n.value].copy()


def ref_load_graph(path: str) -> RefGraph:
    out = C.c_void_p()
    _chk(ref().ref_load_graph(os.fsencode(path), C.byref(out)))
    return RefGraph(out.value)


def ref_validate_roundtrip(b: "RefBvss", g: RefGraph):
    """(#discrepancies, checked_slices) of the reference's validate_roundtrip."""
    checked = C.c_uint64()
    r = ref().ref_validate_roundtrip(b.ptr, g.ptr, C.byref(checked))
    if r < 0:
        raise RefError(r, ref().ref_last_error().decode())
    return r, checked.value
