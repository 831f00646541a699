"""Python mirror of the reference's C++ API for the hot path (R = /root/reference/proj):

    graph load   Graph.from_edges / Graph.from_csr /      R:include/blest/graph.hpp:38-79, :150
                 load_graph, Graph.digest / in_* views,
                 reference_bfs (device, over the CSR)     R:include/blest/graph.hpp:119
    reorder      select_plan / make_permutation / rcm /   R:include/blest/ordering.hpp:12-83
                 jaccard_with_windows / apply_permutation
    BVSS build   build_bvss / bvss_stats / save_bvss /    R:include/blest/bvss.hpp:16-111
                 load_bvss / validate_roundtrip,
                 save_permutation / load_permutation      R:src/graph.cpp:396-417
    bfs(source)  run_eager / run_lazy / run_auto_prebuilt  R:include/blest/bfs_engine.hpp:14-101
                 / run_auto

Same names, argument meaning and error behaviour (ValueError for the reference's
std::invalid_argument, RuntimeError for std::runtime_error, BlestLogicError for
std::logic_error). Every call goes through the C-ABI of libblest_b200.so; there is no
CPU path for any compute step.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

KUNREACHED = 0xFFFFFFFF
RMAT_ABC = (2448131113, 816043786, 816043786)  # Graph500 .57/.19/.19 scaled by 2^32


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a is not None and a.size else 0


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


# ------------------------------------------------------------------------------------
# Graph (R:include/blest/graph.hpp)
# ------------------------------------------------------------------------------------
class Graph:
    """Device-resident CSR out-view; blest::Graph for the hot path."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        n, m, d = C.c_uint32(), C.c_uint64(), C.c_int()
        L.check(L.lib().blest_graph_info(self._h, C.byref(n), C.byref(m), C.byref(d)))
        self._n, self._m, self._directed = n.value, m.value, bool(d.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and L._lib is not None:
            L._lib.blest_graph_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # Graph::from_edges (R:src/graph.cpp:33-55)
    @staticmethod
    def from_edges(n: int, edges, directed: bool = True) -> "Graph":
        if isinstance(edges, tuple) and len(edges) == 2:
            src, dst = _u32(edges[0]), _u32(edges[1])
        else:
            e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
            if (e < 0).any():
                raise ValueError("negative vertex id")
            src, dst = _u32(e[:, 0]), _u32(e[:, 1])
        out = C.c_void_p()
        L.check(L.lib().blest_graph_from_edges(n, _ptr(src), _ptr(dst), len(src), int(directed), 1,
                                               C.byref(out)))
        return Graph(out.value)

    @staticmethod
    def from_csr(n: int, offsets, targets, directed: bool = True) -> "Graph":
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        tgt = _u32(targets)
        out = C.c_void_p()
        L.check(L.lib().blest_graph_from_csr(n, _ptr(off), _ptr(tgt), int(directed), 1, C.byref(out)))
        return Graph(out.value)

    @staticmethod
    def generate_rmat(scale: int, edgefactor: int = 16, seed: int = 1, abc=RMAT_ABC) -> "Graph":
        out = C.c_void_p()
        L.check(L.lib().blest_graph_generate(0, scale, 0, edgefactor << scale, seed, abc[0], abc[1],
                                             abc[2], C.byref(out)))
        return Graph(out.value)

    @staticmethod
    def generate_urand(n: int, num_edges: int, seed: int = 1) -> "Graph":
        out = C.c_void_p()
        L.check(L.lib().blest_graph_generate(1, n, 0, num_edges, seed, 0, 0, 0, C.byref(out)))
        return Graph(out.value)

    @staticmethod
    def generate_grid(rows: int, cols: int) -> "Graph":
        out = C.c_void_p()
        L.check(L.lib().blest_graph_generate(2, rows, cols, 0, 0, 0, 0, 0, C.byref(out)))
        return Graph(out.value)

    def num_vertices(self) -> int:
        return self._n

    def num_edges(self) -> int:
        return self._m

    def directed(self) -> bool:
        return self._directed

    def csr(self):
        off = np.zeros(self._n + 1, np.uint64)
        tgt = np.zeros(max(self._m, 1), np.uint32)
        L.check(L.lib().blest_graph_copy_csr(self._h, _ptr(off), _ptr(tgt)))
        return off, tgt[: self._m]

    def out_offsets(self) -> np.ndarray:
        return self.csr()[0]

    def out_targets(self) -> np.ndarray:
        return self.csr()[1]

    def out_degrees(self) -> np.ndarray:
        d = np.zeros(max(self._n, 1), np.uint32)
        L.check(L.lib().blest_graph_out_degrees(self._h, _ptr(d), 1))
        return d[: self._n]

    def device_csr(self):
        o, t = C.c_void_p(), C.c_void_p()
        L.check(L.lib().blest_graph_device_csr(self._h, C.byref(o), C.byref(t)))
        return o.value, t.value

    def traversed_edges(self, levels_device_ptr: int) -> int:
        e = C.c_uint64()
        L.check(L.lib().blest_graph_traversed_edges(self._h, levels_device_ptr, C.byref(e)))
        return e.value

    # the incoming view (R:include/blest/graph.hpp:54-68): transposed on the device, cached
    def in_csr(self):
        if getattr(self, "_in", None) is None:
            off = np.zeros(self._n + 1, np.uint64)
            src = np.zeros(max(self._m, 1), np.uint32)
            L.check(L.lib().blest_graph_copy_in_csr(self._h, _ptr(off), _ptr(src)))
            self._in = (off, src[: self._m])
        return self._in

    def in_offsets(self) -> np.ndarray:
        return self.in_csr()[0]

    def in_sources(self) -> np.ndarray:
        return self.in_csr()[1]

    def in_neighbors(self, v: int) -> np.ndarray:
        off, src = self.in_csr()
        return src[int(off[v]): int(off[v + 1])]

    def in_degree(self, v: int) -> int:
        off = self.in_csr()[0]
        return int(off[v + 1] - off[v])

    def out_neighbors(self, u: int) -> np.ndarray:
        off, tgt = self._host_csr()
        return tgt[int(off[u]): int(off[u + 1])]

    def out_degree(self, u: int) -> int:
        off = self._host_csr()[0]
        return int(off[u + 1] - off[u])

    def has_edge(self, u: int, v: int) -> bool:
        """Graph::has_edge (R:src/graph.cpp:57-60): binary search in u's sorted out-list."""
        nb = self.out_neighbors(u)
        i = int(np.searchsorted(nb, v))
        return i < len(nb) and int(nb[i]) == v

    def _host_csr(self):
        if getattr(self, "_out", None) is None:
            self._out = self.csr()
        return self._out

    def digest(self) -> int:
        """Graph::digest (R:src/graph.cpp:62-75): FNV-1a over (n, m, arcs), the cache key."""
        d = C.c_uint64()
        L.check(L.lib().blest_graph_digest(self._h, C.byref(d)))
        return d.value

    def pick_sources(self, count: int, seed: int, skip_isolated: bool = True) -> np.ndarray:
        out = np.zeros(max(count, 1), np.uint32)
        L.check(L.lib().blest_pick_sources(self._h, count, seed, int(skip_isolated), _ptr(out)))
        return out[:count]


# ------------------------------------------------------------------------------------
# Permutation (R:include/blest/graph.hpp:81-103)
# ------------------------------------------------------------------------------------
class Permutation:
    def __init__(self, forward: np.ndarray):
        f = _u32(forward)
        n = len(f)
        if n and f.max() >= n:
            raise ValueError("permutation is not a bijection on [0, n)")
        inv = np.full(n, n, dtype=np.uint32)  # O(n) bijection check (np.unique sorts: ~7 s at 2^24)
        inv[f] = np.arange(n, dtype=np.uint32)
        if n and (inv == n).any():
            raise ValueError("permutation is not a bijection on [0, n)")
        self._fwd = f
        self._inv = inv

    @classmethod
    def _trusted(cls, forward: np.ndarray) -> "Permutation":
        """A forward map the library produced (a bijection by construction): no re-check."""
        p = cls.__new__(cls)
        p._fwd = _u32(forward)
        p._inv = np.empty_like(p._fwd)
        p._inv[p._fwd] = np.arange(len(p._fwd), dtype=np.uint32)
        return p

    @staticmethod
    def identity(n: int) -> "Permutation":
        return Permutation(np.arange(n, dtype=np.uint32))

    @staticmethod
    def from_forward(forward) -> "Permutation":
        return Permutation(forward)

    @staticmethod
    def from_inverse(inverse) -> "Permutation":
        inv = _u32(inverse)
        f = np.empty_like(inv)
        f[inv] = np.arange(len(inv), dtype=np.uint32)
        return Permutation(f)

    def size(self) -> int:
        return len(self._fwd)

    def forward(self, old_id: int) -> int:
        return int(self._fwd[old_id])

    def inverse(self, new_id: int) -> int:
        return int(self._inv[new_id])

    def forward_map(self) -> np.ndarray:
        return self._fwd

    def inverse_map(self) -> np.ndarray:
        return self._inv

    def inverted(self) -> "Permutation":
        return Permutation(self._inv)

    @staticmethod
    def composed(first: "Permutation", second: "Permutation") -> "Permutation":
        if first.size() != second.size():
            raise ValueError("cannot compose permutations of different sizes")
        return Permutation(second._fwd[first._fwd])

    def is_identity(self) -> bool:
        return bool(np.array_equal(self._fwd, np.arange(len(self._fwd), dtype=np.uint32)))


def apply_permutation(g: Graph, perm: Permutation) -> Graph:
    """apply_permutation (R:src/graph.cpp:126-134) on the GPU."""
    if perm.size() != g.num_vertices():
        raise ValueError("permutation size does not match vertex count")
    out = C.c_void_p()
    f = perm.forward_map()
    L.check(L.lib().blest_graph_apply_permutation(g.handle, _ptr(f), 1, C.byref(out)))
    return Graph(out.value)


def relabel_permutation(n: int, seed: int) -> Permutation:
    """Harness relabel (GAP-style): rank of splitmix64(seed, i)."""
    f = np.zeros(max(n, 1), np.uint32)
    L.check(L.lib().blest_relabel_permutation(n, seed, _ptr(f), 1))
    return Permutation(f[:n])


# ------------------------------------------------------------------------------------
# Ordering (R:include/blest/ordering.hpp)
# ------------------------------------------------------------------------------------
class OrderingStrategy(enum.Enum):
    JaccardWindows = "jaccard-windows"
    Rcm = "rcm"
    Random = "random"
    Identity = "identity"


class PrePass(enum.Enum):
    None_ = "none"
    BfsLocality = "bfs-locality"


def ordering_strategy_from_string(s: str) -> OrderingStrategy:
    for x in OrderingStrategy:
        if x.value == s:
            return x
    raise ValueError("unknown ordering strategy: " + s)


@dataclass
class SocialLikeReport:
    top1_share: float = 0.0
    top10_share: float = 0.0
    power_law_slope: float = 0.0
    power_law_fit_r2: float = 0.0
    is_social_like: bool = False
    triggered_rules: list = field(default_factory=list)


@dataclass
class OrderingPlan:
    strategy: OrderingStrategy = OrderingStrategy.Identity
    window_size: int = 0
    pre_pass: PrePass = PrePass.None_
    classification: SocialLikeReport = field(default_factory=SocialLikeReport)


@dataclass
class SelectDefaults:
    window_size: int = 1 << 16
    pre_pass: PrePass = PrePass.None_
    force: Optional[OrderingStrategy] = None


def classify_social_like(g: Graph) -> SocialLikeReport:
    """classify_social_like(g, DegreeSide::Out) (R:src/ordering.cpp:346-387)."""
    r = L.SocialReportT()
    L.check(L.lib().blest_classify_social_like(g.handle, C.byref(r)))
    rules = (["heavy-tail"] if r.heavy_tail_fired else []) + (["power-law"] if r.power_law_fired else [])
    return SocialLikeReport(r.top1_share, r.top10_share, r.power_law_slope, r.power_law_fit_r2,
                            bool(r.is_social_like), rules)


def select_plan(g: Graph, sigma: int = 8, defaults: SelectDefaults | None = None) -> OrderingPlan:
    """select_plan (R:src/ordering.cpp:389-405)."""
    defaults = defaults or SelectDefaults()
    plan = OrderingPlan(classification=classify_social_like(g), pre_pass=defaults.pre_pass)
    if defaults.force is not None:
        plan.strategy = defaults.force
    else:
        plan.strategy = (OrderingStrategy.JaccardWindows if plan.classification.is_social_like
                         else OrderingStrategy.Rcm)
    if plan.strategy == OrderingStrategy.JaccardWindows:
        plan.window_size = defaults.window_size
        if plan.window_size == 0 or plan.window_size % sigma != 0:
            raise ValueError("window size must be a positive multiple of sigma")
    return plan


def rcm(g: Graph) -> Permutation:
    f = np.zeros(max(g.num_vertices(), 1), np.uint32)
    L.check(L.lib().blest_order_rcm(g.handle, _ptr(f)))
    return Permutation._trusted(f[: g.num_vertices()])


def jaccard_with_windows(g: Graph, sigma: int, w: int, pre_pass: Permutation | None = None) -> Permutation:
    """jaccard_with_windows (R:src/ordering.cpp:139-166), GPU clusterer."""
    base = g
    if pre_pass is not None and not pre_pass.is_identity():
        base = apply_permutation(g, pre_pass)
    f = np.zeros(max(base.num_vertices(), 1), np.uint32)
    L.check(L.lib().blest_order_jaccard_windows(base.handle, sigma, w, _ptr(f)))
    win = Permutation(f[: base.num_vertices()])
    if base is not g:
        return Permutation.composed(pre_pass, win)
    return win


def random_order(n: int, seed: int) -> Permutation:
    f = np.zeros(max(n, 1), np.uint32)
    L.check(L.lib().blest_order_random(n, seed, _ptr(f)))
    return Permutation(f[:n])


def make_permutation(g: Graph, plan: OrderingPlan, sigma: int = 8, seed: int = 0) -> Permutation:
    """make_permutation (R:src/ordering.cpp:407-422)."""
    if plan.strategy == OrderingStrategy.Identity:
        return Permutation.identity(g.num_vertices())
    if plan.strategy == OrderingStrategy.Random:
        return random_order(g.num_vertices(), seed)
    if plan.strategy == OrderingStrategy.Rcm:
        return rcm(g)
    if plan.pre_pass == PrePass.BfsLocality:
        raise NotImplementedError("bfs-locality pre-pass is out of scope (SURVEY §2)")
    return jaccard_with_windows(g, sigma, plan.window_size)


# ------------------------------------------------------------------------------------
# BVSS (R:include/blest/bvss.hpp)
# ------------------------------------------------------------------------------------
@dataclass
class BvssStats:
    compression_ratio: float
    update_divergence: float
    num_slice_sets: int
    num_vss: int
    num_slices_padded: int
    num_unpadded_slices: int
    connectivity_bits: int
    per_vss_slice_histogram: dict
    bytes_real_ptrs: int
    bytes_virtual_to_real: int
    bytes_row_ids: int
    bytes_masks: int
    bytes_dynamic: int
    bytes_levels: int

    def bytes_static(self) -> int:
        return self.bytes_real_ptrs + self.bytes_virtual_to_real + self.bytes_row_ids + self.bytes_masks


class Bvss:
    """Device-resident BVSS (blest::Bvss) plus its BFS workspace."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        info = L.BvssInfo()
        L.check(L.lib().blest_bvss_get_info(self._h, C.byref(info)))
        self.n = info.n
        self.m = info.m
        self.num_slice_sets = info.num_slice_sets
        self.num_vss = info.num_vss
        self.num_unpadded_slices = info.num_unpadded_slices
        self.sigma = info.sigma
        self.tau = info.tau
        self.producing_permutation: Optional[Permutation] = None
        self.ordering_tag = ""
        self._divergence: Optional[float] = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and L._lib is not None:
            L._lib.blest_bvss_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def sentinel(self) -> int:
        return self.n

    @staticmethod
    def upload(n: int, m: int, real_ptrs, virtual_to_real, row_ids, masks) -> "Bvss":
        rp, v2r, rows, mk = _u32(real_ptrs), _u32(virtual_to_real), _u32(row_ids), _u32(masks)
        nv = len(v2r)
        if len(rows) != nv * 128 or len(mk) != nv * 32 or len(rp) != (n + 7) // 8 + 1:
            raise ValueError("BVSS array lengths do not match numVSS / numSliceSets")
        out = C.c_void_p()
        L.check(L.lib().blest_bvss_upload(n, m, nv, _ptr(rp), _ptr(v2r), _ptr(rows), _ptr(mk), 1,
                                          C.byref(out)))
        return Bvss(out.value)

    def arrays(self):
        rp = np.zeros(self.num_slice_sets + 1, np.uint32)
        v2r = np.zeros(max(self.num_vss, 1), np.uint32)
        rows = np.zeros(max(self.num_vss * 128, 1), np.uint32)
        mk = np.zeros(max(self.num_vss * 32, 1), np.uint32)
        L.check(L.lib().blest_bvss_download(self._h, _ptr(rp), _ptr(v2r), _ptr(rows), _ptr(mk)))
        nv = self.num_vss
        return rp, v2r[:nv], rows[: nv * 128], mk[: nv * 32]

    def update_divergence(self) -> float:
        if self._divergence is None:
            d = C.c_double()
            L.check(L.lib().blest_bvss_update_divergence(self._h, C.byref(d)))
            self._divergence = d.value
        return self._divergence


def save_bvss(b: Bvss, path: str) -> None:
    """save_bvss (R:src/bvss.cpp:250-266): the reference's 'BVSS' v1 binary cache."""
    L.check(L.lib().blest_bvss_save(b.handle, os.fsencode(path)))


def load_bvss(path: str) -> Bvss:
    """load_bvss (R:src/bvss.cpp:268-295)."""
    out = C.c_void_p()
    L.check(L.lib().blest_bvss_load(os.fsencode(path), C.byref(out)))
    return Bvss(out.value)


def save_permutation(p: Permutation, path: str) -> None:
    """save_permutation (R:src/graph.cpp:396-401): one inverse id per line."""
    f = p.forward_map()
    L.check(L.lib().blest_permutation_save(_ptr(f), len(f), os.fsencode(path)))


def load_permutation(path: str) -> Permutation:
    """load_permutation (R:src/graph.cpp:403-417)."""
    n = C.c_uint32(0)
    L.check(L.lib().blest_permutation_load(os.fsencode(path), None, C.byref(n)))
    f = np.zeros(max(n.value, 1), np.uint32)
    L.check(L.lib().blest_permutation_load(os.fsencode(path), _ptr(f), C.byref(n)))
    return Permutation(f[: n.value])


def load_graph(path: str) -> Graph:
    """load_graph (R:src/graph.cpp:390-394): .mtx Matrix Market, else an edge list."""
    out = C.c_void_p()
    L.check(L.lib().blest_graph_load(os.fsencode(path), C.byref(out)))
    return Graph(out.value)


def reference_bfs(g: Graph, src: int) -> "BfsResult":
    """reference_bfs (R:src/graph.cpp:144-167), on the device straight over the CSR (the
    validation oracle the CLI's --validate compares the engines with)."""
    if not 0 <= int(src) < g.num_vertices():
        raise ValueError("bfs source out of range")
    lv = np.zeros(max(g.num_vertices(), 1), np.uint32)
    vis, nl = C.c_uint32(), C.c_uint32()
    L.check(L.lib().blest_graph_bfs(g.handle, int(src), _ptr(lv), C.byref(vis), C.byref(nl)))
    return BfsResult(source=int(src), levels=lv[: g.num_vertices()], visited_count=vis.value,
                     num_levels=nl.value)


@dataclass
class RoundtripReport:
    checked_slices: int = 0
    discrepancies: list = field(default_factory=list)

    def ok(self) -> bool:
        return not self.discrepancies


def validate_roundtrip(b: Bvss, g: Graph) -> RoundtripReport:
    """validate_roundtrip (R:src/bvss.cpp:143-188) on the device: every slot decoded, the
    padding rules checked, the decoded arcs compared with g's incoming view per row. One
    discrepancy entry per violation class (with its count and first offender)."""
    r = L.RoundtripReportT()
    L.check(L.lib().blest_bvss_validate_roundtrip(b.handle, g.handle, C.byref(r)))
    d = []
    if r.padded_nonzero_mask:
        d.append(f"padded slot with nonzero mask at vss {r.first_padded_nonzero_vss} ({r.padded_nonzero_mask} slots)")
    if r.real_zero_mask:
        d.append(f"real slot with zero mask at vss {r.first_zero_mask_vss} ({r.real_zero_mask} slots)")
    if r.mask_bit_beyond_n:
        d.append(f"mask bit beyond n at slice set {r.first_beyond_set} ({r.mask_bit_beyond_n} bits)")
    if r.rows_mismatched:
        d.append(f"incoming list mismatch at row {r.first_mismatched_row} ({r.rows_mismatched} rows)")
    return RoundtripReport(int(r.checked_slices), d)


def build_bvss(g: Graph) -> Bvss:
    """build_bvss (R:src/bvss.cpp:19-101) on the GPU."""
    out = C.c_void_p()
    L.check(L.lib().blest_bvss_build(g.handle, C.byref(out)))
    return Bvss(out.value)


def compression_ratio(b: Bvss) -> float:
    if b.num_unpadded_slices == 0:
        return 0.0
    return b.m / (b.num_unpadded_slices * 8)


def update_divergence(b: Bvss) -> float:
    return b.update_divergence()


def bvss_stats(b: Bvss) -> BvssStats:
    s = L.BvssStatsT()
    L.check(L.lib().blest_bvss_stats(b.handle, C.byref(s)))
    b._divergence = s.update_divergence
    hist = {k: int(s.per_vss_slice_histogram[k]) for k in range(129) if s.per_vss_slice_histogram[k]}
    return BvssStats(s.compression_ratio, s.update_divergence, s.num_slice_sets, s.num_vss,
                     s.num_slices_padded, s.num_unpadded_slices, s.connectivity_bits, hist,
                     s.bytes_real_ptrs, s.bytes_virtual_to_real, s.bytes_row_ids, s.bytes_masks,
                     s.bytes_dynamic, s.bytes_levels)


# ------------------------------------------------------------------------------------
# Engines (R:include/blest/bfs_engine.hpp)
# ------------------------------------------------------------------------------------
class EngineMode(enum.Enum):
    Eager = "eager"
    Lazy = "lazy"
    Auto = "auto"


def engine_mode_from_string(s: str) -> EngineMode:
    for m in EngineMode:
        if m.value == s:
            return m
    raise ValueError("unknown engine mode: " + s)


@dataclass
class EngineConfig:
    num_warps: int = 0  # 0 = the whole persistent grid
    mode: EngineMode = EngineMode.Auto
    lazy_divergence_threshold: float = 25000.0
    max_levels: int = 0
    workers: int = 1  # accepted for API parity; the GPU grid replaces CPU workers
    pull: str = "popc"  # "popc" (CUDA-core) or "mma" (b1 m8n8k128 mma.sync tile)
    grid_ctas: int = 0
    threads_per_cta: int = 0


@dataclass
class LevelTrace:
    level: int = 0
    queue_size: int = 0
    frontier_population: int = 0
    discovered: int = 0
    full_atomics: int = 0
    stage1_full_atomics: int = 0
    relaxed_atomics: int = 0
    queue_pushes: int = 0


@dataclass
class EngineCounters:
    mma_calls: int = 0
    full_atomics: int = 0
    relaxed_atomics: int = 0
    queue_pushes: int = 0
    vss_dequeues: int = 0
    brs_baseline_mma_calls: int = 0
    levels_processed: int = 0
    trace: list = field(default_factory=list)
    trace_truncated: bool = False


@dataclass
class BfsResult:
    source: int = 0
    levels: Optional[np.ndarray] = None
    visited_count: int = 0
    num_levels: int = 0


@dataclass
class FrontierState:
    f_curr: np.ndarray
    levels: np.ndarray
    q_curr: np.ndarray
    v_curr: Optional[np.ndarray] = None
    v_next: Optional[np.ndarray] = None
    current_level: int = 0


def init_state(b: Bvss, src: int, mode: EngineMode) -> FrontierState:
    """init_state (R:src/bfs_engine.cpp:30-49): the seeded state the fused kernel builds."""
    if src >= b.n:
        raise ValueError("bfs source out of range")
    words = (b.n + 31) // 32
    f = np.zeros(words, np.uint32)
    f[src // 32] |= np.uint32(1 << (src % 32))
    lv = np.full(b.n, KUNREACHED, np.uint32)
    lv[src] = 0
    rp = b.arrays()[0]
    q = np.arange(rp[src // 8], rp[src // 8 + 1], dtype=np.uint32)
    if mode == EngineMode.Lazy:
        return FrontierState(f, lv, q, f.copy(), f.copy())
    return FrontierState(f, lv, q)


def _cfg_struct(cfg: EngineConfig, mode: EngineMode) -> L.EngineConfigT:
    if cfg.pull not in ("popc", "mma"):
        raise ValueError("pull must be 'popc' or 'mma'")
    return L.EngineConfigT(L.MODE_LAZY if mode == EngineMode.Lazy else L.MODE_EAGER,
                           L.PULL_MMA if cfg.pull == "mma" else L.PULL_POPC,
                           cfg.max_levels, cfg.num_warps, cfg.grid_ctas, cfg.threads_per_cta)


def _run(b: Bvss, src: int, cfg: EngineConfig, mode: EngineMode, want_levels: bool = True):
    if cfg.num_warps < 0:
        raise ValueError("numWarps must be >= 1")
    cs = _cfg_struct(cfg, mode)
    lv = np.zeros(max(b.n, 1), np.uint32) if want_levels else None
    ctr = L.CountersT()
    cap = 1 << 16
    trace = (L.LevelTraceT * cap)()
    L.check(L.lib().blest_bfs(b.handle, src, C.byref(cs), _ptr(lv) if lv is not None else None,
                              C.byref(ctr), C.cast(trace, C.c_void_p), cap))
    rows = [LevelTrace(*(getattr(trace[i], f) for f, _ in L.LevelTraceT._fields_))
            for i in range(min(ctr.trace_len, cap))]
    res = BfsResult(source=src, levels=lv[: b.n] if lv is not None else None,
                    visited_count=ctr.visited_count, num_levels=ctr.num_levels)
    cnt = EngineCounters(ctr.mma_calls, ctr.full_atomics, ctr.relaxed_atomics, ctr.queue_pushes,
                         ctr.vss_dequeues, ctr.brs_baseline_mma_calls, ctr.levels_processed, rows,
                         bool(ctr.trace_truncated))
    return res, cnt


def run_eager(b: Bvss, src: int, cfg: EngineConfig | None = None):
    """run_eager (R:src/bfs_engine.cpp:155-236): fused persistent kernel, Alg. 2."""
    return _run(b, src, cfg or EngineConfig(), EngineMode.Eager)


def run_lazy(b: Bvss, src: int, cfg: EngineConfig | None = None):
    """run_lazy (R:src/bfs_engine.cpp:238-350): fused persistent kernel, Alg. 3."""
    return _run(b, src, cfg or EngineConfig(), EngineMode.Lazy)


def run_batch(b: Bvss, srcs, mode: EngineMode, cfg: EngineConfig | None = None, out=None):
    """Many sources back to back through blest_bfs_batch (device-pipelined: source k's level
    array is copied to the host while source k+1 runs). Returns (levels [k, n] uint32 —
    `out` if given, e.g. pinned memory — and one EngineCounters per source, trace rows
    omitted). Same results as calling run_eager / run_lazy per source."""
    cfg = cfg or EngineConfig()
    if mode == EngineMode.Auto:
        raise ValueError("run_batch needs a resolved mode (eager or lazy)")
    srcs = np.ascontiguousarray(srcs, np.uint32)
    k = len(srcs)
    lv = out if out is not None else np.zeros((k, max(b.n, 1)), np.uint32)
    if out is not None:  # the library writes k*n 32-bit words through the pointer
        dt = getattr(out, "dtype", None)
        nbytes = out.element_size() if hasattr(out, "element_size") else getattr(dt, "itemsize", 0)
        contig = out.is_contiguous() if hasattr(out, "is_contiguous") else out.flags["C_CONTIGUOUS"]
        numel = out.numel() if hasattr(out, "numel") else out.size
        if nbytes != 4 or not contig or numel < k * b.n:
            raise ValueError("out must be a contiguous 32-bit buffer with at least k*n elements")
    ctr = (L.CountersT * max(k, 1))()
    cs = _cfg_struct(cfg, mode)
    ptr = lv.data_ptr() if hasattr(lv, "data_ptr") else lv.ctypes.data
    L.check(L.lib().blest_bfs_batch(b.handle, _ptr(srcs) if k else None, k, C.byref(cs), C.c_void_p(ptr),
                                    C.cast(ctr, C.c_void_p)))
    cnts = [EngineCounters(c.mma_calls, c.full_atomics, c.relaxed_atomics, c.queue_pushes, c.vss_dequeues,
                           c.brs_baseline_mma_calls, c.levels_processed, [], bool(c.trace_truncated))
            for c in list(ctr)[:k]]
    return lv, cnts


@dataclass
class AutoConfig:
    engine: EngineConfig = field(default_factory=EngineConfig)
    ordering: SelectDefaults = field(default_factory=SelectDefaults)
    seed: int = 0


@dataclass
class AutoResult:
    bfs: BfsResult
    counters: EngineCounters
    plan: OrderingPlan
    stats: Optional[BvssStats]
    chosen_mode: EngineMode


def choose_mode(b: Bvss, plan: OrderingPlan, cfg: EngineConfig) -> EngineMode:
    """Lazy iff social-like and update divergence >= threshold (R:src/bfs_engine.cpp:358-362)."""
    if cfg.mode != EngineMode.Auto:
        return cfg.mode
    if plan.classification.is_social_like and b.update_divergence() >= cfg.lazy_divergence_threshold:
        return EngineMode.Lazy
    return EngineMode.Eager


def run_auto_prebuilt(b: Bvss, plan: OrderingPlan, src: int, cfg: AutoConfig | None = None,
                      with_stats: bool = False) -> AutoResult:
    """run_auto_prebuilt (R:src/bfs_engine.cpp:352-386). The divergence is computed once per
    structure and cached (the reference recomputes bvss_stats on every call, :356)."""
    cfg = cfg or AutoConfig()
    mode = choose_mode(b, plan, cfg.engine)
    perm = b.producing_permutation
    mapped = perm is not None and not perm.is_identity()
    if not 0 <= int(src) < b.n:  # before any permutation lookup (R:src/bfs_engine.cpp:31)
        raise ValueError("bfs source out of range")
    run_src = perm.forward(src) if mapped else src
    res, cnt = _run(b, run_src, cfg.engine, mode)
    if mapped:
        res = BfsResult(source=src, levels=res.levels[perm.forward_map()],
                        visited_count=res.visited_count, num_levels=res.num_levels)
    return AutoResult(res, cnt, plan, bvss_stats(b) if with_stats else None, mode)


def prepare(g: Graph, cfg: AutoConfig | None = None) -> tuple[Bvss, OrderingPlan]:
    """Classify -> order -> permute -> build (the prebuilt half of run_auto, :388-402)."""
    cfg = cfg or AutoConfig()
    plan = select_plan(g, 8, cfg.ordering)
    perm = make_permutation(g, plan, 8, cfg.seed)
    b = build_bvss(g if perm.is_identity() else apply_permutation(g, perm))
    b.ordering_tag = plan.strategy.value
    b.producing_permutation = perm
    return b, plan


def run_auto(g: Graph, src: int, cfg: AutoConfig | None = None) -> AutoResult:
    """run_auto (R:src/bfs_engine.cpp:388-402)."""
    cfg = cfg or AutoConfig()
    b, plan = prepare(g, cfg)
    return run_auto_prebuilt(b, plan, src, cfg, with_stats=True)


def device_info():
    name = C.create_string_buffer(128)
    sms, ma, mi = C.c_int(), C.c_int(), C.c_int()
    L.check(L.lib().blest_device_info(name, 128, C.byref(sms), C.byref(ma), C.byref(mi)))
    return dict(name=name.value.decode(), sm_count=sms.value, cc=f"{ma.value}.{mi.value}")


def tile_pull(masks, alpha) -> np.ndarray:
    """The engines' b1 tile on the device (blest_tile_pull): masks [T, 32] u32, alpha [T] u8
    -> FragC counts [T, 2 rounds, 64] (tc::mma_m8n8k128 semantics, R:src/tc_emu.cpp:9-45)."""
    m = np.ascontiguousarray(masks, np.uint32).reshape(-1, 32)
    a = np.ascontiguousarray(alpha, np.uint8).reshape(-1)
    if len(a) != len(m):
        raise ValueError("one alpha per tile")
    out = np.zeros((max(len(m), 1), 2, 64), np.uint32)
    L.check(L.lib().blest_tile_pull(_ptr(m) if len(m) else None, _ptr(a) if len(a) else None, len(m), _ptr(out)))
    return out[: len(m)]
