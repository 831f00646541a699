"""ctypes binding of the C-ABI in include/blest_b200.h (libblest_b200.so, built in-tree).

There is no fallback: if the shared library is missing or the device is not an sm_100
part, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BLEST_LIB") or os.path.join(HERE, "libblest_b200.so")

BLEST_OK, BLEST_EINVAL, BLEST_ERUNTIME, BLEST_ELOGIC, BLEST_ECUDA, BLEST_ENOMEM = 0, -1, -2, -3, -4, -5
BLEST_EPARSE = -6
MODE_EAGER, MODE_LAZY, MODE_AUTO = 0, 1, 2
PULL_POPC, PULL_MMA = 0, 1


class BlestError(Exception):
    """Base for status codes that are not mapped onto a Python built-in."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class BlestCudaError(BlestError, RuntimeError):
    pass


class BlestLogicError(BlestError, AssertionError):
    """std::logic_error: an engine invariant broke."""


class ParseError(RuntimeError):
    """blest::ParseError (R:include/blest/graph.hpp:23-32): a runtime_error with a line."""

    def __init__(self, msg: str):
        super().__init__(msg)
        import re
        m = re.search(r"\(line (\d+)\)$", msg)
        self.line = int(m.group(1)) if m else 0


class RoundtripReportT(C.Structure):
    _fields_ = [("checked_slices", C.c_uint64), ("padded_nonzero_mask", C.c_uint64),
                ("real_zero_mask", C.c_uint64), ("mask_bit_beyond_n", C.c_uint64),
                ("rows_mismatched", C.c_uint64), ("first_padded_nonzero_vss", C.c_uint64),
                ("first_zero_mask_vss", C.c_uint64), ("first_beyond_set", C.c_uint64),
                ("first_mismatched_row", C.c_uint64)]


class BvssInfo(C.Structure):
    _fields_ = [("n", C.c_uint32), ("num_slice_sets", C.c_uint32), ("num_vss", C.c_uint32),
                ("sigma", C.c_uint32), ("tau", C.c_uint32), ("m", C.c_uint64),
                ("num_unpadded_slices", C.c_uint64)]


class BvssStatsT(C.Structure):
    _fields_ = [("compression_ratio", C.c_double), ("update_divergence", C.c_double),
                ("num_slice_sets", C.c_uint32), ("num_vss", C.c_uint32),
                ("num_slices_padded", C.c_uint64), ("num_unpadded_slices", C.c_uint64),
                ("connectivity_bits", C.c_uint64), ("bytes_real_ptrs", C.c_uint64),
                ("bytes_virtual_to_real", C.c_uint64), ("bytes_row_ids", C.c_uint64),
                ("bytes_masks", C.c_uint64), ("bytes_dynamic", C.c_uint64),
                ("bytes_levels", C.c_uint64), ("per_vss_slice_histogram", C.c_uint64 * 129)]


class SocialReportT(C.Structure):
    _fields_ = [("top1_share", C.c_double), ("top10_share", C.c_double),
                ("power_law_slope", C.c_double), ("power_law_fit_r2", C.c_double),
                ("is_social_like", C.c_int), ("heavy_tail_fired", C.c_int),
                ("power_law_fired", C.c_int)]


class EngineConfigT(C.Structure):
    _fields_ = [("mode", C.c_int), ("pull", C.c_int), ("max_levels", C.c_uint32),
                ("num_warps", C.c_uint32), ("grid_ctas", C.c_uint32), ("threads_per_cta", C.c_uint32)]


class CountersT(C.Structure):
    _fields_ = [("mma_calls", C.c_uint64), ("full_atomics", C.c_uint64),
                ("relaxed_atomics", C.c_uint64), ("queue_pushes", C.c_uint64),
                ("vss_dequeues", C.c_uint64), ("brs_baseline_mma_calls", C.c_uint64),
                ("levels_processed", C.c_uint32), ("num_levels", C.c_uint32),
                ("visited_count", C.c_uint64), ("trace_len", C.c_uint32),
                ("trace_truncated", C.c_uint32)]


class LevelTraceT(C.Structure):
    _fields_ = [("level", C.c_uint64), ("queue_size", C.c_uint64),
                ("frontier_population", C.c_uint64), ("discovered", C.c_uint64),
                ("full_atomics", C.c_uint64), ("stage1_full_atomics", C.c_uint64),
                ("relaxed_atomics", C.c_uint64), ("queue_pushes", C.c_uint64)]


class RowsStatsT(C.Structure):
    _fields_ = [("iterations", C.c_uint32), ("max_level", C.c_uint32), ("queue", C.c_uint64),
                ("discovered", C.c_uint64), ("relaxed", C.c_uint64), ("pushes", C.c_uint64),
                ("unpulled", C.c_uint64)]


# Every symbol include/blest_b200.h declares, with its ctypes signature.
vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
P = C.POINTER
SIGNATURES = {
    "blest_last_error": (C.c_char_p, []),
    "blest_version": (C.c_char_p, []),
    "blest_set_stream": (i32, [vp]),
    "blest_device_info": (i32, [C.c_char_p, i32, P(i32), P(i32), P(i32)]),
    "blest_kernel_launches": (u64, []),
    "blest_graph_from_edges": (i32, [u32, vp, vp, u64, i32, i32, P(vp)]),
    "blest_graph_from_csr": (i32, [u32, vp, vp, i32, i32, P(vp)]),
    "blest_graph_generate": (i32, [i32, u32, u32, u64, u64, u32, u32, u32, P(vp)]),
    "blest_graph_info": (i32, [vp, P(u32), P(u64), P(i32)]),
    "blest_graph_device_csr": (i32, [vp, P(vp), P(vp)]),
    "blest_graph_copy_csr": (i32, [vp, vp, vp]),
    "blest_graph_apply_permutation": (i32, [vp, vp, i32, P(vp)]),
    "blest_graph_out_degrees": (i32, [vp, vp, i32]),
    "blest_graph_traversed_edges": (i32, [vp, vp, P(u64)]),
    "blest_graph_free": (i32, [vp]),
    "blest_classify_social_like": (i32, [vp, P(SocialReportT)]),
    "blest_order_rcm": (i32, [vp, vp]),
    "blest_order_jaccard_windows": (i32, [vp, u32, u32, vp]),
    "blest_order_random": (i32, [u32, u64, vp]),
    "blest_relabel_permutation": (i32, [u32, u64, vp, i32]),
    "blest_pick_sources": (i32, [vp, u32, u64, i32, vp]),
    "blest_bvss_build": (i32, [vp, P(vp)]),
    "blest_bvss_upload": (i32, [u32, u64, u32, vp, vp, vp, vp, i32, P(vp)]),
    "blest_bvss_get_info": (i32, [vp, P(BvssInfo)]),
    "blest_bvss_download": (i32, [vp, vp, vp, vp, vp]),
    "blest_bvss_stats": (i32, [vp, P(BvssStatsT)]),
    "blest_bvss_update_divergence": (i32, [vp, P(C.c_double)]),
    "blest_bvss_free": (i32, [vp]),
    "blest_bfs": (i32, [vp, u32, P(EngineConfigT), vp, P(CountersT), vp, u32]),
    "blest_bfs_launch": (i32, [vp, u32, P(EngineConfigT)]),
    "blest_bfs_finish": (i32, [vp, vp, P(CountersT), vp, u32]),
    "blest_bfs_batch": (i32, [vp, vp, u32, P(EngineConfigT), vp, vp]),
    "blest_bfs_prepare": (i32, [vp, vp, P(u64)]),
    "blest_tile_pull": (i32, [vp, vp, u32, vp]),
    "blest_graph_copy_in_csr": (i32, [vp, vp, vp]),
    "blest_graph_transpose": (i32, [vp, P(vp)]),
    "blest_graph_digest": (i32, [vp, P(u64)]),
    "blest_graph_bfs": (i32, [vp, u32, vp, P(u32), P(u32)]),
    "blest_graph_load": (i32, [C.c_char_p, P(vp)]),
    "blest_bvss_save": (i32, [vp, C.c_char_p]),
    "blest_bvss_load": (i32, [C.c_char_p, P(vp)]),
    "blest_permutation_save": (i32, [vp, u32, C.c_char_p]),
    "blest_permutation_load": (i32, [C.c_char_p, vp, P(u32)]),
    "blest_bvss_validate_roundtrip": (i32, [vp, vp, P(RoundtripReportT)]),
    "blest_bfs_levels_device": (i32, [vp, P(vp)]),
    "blest_bfs_phase_times": (i32, [vp, vp, u32, P(u32)]),
    "blest_bfs_last_geometry": (i32, [vp, P(u32), P(u32)]),
    "blest_bfs_last_unpulled": (i32, [vp, P(u64)]),
    "blest_bvss_build_rows": (i32, [vp, u32, u32, P(vp)]),
    "blest_partition_rows": (i32, [vp, u32, vp, vp]),
    "blest_rows_create": (i32, [vp, u32, u32, vp, P(vp)]),
    "blest_rows_info": (i32, [vp, P(u32), P(u32), P(u32), P(u64)]),
    "blest_rows_ipc_handle": (i32, [vp, vp]),
    "blest_rows_open_peers": (i32, [vp, vp]),
    "blest_rows_set_local_peers": (i32, [vp, u32]),
    "blest_rows_bfs": (i32, [vp, u32]),
    "blest_rows_group_bfs": (i32, [vp, u32, u32]),
    "blest_rows_step": (i32, [vp, u32, u32, vp]),
    "blest_rows_send_buffer": (i32, [vp, P(vp)]),
    "blest_rows_flags": (i32, [vp, P(u32), P(u32), P(u32)]),
    "blest_rows_finish": (i32, [vp, vp, P(RowsStatsT)]),
    "blest_rows_free": (i32, [vp]),
    "blest_rows_phase_times": (i32, [vp, vp, u32, P(u32)]),
}

_lib = None
_lock = threading.Lock()


def build() -> None:
    import subprocess
    root = os.path.dirname(HERE)
    subprocess.check_call(["make", "-s", "-C", root, "-j8", "lib"])


def lib():
    """Load libblest_b200.so (building it first if absent and nvcc is available)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                if os.environ.get("BLEST_LIB") and not hasattr(L, name):
                    continue  # an experiment build (BLEST_LIB) from an older tree may lack newer entries
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == BLEST_OK:
        return
    msg = lib().blest_last_error().decode(errors="replace")
    if rc == BLEST_EINVAL:
        raise ValueError(msg)
    if rc == BLEST_ERUNTIME:
        raise RuntimeError(msg)
    if rc == BLEST_ELOGIC:
        raise BlestLogicError(rc, msg)
    if rc == BLEST_ENOMEM:
        raise MemoryError(msg)
    if rc == BLEST_EPARSE:
        raise ParseError(msg)
    raise BlestCudaError(rc, msg)
