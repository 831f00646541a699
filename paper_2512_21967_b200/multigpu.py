"""Row-partitioned multi-GPU BFS; the reference has no multi-GPU mode (the
paper lists it as future work), so the interface here is new.

One process per GPU. Rank g owns destination rows [32·bounds[g], 32·bounds[g+1]) — ranges
balanced by BVSS slice count (`partition_rows`) — and a BVSS of A[rows_g, all columns]
built on its own device (`RowsEngine`, csrc/rows.cu). Per level every rank pulls its
local VSSs (the lazy stage 1), sweeps its owned V words (levels, frontier diff), and every
rank receives the whole n/8-byte frontier: each word has one writer (its row owner), so an
all-gather suffices (NCCL has no OR-reduction). Termination is consistent because every
rank sweeps the same gathered frontier.

Two exchange modes over one CUDA kernel:
  * stepped (`SteppedBfs`): one cooperative launch per level; the frontier all-gather is a
    torch.distributed collective (NCCL over NVLink on B200s) enqueued on the same stream.
    The host never waits for a level: it reads the termination flag the kernels write to
    mapped host memory and runs at most `ahead` levels in front (launches past the end are
    no-ops). Every rank issues the same number of collectives (iterations + 1 + ahead).
  * fused (`RowsEngine.bfs`): one launch per BFS per rank; diff words are stored straight
    into every peer's frontier buffer through CUDA IPC mappings, with a cross-rank arrival
    barrier inside the kernel. `group_bfs` runs G virtual ranks of one GPU in one launch.

`SteppedBfs` is backend-agnostic: tests/partition_cpu.py provides a numpy backend with the
same step semantics, so the gloo CPU tests exercise exactly this host protocol.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib as L


def partition_rows_even(n: int, world: int) -> list[int]:
    """Word bounds (frontier words of 32 rows) with equal word counts per rank."""
    words = (n + 31) // 32
    per = (words + world - 1) // world if world else 0
    return [min(r * per, words) for r in range(world)] + [words]


def partition_rows(graph, world: int) -> tuple[list[int], list[int]]:
    """Word bounds balanced by BVSS slice count (a slice = one (column slice set, row)
    pair: the unit of pull work and of BVSS storage), computed on the device; and each
    rank's slice count."""
    if world < 1:
        raise ValueError("world size must be positive")
    b = (C.c_uint64 * (world + 1))()
    s = (C.c_uint64 * world)()
    L.check(L.lib().blest_partition_rows(graph.handle, world, C.cast(b, C.c_void_p), C.cast(s, C.c_void_p)))
    return list(b), list(s)


def rows_of(bounds: list[int], rank: int, n: int) -> tuple[int, int]:
    return min(32 * bounds[rank], n), min(32 * bounds[rank + 1], n)


@dataclass
class RowsResult:
    levels: np.ndarray  # owned rows' levels (u32, 0xFFFFFFFF = unreached)
    row_lo: int
    row_hi: int
    iterations: int     # level iterations (the last one discovered nothing)
    discovered: int     # owned rows discovered (source excluded)
    queue: int          # Σ local VSS queue over the levels
    collectives: int = 0
    unpulled: int = 0   # local VSSs of a barren last level counted in queue, not pulled (exhaustion exit)


class _DevArray:
    """__cuda_array_interface__ view of a library-owned device buffer of u32 words, typed
    int32 (the bit pattern is what matters; gloo and NCCL collectives take int32)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<i4", "data": (ptr, False), "version": 3}


class RowsEngine:
    """One rank's engine (csrc/rows.cu) over its BVSS slice, built on the current device."""

    def __init__(self, graph, rank: int, world: int, bounds: list[int]):
        self.n = graph.num_vertices()
        self.rank, self.world = rank, world
        self.bounds = list(bounds)
        h = C.c_void_p()
        arr = (C.c_uint64 * (world + 1))(*bounds)
        L.check(L.lib().blest_rows_create(graph.handle, rank, world, C.cast(arr, C.c_void_p), C.byref(h)))
        self._h = h
        lo, hi, nv, per = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint64()
        L.check(L.lib().blest_rows_info(h, C.byref(lo), C.byref(hi), C.byref(nv), C.byref(per)))
        self.row_lo, self.row_hi, self.num_vss, self.per = lo.value, hi.value, nv.value, per.value
        self._send = None

    def __del__(self):
        if getattr(self, "_h", None) and L._lib is not None:
            L._lib.blest_rows_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # ---- fused (P2P) mode ----
    def ipc_handle(self) -> bytes:
        buf = (C.c_char * 64)()
        L.check(L.lib().blest_rows_ipc_handle(self._h, buf))
        return bytes(buf)

    def open_peers(self, handles: list[bytes]):
        blob = b"".join(handles)
        if len(blob) != 64 * self.world:
            raise ValueError("one 64-byte IPC handle per rank expected")
        L.check(L.lib().blest_rows_open_peers(self._h, C.c_char_p(blob)))

    def bfs(self, src: int):
        """Fused BFS launch (async; every rank must launch it)."""
        L.check(L.lib().blest_rows_bfs(self._h, int(src)))

    # ---- stepped (NCCL) mode ----
    def send(self):
        """The rank's send buffer (per_words u32, device) as a torch tensor view."""
        if self._send is None:
            import torch
            p = C.c_void_p()
            L.check(L.lib().blest_rows_send_buffer(self._h, C.byref(p)))
            self._send = torch.as_tensor(_DevArray(p.value, self.per), device="cuda")
        return self._send

    def step(self, level: int, src: int, recv=None):
        ptr = None if recv is None else C.c_void_p(recv.data_ptr())
        L.check(L.lib().blest_rows_step(self._h, level, int(src), ptr))

    def flags(self) -> tuple[int, int, int]:
        a, b, c = C.c_uint32(), C.c_uint32(), C.c_uint32()
        L.check(L.lib().blest_rows_flags(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def phase_times(self, cap: int = 4096) -> np.ndarray:
        """Timeline of the last fused BFS: rows of (start, stage-1 end, exchange end, level
        end) in %globaltimer ns, one per level."""
        out = (C.c_uint64 * (4 * cap))()
        rows = C.c_uint32()
        L.check(L.lib().blest_rows_phase_times(self._h, C.cast(out, C.c_void_p), cap, C.byref(rows)))
        return np.array(out[: 4 * rows.value], np.uint64).reshape(-1, 4)

    def finish(self, levels: bool = True) -> RowsResult:
        out = np.zeros(max(self.row_hi - self.row_lo, 1), np.uint32) if levels else None
        st = L.RowsStatsT()
        L.check(L.lib().blest_rows_finish(self._h, out.ctypes.data if levels else None, C.byref(st)))
        return RowsResult(out[: self.row_hi - self.row_lo] if levels else None, self.row_lo, self.row_hi,
                          st.iterations, st.discovered, st.queue, unpulled=st.unpulled)


def set_local_peers(engines: list[RowsEngine]):
    arr = (C.c_void_p * len(engines))(*[e.handle.value for e in engines])
    L.check(L.lib().blest_rows_set_local_peers(C.cast(arr, C.c_void_p), len(engines)))


def group_bfs(engines: list[RowsEngine], src: int):
    """G virtual ranks of one device: one cooperative launch runs the fused BFS of all."""
    arr = (C.c_void_p * len(engines))(*[e.handle.value for e in engines])
    L.check(L.lib().blest_rows_group_bfs(C.cast(arr, C.c_void_p), len(engines), int(src)))


def run_stepped_local(engines: list[RowsEngine], src: int) -> list[RowsResult]:
    """Stepped mode with every rank on this device (virtual ranks): the all-gather is a
    device concatenation of the send buffers; lock-step, one host check per level."""
    import torch
    for e in engines:
        e.step(1, src, None)
    level = 1
    while True:
        recv = torch.cat([e.send() for e in engines])
        level += 1
        for e in engines:
            e.step(level, src, recv)
        torch.cuda.synchronize()
        done = [e.flags()[1] for e in engines]
        if all(done):
            if len(set(done)) != 1:
                raise AssertionError(f"ranks disagree on the termination level: {done}")
            break
        if any(done):
            raise AssertionError(f"ranks disagree on termination: {done}")
    return [e.finish() for e in engines]


def assemble(results: list[RowsResult], n: int) -> np.ndarray:
    out = np.full(n, 0xFFFFFFFF, np.uint32)
    for r in results:
        out[r.row_lo:r.row_hi] = r.levels
    return out


class SteppedBfs:
    """Host protocol of the stepped mode. backend: step(level, src, recv) / send() ->
    per-word tensor / flags() -> (progress, done, status) / finish(). allgather(send) ->
    recv (world × per words, rank-major); it must be stream-ordered after the step that
    wrote `send` (torch.distributed NCCL collectives are)."""

    def __init__(self, backend, allgather: Callable, ahead: int = 2, max_levels: int = 0):
        self.backend = backend
        self.allgather = allgather
        self.ahead = max(0, ahead)
        self.cap = max_levels

    def run(self, src: int, levels: bool = True) -> RowsResult:
        b = self.backend
        b.step(1, src, None)
        issued, done, target = 0, 0, None
        while target is None or issued < target:
            while True:  # run-ahead limit: the launch `issued + 1 - ahead` has started
                prog, d, status = b.flags()
                if d and target is None:
                    done = d
                    target = done + 1 + self.ahead  # identical on every rank
                if prog >= issued + 1 - self.ahead or target is not None:
                    break
                time.sleep(0)
            if target is not None and issued >= target:
                break
            if self.cap and issued >= self.cap:
                raise RuntimeError(f"BFS ran past the level safety cap at level {issued + 1}")
            recv = self.allgather(b.send())
            issued += 1
            b.step(issued + 1, src, recv)
        r = b.finish(levels)
        r.collectives = issued
        if r.iterations != done:
            raise AssertionError(f"terminated at {done} iterations but the engine reports {r.iterations}")
        return r


def torch_allgather(group=None):
    """all_gather_into_tensor over torch.distributed (NCCL on GPUs, stream-ordered); other
    backends (gloo: several ranks sharing one GPU in tests) go through host memory."""
    import torch
    import torch.distributed as dist
    bufs = {}

    def gather(local):
        world = dist.get_world_size(group)
        key = (local.numel(), local.device)
        if key not in bufs:
            bufs[key] = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
        out = bufs[key]
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(out, local, group=group)
            return out
        host = local.cpu()
        parts = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(parts, host, group=group)
        out.copy_(torch.cat(parts))
        return out
    return gather


def exchange_ipc_handles(engine: RowsEngine, group=None):
    """All ranks' IPC handles (torch.distributed all_gather_object), then map the peers."""
    import torch.distributed as dist
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, engine.ipc_handle(), group=group)
    engine.open_peers(handles)
