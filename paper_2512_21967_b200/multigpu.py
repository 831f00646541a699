"""Row-partitioned multi-GPU BFS: one process per GPU, rank g owns the
destination rows [row_lo, row_hi) (32-aligned) and a BVSS of A[rows_g, all columns]; per
level every rank pulls its local queue, sweeps its owned frontier words, and an all-gather
(NCCL over NVLink on B200s; any torch.distributed backend works) gives every rank the full
n/8-byte frontier diff, from which it queues its local VSSs for the next level. Each diff
word has a single writer (its row owner), so no OR-reduction is needed — NCCL has none.

The level loop is backend-agnostic: `GpuPartition` drives libblest_b200's partition
kernels through the C-ABI; the CPU tests plug an oracle-backed backend into the same loop
under gloo to check the partition/exchange protocol with world_size 2.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib as L


def partition_rows(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous 32-aligned row ranges, one per rank (equal frontier-word counts)."""
    words = (n + 31) // 32
    per = (words + world - 1) // world
    return [(min(r * per * 32, n), min((r + 1) * per * 32, n)) for r in range(world)]


def words_per_rank(n: int, world: int) -> int:
    return ((n + 31) // 32 + world - 1) // world


@dataclass
class PartitionedResult:
    levels: np.ndarray      # owned rows' levels (u32, kUnreached where not reached)
    row_lo: int
    row_hi: int
    iterations: int         # level iterations run (the last one discovered nothing)
    discovered: int         # vertices discovered over all ranks (source excluded)


class RowPartitionedBfs:
    """The per-level protocol. backend: begin(src) / pull() / sweep(level) -> local diff
    words (length words_per_rank) / enqueue(full_diff) -> (queue_len, total_bits) /
    levels(). allgather(local) -> concatenation over ranks (length world * per)."""

    def __init__(self, backend, n: int, allgather: Callable, max_levels: int = 0):
        self.backend = backend
        self.n = n
        self.allgather = allgather
        self.cap = max_levels or n + 1

    def run(self, src: int) -> PartitionedResult:
        if not 0 <= src < self.n:
            raise ValueError("bfs source out of range")
        b = self.backend
        b.begin(src)
        level, total = 1, 0
        while True:
            if level > self.cap:
                raise RuntimeError(f"BFS ran past the level safety cap at level {level}")
            b.pull()
            local = b.sweep(level)
            full = self.allgather(local)
            _, bits = b.enqueue(full)
            total += bits
            if bits == 0:
                break
            level += 1
        lo, hi = b.row_range()
        return PartitionedResult(b.levels(), lo, hi, level, total)


class GpuPartition:
    """Backend over the C-ABI partition kernels (blest_bvss_build_rows / blest_part_*)."""

    def __init__(self, graph, row_lo: int, row_hi: int, per_words: int, device=None):
        import torch
        self.torch = torch
        h = C.c_void_p()
        L.check(L.lib().blest_bvss_build_rows(graph.handle, row_lo, row_hi, C.byref(h)))
        self._h = h
        self.local = torch.zeros(per_words, dtype=torch.int32, device=device or "cuda")
        lo, hi, wlo, whi = C.c_uint32(), C.c_uint32(), C.c_uint64(), C.c_uint64()
        L.check(L.lib().blest_part_range(h, C.byref(lo), C.byref(hi), C.byref(wlo), C.byref(whi)))
        self.lo, self.hi = lo.value, hi.value

    def __del__(self):
        if getattr(self, "_h", None) and L._lib is not None:
            L._lib.blest_bvss_free(self._h)
            self._h = None

    def row_range(self):
        return self.lo, self.hi

    def begin(self, src: int):
        q = C.c_uint64()
        L.check(L.lib().blest_part_begin(self._h, src, C.byref(q)))
        return q.value

    def pull(self):
        L.check(L.lib().blest_part_pull(self._h))

    def sweep(self, level: int):
        self.local.zero_()
        d = C.c_uint64()
        L.check(L.lib().blest_part_sweep(self._h, level, C.c_void_p(self.local.data_ptr()), C.byref(d)))
        return self.local

    def enqueue(self, full):
        q, bits = C.c_uint64(), C.c_uint64()
        L.check(L.lib().blest_part_enqueue(self._h, C.c_void_p(full.data_ptr()), C.byref(q), C.byref(bits)))
        return q.value, bits.value

    def levels(self) -> np.ndarray:
        out = np.zeros(max(self.hi - self.lo, 1), np.uint32)
        L.check(L.lib().blest_part_levels(self._h, out.ctypes.data))
        return out[: self.hi - self.lo]


def nccl_allgather(group=None):
    """all_gather_into_tensor over torch.distributed (NCCL on GPUs)."""
    import torch
    import torch.distributed as dist

    def gather(local):
        world = dist.get_world_size(group)
        if dist.get_backend(group) == "nccl":
            out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
            dist.all_gather_into_tensor(out, local, group=group)
            return out
        # gloo (several ranks sharing one GPU in tests): through host memory
        host = local.cpu()
        parts = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(parts, host, group=group)
        return torch.cat(parts).to(local.device)
    return gather


def run_lockstep(backends, n: int, src: int, max_levels: int = 0):
    """All ranks of a partition driven in one process (G virtual ranks on one GPU, or CPU
    backends): same protocol as RowPartitionedBfs, the all-gather being a concatenation.
    Returns the assembled level array and the number of level iterations."""
    import torch
    cap = max_levels or n + 1
    for b in backends:
        b.begin(src)
    level = 1
    while True:
        if level > cap:
            raise RuntimeError(f"BFS ran past the level safety cap at level {level}")
        for b in backends:
            b.pull()
        locals_ = [b.sweep(level).clone() for b in backends]
        full = torch.cat(locals_)
        bits = [b.enqueue(full)[1] for b in backends]
        if len(set(bits)) != 1:
            raise AssertionError("ranks disagree on the gathered frontier")
        if bits[0] == 0:
            break
        level += 1
    out = np.full(n, 0xFFFFFFFF, np.uint32)
    for b in backends:
        lo, hi = b.row_range()
        out[lo:hi] = b.levels()
    return out, level
