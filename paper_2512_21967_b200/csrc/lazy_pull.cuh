// Lazy stage 1 (BLEST Alg. 3 pull, run_lazy R:src/bfs_engine.cpp:273-292; pull_vss
// :131-146) as warp-level device functions shared by the single-GPU lazy kernel
// (bfs_lazy.cu) and the row-partitioned multi-GPU kernel (rows.cu).
//
// Input: the level's active slice sets SL (ascending, entry = first queue position << 32 |
// set id), S of them, len VSSs in total, and the frontier bytes Fd8 (α of set s = Fd8[s]).
// A sparse level (len < dense_min) is pulled straight from registers: every warp expands
// its own contiguous share of queue positions and pulls it. A dense level first expands SL
// into the materialised queue Q (equal contiguous share per warp; the caller then places a
// grid barrier) and pulls Q round-robin like the reference (p ≡ warp mod #warps, :190),
// the last 1/tail_div handed out dynamically in 32-position chunks.
//
// Per VSS: one coalesced 128 B mask line and four 128 B row-id lines (streaming loads),
// AND with α, and for every nonzero column the visited test of the row in the test bitmap
// W, then a fire-and-forget RED into V_next for a bit still clear (legal per SURVEY §8(a)
// pitfall 7). The tests of a warp's batch of kBatchLazy VSSs run as phases (all loads, then
// all REDs), so a batch pays each latency once, not once per VSS.
#pragma once

#include "bfs_device.cuh"

namespace blestgpu {
namespace bfsdev {

// Visited tests of one batch (kBatchLazy VSSs × 4 columns per lane) in batch-wide phases,
// each phase's memory operations in flight together: (A) every (VSS, column) slot's word of
// the test bitmap W — the row's word when the lane's pull hit the column, else the sentinel
// word `sent` (all ones, L1-resident), so the load is unconditional and needs no default
// move; (B) optionally (recheck) the words still clear re-read from V_next at L2; (C) a
// fire-and-forget RED into V_next for every bit still clear. Default W = V_next without
// (B): V_next ⊇ V_curr, so a set bit means "visited before, or already marked this level",
// and an L1 copy lagging this level's REDs from other SMs only costs an extra idempotent
// RED (the grid barrier invalidates L1 between levels). W = V_curr with (B) is the older
// scheme (V_curr is frozen within the level; the L2 re-check spares REDs). hit(j, c) says
// whether the lane's pull hit column c of VSS j; rw[j] holds its row ids. Returns the REDs
// issued. The stage is instruction-issue bound as much as latency bound (C2 level 3:
// ~124 warp instructions per VSS at ~74 % of the SM issue rate before this form), so every
// phase is a straight line of LOP3 / SHF / SEL / IMAD.WIDE / LDG per slot.
// (Codegen note: the optional phase B branch also keeps ptxas from interleaving phase A's
// result moves with its later loads — without it the same default path measured 5.3 ms
// per BFS instead of 2.0.)
// LOG (sparse levels of the single-GPU kernel): every word a RED went to is appended to the
// level's dirty-word log (one reservation per warp and batch), so a small stage 2 can visit
// just those words instead of sweeping all n/32 (bfs_device.cuh small_stage2).
struct RedLog {
    uint32_t* words;             // log entries (engine word index; duplicates allowed)
    unsigned long long* count;   // entries reserved (may exceed cap: then the log is incomplete)
    uint32_t cap;
};

template <bool LOG = false, typename Hit>
__device__ __forceinline__ uint32_t check_batch(const uint32_t* W, uint32_t* Vn, bool recheck, uint32_t sent,
                                                const uint4 (&rw)[kBatchLazy], Hit hit, const RedLog* log = nullptr,
                                                bool* log_on = nullptr) {
    uint32_t vw[4 * kBatchLazy];
#pragma unroll
    for (int j = 0; j < kBatchLazy; ++j) {
        const uint32_t u[4] = {rw[j].x, rw[j].y, rw[j].z, rw[j].w};
#pragma unroll
        for (int c = 0; c < 4; ++c) vw[4 * j + c] = W[hit(j, c) ? (u[c] >> 5) : sent];
    }
    if (recheck) {
#pragma unroll
        for (int j = 0; j < kBatchLazy; ++j) {
            const uint32_t u[4] = {rw[j].x, rw[j].y, rw[j].z, rw[j].w};
#pragma unroll
            for (int c = 0; c < 4; ++c) vw[4 * j + c] = recheck_word(Vn, u[c], vw[4 * j + c]);
        }
    }
    uint32_t reds = 0, issued = 0;
#pragma unroll
    for (int j = 0; j < kBatchLazy; ++j) {
        const uint32_t u[4] = {rw[j].x, rw[j].y, rw[j].z, rw[j].w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            // ptxas never predicates a global RED (it branches around it), so the count
            // lives inside the same branch: executed only when some lane issues the RED
            const uint32_t bit = __funnelshift_l(0u, 1u, u[c]);
            if (!(vw[4 * j + c] & bit)) {
                red_or(Vn + (u[c] >> 5), bit);
                ++reds;
                if (LOG) issued |= 1u << (4 * j + c);
            }
        }
    }
    if (LOG && *log_on && __any_sync(0xffffffffu, issued != 0)) {
        const uint32_t n = __popc(issued);
        const uint32_t incl = warp_incl_scan(n);
        unsigned long long base = 0;
        if (lane_id() == 31) base = atomicAdd(log->count, (unsigned long long)incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        if (base + __shfl_sync(0xffffffffu, incl, 31) > log->cap) *log_on = false;  // full: stop logging
        base += incl - n;
#pragma unroll
        for (int j = 0; j < kBatchLazy; ++j) {
            const uint32_t u[4] = {rw[j].x, rw[j].y, rw[j].z, rw[j].w};
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if ((issued >> (4 * j + c)) & 1u) {
                    if (base < log->cap) log->words[base] = u[c] >> 5;
                    ++base;
                }
        }
    }
    return reds;
}

// Everything stage 1 of one level needs (one per warp, built from kernel parameters).
struct PullCtx {
    const uint32_t* __restrict__ rp;     // real_ptrs
    const uint32_t* __restrict__ masks;  // 32 words per VSS
    const uint4* __restrict__ rows4;     // 32 uint4 per VSS (lane t's 4 row ids)
    const uint8_t* Fd8;                  // α of set s = Fd8[s]
    const unsigned long long* SL;        // active sets, ascending
    unsigned long long* Q;               // materialised queue (dense levels)
    unsigned long long* tail_ctr;        // dense tail chunk counter (zeroed before the level)
    const uint32_t* W;                   // test bitmap (V_next, or V_curr with recheck)
    uint32_t* Vn;                        // V_next
    uint64_t len;                        // VSSs queued
    uint32_t S;                          // sets queued
    uint32_t sent;                       // sentinel word index (all ones) of W
    bool recheck;
    uint32_t tail_div;
    uint32_t gw, NW, all_warps;          // this warp, pulling warps, all warps of the grid
    uint64_t pol;                        // L2 evict-first policy for the BVSS stream
    RedLog log;                          // pull_sparse<PULL, true>: dirty-word log
};

// Every pointer of the context addresses global memory. Callers whose pointers come from a
// struct in global memory (the row-partitioned kernel's per-rank parameters) would
// otherwise get generic LD instead of LDG for the visited tests and queue reads.
__device__ __forceinline__ void assume_global(const PullCtx& c) {
    __builtin_assume(__isGlobal(c.rp));
    __builtin_assume(__isGlobal(c.masks));
    __builtin_assume(__isGlobal(c.rows4));
    __builtin_assume(__isGlobal(c.Fd8));
    __builtin_assume(__isGlobal(c.SL));
    __builtin_assume(__isGlobal(c.Q));
    __builtin_assume(__isGlobal(c.tail_ctr));
    __builtin_assume(__isGlobal(c.W));
    __builtin_assume(__isGlobal(c.Vn));
}

// One warp's view of 32 consecutive SL entries.
struct SetWindow {
    uint32_t base;   // SL index held by lane 0
    uint64_t first;  // lane's first queue position (UINT64_MAX past the list)
    uint32_t b;      // lane's first VSS id (real_ptrs[s])
    uint32_t alpha;  // lane's frontier byte
    uint64_t wend;   // one past the last position covered by the window
};

__device__ __forceinline__ void load_window(const unsigned long long* SL, const uint32_t* rp, const uint8_t* Fd8,
                                            uint32_t base, uint32_t S, uint64_t T, SetWindow& w) {
    const unsigned lane = lane_id();
    const uint32_t k = base + lane;
    uint64_t first = ~0ull, nxt = T;
    uint32_t b = 0, alpha = 0;
    if (k < S) {
        const unsigned long long e = SL[k];
        first = e >> 32;
        const uint32_t ss = (uint32_t)e;
        b = rp[ss];
        alpha = Fd8[ss];
        if (lane == 31 && k + 1 < S) nxt = SL[k + 1] >> 32;
    }
    w.base = base;
    w.first = first;
    w.b = b;
    w.alpha = alpha;
    w.wend = (base + 32 < S) ? __shfl_sync(0xffffffffu, nxt, 31) : T;
}

// Largest SL index k with first(k) <= pos (first(0) = 0, entries ascending).
__device__ __forceinline__ uint32_t find_set(const unsigned long long* SL, uint32_t S, uint64_t pos) {
    const unsigned lane = lane_id();
    uint32_t lo = 0, hi = S;
    while (hi - lo > 32) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t idx = lo + lane * step;
        const bool ok = idx < hi && (SL[idx] >> 32) <= pos;
        const unsigned ball = __ballot_sync(0xffffffffu, ok);
        lo = lo + (31 - __clz(ball)) * step;
        hi = min(hi, lo + step);
    }
    const uint32_t idx = lo + lane;
    const bool ok = idx < hi && (SL[idx] >> 32) <= pos;
    return lo + (31 - __clz(__ballot_sync(0xffffffffu, ok)));
}

// Queue entry (α << 32 | VSS) of position c0 + lane; `win` is slid forward as needed.
__device__ __forceinline__ unsigned long long entry_at(const PullCtx& c, uint64_t c0, SetWindow& win) {
    const unsigned lane = lane_id();
    if (c0 + 31 >= win.wend && win.wend < c.len) {  // slide to the set holding c0
        const unsigned own = __ballot_sync(0xffffffffu, win.first <= c0);
        const uint32_t nb = (c0 >= win.wend) ? win.base + 32 : win.base + (31 - __clz(own));
        load_window(c.SL, c.rp, c.Fd8, nb, c.S, c.len, win);
    }
    const uint64_t q = c0 + lane;
    int l = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
        const uint64_t f = __shfl_sync(0xffffffffu, win.first, l + step);
        if (f <= q) l += step;
    }
    const uint32_t v = __shfl_sync(0xffffffffu, win.b, l) + (uint32_t)(q - __shfl_sync(0xffffffffu, win.first, l));
    const uint32_t a = __shfl_sync(0xffffffffu, win.alpha, l);
    return ((unsigned long long)a << 32) | v;
}

// Loads of the VSSs named by lanes 0..kBatchLazy-1 of e, then their visited tests. An
// absent batch slot carries entry 0 (VSS 0 with α = 0): its loads are harmless and its
// pull finds no candidate, so no per-slot predication is needed.
template <int PULL, bool LOG = false>
__device__ __forceinline__ uint32_t pull_batch(const PullCtx& c, unsigned long long e, bool* log_on = nullptr) {
    const unsigned lane = lane_id();
    uint32_t mk[kBatchLazy], a[kBatchLazy];
    uint4 rw[kBatchLazy];
#pragma unroll
    for (int j = 0; j < kBatchLazy; ++j) {
        const uint32_t v = __shfl_sync(0xffffffffu, (uint32_t)e, j);
        a[j] = __shfl_sync(0xffffffffu, (uint32_t)(e >> 32), j);  // α (0 when absent)
        mk[j] = ld_stream_u32(c.masks + 32 * (uint64_t)v + lane, c.pol);
        rw[j] = ld_stream_u4(c.rows4 + 32 * (uint64_t)v + lane, c.pol);
    }
    if (PULL == 0) {
        uint32_t x[kBatchLazy];  // mask & α in every column byte
#pragma unroll
        for (int j = 0; j < kBatchLazy; ++j) x[j] = mk[j] & (a[j] * 0x01010101u);
        return check_batch<LOG>(c.W, c.Vn, c.recheck, c.sent, rw,
                                [&](int j, int col) { return (x[j] & (0xFFu << (8 * col))) != 0u; }, &c.log, log_on);
    }
    uint32_t cm[kBatchLazy];  // column hits from the b1 tile (bit c = column c)
#pragma unroll
    for (int j = 0; j < kBatchLazy; ++j) {
        uint32_t cnt[4];
        column_counts<PULL>(mk[j], a[j], cnt);
        cm[j] = (cnt[0] != 0) | ((cnt[1] != 0) << 1) | ((cnt[2] != 0) << 2) | ((cnt[3] != 0) << 3);
    }
    return check_batch<LOG>(c.W, c.Vn, c.recheck, c.sent, rw,
                            [&](int j, int col) { return ((cm[j] >> col) & 1u) != 0u; }, &c.log, log_on);
}

// Sparse level: the warp expands its own contiguous share of the queue and pulls it
// straight from registers — no materialised queue, no barrier. Returns REDs issued.
template <int PULL, bool LOG = false>
__device__ __forceinline__ uint32_t pull_sparse(const PullCtx& c) {
    assume_global(c);
    uint32_t reds = 0;
    if (c.gw >= c.NW) return 0;
    const unsigned lane = lane_id();
    const uint64_t lo = (uint64_t)c.gw * c.len / c.NW, hi = (uint64_t)(c.gw + 1) * c.len / c.NW;
    if (lo >= hi) return 0;
    SetWindow win;
    load_window(c.SL, c.rp, c.Fd8, find_set(c.SL, c.S, lo), c.S, c.len, win);
    bool log_on = true;  // LOG: until the log is full (then stage 2 sweeps anyway)
    for (uint64_t c0 = lo; c0 < hi; c0 += 32) {
        const unsigned long long mine = entry_at(c, c0, win);
        const uint32_t cnt = (hi - c0 < 32) ? (uint32_t)(hi - c0) : 32u;
        for (uint32_t k = 0; k < cnt; k += kBatchLazy) {
            unsigned long long e = __shfl_sync(0xffffffffu, mine, (lane + k) & 31);
            if (lane >= (uint32_t)kBatchLazy || k + lane >= cnt) e = 0;  // absent
            reds += pull_batch<PULL, LOG>(c, e, &log_on);
        }
    }
    return reds;
}

// Dense level, part 1: SL expanded into Q, an equal contiguous share per warp of the whole
// grid (a hub set with thousands of VSSs is spread over all warps). A grid barrier must
// follow before pull_dense.
__device__ __forceinline__ void expand_queue(const PullCtx& c) {
    assume_global(c);
    const unsigned lane = lane_id();
    const uint64_t lo = (uint64_t)c.gw * c.len / c.all_warps, hi = (uint64_t)(c.gw + 1) * c.len / c.all_warps;
    if (lo >= hi) return;
    SetWindow win;
    load_window(c.SL, c.rp, c.Fd8, find_set(c.SL, c.S, lo), c.S, c.len, win);
    for (uint64_t c0 = lo; c0 < hi; c0 += 32) {
        const unsigned long long e = entry_at(c, c0, win);
        if (c0 + lane < hi) c.Q[c0 + lane] = e;
    }
}

// Dense level, part 2: batches of kBatchLazy queue positions q0, q0+qs, ... < qe, the next
// batch's queue entries fetched while this batch is processed. Positions [0, len - tail)
// go round-robin over the warps like the reference (p ≡ warp mod #warps, :190); the last
// 1/tail_div (whole grid only) is handed out in chunks of 32 consecutive positions from a
// counter, so warps that finish early absorb the tail instead of waiting at the barrier.
template <int PULL>
__device__ __forceinline__ uint32_t pull_dense(const PullCtx& c) {
    assume_global(c);
    uint32_t reds = 0;
    if (c.gw >= c.NW) return 0;
    const unsigned lane = lane_id();
    auto run = [&](uint64_t q0, uint64_t qs, uint64_t qe) {
        const uint64_t step = qs * kBatchLazy;
        auto qload = [&](uint64_t base) -> unsigned long long {
            const uint64_t pos = base + (uint64_t)lane * qs;
            return (lane < kBatchLazy && pos < qe) ? c.Q[pos] : 0ull;  // 0: absent
        };
        unsigned long long e_next = qload(q0);
        for (uint64_t p0 = q0; p0 < qe; p0 += step) {
            const unsigned long long e = e_next;
            e_next = qload(p0 + step);
            reds += pull_batch<PULL>(c, e);
        }
    };
    const uint64_t tail = (c.NW == c.all_warps && c.tail_div) ? c.len / c.tail_div : 0;
    const uint64_t stat = c.len - tail;
    run(c.gw, c.NW, stat);
    if (tail) {
        for (;;) {
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(c.tail_ctr, 32ull);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= tail) break;
            run(stat + t, 1, stat + min(t + 32, (unsigned long long)tail));
        }
    }
    return reds;
}

}  // namespace bfsdev
}  // namespace blestgpu
