// Lazy engine (BLEST Alg. 3; run_lazy, R:src/bfs_engine.cpp:238-350) as one fused
// persistent cooperative kernel.
//
// Stage 1 (pull, :273-292). Warps take queue positions round-robin exactly like the
// reference (p ≡ warp mod #warps, :190), kBatchLazy at a time, so neighbouring warps stream
// neighbouring VSSs. Queue entries carry the set's frontier byte α (final when stage 2
// enqueued it). Per VSS: one coalesced 128 B mask line and four 128 B row-id lines
// (streaming loads), AND with α, and for every nonzero column the visited test: V_curr
// (frozen during the stage, L1-cached) and, if clear, V_next at L2; only then a
// fire-and-forget RED sets the V_next bit (legal per SURVEY §8(a) pitfall 7). The tests
// of a warp's whole batch run as three phases (all V_curr loads, then the V_next
// re-checks, then the REDs), so a batch pays each latency once, not once per VSS.
//
// Stage 2 (word sweep, :296-338) is lazy_stage2 (bfs_device.cuh): balanced, no contended
// atomics; it emits the next queue as the ascending list SL of active slice sets (set id,
// first queue position). A dense level first expands SL into the materialised queue —
// every warp writes an equal contiguous share of positions, resolving sets with a
// 32-set window in its lanes — then a grid barrier, then stage 1. A hub set with
// thousands of VSSs is thus spread over all warps instead of one. A sparse level
// (T < dense_min) skips the queue and the barrier: each warp expands its own contiguous
// share into registers and pulls it directly. The frontier words alternate between B2
// and B3 by level parity, so the next level's can be cleared while this one is read.
#include "bfs.cuh"
#include "bfs_device.cuh"

namespace blestgpu {

namespace {
using namespace bfsdev;


#ifndef BLEST_MINB
#define BLEST_MINB 1
#endif
// Visited tests of one batch (kBatchLazy VSSs × 4 columns per lane) in batch-wide phases,
// each phase's memory operations in flight together (one latency per phase, not one per
// VSS): (A) every (VSS, column) slot's word of the test bitmap W — the row's word when the
// lane's pull hit the column, else the sentinel word `sent` (all ones, L1-resident), so the
// load is unconditional and needs no default move; (B) optionally (Params::recheck) the
// words still clear re-read from V_next at L2; (C) a fire-and-forget RED into V_next for
// every bit still clear (legal per SURVEY §8(a) pitfall 7). Default W = V_next without (B):
// V_next ⊇ V_curr, so a set bit means "visited before, or already marked this level", and
// an L1 copy lagging this level's REDs from other SMs only costs an extra idempotent RED
// (the grid barrier invalidates L1 between levels). W = V_curr with (B) is the older
// scheme (V_curr is frozen within the level; the L2 re-check spares REDs). hit[j] holds
// the lane's 4 column hits of VSS j in bits 0..3; rw[j] its row ids. Returns the REDs
// issued. The stage is instruction-issue bound as much as latency bound (C2 level 3:
// ~124 warp instructions per VSS at ~74 % of the SM issue rate), so every phase is a
// straight line of LOP3 / SHF / SEL / IMAD.WIDE / LDG|RED per slot.
// (Codegen note: the optional phase B branch also keeps ptxas from interleaving phase
// A's result moves with its later loads — without it the same default path measured
// 5.3 ms per BFS.)
template <typename Hit>
__device__ __forceinline__ uint32_t check_batch(const uint32_t* W, uint32_t* Vn, bool recheck, uint32_t sent,
                                                const uint4 (&rw)[kBatchLazy], Hit hit) {
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
    uint32_t reds = 0;
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
            }
        }
    }
    return reds;
}

template <int PULL, int THREADS, bool SIGMA>
#ifndef BLEST_LAZY_MINB
#define BLEST_LAZY_MINB (BLEST_MINB > 1 ? BLEST_MINB : 1024 / THREADS)
#endif
__global__ void __launch_bounds__(THREADS, BLEST_LAZY_MINB) k_bfs_lazy(Params p) {
    constexpr int WPC = THREADS / 32;
    __shared__ Smem<THREADS, 1> sm;
    const unsigned lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t gtid = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    const uint64_t gthreads = (uint64_t)gridDim.x * THREADS;
    const uint32_t gw = blockIdx.x * WPC + warp;
    const uint32_t all_warps = gridDim.x * WPC;
    const uint32_t NW = (p.num_warps && p.num_warps < all_warps) ? p.num_warps : all_warps;
    unsigned gen = 0;
    const uint64_t pol = evict_first_policy();
    if (threadIdx.x < 4) sm.ctr[threadIdx.x] = 0;
    uint32_t* Vc = p.B0;
    uint32_t* Vn = p.B1;
    const uint4* __restrict__ rows4 = p.rows4;  // SIGMA: the σ view's row ids

    // ---- init_state (R:src/bfs_engine.cpp:30-49), fused ----
    const uint32_t src = p.src;
    const uint32_t sset = src / kSigma;
    const uint32_t seed_b = p.rp[sset], seed_e = p.rp[sset + 1];
    const uint32_t vsrc = SIGMA ? p.sig[src] : src;  // the source's engine id (hot rank or row)
    for (uint64_t i = gtid; i < p.n; i += gthreads) p.L[i] = (i == src) ? 0u : kInf;
    const uint32_t src_word = src >> 5, src_bit = 1u << (src & 31);
    const uint64_t vs_word = vsrc >> 5;
    const uint32_t vs_bit = 1u << (vsrc & 31);
    const uint64_t vwords = p.words + (SIGMA ? p.hot_words : 0);  // visited bitmap words
    for (uint64_t w = gtid; w < vwords; w += gthreads) {
        const uint32_t seed = (w == vs_word) ? vs_bit : 0u;
        Vc[w] = seed;
        Vn[w] = seed;
        if (w < p.words) p.B2[w] = (w == src_word) ? src_bit : 0u;  // α of the source's set, level 1
    }
    if (gtid == 0) {  // sentinel word after the visited bitmaps: "visited" for every bit
        Vc[vwords] = ~0u;
        Vn[vwords] = ~0u;
    }
    if (threadIdx.x == 0) {
        p.agg[blockIdx.x] = 0;
        p.aggS[blockIdx.x] = 0;
    }
    if (gtid == 0) {
        p.SL[0] = sset;                        // first position 0
        p.ctl[0] = seed_e - seed_b;            // T: VSSs queued for the level
        p.ctl[1] = (seed_e > seed_b) ? 1 : 0;  // S: slice sets queued
        for (int i = 2; i < 8; ++i) p.ctl[i] = 0;
        for (int i = 0; i < 8; ++i) p.trace[i] = 0;
    }
    uint32_t next_T = grid_barrier_pay(p.bar, gen, &p.ctl[0]);

    uint32_t ctr[4] = {0, 0, 0, 0};  // discovered, full, relaxed, pushes
    uint32_t level = 1;
    for (;; ++level) {
        const unsigned long long len = next_T;  // broadcast by the barrier
        const uint32_t S = (uint32_t)ld_relaxed_gpu_u64(&p.ctl[1]);
        if (len == 0) break;
        if (level > p.cap) {  // runaway (R:src/bfs_engine.cpp:72-75)
            if (gtid == 0) p.ctl[6] = 1;
            break;
        }
        if (gtid == 0) {
            p.ctl[7] = 0;  // stage-1 tail chunk counter (read after the expansion barrier)
            if (level - 1 < p.trace_cap) {
                p.trace[8ull * (level - 1) + 0] = level;
                p.trace[8ull * (level - 1) + 1] = len;
                p.tstamp[3ull * (level - 1)] = globaltimer();
            } else {
                atomicAdd(&p.trace[8ull * (p.trace_cap - 1) + 1], len);
            }
            if (level < p.trace_cap)
                for (int i = 0; i < 8; ++i) p.trace[8ull * level + i] = 0;
        }
        unsigned long long* Qc = p.Q0;
        // the level's frontier words (α) and the next level's: B2/B3 alternate, so the next
        // frontier can be cleared while this one is still being read (no barrier between)
        const uint32_t* Fd = (level & 1) ? p.B2 : p.B3;
        uint32_t* Fn = (level & 1) ? p.B3 : p.B2;
        const uint8_t* Fd8 = reinterpret_cast<const uint8_t*>(Fd);
        // queue entry (α << 32 | VSS) of position c0 + lane; `win` is slid forward as needed
        auto entry_at = [&](uint64_t c0, SetWindow& win) -> unsigned long long {
            if (c0 + 31 >= win.wend && win.wend < len) {  // slide to the set holding c0
                const unsigned own = __ballot_sync(0xffffffffu, win.first <= c0);
                const uint32_t nb = (c0 >= win.wend) ? win.base + 32 : win.base + (31 - __clz(own));
                load_window(p, Fd8, nb, S, len, win);
            }
            const uint64_t q = c0 + lane;
            int l = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint64_t f = __shfl_sync(0xffffffffu, win.first, l + step);
                if (f <= q) l += step;
            }
            const uint32_t v = __shfl_sync(0xffffffffu, win.b, l) +
                               (uint32_t)(q - __shfl_sync(0xffffffffu, win.first, l));
            const uint32_t a = __shfl_sync(0xffffffffu, win.alpha, l);
            return ((unsigned long long)a << 32) | v;
        };
        const bool recheck = p.lazy_recheck != 0;  // W = V_curr + V_next re-check (older scheme)
        const uint32_t* W = recheck ? Vc : Vn;
        // Loads of the VSSs named by lanes 0..kBatchLazy-1 of e, then their visited tests.
        // An absent batch slot carries entry 0 (VSS 0 with α = 0): its loads are harmless
        // and its pull finds no candidate, so no per-slot predication is needed.
        const uint32_t sent = (uint32_t)vwords;  // sentinel word (all ones) after the bitmap
        auto pull_batch = [&](unsigned long long e) {
            uint32_t mk[kBatchLazy], a[kBatchLazy];
            uint4 rw[kBatchLazy];
#pragma unroll
            for (int j = 0; j < kBatchLazy; ++j) {
                const uint32_t v = __shfl_sync(0xffffffffu, (uint32_t)e, j);
                a[j] = __shfl_sync(0xffffffffu, (uint32_t)(e >> 32), j);  // α (0 when absent)
                mk[j] = ld_stream_u32(p.masks + 32 * (uint64_t)v + lane, pol);
                rw[j] = ld_stream_u4(rows4 + 32 * (uint64_t)v + lane, pol);
            }
            if (PULL == 0) {
                uint32_t x[kBatchLazy];  // mask & α in every column byte
#pragma unroll
                for (int j = 0; j < kBatchLazy; ++j) x[j] = mk[j] & (a[j] * 0x01010101u);
                ctr[2] += check_batch(W, Vn, recheck, sent, rw,
                                      [&](int j, int c) { return (x[j] & (0xFFu << (8 * c))) != 0u; });
            } else {
                uint32_t cm[kBatchLazy];  // column hits from the b1 tile (bit c = column c)
#pragma unroll
                for (int j = 0; j < kBatchLazy; ++j) {
                    uint32_t cnt[4];
                    column_counts<PULL>(mk[j], a[j], cnt);
                    cm[j] = (cnt[0] != 0) | ((cnt[1] != 0) << 1) | ((cnt[2] != 0) << 2) | ((cnt[3] != 0) << 3);
                }
                ctr[2] += check_batch(W, Vn, recheck, sent, rw,
                                      [&](int j, int c) { return ((cm[j] >> c) & 1u) != 0u; });
            }
        };
        if (len < p.dense_min) {
            // ---- sparse level: every warp expands its own contiguous share of the queue
            // and pulls it straight from registers — no materialised queue, no barrier ----
            if (SIGMA)
                for (uint64_t w = gtid; w < p.words; w += gthreads) Fn[w] = 0;
            if (gw < NW) {
                const uint64_t lo = (uint64_t)gw * len / NW, hi = (uint64_t)(gw + 1) * len / NW;
                if (lo < hi) {
                    SetWindow win;
                    load_window(p, Fd8, find_set(p, S, lo), S, len, win);
                    for (uint64_t c0 = lo; c0 < hi; c0 += 32) {
                        const unsigned long long mine = entry_at(c0, win);
                        const uint32_t cnt = (hi - c0 < 32) ? (uint32_t)(hi - c0) : 32u;
                        for (uint32_t k = 0; k < cnt; k += kBatchLazy) {
                            unsigned long long e = __shfl_sync(0xffffffffu, mine, (lane + k) & 31);
                            if (lane >= (uint32_t)kBatchLazy || k + lane >= cnt) e = 0;  // absent
                            pull_batch(e);
                        }
                    }
                }
            }
        } else {
            // ---- dense level: expand SL into the queue, equal contiguous share per warp ----
            {
                const uint64_t lo = (uint64_t)gw * len / all_warps, hi = (uint64_t)(gw + 1) * len / all_warps;
                if (lo < hi) {
                    SetWindow win;
                    load_window(p, Fd8, find_set(p, S, lo), S, len, win);
                    for (uint64_t c0 = lo; c0 < hi; c0 += 32) {
                        const unsigned long long e = entry_at(c0, win);
                        if (c0 + lane < hi) Qc[c0 + lane] = e;
                    }
                }
            }
            if (SIGMA)  // Fn is the previous level's α: its readers finished long ago
                for (uint64_t w = gtid; w < p.words; w += gthreads) Fn[w] = 0;
            grid_barrier(p.bar, gen);

            // ---- stage 1: pull (pull_vss, R:src/bfs_engine.cpp:131-146) ----
            if (gw < NW) {
                // Batches of kBatchLazy queue positions q0, q0+qs, ... < qe: mask words and row
                // ids loaded together (streaming loads), the next batch's queue entries fetched
                // while this batch is processed.
                auto run = [&](uint64_t q0, uint64_t qs, uint64_t qe) {
                    const uint64_t step = qs * kBatchLazy;
                    auto qload = [&](uint64_t base) -> unsigned long long {
                        const uint64_t pos = base + (uint64_t)lane * qs;
                        return (lane < kBatchLazy && pos < qe) ? Qc[pos] : 0ull;  // 0: absent
                    };
                    unsigned long long e_next = qload(q0);
                    for (uint64_t p0 = q0; p0 < qe; p0 += step) {
                        const unsigned long long e = e_next;
                        e_next = qload(p0 + step);
                        pull_batch(e);
                    }
                };
                // Positions [0, len - tail): round-robin over the warps like the reference
                // (p ≡ warp mod #warps, :190). The last 1/tail_div (8; whole grid) is handed
                // out in chunks of 32 consecutive positions from a counter, so warps that
                // finish early absorb the tail instead of waiting at the barrier.
                const uint64_t tail = (NW == all_warps && p.tail_div) ? len / p.tail_div : 0;
                const uint64_t stat = len - tail;
                run(gw, NW, stat);
                if (tail) {
                    for (;;) {
                        unsigned long long c = 0;
                        if (lane == 0) c = atomicAdd(&p.ctl[7], 32ull);
                        c = __shfl_sync(0xffffffffu, c, 0);
                        if (c >= tail) break;
                        run(stat + c, 1, stat + min(c + 32, (unsigned long long)tail));
                    }
                }
            }
        }
        level_barrier(p, sm, gen, level, ctr, 1);

        if (SIGMA)
            lazy_stage2_hot<THREADS>(p, sm, level, ctr, gen, Fn);
        else
            lazy_stage2<THREADS>(p, sm, level, ctr, Fn);
        next_T = level_barrier(p, sm, gen, level, ctr, 2, &p.ctl[0]);
    }
    if (gtid == 0) p.ctl[4] = level - 1;
}

}  // namespace

void* lazy_kernel(int pull, int threads, bool sigma) {
#define BLEST_LAZY_CASES(PULL, SIGMA)                         \
    switch (threads) {                                        \
        case 256: return (void*)k_bfs_lazy<PULL, 256, SIGMA>;   \
        case 512: return (void*)k_bfs_lazy<PULL, 512, SIGMA>;   \
        case 1024: return (void*)k_bfs_lazy<PULL, 1024, SIGMA>; \
    }
    if (pull == 1) {
        if (sigma) { BLEST_LAZY_CASES(1, true) } else { BLEST_LAZY_CASES(1, false) }
    } else {
        if (sigma) { BLEST_LAZY_CASES(0, true) } else { BLEST_LAZY_CASES(0, false) }
    }
#undef BLEST_LAZY_CASES
    throw InvalidArgument("threads per CTA must be 256, 512 or 1024");
}

}  // namespace blestgpu
