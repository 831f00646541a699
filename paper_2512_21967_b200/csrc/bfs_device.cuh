// Device-side pieces shared by the eager (bfs.cu) and lazy (bfs_lazy.cu) kernels.
#pragma once

#include <atomic>

#include "bfs.cuh"

namespace blestgpu {
namespace bfsdev {

#ifndef BLEST_KBATCH
#define BLEST_KBATCH 4
#endif
constexpr int kBatch = BLEST_KBATCH;  // VSSs in flight per warp
constexpr int kPushCap = 64;      // per-warp push buffer entries (eager)
constexpr unsigned long long kNoEntry = ~0ull;

struct Params {
    uint32_t n, num_sets;
    uint64_t words;
    const uint32_t* __restrict__ rp;
    const uint32_t* __restrict__ masks;
    const uint4* __restrict__ rows4;
    uint32_t* L;
    uint32_t* B0;  // eager F0 | lazy V_curr
    uint32_t* B1;  // eager F1 | lazy V_next
    uint32_t* B2;  // eager F2 | lazy per-level diff
    unsigned long long* Q0;
    unsigned long long* Q1;
    unsigned long long* Q2;
    unsigned long long* ctl;    // [0..3] qlen ring, [4] iterations, [5] max level, [6] status
    unsigned long long* agg;    // lazy stage 2: per-CTA (level << 40 | VSS count)
    unsigned long long* aggS;   // lazy stage 2: per-CTA (level << 40 | slice-set count)
    unsigned long long* SL;     // lazy queue: frontier slice sets (first VSS position << 32 | set)
    unsigned* bar;
    unsigned long long* trace;
    unsigned long long* tstamp;  // per level: [start, stage-1 end, level end] (%globaltimer ns)
    uint32_t trace_cap;
    uint32_t src;
    uint32_t cap;
    uint32_t num_warps;
    uint32_t hub_words;      // lazy: V_curr words [0, hub_words) staged in shared memory on
                             // dense levels (0 = off; the L1 then caches the hub prefix)
    uint64_t dense_min;      // queue length from which a level stages the hub prefix
    uint32_t xflags;  // experiment switches (BLEST_XFLAGS env; timing studies only)
};

template <int THREADS, int MODE = 0>
struct Smem {
    unsigned long long push[THREADS / 32][MODE == 0 ? kPushCap : 1];  // eager: ss | ss << 32
    unsigned long long ctr[4];                         // discovered, full, relaxed, pushes
    unsigned long long red[THREADS / 32];              // block reductions / scans
    unsigned long long base;
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Fire-and-forget OR (REDG): the lazy scheme's "relaxed atomic" (R:src/bfs_engine.cpp:287-288).
__device__ __forceinline__ void red_or(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v));
}

template <int MODE>
__device__ __forceinline__ unsigned long long* queue_at(const Params& p, uint32_t idx) {
    if (MODE == 0) {
        const uint32_t k = idx % 3;
        return k == 0 ? p.Q0 : (k == 1 ? p.Q1 : p.Q2);
    }
    return (idx & 1) ? p.Q1 : p.Q0;
}

__device__ __forceinline__ uint32_t* fbuf(const Params& p, uint32_t idx) {
    const uint32_t k = idx % 3;
    return k == 0 ? p.B0 : (k == 1 ? p.B1 : p.B2);
}

// Block-wide exclusive scan of a u64 per thread; returns the thread's offset, *total the sum.
template <int THREADS, int MODE>
__device__ __forceinline__ unsigned long long block_excl_scan(Smem<THREADS, MODE>& sm, unsigned long long x,
                                                              unsigned long long* total) {
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    unsigned long long incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += y;
    }
    __syncthreads();  // protect sm.red from a previous use
    if (lane == 31) sm.red[warp] = incl;
    __syncthreads();
    unsigned long long before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < THREADS / 32; ++w) {
        const unsigned long long t = sm.red[w];
        if (w < (int)warp) before += t;
        all += t;
    }
    *total = all;
    return before + incl - x;
}

// Warp flush (eager): reserve room for the buffered slice sets' VSS ranges with one
// atomicAdd and write the expanded entries. Returns VSS entries written.
__device__ __forceinline__ uint32_t flush_pushes(const Params& p, unsigned long long* buf, uint32_t& count,
                                 unsigned long long* Qn, unsigned long long* qlen_next) {
    const unsigned lane = lane_id();
    uint32_t total = 0;
    uint32_t my_off[kPushCap / 32], my_b[kPushCap / 32], my_len[kPushCap / 32];
#pragma unroll
    for (int k = 0; k < kPushCap / 32; ++k) {
        const uint32_t i = k * 32 + lane;
        uint32_t b = 0, len = 0;
        if (i < count) {
            const uint32_t ss = (uint32_t)buf[i];
            b = p.rp[ss];
            len = p.rp[ss + 1] - b;
        }
        const uint32_t incl = warp_incl_scan(len);
        my_off[k] = total + incl - len;
        my_b[k] = b;
        my_len[k] = len;
        total += __shfl_sync(0xffffffffu, incl, 31);
    }
    unsigned long long base = 0;
    if (lane == 0 && total) base = atomicAdd(qlen_next, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (uint32_t i = 0; i < count; ++i) {
        const int k = i >> 5;
        const uint32_t src_lane = i & 31;
        uint32_t off = 0, b = 0, len = 0;
#pragma unroll
        for (int kk = 0; kk < kPushCap / 32; ++kk)
            if (kk == k) {
                off = __shfl_sync(0xffffffffu, my_off[kk], src_lane);
                b = __shfl_sync(0xffffffffu, my_b[kk], src_lane);
                len = __shfl_sync(0xffffffffu, my_len[kk], src_lane);
            }
        const unsigned long long aux = buf[i] & 0xFFFFFFFF00000000ull;
        for (uint32_t t = lane; t < len; t += 32) Qn[base + off + t] = aux | (unsigned long long)(b + t);
    }
    __syncwarp();
    count = 0;
    return total;
}

// Append per-lane push flags for one column to the warp buffer (flushing first if full).
__device__ __forceinline__ void push_column(const Params& p, bool flag, unsigned long long item,
                                            unsigned long long* buf, uint32_t& count,
                                            unsigned long long* Qn, unsigned long long* qlen_next,
                                            uint32_t& pushes, uint32_t& full) {
    const unsigned ball = __ballot_sync(0xffffffffu, flag);
    if (!ball) return;
    const uint32_t k = __popc(ball);
    if (count + k > kPushCap) {
        const uint32_t t = flush_pushes(p, buf, count, Qn, qlen_next);
        if (lane_id() == 0) {  // per-warp quantities: count once, not per lane
            pushes += t;
            full += 1;
        }
    }
    if (flag) buf[count + __popc(ball & ((1u << lane_id()) - 1))] = item;
    __syncwarp();
    count += k;
}

template <int PULL>
__device__ __forceinline__ void column_counts(uint32_t m, uint32_t alpha, uint32_t (&cnt)[4]) {
    if (PULL == 0) {
        // CUDA-core path: AND with the broadcast frontier byte, per-byte nonzero test.
        const uint32_t x = m & (alpha * 0x01010101u);
        cnt[0] = x & 0xFFu;
        cnt[1] = (x >> 8) & 0xFFu;
        cnt[2] = (x >> 16) & 0xFFu;
        cnt[3] = x >> 24;
    } else {
        // BLEST tile: 2 × m8n8k128 b1 AND+POPC per VSS. fragB: lanes 9r hold α, lanes 9r+4
        // hold α<<8 (build_fragB, R:src/tc_emu.cpp:22-29); fragA = the lane's low/high 16
        // mask bits per round (pack_fragA_round :31-38); lane t gets its own two column
        // popcounts (lane_dot_products :40-45).
        const unsigned lane = lane_id();
        const uint32_t r9 = lane % 9;
        const uint32_t b = (r9 == 0) ? alpha : ((r9 == 4) ? (alpha << 8) : 0u);
#pragma unroll
        for (int round = 0; round < 2; ++round) {
            const uint32_t a = round ? (m >> 16) : (m & 0xFFFFu);
            int d0 = 0, d1 = 0;
            asm volatile(
                "mma.sync.aligned.m8n8k128.row.col.s32.b1.b1.s32.and.popc "
                "{%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+r"(d0), "+r"(d1)
                : "r"(a), "r"(b));
            cnt[2 * round] = (uint32_t)d0;
            cnt[2 * round + 1] = (uint32_t)d1;
        }
    }
}

// Flush per-thread counters into the CTA's shared counters, then (thread 0) into the
// level's trace row; then the grid barrier; block 0 stamps the time.
template <int THREADS, int MODE>
__device__ __forceinline__ void level_barrier(const Params& p, Smem<THREADS, MODE>& sm, unsigned& gen,
                                              uint32_t level, uint32_t (&c)[4], int stamp_slot) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t s = warp_sum(c[i]);
        if (lane_id() == 0 && s) atomicAdd(&sm.ctr[i], (unsigned long long)s);
        c[i] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t row = min(level - 1, p.trace_cap - 1);
        unsigned long long* t = p.trace + 8ull * row;
        if (sm.ctr[0]) {
            atomicAdd(&t[3], sm.ctr[0]);
            atomicMax(&p.ctl[5], (unsigned long long)level);
        }
        if (sm.ctr[1]) atomicAdd(&t[4], sm.ctr[1]);
        if (sm.ctr[2]) atomicAdd(&t[6], sm.ctr[2]);
        if (sm.ctr[3]) atomicAdd(&t[7], sm.ctr[3]);
#pragma unroll
        for (int i = 0; i < 4; ++i) sm.ctr[i] = 0;
    }
    grid_barrier(p.bar, gen);
    if (blockIdx.x == 0 && threadIdx.x == 0 && level - 1 < p.trace_cap)
        p.tstamp[3ull * (level - 1) + stamp_slot] = globaltimer();
}


}  // namespace bfsdev
}  // namespace blestgpu
