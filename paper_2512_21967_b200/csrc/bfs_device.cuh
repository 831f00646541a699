// Device-side pieces shared by the eager (bfs.cu) and lazy (bfs_lazy.cu) kernels.
#pragma once

#include <atomic>

#include "bfs.cuh"

namespace blestgpu {
namespace bfsdev {

#ifndef BLEST_KBATCH
#define BLEST_KBATCH 2
#endif
#ifndef BLEST_KBATCH_LAZY
#define BLEST_KBATCH_LAZY 3
#endif
// eager: VSSs per warp batch. The sparse levels of high-diameter graphs are a dependent
// chain per warp, and a smaller batch spreads a level's VSSs over more warps: 2 vs 4 gives
// C4 68.3 → 61.0 ms, C1 0.092 → 0.085 ms, C3 with the eager engine 3.97 → 4.11 ms (1: C4
// 60.8, C3 eager 5.06; 3: 64.2 / 3.75; one build with 3 on dense and 1 on sparse levels
// spilled and lost both ways: 62.5 / 4.03 — profiles/r02_ekb_ab/)
constexpr int kBatch = BLEST_KBATCH;
constexpr int kBatchLazy = BLEST_KBATCH_LAZY;  // lazy (C2: 3 → 1.73 ms, 4 → 1.87, 2 → 2.03)
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
    uint32_t* B3;  // eager visited bitmap VIS
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
    uint64_t dense_min;  // queue length from which a level counts as dense (eager re-checks)
    // lazy hot-row view (sigma.cuh): V_curr / V_next (B0, B1) = [hot prefix, hot_words
    // words | row words]; inv: hot rank -> row; sig: row -> engine id (source seeding)
    const uint32_t* __restrict__ inv;
    const uint32_t* __restrict__ sig;
    uint64_t hot_words;
    uint32_t xflags;  // experiment switches (BLEST_XFLAGS env; timing studies only)
    uint32_t lazy_recheck;  // lazy: test V_curr and re-check V_next at L2 (BLEST_LAZY_RECHECK)
    uint32_t tail_div;      // lazy: dense levels hand out their last 1/tail_div dynamically (0 = off)
    uint32_t log_cap;       // lazy: dirty-word log entries (in Q0) for the small stage 2 (0 = off)
    // lazy exhaustion exit: rows present in the BVSS (bitmap, original ids) and their count;
    // once 1 + Σ discovered covers every discoverable vertex the next level is barren
    const uint32_t* __restrict__ present;
    uint64_t present_rows;  // 0 = off
};

template <int THREADS, int MODE = 0>
struct Smem {
    unsigned long long push[THREADS / 32][MODE == 0 ? kPushCap : 1];  // eager: ss | ss << 32
    unsigned long long ctr[4];                         // discovered, full, relaxed, pushes
    unsigned long long red[THREADS / 32];              // block reductions / scans
    unsigned long long base;
    unsigned long long nz;                             // stage 2: chunks with a frontier word
};

// Block-wide OR of a per-thread chunk mask into sm.nz (thread 0 must have zeroed it before a
// __syncthreads that precedes this call; read it after a later __syncthreads).
template <int THREADS, int MODE>
__device__ __forceinline__ void block_or_nz(Smem<THREADS, MODE>& sm, unsigned long long m) {
    const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)m);
    const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(m >> 32));
    if ((threadIdx.x & 31) == 0 && (lo | hi)) atomicOr(&sm.nz, ((unsigned long long)hi << 32) | lo);
}
// bit of chunk i (relative to the CTA's first chunk) in the masks; chunks from 63 on share bit 63
__device__ __forceinline__ unsigned long long chunk_bit(uint64_t i) { return 1ull << (i < 63 ? i : 63); }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Timing study (BLEST_XFLAGS bit `bit`): CTA 0's thread 0 stamps tstamp slot 1 of the level
// once `dep` (a loaded value) has arrived — the volatile shared store consumes it first.
__device__ __forceinline__ void probe(const Params& p, uint32_t level, uint32_t bit, uint32_t dep, bool first) {
    if ((p.xflags & bit) && first && threadIdx.x == 0 && blockIdx.x == 0 && level - 1 < p.trace_cap) {
        __shared__ uint32_t sink;
        asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&sink)), "r"(dep)
                     : "memory");
        p.tstamp[3ull * (level - 1) + 1] = globaltimer();
    }
}

// Fire-and-forget OR (REDG): the lazy scheme's "relaxed atomic" (R:src/bfs_engine.cpp:287-288).
__device__ __forceinline__ void red_or(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v));
}

// Visited-test building blocks, written in PTX so each is a handful of SASS instructions
// with no branch: 32-bit word index, one IMAD.WIDE for the address, SHF.L.W for the bit.
// cand_word: the bitmap word holding bit x if `m & sel` (the lane's pull hit column x),
// else all ones (= "visited", nothing more to do). Plain ld.global: L1-cached.
__device__ __forceinline__ uint32_t cand_word(const uint32_t* base, uint32_t x, uint32_t m, uint32_t sel) {
    uint32_t v;
    asm("{\n\t.reg .pred q;\n\t.reg .b64 a;\n\t.reg .b32 t;\n\t"
        "and.b32 t, %3, %4;\n\tsetp.ne.u32 q, t, 0;\n\t"
        "shr.u32 t, %2, 5;\n\tmul.wide.u32 a, t, 4;\n\tadd.s64 a, a, %1;\n\t"
        "mov.b32 %0, -1;\n\t@q ld.global.u32 %0, [a];\n\t}"
        : "=r"(v)
        : "l"(base), "r"(x), "r"(m), "r"(sel));
    return v;
}
// recheck_word: v if it has bit x, else the word re-read at L2 (ld.relaxed.gpu).
__device__ __forceinline__ uint32_t recheck_word(const uint32_t* base, uint32_t x, uint32_t v) {
    uint32_t r;
    asm("{\n\t.reg .pred q;\n\t.reg .b64 a;\n\t.reg .b32 t, b;\n\t"
        "shf.l.wrap.b32 b, 0, 1, %2;\n\tand.b32 t, %3, b;\n\tsetp.eq.u32 q, t, 0;\n\t"
        "shr.u32 t, %2, 5;\n\tmul.wide.u32 a, t, 4;\n\tadd.s64 a, a, %1;\n\t"
        "mov.b32 %0, %3;\n\t@q ld.relaxed.gpu.global.u32 %0, [a];\n\t}"
        : "=r"(r)
        : "l"(base), "r"(x), "r"(v));
    return r;
}
// red_if_clear: if v lacks bit x, RED it into the bitmap; returns 1 if a RED was issued.
__device__ __forceinline__ uint32_t red_if_clear(uint32_t* base, uint32_t x, uint32_t v) {
    uint32_t issued;
    asm volatile("{\n\t.reg .pred q;\n\t.reg .b64 a;\n\t.reg .b32 t, b;\n\t"
        "shf.l.wrap.b32 b, 0, 1, %2;\n\tand.b32 t, %3, b;\n\tsetp.eq.u32 q, t, 0;\n\t"
        "shr.u32 t, %2, 5;\n\tmul.wide.u32 a, t, 4;\n\tadd.s64 a, a, %1;\n\t"
        "@q red.relaxed.gpu.global.or.b32 [a], b;\n\tselp.u32 %0, 1, 0, q;\n\t}"
        : "=r"(issued)
        : "l"(base), "r"(x), "r"(v));
    return issued;
}

// atom_if_clear: if v lacks bit x, atomicOr the bit into the bitmap and return the old
// word (its bit clear ⇒ this lane set it); else return all ones.
__device__ __forceinline__ uint32_t atom_if_clear(uint32_t* base, uint32_t x, uint32_t v) {
    uint32_t r;
    asm volatile("{\n\t.reg .pred q;\n\t.reg .b64 a;\n\t.reg .b32 t, b;\n\t"
        "shf.l.wrap.b32 b, 0, 1, %2;\n\tand.b32 t, %3, b;\n\tsetp.eq.u32 q, t, 0;\n\t"
        "shr.u32 t, %2, 5;\n\tmul.wide.u32 a, t, 4;\n\tadd.s64 a, a, %1;\n\t"
        "mov.b32 %0, -1;\n\t@q atom.relaxed.gpu.global.or.b32 %0, [a], b;\n\t}"
        : "=r"(r)
        : "l"(base), "r"(x), "r"(v));
    return r;
}

// Predicated RED (no branch / reconvergence point per call site).
__device__ __forceinline__ void red_or_if(bool pred, uint32_t* p, uint32_t v) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.relaxed.gpu.global.or.b32 [%0], %1;\n\t}" ::"l"(p),
        "r"(v), "r"((uint32_t)pred));
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
                                 unsigned long long* Qn, unsigned long long* qlen_next, bool pf) {
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
        for (uint32_t t = lane; t < len; t += 32) {
            Qn[base + off + t] = aux | (unsigned long long)(b + t);
            if (pf) {  // sparse level: pull the next level's VSS lines into L2
                const uint64_t v = b + t;
                asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p.masks + 32 * v));
#pragma unroll
                for (int l = 0; l < 4; ++l) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p.rows4 + 32 * v + 8 * l));
            }
        }
    }
    __syncwarp();
    count = 0;
    return total;
}

// Append per-lane push flags for one column to the warp buffer (flushing first if full).
__device__ __forceinline__ void push_column(const Params& p, bool flag, unsigned long long item,
                                            unsigned long long* buf, uint32_t& count,
                                            unsigned long long* Qn, unsigned long long* qlen_next,
                                            uint32_t& pushes, uint32_t& full, bool pf) {
    const unsigned ball = __ballot_sync(0xffffffffu, flag);
    if (!ball) return;
    const uint32_t k = __popc(ball);
    if (count + k > kPushCap) {
        const uint32_t t = flush_pushes(p, buf, count, Qn, qlen_next, pf);
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

// Flush per-thread counters into the CTA's shared counters, the grid barrier, then
// (thread 0) the CTA's counters into the level's trace row; block 0 stamps the time. The
// trace atomics follow the barrier so its fence never waits on them (one L2 round trip
// less per level; they land before the kernel ends, and row `level` is not reset again).
template <int THREADS, int MODE>
__device__ __forceinline__ uint32_t level_barrier(const Params& p, Smem<THREADS, MODE>& sm, unsigned& gen,
                                                  uint32_t level, uint32_t (&c)[4], int stamp_slot,
                                                  const unsigned long long* payload = nullptr,
                                                  unsigned long long* red_flag = nullptr,
                                                  unsigned long long* vis_total = nullptr,
                                                  unsigned long long* vis_out = nullptr,
                                                  bool disc_before = false) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t s = warp_sum(c[i]);
        if (lane_id() == 0 && s) atomicAdd(&sm.ctr[i], (unsigned long long)s);
        c[i] = 0;
    }
    __syncthreads();
    unsigned long long mine[4] = {0, 0, 0, 0};
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            mine[i] = sm.ctr[i];
            sm.ctr[i] = 0;
        }
    }
    // red_flag: set (plain store, every writer stores 1) when the CTA issued a stage-1 RED;
    // read back as the payload after the barrier
    if (red_flag && threadIdx.x == 0 && mine[2]) *red_flag = 1ull;
    // vis_total: running 1 + Σ discovered, added before the barrier, read back with the payload
    if (vis_total && threadIdx.x == 0 && mine[0]) atomicAdd(vis_total, mine[0]);
    // disc_before (eager exhaustion exit, dense levels): the trace row's discoveries are
    // added before the barrier, so the row is final once the barrier is passed
    if (disc_before && threadIdx.x == 0 && mine[0])
        atomicAdd(&p.trace[8ull * min(level - 1, p.trace_cap - 1) + 3], mine[0]);
    probe(p, level, 1u << 17, (uint32_t)mine[0], true);
    const uint32_t pay = grid_barrier_pay(p.bar, gen, red_flag ? red_flag : payload, vis_total, vis_out);
    probe(p, level, 1u << 18, pay, true);
    if (threadIdx.x == 0) {
        const uint32_t row = min(level - 1, p.trace_cap - 1);
        unsigned long long* t = p.trace + 8ull * row;
        if (mine[0]) {
            if (!disc_before) atomicAdd(&t[3], mine[0]);
            atomicMax(&p.ctl[5], (unsigned long long)level);
        }
        if (mine[1]) atomicAdd(&t[4], mine[1]);
        if (mine[2]) atomicAdd(&t[6], mine[2]);
        if (mine[3]) atomicAdd(&t[7], mine[3]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && level - 1 < p.trace_cap)
        p.tstamp[3ull * (level - 1) + stamp_slot] = globaltimer();
    return pay;
}


// Lazy stage 2 (R:src/bfs_engine.cpp:296-338), shared by both lazy kernels. The ⌈n/32⌉
// words are cut into chunks of 4·THREADS (one uint4 of words per thread) and each CTA owns
// a contiguous run of chunks. Pass A, per chunk: diff = V_next & ~V_curr, V_curr = V_next,
// diff words stored in Fd (α of the next level, like the reference's in-place F_curr,
// :310-311), levels written with one coalesced 128 B store per changed word, and the
// thread's active slice sets / their VSSs counted (real_ptrs lookups only for nonzero diff
// bytes). The CTA publishes both counts (tagged with the level, so no reset) and sums its
// predecessors'; pass B writes its SL entries (set | first position << 32) in ascending
// order, reusing the diff words held in registers when the CTA owns one chunk. The last
// CTA stores the grid totals (the next level's T, S) in ctl[0], ctl[1].
// The 17 real_ptrs entries bounding the 16 slice sets of words w0 … w0+3 (sets 4·w0 …
// 4·w0+15), issued together — four 16-byte loads (4·w0 is a multiple of 16) and one word —
// instead of up to 16 dependent pairs behind per-byte branches. Past the last set the
// bound repeats (count 0).
__device__ __forceinline__ void s2_rp(const uint32_t* rp, uint64_t num_sets, uint64_t w0, uint32_t (&r)[17]) {
    const uint64_t s0 = 4 * w0;
    if (s0 + 16 <= num_sets) {
        const uint4* q = reinterpret_cast<const uint4*>(rp + s0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 v = __ldg(q + i);
            r[4 * i] = v.x;
            r[4 * i + 1] = v.y;
            r[4 * i + 2] = v.z;
            r[4 * i + 3] = v.w;
        }
        r[16] = __ldg(rp + s0 + 16);
    } else {
#pragma unroll
        for (int i = 0; i < 17; ++i) r[i] = __ldg(rp + min(s0 + i, num_sets));
    }
}

template <int THREADS>
__device__ __forceinline__ void s2_counts(const Params& p, uint64_t w0, const uint32_t (&d)[4],
                                          unsigned long long& nv, unsigned long long& ns) {
    if (!(d[0] | d[1] | d[2] | d[3])) return;
    uint32_t r[17];
    s2_rp(p.rp, p.num_sets, w0, r);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t c = ((d[k] >> (8 * b)) & 0xFFu) ? r[4 * k + b + 1] - r[4 * k + b] : 0u;
            nv += c;
            ns += c != 0;  // sets without VSSs push nothing
        }
    }
}

template <int THREADS>
__device__ __forceinline__ void s2_load(const Params& p, const uint32_t* src, uint64_t w0, uint32_t (&d)[4], bool cg) {
    if (w0 + 4 <= p.words) {
        const uint4 v = cg ? __ldcg(reinterpret_cast<const uint4*>(src + w0)) : *reinterpret_cast<const uint4*>(src + w0);
        d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) d[k] = (w0 + k < p.words) ? (cg ? __ldcg(src + w0 + k) : src[w0 + k]) : 0u;
    }
}

// Second half of stage 2 (shared by both stage-2 variants): publish the CTA's (VSS, set)
// counts tagged with the level, sum its predecessors', and write its SL entries from the
// frontier diff words of its chunks (`keep` holds them when the CTA owns one chunk).
// The (VSS, set) count pairs are scanned packed into one u64 (sets in the top kSetBits bits,
// VSSs below): one block scan per phase instead of two (C2: 7 levels × 3 phases).
constexpr int kSetBits = 25;  // up to 2^25 slice sets (n < 2^28)
constexpr unsigned long long kVssMask = (1ull << (64 - kSetBits)) - 1;
__device__ __forceinline__ unsigned long long pack_vs(unsigned long long v, unsigned long long s) {
    return (s << (64 - kSetBits)) | v;
}

template <int THREADS>
__device__ __forceinline__ void s2_enqueue(const Params& p, Smem<THREADS, 1>& sm, uint32_t level, uint32_t (&ctr)[4],
                                           uint64_t k0, uint64_t k1, bool single, const uint32_t (&keep)[4],
                                           unsigned long long my_vss, unsigned long long my_sets,
                                           const uint32_t* Fd, unsigned long long nzm) {
    constexpr unsigned long long kTagMask = (1ull << 40) - 1;
    constexpr uint64_t CH = 4ull * THREADS;
    // Fd: the frontier words being built this level (parameter)
    if (threadIdx.x == 0) sm.nz = 0;
    unsigned long long cta = 0;
    block_excl_scan(sm, pack_vs(my_vss, my_sets), &cta);
    block_or_nz(sm, nzm);
    const unsigned long long cta_vss = cta & kVssMask, cta_sets = cta >> (64 - kSetBits);
    if (threadIdx.x == 0) {
        const unsigned long long tag = (unsigned long long)level << 40;
        p.aggS[blockIdx.x] = tag | cta_sets;
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.agg + blockIdx.x), "l"(tag | cta_vss) : "memory");
    }
    unsigned long long bv = 0, bs = 0;
    for (uint32_t c = threadIdx.x; c < blockIdx.x; c += THREADS) {
        unsigned long long x;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p.agg + c) : "memory");
        } while ((x >> 40) != level);
        bv += x & kTagMask;
        bs += ld_relaxed_gpu_u64(p.aggS + c) & kTagMask;
    }
    unsigned long long run = 0;
    block_excl_scan(sm, pack_vs(bv, bs), &run);
    unsigned long long run_vss = run & kVssMask, run_sets = run >> (64 - kSetBits);
    if (threadIdx.x == 0) {
        ctr[3] += (uint32_t)cta_vss;
        if (blockIdx.x == gridDim.x - 1) {  // grid totals: the next level's T, S
            p.ctl[0] = run_vss + cta_vss;
            p.ctl[1] = run_sets + cta_sets;
        }
    }
    // pass B: SL entries of the CTA's active sets, ascending; chunks without a frontier
    // word contribute nothing (no loads, no scans — the skip is uniform over the CTA)
    const unsigned long long nz = sm.nz;  // after the scans' __syncthreads
    for (uint64_t ch = k0; ch < k1; ++ch) {
        if (!(nz & chunk_bit(ch - k0))) continue;
        const uint64_t w0 = ch * CH + 4ull * threadIdx.x;
        uint32_t d[4];
        if (single) {
#pragma unroll
            for (int k = 0; k < 4; ++k) d[k] = keep[k];
        } else {
            s2_load<THREADS>(p, Fd, w0, d, true);
        }
        unsigned long long nv = 0, ns = 0;
        s2_counts<THREADS>(p, w0, d, nv, ns);
        unsigned long long it = 0;
        const unsigned long long pos = block_excl_scan(sm, pack_vs(nv, ns), &it);
        unsigned long long pv = run_vss + (pos & kVssMask);
        unsigned long long ps = run_sets + (pos >> (64 - kSetBits));
        if (ns) {
            uint32_t r[17];
            s2_rp(p.rp, p.num_sets, w0, r);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const uint32_t c = ((d[k] >> (8 * b)) & 0xFFu) ? r[4 * k + b + 1] - r[4 * k + b] : 0u;
                    if (c) {
                        p.SL[ps++] = (pv << 32) | (4 * (w0 + k) + b);
                        pv += c;
                    }
                }
            }
        }
        run_vss += it & kVssMask;
        run_sets += it >> (64 - kSetBits);
    }
}

// HOT (hot-row view, sigma.cuh): the visited words of row r live at word r/32 + hot_words
// (after the hot prefix), and Fd already holds the hot rows' discoveries (REDs of
// hot_stage2), which are merged into the frontier words; their levels are already stored.
template <int THREADS, bool HOT = false>
__device__ __forceinline__ void lazy_stage2(const Params& p, Smem<THREADS, 1>& sm, uint32_t level,
                                            uint32_t (&ctr)[4], uint32_t* Fd_out = nullptr) {
    constexpr unsigned long long kTagMask = (1ull << 40) - 1;
    constexpr uint64_t CH = 4ull * THREADS;
    const unsigned lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    uint32_t* Vc = p.B0 + (HOT ? p.hot_words : 0);  // 16-byte aligned: hot_words % 4 == 0
    uint32_t* Vn = p.B1 + (HOT ? p.hot_words : 0);
    uint32_t* Fd = Fd_out ? Fd_out : p.B2;  // the next level's frontier words
    const uint64_t chunks = (p.words + CH - 1) / CH;
    const uint64_t k0 = (uint64_t)blockIdx.x * chunks / gridDim.x, k1 = (uint64_t)(blockIdx.x + 1) * chunks / gridDim.x;
    const bool single = k1 - k0 <= 1;
    uint32_t keep[4] = {0, 0, 0, 0};  // frontier words of the CTA's only chunk
    unsigned long long my_vss = 0, my_sets = 0, nzm = 0;
    // pass A
    for (uint64_t ch = k0; ch < k1; ++ch) {
        const uint64_t w0 = ch * CH + 4ull * threadIdx.x;
        uint32_t nx[4], cu[4], d[4], f[4];
        s2_load<THREADS>(p, Vn, w0, nx, true);  // REDs landed in L2
        s2_load<THREADS>(p, Vc, w0, cu, false);
        if (HOT) s2_load<THREADS>(p, Fd, w0, f, true);  // hot rows' discoveries (REDs)
        bool any = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            d[k] = nx[k] & ~cu[k];
            any |= d[k] != 0;
            ctr[0] += __popc(d[k]);
            if (HOT) f[k] |= d[k];
            else f[k] = d[k];
            keep[k] = f[k];
        }
        if (w0 + 4 <= p.words) {
            *reinterpret_cast<uint4*>(Fd + w0) = make_uint4(f[0], f[1], f[2], f[3]);
            if (any) *reinterpret_cast<uint4*>(Vc + w0) = make_uint4(nx[0], nx[1], nx[2], nx[3]);
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (w0 + k < p.words) {
                    Fd[w0 + k] = f[k];
                    if (d[k]) Vc[w0 + k] = nx[k];
                }
        }
        s2_counts<THREADS>(p, w0, f, my_vss, my_sets);
        const bool fany = (f[0] | f[1] | f[2] | f[3]) != 0u;
        if (fany) nzm |= chunk_bit(ch - k0);
        // levels of every discovery of the word — cold (d) and, with the hot view, the hot
        // rows merged into f: one coalesced 128 B store per changed word (lane = bit)
        unsigned ball = __ballot_sync(0xffffffffu, HOT ? fany : any);
        const uint64_t wwarp = ch * CH + 128ull * warp;
        while (ball) {
            const int src = __ffs(ball) - 1;
            ball &= ball - 1;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t dk = __shfl_sync(0xffffffffu, HOT ? f[k] : d[k], src);
                if ((dk >> lane) & 1u) p.L[32 * (wwarp + 4 * src + k) + lane] = level;
            }
        }
    }
    s2_enqueue<THREADS>(p, sm, level, ctr, k0, k1, single, keep, my_vss, my_sets, Fd, nzm);
}

// Hot-row stage 2 (sigma.cuh): the hot prefix of the visited bitmaps (hot_words words,
// one per thread) — diff, V_curr update, and each hot discovery mapped back (σ⁻¹) to RED
// its bit into the original-space frontier Fd (zeroed during stage 1); a grid barrier;
// then lazy_stage2<HOT> sweeps the row words, merges Fd and writes the levels of both
// (coalesced, instead of one scattered store per hot discovery).
template <int THREADS>
__device__ __forceinline__ void lazy_stage2_hot(const Params& p, Smem<THREADS, 1>& sm, uint32_t level,
                                                uint32_t (&ctr)[4], unsigned& gen, uint32_t* Fd) {
    uint32_t* Vc = p.B0;
    uint32_t* Vn = p.B1;
    // word w goes to CTA w mod G: the dense, hottest words (most of the early levels'
    // discoveries) spread over every CTA instead of the first hot_words / THREADS ones
    for (uint64_t w = blockIdx.x + (uint64_t)threadIdx.x * gridDim.x; w < p.hot_words;
         w += (uint64_t)THREADS * gridDim.x) {
        const uint32_t nx = __ldcg(Vn + w), d = nx & ~Vc[w];
        if (!d) continue;
        Vc[w] = nx;
        ctr[0] += __popc(d);
        for (uint32_t rest = d; rest;) {  // σ⁻¹ reads 8 at a time, then their stores / REDs
            uint32_t rr[8], bits = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                rr[t] = 0;
                if (rest) {
                    const int b = __ffs(rest) - 1;
                    rest &= rest - 1;
                    rr[t] = __ldg(p.inv + 32 * w + b);
                    bits |= 1u << t;
                }
            }
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if ((bits >> t) & 1u) red_or(Fd + (rr[t] >> 5), 1u << (rr[t] & 31));  // level: row sweep
        }
    }
    grid_barrier(p.bar, gen);  // the hot discoveries are in Fd
    if ((p.xflags & 32) && blockIdx.x == 0 && threadIdx.x == 0 && level - 1 < p.trace_cap)
        p.tstamp[3ull * (level - 1) + 1] = globaltimer();  // timing study: hot pass end
    lazy_stage2<THREADS, true>(p, sm, level, ctr, Fd);
}

// Small stage 2 (a sparse level whose stage-1 REDs all went into the dirty-word log,
// lazy_pull.cuh RedLog): the same outputs as lazy_stage2(_hot) — V_curr = V_next, levels,
// the next frontier words Fn (all zero beforehand) and the next level's SL — from the
// logged words only, no Θ(n/32) sweep, no block scans, no extra grid barrier. Each logged
// word is claimed with atomicOr(V_curr, V_next) (duplicates in the log find nothing new);
// each discovery ORs its bit into Fn, and the lane that turns its set's byte nonzero owns
// the set: it appends (first position << 32 | set) to SL with one warp-aggregated atomic on
// the packed (sets, VSSs) counter `packed`, so SL stays ordered by first position (not by
// set id) and exactly-once. Totals: packed's VSS part is the next T, its set part the next S.
template <int THREADS, bool SIGMA>
__device__ __forceinline__ void small_stage2(const Params& p, uint32_t level, uint32_t (&ctr)[4], uint32_t* Fn,
                                             const uint32_t* log, uint32_t cnt, unsigned long long* packed) {
    const unsigned lane = lane_id();
    const uint32_t gw = blockIdx.x * (THREADS / 32) + (threadIdx.x >> 5);
    const uint32_t all_warps = gridDim.x * (THREADS / 32);
    const uint64_t hw = SIGMA ? p.hot_words : 0;
    uint32_t* Vc = p.B0;
    const uint32_t* Vn = p.B1;
    for (uint64_t base = (uint64_t)gw * 32; base < cnt; base += (uint64_t)all_warps * 32) {
        const uint64_t i = base + lane;
        uint32_t d = 0, we = 0;
        if (i < cnt) {
            we = log[i];
            const uint32_t nx = __ldcg(Vn + we);
            d = nx & ~atomicOr(Vc + we, nx);
        }
        // the warp's discoveries, 32 per round, whatever word they sit in (a hub word of the
        // hot prefix holds up to 32): lane k takes the k-th set bit of the concatenation
        const uint32_t nb = __popc(d);
        ctr[0] += nb;
        const uint32_t incl = warp_incl_scan(nb), excl = incl - nb;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t k0 = 0; k0 < total; k0 += 32) {
            const uint32_t k = k0 + lane;
            int l = 0;  // the last lane with excl <= k: the word holding discovery k
#pragma unroll
            for (int step = 16; step > 0; step >>= 1)
                if (__shfl_sync(0xffffffffu, excl, l + step) <= k) l += step;
            const uint32_t dw = __shfl_sync(0xffffffffu, d, l), wl = __shfl_sync(0xffffffffu, we, l);
            const uint32_t jth = k - __shfl_sync(0xffffffffu, excl, l);
            bool own = false;
            uint32_t r = 0;
            if (k < total) {
                const uint32_t b = __fns(dw, 0, jth + 1);
                r = (SIGMA && wl < hw) ? __ldg(p.inv + 32ull * wl + b) : 32u * (uint32_t)(wl - hw) + b;
                p.L[r] = level;
                const uint32_t o = atomicOr(Fn + (r >> 5), 1u << (r & 31));
                own = ((o >> (8 * ((r >> 3) & 3))) & 0xFFu) == 0;
            }
            const uint32_t ss = r >> 3;
            uint32_t c = 0;
            if (own) c = __ldg(p.rp + ss + 1) - __ldg(p.rp + ss);
            const unsigned long long v = c ? pack_vs(c, 1) : 0ull;
            unsigned long long vin = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, vin, o);
                if (lane >= (unsigned)o) vin += y;
            }
            unsigned long long at = 0;
            if (lane == 31 && vin) at = atomicAdd(packed, vin);
            at = __shfl_sync(0xffffffffu, at, 31) + vin - v;
            if (c) {
                p.SL[at >> (64 - kSetBits)] = ((at & kVssMask) << 32) | ss;
                ctr[3] += c;
            }
        }
    }
}

}  // namespace bfsdev
}  // namespace blestgpu
