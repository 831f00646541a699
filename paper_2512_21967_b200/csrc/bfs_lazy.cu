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
#include "lazy_pull.cuh"

namespace blestgpu {

namespace {
using namespace bfsdev;


#ifndef BLEST_MINB
#define BLEST_MINB 1
#endif
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
        for (int i = 2; i < 16; ++i) p.ctl[i] = 0;
        p.ctl[12] = 1;  // vertices visited so far (the source)
        for (int i = 0; i < 8; ++i) p.trace[i] = 0;
    }
    // Exhaustion exit: a vertex can only be discovered through a BVSS row, so once the
    // visited count reaches |rows ∪ {src}| no level can discover anything — the next level
    // is the barren last one, and its trace row (queue = T, every other count 0) is known
    // without pulling it (urand C3: the 2.2 M-VSS final level; BLEST_EXHAUST=0 disables).
    const uint64_t reach = p.present_rows
                               ? p.present_rows + (((p.present[src >> 5] >> (src & 31)) & 1u) ? 0u : 1u)
                               : ~0ull;
    unsigned long long visited = 1;
    uint32_t next_T = grid_barrier_pay(p.bar, gen, &p.ctl[0]);
    // The level array (4n bytes, the bulk of init_state) is written after the init barrier:
    // its stores drain while level 1's stage 1 runs (nothing reads L), and the barrier after
    // that stage orders them before stage 2's first level stores (~5 µs per BFS).
    for (uint64_t i = gtid; i < p.n; i += gthreads) p.L[i] = (i == src) ? 0u : kInf;

    uint32_t ctr[4] = {0, 0, 0, 0};  // discovered, full, relaxed, pushes
    bool prev_small = false;  // the last stage 2 was small_stage2 (uniform over the grid)
    uint32_t level = 1;
    for (;; ++level) {
        const unsigned long long len = next_T;  // broadcast by the barrier
        // S: the full stage 2 stores it in ctl[1]; small_stage2 packs it with T (ctl[8|9])
        const uint32_t S = prev_small
                               ? (uint32_t)(ld_relaxed_gpu_u64(&p.ctl[8 + ((level - 1) & 1)]) >> (64 - kSetBits))
                               : (uint32_t)ld_relaxed_gpu_u64(&p.ctl[1]);
        if (len == 0) break;
        if (level > p.cap) {  // runaway (R:src/bfs_engine.cpp:72-75)
            if (gtid == 0) p.ctl[6] = 1;
            break;
        }
        if (gtid == 0) {
            p.ctl[7] = 0;  // stage-1 tail chunk counter (read after the expansion barrier)
            p.ctl[2 + ((level + 1) & 1)] = 0;  // the next level's RED flag (last read at level - 1)
            p.ctl[8 + (level & 1)] = 0;         // small stage 2 counter (last read at level - 1's start)
            p.ctl[10 + ((level + 1) & 1)] = 0;  // the next level's dirty-word log count
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
        if (visited >= reach) {  // barren by exhaustion (uniform: every thread read the same count)
            if (gtid == 0) {
                p.ctl[13] = len;  // VSSs accounted without a pull (bench: bytes actually streamed)
                if (level - 1 < p.trace_cap) {
                    const unsigned long long t = globaltimer();
                    p.tstamp[3ull * (level - 1) + 1] = t;
                    p.tstamp[3ull * (level - 1) + 2] = t;
                }
            }
            ++level;  // the barren level counts as an iteration (R:src/bfs_engine.cpp:117-124)
            break;
        }
        unsigned long long* Qc = p.Q0;
        // the level's frontier words (α) and the next level's: B2/B3 alternate, so the next
        // frontier can be cleared while this one is still being read (no barrier between)
        const uint32_t* Fd = (level & 1) ? p.B2 : p.B3;
        uint32_t* Fn = (level & 1) ? p.B3 : p.B2;
        const uint8_t* Fd8 = reinterpret_cast<const uint8_t*>(Fd);
        const bool recheck = p.lazy_recheck != 0;  // W = V_curr + V_next re-check (older scheme)
        PullCtx pc;
        pc.rp = p.rp;
        pc.masks = p.masks;
        pc.rows4 = rows4;
        pc.Fd8 = Fd8;
        pc.SL = p.SL;
        pc.Q = Qc;
        pc.tail_ctr = &p.ctl[7];
        pc.W = recheck ? Vc : Vn;
        pc.Vn = Vn;
        pc.len = len;
        pc.S = S;
        pc.sent = (uint32_t)vwords;  // sentinel word (all ones) after the bitmap
        pc.recheck = recheck;
        pc.tail_div = p.tail_div;
        pc.gw = gw;
        pc.NW = NW;
        pc.all_warps = all_warps;
        pc.pol = pol;
        const bool sparse = len < p.dense_min;
        if (sparse) {
            // Fn is the previous level's α (its readers finished long ago): cleared here for
            // the hot view's stage 2 and for small_stage2, which writes only discoveries
            for (uint64_t w = gtid; w < p.words; w += gthreads) Fn[w] = 0;
            pc.log.words = reinterpret_cast<uint32_t*>(p.Q0);  // the queue is unused on sparse levels
            pc.log.count = &p.ctl[10 + (level & 1)];
            pc.log.cap = p.log_cap;
            ctr[2] += pull_sparse<PULL, true>(pc);
        } else {
            expand_queue(pc);
            if (SIGMA)
                for (uint64_t w = gtid; w < p.words; w += gthreads) Fn[w] = 0;
            grid_barrier(p.bar, gen);
            // ---- stage 1: pull (pull_vss, R:src/bfs_engine.cpp:131-146) ----
            ctr[2] += pull_dense<PULL>(pc);
        }
        // No RED this level ⇔ no discovery (a RED is the only way a V_next bit gets set, and
        // the barrier before the stage made every earlier bit visible to the tests): the
        // level is the barren last one — skip its Θ(n/32) stage 2 (one per BFS, ~17 µs).
        // (sparse levels: the payload is the dirty-word log count, zero iff no RED)
        const uint32_t s1 = sparse ? level_barrier(p, sm, gen, level, ctr, 1, &p.ctl[10 + (level & 1)])
                                   : level_barrier(p, sm, gen, level, ctr, 1, nullptr, &p.ctl[2 + (level & 1)]);
        if (s1 == 0) {
            if (gtid == 0 && level - 1 < p.trace_cap) p.tstamp[3ull * (level - 1) + 2] = globaltimer();
            ++level;  // the barren level counts as an iteration (R:src/bfs_engine.cpp:117-124)
            break;
        }

        prev_small = sparse && s1 <= p.log_cap;  // the log holds every RED'd word
        if (prev_small) {
            small_stage2<THREADS, SIGMA>(p, level, ctr, Fn, reinterpret_cast<const uint32_t*>(p.Q0), s1,
                                         &p.ctl[8 + (level & 1)]);
            next_T = level_barrier(p, sm, gen, level, ctr, 2, &p.ctl[8 + (level & 1)], nullptr, &p.ctl[12], &visited);
        } else {
            if (SIGMA)
                lazy_stage2_hot<THREADS>(p, sm, level, ctr, gen, Fn);
            else
                lazy_stage2<THREADS>(p, sm, level, ctr, Fn);
            next_T = level_barrier(p, sm, gen, level, ctr, 2, &p.ctl[0], nullptr, &p.ctl[12], &visited);
        }
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
