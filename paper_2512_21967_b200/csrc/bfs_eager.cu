// Eager engine (BLEST Alg. 2; run_eager, R:src/bfs_engine.cpp:155-236) as one fused
// persistent cooperative kernel: init_state and every level in one launch, one grid
// barrier per level (it also broadcasts the next queue length).
//
// Work unit = one VSS handled by one warp (lane t: its mask word, one coalesced 128 B line
// per VSS, and its 4 row ids, one 16 B load; streaming loads). Warps take queue positions
// round-robin exactly like the reference (p ≡ warp mod #warps, :190), kBatch at a time.
// Queue entries are 64-bit: low = VSS id, high = slice set (saves virtual_to_real, :192);
// α is the set's byte of F_curr (frontier_byte :148-151), loaded beside the mask/row loads.
//
// Sink (:198-211): the reference's levels[u] test becomes one visited bitmap VIS
// (n/8 bytes, L1/L2-resident, unlike the 4n-byte level array) holding every discovery of
// the previous levels (and, lagging, of this one). A clear VIS bit goes to an atomicOr on
// F_next, which ELECTS the discoverer (old bit clear) and, through its old byte, tells
// whether u is its slice set's first discovery this level (:204-205) ⇒ push the set's VSS
// range; the discoverer stores levels[u] = ℓ and REDs u into VIS. The tests of a warp's
// whole batch (kBatch VSSs × 4 columns per lane) run as phases — all VIS loads, then (dense
// levels) the F_next re-checks at L2, then the atomics — so each phase costs one latency.
// Pushes gather in a per-warp shared buffer; a flush reserves queue space with ONE
// atomicAdd per buffer (warp-aggregated reservation) and expands [real_ptrs[s], real_ptrs[s+1]).
//
// Frontier bitmaps are triple-buffered: level ℓ reads F[ℓ%3], ORs into F[(ℓ+1)%3], and
// zeroes the bytes of F[(ℓ+2)%3] that level ℓ-1 read (set ids fetched from queue ℓ-1 at
// the level's start, stores issued after the pull), so no Θ(n) clear is ever needed
// (the reference clears every word, :227-228) and nothing sits on the level's critical path.
#include <atomic>

#include "bfs.cuh"
#include "bfs_device.cuh"

namespace blestgpu {

namespace {
using namespace bfsdev;

// Row id of flat candidate k (VSS k / 4, column k % 4); constant-folded when unrolled.
__device__ __forceinline__ uint32_t row_of(const uint4 (&rw)[kBatch], int k) {
    const uint4& r = rw[k >> 2];
    return (k & 3) == 0 ? r.x : (k & 3) == 1 ? r.y : (k & 3) == 2 ? r.z : r.w;
}

template <int PULL, int THREADS>
#ifndef BLEST_EAGER_MINB
#define BLEST_EAGER_MINB 1
#endif
__global__ void __launch_bounds__(THREADS, BLEST_EAGER_MINB) k_bfs_eager(Params p) {
    constexpr int WPC = THREADS / 32;
    __shared__ Smem<THREADS, 0> sm;
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
    uint32_t* VIS = p.B3;

    // ---- init_state (R:src/bfs_engine.cpp:30-49), fused ----
    const uint32_t src = p.src;
    const uint32_t sset = src / kSigma;
    const uint32_t seed_b = p.rp[sset], seed_e = p.rp[sset + 1];
    for (uint64_t i = gtid; i < p.n; i += gthreads) p.L[i] = (i == src) ? 0u : kInf;
    const uint32_t src_word = src >> 5, src_bit = 1u << (src & 31);
    for (uint64_t w = gtid; w < p.words; w += gthreads) {
        const uint32_t seed = (w == src_word) ? src_bit : 0u;
        p.B0[w] = 0;
        p.B1[w] = seed;  // F[1] = F_curr of level 1
        p.B2[w] = 0;
        VIS[w] = seed;  // every discovery so far (the source)
    }
    {
        const unsigned long long aux = (unsigned long long)sset << 32;
        for (uint64_t i = gtid; i < seed_e - seed_b; i += gthreads) p.Q1[i] = aux | (seed_b + i);
    }
    if (gtid == 0) {
        p.ctl[0] = 0;
        p.ctl[1] = seed_e - seed_b;
        for (int i = 2; i < 8; ++i) p.ctl[i] = 0;
        p.ctl[13] = 0;  // VSSs of a barren level accounted without a pull
        for (int i = 0; i < 8; ++i) p.trace[i] = 0;
    }
    // Exhaustion exit (as in the lazy kernel): the next level is barren once 1 + Σ discovered
    // reaches |BVSS rows ∪ {src}|. Nothing is added to a sparse level (C4 runs 8.6 K of them;
    // reading the trace rows at every barrier cost it 8 %): after a DENSE level, whose CTAs
    // add their discoveries to its trace row before the barrier, thread 0 of every CTA sums
    // the trace rows not summed yet — all final then — so the count is exact after a dense
    // level and stale (low: never an early exit) after a sparse one.
    // (state in shared memory: registers are what this kernel is short of)
    __shared__ unsigned long long s_vis, s_reach;  // 1 + Σ discovered of trace rows [0, s_summed)
    __shared__ uint32_t s_summed;
    if (threadIdx.x == 0) {
        s_reach = p.present_rows ? p.present_rows + (((p.present[src >> 5] >> (src & 31)) & 1u) ? 0u : 1u) : ~0ull;
        s_vis = 1;
        s_summed = 0;
    }
    uint32_t next_len = grid_barrier_pay(p.bar, gen, &p.ctl[1]);

    unsigned long long* pbuf = sm.push[warp];
    uint32_t pcount = 0;
    uint32_t ctr[4] = {0, 0, 0, 0};  // discovered, full, relaxed, pushes
    unsigned long long prev_len = 0;  // length of queue ℓ-1 (its sets' F bytes get zeroed)
    uint32_t level = 1;
    for (;; ++level) {
        const unsigned long long len = next_len;
        if (len == 0) break;
        if (level > p.cap) {  // runaway (R:src/bfs_engine.cpp:72-75)
            if (gtid == 0) p.ctl[6] = 1;
            break;
        }
        if (gtid == 0) {
            p.ctl[(level + 2) & 3] = 0;
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
        if (s_vis >= s_reach) {  // barren by exhaustion (uniform: every CTA read the same rows)
            if (gtid == 0) {
                p.ctl[13] = len;
                if (level - 1 < p.trace_cap) {
                    const unsigned long long t = globaltimer();
                    p.tstamp[3ull * (level - 1) + 1] = t;
                    p.tstamp[3ull * (level - 1) + 2] = t;
                }
            }
            ++level;  // the barren level counts as an iteration (R:src/bfs_engine.cpp:117-124)
            break;
        }
        // triple buffers by select (a runtime-indexed array would live in local memory)
        auto qsel = [&](uint32_t k) { return k == 0 ? p.Q0 : (k == 1 ? p.Q1 : p.Q2); };
        auto fsel = [&](uint32_t k) { return k == 0 ? p.B0 : (k == 1 ? p.B1 : p.B2); };
        const uint32_t k0 = level % 3, k1 = (level + 1) % 3, k2 = (level + 2) % 3;
        const unsigned long long* Qc = qsel(k0);
        unsigned long long* Qn = qsel(k1);
        const uint8_t* Fc8 = reinterpret_cast<const uint8_t*>(fsel(k0));
        uint32_t* Fn = fsel(k1);
        unsigned long long* qlen_next = &p.ctl[(level + 1) & 3];
        // Frontier bytes level ℓ-1 read (sets of queue ℓ-1) become F_next at ℓ+1: fetch this
        // thread's set id now, store the zero after the pull (latency hidden by the pull).
        uint8_t* Fz = reinterpret_cast<uint8_t*>(fsel(k2));
        const unsigned long long* Qz = qsel(k2);
        const uint32_t zss = (gtid < prev_len) ? (uint32_t)(Qz[gtid] >> 32) : 0xFFFFFFFFu;

        const bool recheck = len >= p.dense_min;  // sparse levels: straight to the atomic
        // ---- pull over the queue (pull_vss, R:src/bfs_engine.cpp:131-146) ----
        if (gw < NW) {
            // queue entries two batches ahead; on dense levels the lines of batch i+2 are
            // prefetched into L2 once batch i's tests are issued (see the lazy kernel)
            auto qload = [&](uint64_t base) -> unsigned long long {
                const uint64_t pos = base + (uint64_t)lane * NW;
                return (lane < kBatch && pos < len) ? Qc[pos] : kNoEntry;
            };
            const uint64_t step = (uint64_t)NW * kBatch;
            const bool pf = recheck && !(p.xflags & 512);
            unsigned long long e_next = qload(gw), e_next2 = qload(gw + step);
            for (uint64_t p0 = gw; p0 < len; p0 += step) {
                const unsigned long long e = e_next;
                e_next = e_next2;
                e_next2 = qload(p0 + 2 * step);
                const uint32_t alpha_l = (e != kNoEntry) ? Fc8[e >> 32] : 0u;  // frontier_byte
                uint32_t mk[kBatch];
                uint4 rw[kBatch];
                unsigned long long ej[kBatch];
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    ej[j] = __shfl_sync(0xffffffffu, e, j);
                    mk[j] = 0;
                    rw[j] = make_uint4(0, 0, 0, 0);
                    if (ej[j] != kNoEntry) {
                        const uint64_t v = (uint32_t)ej[j];
                        mk[j] = ld_stream_u32(p.masks + 32 * v + lane, pol);
                        rw[j] = ld_stream_u4(p.rows4 + 32 * v + lane, pol);
                    }
                }
                // Sink (R:src/bfs_engine.cpp:198-211) in batch-wide phases, each phase's
                // memory operations in flight together (branch-free PTX blocks): (A) VIS word
                // (L1) of every column with a nonzero pull; (B) dense levels only: F_next at
                // L2 for the rest (claimed this level already?) to spare the atomic; (C)
                // atomicOr on F_next elects the discoverer (old bit clear) and its old byte
                // says whether it is the set's first discovery this level (push, :204-205);
                // (D) the discoverer stores the level and REDs its VIS bit.
                const bool first = p0 == gw;
                probe(p, level, 4096, mk[0] ^ rw[0].x ^ alpha_l, first);
                uint32_t vw[4 * kBatch];
                if (PULL == 0) {
#pragma unroll
                    for (int j = 0; j < kBatch; ++j) {  // absent entries: no candidates
                        const uint32_t a = ej[j] != kNoEntry ? __shfl_sync(0xffffffffu, alpha_l, j) : 0u;
                        const uint32_t m = mk[j] & (a * 0x01010101u);
#pragma unroll
                        for (int c = 0; c < 4; ++c) vw[4 * j + c] = cand_word(VIS, row_of(rw, 4 * j + c), m, 0xFFu << (8 * c));
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < kBatch; ++j) {
                        uint32_t cnt[4] = {0, 0, 0, 0};
                        const uint32_t a = __shfl_sync(0xffffffffu, alpha_l, j);
                        if (ej[j] != kNoEntry) column_counts<PULL>(mk[j], a, cnt);  // warp-uniform
#pragma unroll
                        for (int c = 0; c < 4; ++c) vw[4 * j + c] = cand_word(VIS, row_of(rw, 4 * j + c), cnt[c], ~0u);
                    }
                }
                if (recheck) {
#pragma unroll
                    for (int k = 0; k < 4 * kBatch; ++k) vw[k] = recheck_word(Fn, row_of(rw, k), vw[k]);
                }
                probe(p, level, 8192, vw[0] ^ vw[1] ^ vw[2] ^ vw[3], first);
#pragma unroll
                for (int k = 0; k < 4 * kBatch; ++k) {
                    const uint32_t x = row_of(rw, k);
                    ctr[1] += ((vw[k] >> (x & 31)) & 1u) ^ 1u;  // full atomics (R:src/bfs_engine.cpp:203)
                    vw[k] = atom_if_clear(Fn, x, vw[k]);
                }
                probe(p, level, 16384, vw[0] ^ vw[1] ^ vw[2] ^ vw[3], first);
                uint32_t disc = 0;
#pragma unroll
                for (int k = 0; k < 4 * kBatch; ++k) {
                    const uint32_t x = row_of(rw, k);
                    if (!((vw[k] >> (x & 31)) & 1u)) {  // rare: this lane discovered x
                        disc |= 1u << k;
                        p.L[x] = level;
                        red_or(VIS + (x >> 5), 1u << (x & 31));
                    }
                }
                ctr[0] += __popc(disc);
                if (pf) {  // lane 5j + l: line l of VSS j of batch i+2 (l = 0: masks, 1-4: row ids)
                    const int jj = (int)lane / 5, l = (int)lane % 5;
                    const unsigned long long ej = __shfl_sync(0xffffffffu, e_next2, jj < kBatch ? jj : 0);
                    if (jj < kBatch && ej != kNoEntry) {
                        const uint64_t v = (uint32_t)ej;
                        const void* a = l == 0 ? (const void*)(p.masks + 32 * v) : (const void*)(p.rows4 + 32 * v + 8 * (l - 1));
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
                    }
                }
                if (__any_sync(0xffffffffu, disc != 0)) {
#pragma unroll
                    for (int k = 0; k < 4 * kBatch; ++k) {
                        const uint32_t x = row_of(rw, k);
                        const bool push = ((disc >> k) & 1u) && ((vw[k] >> (8 * ((x >> 3) & 3))) & 0xFFu) == 0;
                        push_column(p, push, (unsigned long long)(x >> 3) << 32 | (x >> 3), pbuf, pcount, Qn,
                                    qlen_next, ctr[3], ctr[1], !recheck && !(p.xflags & 1024));
                    }
                }
            }
        }
        if (pcount) {
            const uint32_t t = flush_pushes(p, pbuf, pcount, Qn, qlen_next, !recheck && !(p.xflags & 1024));
            if (lane == 0) {
                ctr[3] += t;
                ctr[1] += 1;
            }
        }
        probe(p, level, 32768, pcount, true);
        if (zss != 0xFFFFFFFFu) Fz[zss] = 0;
        for (uint64_t i = gtid + gthreads; i < prev_len; i += gthreads) Fz[Qz[i] >> 32] = 0;
        prev_len = len;
        probe(p, level, 65536, ctr[0], true);
        if ((p.xflags & (1u << 19)) && blockIdx.x == 0 && lane == 0 && level - 1 < p.trace_cap)  // timing study:
            atomicMax(&p.tstamp[3ull * (level - 1) + 1], globaltimer());                      // CTA 0's last warp
        if ((p.xflags & (1u << 20)) && lane == 0 && level - 1 < p.trace_cap)  // timing study: the grid's last warp
            atomicMax(&p.tstamp[3ull * (level - 1) + 1], globaltimer());
        if ((p.xflags & 64) && threadIdx.x == 0 && level - 1 < p.trace_cap)  // timing study:
            atomicMax(&p.tstamp[3ull * (level - 1) + 1], globaltimer());      // last CTA's pull end
        const bool track = p.present_rows && recheck && level < p.trace_cap;  // row level-1 not clamped
        next_len = level_barrier(p, sm, gen, level, ctr, 2, qlen_next, nullptr, nullptr, nullptr, track);
        if (track) {  // uniform: rows [s_summed, level) are final now
            if (threadIdx.x == 0) {
                unsigned long long add = 0;
                for (uint32_t k = s_summed; k < level; ++k) add += ld_relaxed_gpu_u64(&p.trace[8ull * k + 3]);
                s_vis += add;
                s_summed = level;
            }
            __syncthreads();
        }
    }
    if (gtid == 0) p.ctl[4] = level - 1;
}

}  // namespace

void* eager_kernel(int pull, int threads) {
    if (pull == 1) {
        switch (threads) {
            case 256: return (void*)k_bfs_eager<1, 256>;
            case 512: return (void*)k_bfs_eager<1, 512>;
            case 1024: return (void*)k_bfs_eager<1, 1024>;
        }
    } else {
        switch (threads) {
            case 256: return (void*)k_bfs_eager<0, 256>;
            case 512: return (void*)k_bfs_eager<0, 512>;
            case 1024: return (void*)k_bfs_eager<0, 1024>;
        }
    }
    throw InvalidArgument("threads per CTA must be 256, 512 or 1024");
}

}  // namespace blestgpu
