// Lazy engine (BLEST Alg. 3; run_lazy, R:src/bfs_engine.cpp:238-350), TMA-pipelined:
// one fused persistent cooperative kernel per source.
//
// Queue. The level's queue is the ascending list SL of active slice sets, each entry the
// set id and the queue position of its first VSS; positions in between are implicit
// (v = real_ptrs[s] + offset). The dequeued VSS multiset — hence every counter — is the
// reference's (:323-330 pushes each set's whole VSS range), but stage 2 writes one entry
// per set, so it is balanced even when a hub set owns thousands of VSSs.
//
// Stage 1 (pull, :273-292), warp-specialised per CTA:
//   producer warp  — owns the CTA's contiguous queue positions [c·T/G, (c+1)·T/G), walks
//                    SL with a 32-set window in its lanes, and for every stage of kSB
//                    positions issues cp.async.bulk copies of each VSS's 128 B mask line
//                    and 512 B row-id block into a shared-memory ring slot, completing on
//                    that slot's mbarrier (expect_tx); α of each VSS rides in a slot header;
//   consumer warps — take ring slots round-robin, copy the slot to registers, release it,
//                    AND each lane's masks with α and run the visited test per nonzero
//                    column: V_curr (frozen during the stage, L1-cached), then V_next at L2,
//                    then a fire-and-forget RED (legal per SURVEY §8(a) pitfall 7).
// The HBM stream thus runs kNS stages ahead of the latency-bound visited checks instead of
// waiting behind them.
//
// Stage 2 (word sweep, :296-338): each CTA owns a contiguous chunk of the ⌈n/32⌉ words.
// Pass A: diff = V_next & ~V_curr, V_curr |= diff, diff words kept (they carry α for the
// next level, like the reference's in-place F_curr :310-311), levels written with one
// coalesced 128 B store per changed word, set/VSS counts reduced. The CTA publishes both
// counts (tagged with the level) and sums its predecessors'; pass B writes its SL entries.
#include "bfs.cuh"
#include "bfs_device.cuh"
#include "lazy_pull.cuh"

namespace blestgpu {

namespace {
using namespace bfsdev;

constexpr int kSB = 16;                        // VSSs per ring slot
// Ring slots per CTA = consumer warps: stage g uses slot g % NC and consumer g % NC, so
// every slot is only ever refilled for the warp that emptied it (a consumer can never
// wait on a later phase of a slot before the earlier one was consumed).
constexpr int kCB = 4;                         // VSSs a consumer holds in registers at once
constexpr uint32_t kSlotBytes = kSB * 640;     // 16 x (128 B masks + 512 B row ids)

struct SlotHdr {
    uint32_t count;
    uint32_t alpha[kSB / 4];  // frontier bytes, 4 per word
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    uint32_t done = 0;
    uint64_t t0 = 0;
    for (uint32_t spins = 0;; ++spins) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
        if (done) break;
        if ((spins & 1023) == 0) {  // watchdog: abort the launch instead of hanging the GPU
            uint64_t t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            if (!t0) t0 = t;
            else if (t - t0 > 4000000000ull) __trap();
        }
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}

template <int PULL, int NC>
__global__ void __launch_bounds__(32 * (NC + 1)) k_bfs_lazy_tma(Params p) {
    constexpr int THREADS = 32 * (NC + 1);
    __shared__ Smem<THREADS, 1> sm;
    constexpr int kNS = NC;
    __shared__ __align__(8) uint64_t full[kNS], empty[kNS];
    __shared__ SlotHdr hdr[kNS];
    extern __shared__ __align__(128) uint8_t ring[];  // kNS slots of kSlotBytes
    const unsigned lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t gtid = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    const uint64_t gthreads = (uint64_t)gridDim.x * THREADS;
    unsigned gen = 0;
    const uint64_t pol = evict_first_policy();
    uint32_t* Vc = p.B0;
    uint32_t* Vn = p.B1;
    uint32_t* Fd = p.B2;
    const uint8_t* Fd8 = reinterpret_cast<const uint8_t*>(Fd);
    if (threadIdx.x < 4) sm.ctr[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // ---- init_state (R:src/bfs_engine.cpp:30-49), fused ----
    const uint32_t src = p.src;
    const uint32_t sset = src / kSigma;
    const uint32_t seed_b = p.rp[sset], seed_e = p.rp[sset + 1];
    for (uint64_t i = gtid; i < p.n; i += gthreads) p.L[i] = (i == src) ? 0u : kInf;
    const uint32_t src_word = src >> 5, src_bit = 1u << (src & 31);
    for (uint64_t w = gtid; w < p.words; w += gthreads) {
        const uint32_t seed = (w == src_word) ? src_bit : 0u;
        Vc[w] = seed;
        Vn[w] = seed;
        Fd[w] = seed;  // α of the source's set for level 1
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
    grid_barrier(p.bar, gen);

    uint32_t ctr[4] = {0, 0, 0, 0};  // discovered, full, relaxed, pushes
    uint32_t ring_base = 0;           // slots consumed by earlier levels (same in every warp)
    uint32_t level = 1;
    for (;; ++level) {
        const unsigned long long T = ld_relaxed_gpu_u64(&p.ctl[0]);
        const uint32_t S = (uint32_t)ld_relaxed_gpu_u64(&p.ctl[1]);
        if (T == 0) break;
        if (level > p.cap) {  // runaway (R:src/bfs_engine.cpp:72-75)
            if (gtid == 0) p.ctl[6] = 1;
            break;
        }
        if (gtid == 0) {
            if (level - 1 < p.trace_cap) {
                p.trace[8ull * (level - 1) + 0] = level;
                p.trace[8ull * (level - 1) + 1] = T;
                p.tstamp[3ull * (level - 1)] = globaltimer();
            } else {
                atomicAdd(&p.trace[8ull * (p.trace_cap - 1) + 1], T);
            }
            if (level < p.trace_cap)
                for (int i = 0; i < 8; ++i) p.trace[8ull * level + i] = 0;
        }

        // ---- stage 1 ----
        const uint64_t lo = (uint64_t)blockIdx.x * T / gridDim.x;
        const uint64_t hi = (uint64_t)(blockIdx.x + 1) * T / gridDim.x;
        const uint32_t nst = (uint32_t)((hi - lo + kSB - 1) / kSB);
        if (warp == 0) {
            // producer
            if (nst) {
                SetWindow win;
                load_window(p.SL, p.rp, Fd8, find_set(p.SL, S, lo), S, T, win);
                for (uint32_t i = 0; i < nst; ++i) {
                    const uint32_t g = ring_base + i, s = g % kNS;
                    const uint64_t sp = lo + (uint64_t)i * kSB;
                    const uint32_t cnt = (hi - sp < (uint64_t)kSB) ? (uint32_t)(hi - sp) : (uint32_t)kSB;
                    if (sp + cnt - 1 >= win.wend) {  // slide the window to the set holding sp
                        const unsigned own = __ballot_sync(0xffffffffu, win.first <= sp);
                        const uint32_t nb = (sp >= win.wend) ? win.base + 32 : win.base + (31 - __clz(own));
                        load_window(p.SL, p.rp, Fd8, nb, S, T, win);
                    }
                    // lane j < kSB resolves position sp + j: binary search of the
                    // window's first positions (5 shuffle steps, all lanes at once)
                    const uint64_t q = sp + (lane < kSB ? lane : 0);
                    int l = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const uint64_t f = __shfl_sync(0xffffffffu, win.first, l + step);
                        if (f <= q) l += step;
                    }
                    const uint32_t myv = __shfl_sync(0xffffffffu, win.b, l) +
                                         (uint32_t)(q - __shfl_sync(0xffffffffu, win.first, l));
                    const uint32_t la = __shfl_sync(0xffffffffu, win.alpha, l);  // all lanes shuffle
                    const uint32_t mya = (lane < cnt) ? la : 0u;
                    // runs of consecutive VSS ids become one bulk copy each
                    const uint32_t prevv = __shfl_up_sync(0xffffffffu, myv, 1);
                    const bool start = lane < cnt && (lane == 0 || prevv + 1 != myv);
                    const unsigned starts = __ballot_sync(0xffffffffu, start) | (1u << cnt);
                    const uint32_t run = start ? (__ffs(starts & ~((2u << lane) - 1)) - 1 - lane) : 0u;
                    if (g >= kNS) mbar_wait(&empty[s], ((g / kNS) - 1) & 1);
                    const uint32_t a4 = mya | (__shfl_down_sync(0xffffffffu, mya, 1) << 8) |
                                        (__shfl_down_sync(0xffffffffu, mya, 2) << 16) |
                                        (__shfl_down_sync(0xffffffffu, mya, 3) << 24);
                    if (lane < kSB && (lane & 3) == 0) hdr[s].alpha[lane >> 2] = a4;
                    if (lane == 0) hdr[s].count = cnt;
                    __syncwarp();
                    if (lane == 0) mbar_arrive_expect_tx(&full[s], cnt * 640);
                    __syncwarp();
                    if (start) {
                        uint8_t* slot = ring + (size_t)s * kSlotBytes;
                        bulk_g2s(slot + lane * 128, p.masks + 32ull * myv, run * 128, &full[s], pol);
                        bulk_g2s(slot + kSB * 128 + lane * 512, p.rows4 + 32ull * myv, run * 512, &full[s], pol);
                    }
                }
            }
        } else {
            // consumers
            for (uint32_t i = warp - 1; i < nst; i += NC) {
                const uint32_t g = ring_base + i, s = g % kNS;
                mbar_wait(&full[s], (g / kNS) & 1);
                const uint32_t cnt = hdr[s].count;
                const uint8_t* slot = ring + (size_t)s * kSlotBytes;
                for (int j0 = 0; j0 < (int)cnt; j0 += kCB) {
                    const uint32_t alphas = hdr[s].alpha[j0 >> 2];
                    uint32_t mk[kCB];
                    uint4 rw[kCB];
#pragma unroll
                    for (int j = 0; j < kCB; ++j) {
                        mk[j] = reinterpret_cast<const uint32_t*>(slot + (j0 + j) * 128)[lane];
                        rw[j] = reinterpret_cast<const uint4*>(slot + kSB * 128 + (j0 + j) * 512)[lane];
                    }
                    if (j0 + kCB >= (int)cnt) {  // slot fully copied out: hand it back
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[s]);
                    }
#pragma unroll
                    for (int j = 0; j < kCB; ++j) {
                        if (j0 + j >= (int)cnt) break;  // warp-uniform
                        uint32_t c4[4];
                        column_counts<PULL>(mk[j], (alphas >> (8 * j)) & 0xFFu, c4);
                        const uint32_t u[4] = {rw[j].x, rw[j].y, rw[j].z, rw[j].w};
                        uint32_t vw[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) vw[c] = c4[c] ? Vc[u[c] >> 5] : ~0u;
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if (!((vw[c] >> (u[c] & 31)) & 1u)) vw[c] = ld_l2_u32(Vn + (u[c] >> 5));
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            if (!((vw[c] >> (u[c] & 31)) & 1u)) {
                                red_or(Vn + (u[c] >> 5), 1u << (u[c] & 31));
                                ++ctr[2];
                            }
                        }
                    }
                }
            }
        }
        ring_base += nst;
        level_barrier(p, sm, gen, level, ctr, 1);

        lazy_stage2<THREADS>(p, sm, level, ctr);
        level_barrier(p, sm, gen, level, ctr, 2);
    }
    if (gtid == 0) p.ctl[4] = level - 1;
}

}  // namespace

size_t lazy_tma_smem(int consumers) { return (size_t)consumers * kSlotBytes; }

void* lazy_tma_kernel(int pull, int consumers) {
    if (consumers == 8) return pull == 1 ? (void*)k_bfs_lazy_tma<1, 8> : (void*)k_bfs_lazy_tma<0, 8>;
    if (consumers == 16) return pull == 1 ? (void*)k_bfs_lazy_tma<1, 16> : (void*)k_bfs_lazy_tma<0, 16>;
    throw InvalidArgument("consumer warps per CTA must be 8 or 16");
}

}  // namespace blestgpu
