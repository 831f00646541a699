// Lazy engine (BLEST Alg. 3; run_lazy, R:src/bfs_engine.cpp:238-350) as one fused
// persistent cooperative kernel.
//
// Queue. The reference pushes every VSS of each newly active slice set (:323-330). Here the
// level's queue is the ascending list of active slice sets SL, each entry holding the
// set id and the queue position of its first VSS; the VSS positions in between are
// implicit (v = real_ptrs[s] + position offset). The dequeued VSS multiset — and so
// every counter — is exactly the reference's, but stage 2 writes one 8-byte entry per
// set instead of one per VSS, and stage 1 can split positions evenly over warps.
//
// Stage 1 (pull, :273-292). Warp w owns the contiguous positions [w·T/W, (w+1)·T/W)
// (balanced to one VSS, the reference's load-balance contract :190). It locates its
// first set with a 32-ary search of SL, keeps a window of 32 consecutive sets in its
// lanes (set id, first position, first VSS, frontier byte α read from this level's diff
// words), and resolves each position with one ballot. Per VSS: one coalesced 128 B mask
// line and four 128 B row-id lines (streaming loads), AND with α, and for every nonzero
// column the visited test: V_curr (frozen during the stage, L1-cached) and, if clear,
// V_next at L2; only then a fire-and-forget RED sets the V_next bit (legal per SURVEY
// §8(a) pitfall 7).
//
// Stage 2 (word sweep, :296-338). Each CTA owns a contiguous chunk of the ⌈n/32⌉ words.
// Pass A: diff = V_next & ~V_curr, V_curr |= diff, diff words kept (they carry α for the
// next stage 1, as the reference's in-place F_curr, :310-311), levels written with one
// coalesced 128 B store per changed word, and the chunk's set and VSS counts reduced.
// The CTA publishes both counts (tagged with the level) and sums its predecessors';
// pass B writes its SL entries at that offset. No contended atomics; deterministic.
#include "bfs.cuh"
#include "bfs_device.cuh"

namespace blestgpu {

namespace {
using namespace bfsdev;

constexpr unsigned long long kTagMask = (1ull << 40) - 1;

// One warp's view of 32 consecutive SL entries.
struct SetWindow {
    uint32_t base;   // SL index held by lane 0
    uint64_t first;  // lane's first queue position (UINT64_MAX past the list)
    uint32_t b;      // lane's first VSS id (real_ptrs[s])
    uint32_t alpha;  // lane's frontier byte
    uint64_t wend;   // one past the last position covered by the window
};

__device__ __forceinline__ void load_window(const Params& p, const uint8_t* Fd8, uint32_t base, uint32_t S,
                                            uint64_t T, SetWindow& w) {
    const unsigned lane = lane_id();
    const uint32_t k = base + lane;
    uint64_t first = ~0ull;
    uint32_t b = 0, alpha = 0;
    if (k < S) {
        const unsigned long long e = p.SL[k];
        first = e >> 32;
        const uint32_t ss = (uint32_t)e;
        b = p.rp[ss];
        alpha = Fd8[ss];
    }
    // end of lane 31's set: next entry's first position, or T
    uint64_t nxt = T;
    if (lane == 31 && k + 1 < S) nxt = p.SL[k + 1] >> 32;
    w.base = base;
    w.first = first;
    w.b = b;
    w.alpha = alpha;
    const uint64_t last_first = __shfl_sync(0xffffffffu, first, 31);
    w.wend = (base + 32 < S) ? __shfl_sync(0xffffffffu, nxt, 31) : T;
    (void)last_first;
}

// Largest SL index k with first(k) <= pos (SL sorted by first; first(0) = 0).
__device__ __forceinline__ uint32_t find_set(const Params& p, uint32_t S, uint64_t pos) {
    const unsigned lane = lane_id();
    uint32_t lo = 0, hi = S;  // answer in [lo, hi)
    while (hi - lo > 32) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t idx = lo + lane * step;
        const bool ok = idx < hi && (p.SL[idx] >> 32) <= pos;
        const unsigned ball = __ballot_sync(0xffffffffu, ok);
        const uint32_t last = 31 - __clz(ball);  // lane 0 always ok (first(lo) <= pos)
        lo = lo + last * step;
        hi = min(hi, lo + step);
    }
    const uint32_t idx = lo + lane;
    const bool ok = idx < hi && (p.SL[idx] >> 32) <= pos;
    const unsigned ball = __ballot_sync(0xffffffffu, ok);
    return lo + (31 - __clz(ball));
}

template <int PULL, int THREADS>
__global__ void __launch_bounds__(THREADS) k_bfs_lazy(Params p) {
    constexpr int WPC = THREADS / 32;
    __shared__ Smem<THREADS, 1> sm;
    extern __shared__ uint32_t hub[];  // optional: V_curr bits of the hub prefix
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
    uint32_t* Fd = p.B2;
    const uint8_t* Fd8 = reinterpret_cast<const uint8_t*>(Fd);

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
        p.SL[0] = sset;  // first position 0
        p.ctl[0] = seed_e - seed_b;             // T: VSSs queued for the level
        p.ctl[1] = (seed_e > seed_b) ? 1 : 0;   // S: slice sets queued
        for (int i = 2; i < 8; ++i) p.ctl[i] = 0;
        for (int i = 0; i < 8; ++i) p.trace[i] = 0;
    }
    grid_barrier(p.bar, gen);

    uint32_t ctr[4] = {0, 0, 0, 0};  // discovered, full, relaxed, pushes
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
        const bool hubs = p.hub_words && T >= p.dense_min;
        const uint32_t hub_n = hubs ? 32u * p.hub_words : 0u;
        if (hubs) {
            const uint4* src4 = reinterpret_cast<const uint4*>(Vc);
            uint4* dst4 = reinterpret_cast<uint4*>(hub);
            for (uint32_t i = threadIdx.x; i < p.hub_words / 4; i += THREADS) dst4[i] = src4[i];
            __syncthreads();
        }

        // ---- stage 1: pull over this warp's contiguous queue positions ----
        if (gw < NW) {
            const uint64_t lo = (uint64_t)gw * T / NW, hi = (uint64_t)(gw + 1) * T / NW;
            if (lo < hi) {
                SetWindow win;
                load_window(p, Fd8, find_set(p, S, lo), S, T, win);
                for (uint64_t pos = lo; pos < hi; pos += kBatch) {
                    const uint64_t last = min(pos + kBatch, hi) - 1;
                    if (last >= win.wend) {  // slide the window to the set holding pos
                        const unsigned own = __ballot_sync(0xffffffffu, win.first <= pos);
                        const uint32_t nb = (pos >= win.wend) ? win.base + 32 : win.base + (31 - __clz(own));
                        load_window(p, Fd8, nb, S, T, win);
                    }
                    uint32_t vj[kBatch], aj[kBatch];
                    uint32_t mk[kBatch];
                    uint4 rw[kBatch];
#pragma unroll
                    for (int j = 0; j < kBatch; ++j) {
                        const uint64_t q = pos + j;
                        const unsigned own = __ballot_sync(0xffffffffu, win.first <= q);
                        const int l = 31 - __clz(own);
                        const uint64_t f = __shfl_sync(0xffffffffu, win.first, l);
                        vj[j] = __shfl_sync(0xffffffffu, win.b, l) + (uint32_t)(q - f);
                        aj[j] = __shfl_sync(0xffffffffu, win.alpha, l);
                        mk[j] = 0;
                        rw[j] = make_uint4(0, 0, 0, 0);
                        if (q <= last) {
                            const uint64_t v = vj[j];
                            mk[j] = ld_stream_u32(p.masks + 32 * v + lane, pol);
                            rw[j] = ld_stream_u4(p.rows4 + 32 * v + lane, pol);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < kBatch; ++j) {
                        if (pos + j > last) break;  // warp-uniform
                        uint32_t cnt[4];
                        column_counts<PULL>(mk[j], aj[j], cnt);
                        const uint32_t u[4] = {rw[j].x, rw[j].y, rw[j].z, rw[j].w};
                        // visited before this level? (V_curr, frozen; hub prefix from smem)
                        uint32_t vw[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            bool need = cnt[c] != 0;
                            if (need && u[c] < hub_n) need = !((hub[u[c] >> 5] >> (u[c] & 31)) & 1u);
                            vw[c] = (need && !(p.xflags & 1)) ? Vc[u[c] >> 5] : (need ? 0u : ~0u);
                        }
                        // not yet: already marked this level by anyone? (V_next at L2)
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if (!((vw[c] >> (u[c] & 31)) & 1u) && !(p.xflags & 2))
                                vw[c] = ld_relaxed_gpu(Vn + (u[c] >> 5));
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
        level_barrier(p, sm, gen, level, ctr, 1);

        // ---- stage 2: chunked word sweep ----
        const uint64_t per = ((p.words + gridDim.x - 1) / gridDim.x + THREADS - 1) / THREADS * THREADS;
        const uint64_t w0 = (uint64_t)blockIdx.x * per;
        const uint64_t w1 = min(w0 + per, p.words);
        unsigned long long my_vss = 0, my_sets = 0;
        // pass A
        for (uint64_t wb = w0; wb < w1; wb += THREADS) {
            const uint64_t w = wb + threadIdx.x;
            uint32_t diff = 0;
            if (w < w1) {
                const uint32_t nx = Vn[w];
                diff = nx & ~Vc[w];
                Fd[w] = diff;
                if (diff) Vc[w] = nx;
                for (uint32_t d = diff; d;) {
                    const int bsel = (__ffs(d) - 1) >> 3;
                    d &= ~(0xFFu << (8 * bsel));
                    const uint64_t ss = 4 * w + bsel;
                    const uint32_t c = p.rp[ss + 1] - p.rp[ss];
                    my_vss += c;
                    my_sets += c != 0;  // sets without VSSs push nothing (empty range)
                }
            }
            ctr[0] += __popc(diff);
            const uint64_t wwarp = wb + 32 * warp;
            unsigned ball = __ballot_sync(0xffffffffu, diff != 0);
            while (ball) {
                const int k = __ffs(ball) - 1;
                ball &= ball - 1;
                const uint32_t dk = __shfl_sync(0xffffffffu, diff, k);
                if ((dk >> lane) & 1u) p.L[32 * (wwarp + k) + lane] = level;
            }
        }
        unsigned long long cta_vss = 0, cta_sets = 0;
        block_excl_scan(sm, my_vss, &cta_vss);
        block_excl_scan(sm, my_sets, &cta_sets);
        __syncthreads();  // every warp is done reading sm.red
        if (threadIdx.x == 0) {
            const unsigned long long tag = (unsigned long long)level << 40;
            p.aggS[blockIdx.x] = tag | cta_sets;
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.agg + blockIdx.x), "l"(tag | cta_vss)
                         : "memory");
        }
        if (warp == 0) {
            unsigned long long bv = 0, bs = 0;
            for (uint32_t c = lane; c < blockIdx.x; c += 32) {
                unsigned long long x;
                do {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p.agg + c) : "memory");
                } while ((x >> 40) != level);
                bv += x & kTagMask;
                bs += ld_relaxed_gpu_u64(p.aggS + c) & kTagMask;
            }
            bv = warp_sum(bv);
            bs = warp_sum(bs);
            if (lane == 0) {
                sm.base = bv;
                sm.red[0] = bs;  // consumed below before any further scan
            }
        }
        __syncthreads();
        unsigned long long run_vss = sm.base, run_sets = sm.red[0];
        __syncthreads();
        if (threadIdx.x == 0) {
            ctr[3] += (uint32_t)cta_vss;
            if (blockIdx.x == gridDim.x - 1) {  // the grid totals become the next level's T, S
                p.ctl[0] = run_vss + cta_vss;
                p.ctl[1] = run_sets + cta_sets;
            }
        }
        // pass B: SL entries of the chunk's active slice sets, in ascending order
        for (uint64_t wb = w0; wb < w1; wb += THREADS) {
            const uint64_t w = wb + threadIdx.x;
            const uint32_t diff = (w < w1) ? Fd[w] : 0u;
            unsigned long long nv = 0, ns = 0;
            uint32_t cnts[4];
#pragma unroll
            for (int bsel = 0; bsel < 4; ++bsel) {
                cnts[bsel] = 0;
                if ((diff >> (8 * bsel)) & 0xFFu) {
                    const uint64_t ss = 4 * w + bsel;
                    cnts[bsel] = p.rp[ss + 1] - p.rp[ss];
                    nv += cnts[bsel];
                    ns += cnts[bsel] != 0;
                }
            }
            unsigned long long it_v = 0, it_s = 0;
            unsigned long long pv = run_vss + block_excl_scan(sm, nv, &it_v);
            unsigned long long ps = run_sets + block_excl_scan(sm, ns, &it_s);
#pragma unroll
            for (int bsel = 0; bsel < 4; ++bsel) {
                if (cnts[bsel]) {
                    p.SL[ps++] = (pv << 32) | (4 * w + bsel);
                    pv += cnts[bsel];
                }
            }
            run_vss += it_v;
            run_sets += it_s;
        }
        level_barrier(p, sm, gen, level, ctr, 2);
    }
    if (gtid == 0) p.ctl[4] = level - 1;
}

}  // namespace

void* lazy_kernel(int pull, int threads) {
    if (pull == 1) {
        switch (threads) {
            case 256: return (void*)k_bfs_lazy<1, 256>;
            case 512: return (void*)k_bfs_lazy<1, 512>;
            case 1024: return (void*)k_bfs_lazy<1, 1024>;
        }
    } else {
        switch (threads) {
            case 256: return (void*)k_bfs_lazy<0, 256>;
            case 512: return (void*)k_bfs_lazy<0, 512>;
            case 1024: return (void*)k_bfs_lazy<0, 1024>;
        }
    }
    throw InvalidArgument("threads per CTA must be 256, 512 or 1024");
}

}  // namespace blestgpu
