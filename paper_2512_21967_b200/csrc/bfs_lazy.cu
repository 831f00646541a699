// Lazy engine (BLEST Alg. 3; run_lazy, R:src/bfs_engine.cpp:238-350) as one fused
// persistent cooperative kernel.
//
// Stage 1 (pull, :273-292). Warps take queue positions round-robin exactly like the
// reference (p ≡ warp mod #warps, :190), kBatch at a time, so neighbouring warps stream
// neighbouring VSSs. Queue entries carry the set's frontier byte α (final when stage 2
// enqueued it). Per VSS: one coalesced 128 B mask line and four 128 B row-id lines
// (streaming loads), AND with α, and for every nonzero column the visited test: V_curr
// (frozen during the stage, L1-cached) and, if clear, V_next at L2; only then a
// fire-and-forget RED sets the V_next bit (legal per SURVEY §8(a) pitfall 7).
//
// Stage 2 (word sweep, :296-338). Each CTA owns a contiguous chunk of the ⌈n/32⌉ words.
// Pass A: diff = V_next & ~V_curr, V_curr |= diff, diff words kept, levels written with
// one coalesced 128 B store per changed word, and the chunk's VSS count reduced. The CTA
// publishes its count (tagged with the level, so no reset) and sums its predecessors';
// pass B expands its sets' VSS ranges [real_ptrs[s], real_ptrs[s+1]) at that offset,
// each warp writing its items' ranges with all 32 lanes (a hub set with thousands of
// VSSs costs one warp a few µs, not one thread). The next queue is in ascending
// slice-set order (deterministic; stage 1 then streams the BVSS in address order) and
// no contended atomic is involved.
#include "bfs.cuh"
#include "bfs_device.cuh"

namespace blestgpu {

namespace {
using namespace bfsdev;

constexpr unsigned long long kTagMask = (1ull << 40) - 1;

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
    }
    {
        const unsigned long long aux = (unsigned long long)(1u << (src & 7)) << 32;
        for (uint64_t i = gtid; i < seed_e - seed_b; i += gthreads) p.Q1[i] = aux | (seed_b + i);
    }
    if (threadIdx.x == 0) p.agg[blockIdx.x] = 0;
    if (gtid == 0) {
        p.ctl[0] = seed_e - seed_b;  // queue length of the level
        for (int i = 1; i < 8; ++i) p.ctl[i] = 0;
        for (int i = 0; i < 8; ++i) p.trace[i] = 0;
    }
    grid_barrier(p.bar, gen);

    uint32_t ctr[4] = {0, 0, 0, 0};  // discovered, full, relaxed, pushes
    uint32_t level = 1;
    for (;; ++level) {
        const unsigned long long len = ld_relaxed_gpu_u64(&p.ctl[0]);
        if (len == 0) break;
        if (level > p.cap) {  // runaway (R:src/bfs_engine.cpp:72-75)
            if (gtid == 0) p.ctl[6] = 1;
            break;
        }
        if (gtid == 0) {
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
        const unsigned long long* Qc = (level & 1) ? p.Q1 : p.Q0;
        unsigned long long* Qn = (level & 1) ? p.Q0 : p.Q1;
        const bool hubs = p.hub_words && len >= p.dense_min;
        const uint32_t hub_n = hubs ? 32u * p.hub_words : 0u;
        if (hubs) {
            const uint4* src4 = reinterpret_cast<const uint4*>(Vc);
            uint4* dst4 = reinterpret_cast<uint4*>(hub);
            for (uint32_t i = threadIdx.x; i < p.hub_words / 4; i += THREADS) dst4[i] = src4[i];
            __syncthreads();
        }

        // ---- stage 1: pull (pull_vss, R:src/bfs_engine.cpp:131-146) ----
        if (gw < NW) {
            // queue entries of the next batch are fetched while this batch is processed
            unsigned long long e_next = kNoEntry;
            if (lane < kBatch && gw + (uint64_t)lane * NW < len) e_next = Qc[gw + (uint64_t)lane * NW];
            for (uint64_t p0 = gw; p0 < len; p0 += (uint64_t)NW * kBatch) {
                const unsigned long long e = e_next;
                e_next = kNoEntry;
                if (lane < kBatch) {
                    const uint64_t pos = p0 + (uint64_t)NW * kBatch + (uint64_t)lane * NW;
                    if (pos < len) e_next = Qc[pos];
                }
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
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    if (ej[j] == kNoEntry) continue;  // warp-uniform
                    uint32_t cnt[4];
                    column_counts<PULL>(mk[j], (uint32_t)((ej[j] >> 32) & 0xFFu), cnt);
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
                        if (!((vw[c] >> (u[c] & 31)) & 1u) && !(p.xflags & 2)) vw[c] = ld_l2_u32(Vn + (u[c] >> 5));
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
        level_barrier(p, sm, gen, level, ctr, 1);

        // ---- stage 2: chunked word sweep ----
        const uint64_t per = ((p.words + gridDim.x - 1) / gridDim.x + THREADS - 1) / THREADS * THREADS;
        const uint64_t w0 = (uint64_t)blockIdx.x * per;
        const uint64_t w1 = min(w0 + per, p.words);
        unsigned long long my_vss = 0;
        // pass A: diff, V_curr update, levels, VSS count of the sets to enqueue
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
                    my_vss += p.rp[ss + 1] - p.rp[ss];
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
        unsigned long long cta_vss = 0;
        block_excl_scan(sm, my_vss, &cta_vss);
        if (threadIdx.x == 0) {
            const unsigned long long tag = ((unsigned long long)level << 40) | cta_vss;
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.agg + blockIdx.x), "l"(tag) : "memory");
        }
        // sum the predecessors' counts with every thread (one or two rounds of loads)
        unsigned long long before = 0;
        for (uint32_t c = threadIdx.x; c < blockIdx.x; c += THREADS) {
            unsigned long long x;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p.agg + c) : "memory");
            } while ((x >> 40) != level);
            before += x & kTagMask;
        }
        unsigned long long running = 0;
        block_excl_scan(sm, before, &running);
        if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) p.ctl[0] = running + cta_vss;  // next length
        if (threadIdx.x == 0) ctr[3] += (uint32_t)cta_vss;
        // pass B: expand the chunk's sets into the queue, slice-set order; warp-cooperative
        for (uint64_t wb = w0; wb < w1; wb += THREADS) {
            const uint64_t w = wb + threadIdx.x;
            const uint32_t diff = (w < w1) ? Fd[w] : 0u;
            uint32_t b[4], c4[4];
            unsigned long long cnt = 0;
#pragma unroll
            for (int bsel = 0; bsel < 4; ++bsel) {
                b[bsel] = c4[bsel] = 0;
                if ((diff >> (8 * bsel)) & 0xFFu) {
                    const uint64_t ss = 4 * w + bsel;
                    b[bsel] = p.rp[ss];
                    c4[bsel] = p.rp[ss + 1] - b[bsel];
                    cnt += c4[bsel];
                }
            }
            unsigned long long it_total = 0;
            unsigned long long pos = running + block_excl_scan(sm, cnt, &it_total);
            unsigned ball = __ballot_sync(0xffffffffu, cnt != 0);
            while (ball) {
                const int k = __ffs(ball) - 1;
                ball &= ball - 1;
                unsigned long long at = __shfl_sync(0xffffffffu, pos, k);
                const uint32_t dk = __shfl_sync(0xffffffffu, diff, k);
#pragma unroll
                for (int bsel = 0; bsel < 4; ++bsel) {
                    const uint32_t bb = __shfl_sync(0xffffffffu, b[bsel], k);
                    const uint32_t cc = __shfl_sync(0xffffffffu, c4[bsel], k);
                    const unsigned long long aux = (unsigned long long)((dk >> (8 * bsel)) & 0xFFu) << 32;
                    for (uint32_t t = lane; t < cc; t += 32) Qn[at + t] = aux | (bb + t);
                    at += cc;
                }
            }
            running += it_total;
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
