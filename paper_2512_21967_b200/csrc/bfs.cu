// Fused persistent BFS kernel for sm_100a: one cooperative launch per source runs
// init_state and every level, with a grid barrier replacing the reference's per-level
// fork/join (R:src/bfs_engine.cpp:187, :273, :299).
//
// Work unit = one VSS (R:include/blest/bvss.hpp:34-63) handled by one warp: lane t reads
// its mask word (one coalesced 128 B line per VSS) and its 4 row ids (one 16 B load; four
// 128 B lines per VSS), both with streaming (evict-first, no-L1) loads. Warps take queue
// positions round-robin exactly like the reference (p ≡ warp mod #warps, :190), B
// positions at a time so each lane keeps 2·B independent HBM loads in flight.
//
// Queue entries are 64-bit: low = VSS id, high = aux. Eager: aux = slice set (saves the
// virtual_to_real lookup, :192). Lazy: aux = the slice set's frontier byte α, final when
// stage 2 enqueues (saves the F_curr read, :281-282).
//
// Eager (Alg. 2, :155-236): one grid barrier per level. Frontier bitmaps F are
// triple-buffered: level ℓ reads F[ℓ%3] (α), atomically ORs discoveries into F[(ℓ+1)%3],
// and zeroes the bytes of F[(ℓ+2)%3] that level ℓ-1 used (found from queue ℓ-1), so no
// Θ(n) clear is ever needed (the reference clears all words per level, :227-228).
// Enqueue: lanes append slice sets to a per-warp shared-memory buffer; a flush reserves
// queue space with ONE atomicAdd per warp buffer and expands [real_ptrs[s], real_ptrs[s+1]).
//
// Lazy (Alg. 3, :238-350): visited words are interleaved {V_curr, V_next} so one 8-byte
// load answers "visited before this level, or already marked this level?"; only then a
// fire-and-forget RED sets the V_next bit (stage 1, :286-289). Stage 2 (:296-338) gives
// every CTA one contiguous chunk of words: pass A computes diff = V_next & ~V_curr,
// writes levels with coalesced 128 B stores, and counts the VSSs to enqueue; the CTA
// publishes its count and sums its predecessors' (tagged with the level, so no reset);
// pass B writes its slice sets' VSS ranges at that offset. The next queue is therefore in
// ascending slice-set order — deterministic, and stage 1 then streams the BVSS in address
// order — with no contended queue-tail atomic at all.
#include <algorithm>
#include <atomic>
#include <string>

#include "bfs.cuh"
#include "bfs_device.cuh"

namespace blestgpu {

extern std::atomic<uint64_t> g_launches;

void* lazy_kernel(int pull, int threads);        // bfs_lazy.cu (register-pipelined variant)
void* lazy_tma_kernel(int pull, int consumers);  // bfs_lazy_tma.cu (TMA producer/consumer)
size_t lazy_tma_smem(int consumers);

namespace {
using namespace bfsdev;

template <int MODE, int PULL, int THREADS>
__global__ void __launch_bounds__(THREADS) k_bfs(Params p) {
    constexpr int WPC = THREADS / 32;
    __shared__ Smem<THREADS, MODE> sm;
    extern __shared__ uint32_t hub[];  // lazy: V_curr bits of the hub prefix [0, 32*hub_words)
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
    uint32_t* Vc = p.B0;  // lazy V_curr: frozen during stage 1 (L1-cacheable)
    uint32_t* Vn = p.B1;  // lazy V_next: REDs at L2, read with L1-bypassing loads

    // ---- init_state (R:src/bfs_engine.cpp:30-49), fused ----
    const uint32_t src = p.src;
    const uint32_t sset = src / kSigma;
    const uint32_t seed_b = p.rp[sset], seed_e = p.rp[sset + 1];
    for (uint64_t i = gtid; i < p.n; i += gthreads) p.L[i] = (i == src) ? 0u : kInf;
    const uint32_t src_word = src >> 5, src_bit = 1u << (src & 31);
    for (uint64_t w = gtid; w < p.words; w += gthreads) {
        const uint32_t seed = (w == src_word) ? src_bit : 0u;
        if (MODE == 0) {
            p.B0[w] = 0;
            p.B1[w] = seed;  // F[1] = F_curr of level 1
            p.B2[w] = 0;
        } else {
            Vc[w] = seed;
            Vn[w] = seed;
        }
    }
    {
        unsigned long long* Q1 = p.Q1;
        const unsigned long long aux =
            (MODE == 0) ? ((unsigned long long)sset << 32)
                        : ((unsigned long long)(1u << (src & 7)) << 32);
        for (uint64_t i = gtid; i < seed_e - seed_b; i += gthreads) Q1[i] = aux | (seed_b + i);
    }
    if (threadIdx.x == 0) p.agg[blockIdx.x] = 0;  // stage-2 tags are per run
    if (gtid == 0) {
        p.ctl[0] = 0;
        p.ctl[1] = seed_e - seed_b;
        p.ctl[2] = 0;
        p.ctl[3] = 0;
        p.ctl[4] = 0;
        p.ctl[5] = 0;
        p.ctl[6] = 0;
        for (int i = 0; i < 8; ++i) p.trace[i] = 0;
    }
    grid_barrier(p.bar, gen);

    unsigned long long* pbuf = sm.push[warp];
    uint32_t pcount = 0;
    uint32_t ctr[4] = {0, 0, 0, 0};  // discovered, full, relaxed, pushes
    uint32_t level = 1;
    for (;; ++level) {
        const unsigned long long len = ld_relaxed_gpu_u64(&p.ctl[level & 3]);
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
        unsigned long long* Qc = queue_at<MODE>(p, level);
        unsigned long long* Qn = queue_at<MODE>(p, level + 1);
        unsigned long long* qlen_next = &p.ctl[(level + 1) & 3];
        const uint32_t* Fc = (MODE == 0) ? fbuf(p, level) : nullptr;
        uint32_t* Fn = (MODE == 0) ? fbuf(p, level + 1) : nullptr;

        if (MODE == 0) {
            // Zero the frontier bytes level ℓ-1 read: they become F_next at ℓ+1.
            uint8_t* Fz = reinterpret_cast<uint8_t*>(fbuf(p, level + 2));
            const unsigned long long* Qz = queue_at<MODE>(p, level + 2);
            const unsigned long long zlen = ld_relaxed_gpu_u64(&p.ctl[(level + 3) & 3]);
            for (uint64_t i = gtid; i < zlen; i += gthreads) Fz[Qz[i] >> 32] = 0;
        }

        // ---- pull over the queue (pull_vss, R:src/bfs_engine.cpp:131-146) ----
        // Dense lazy levels: stage the frozen V_curr bits of the hub prefix in shared memory,
        // so the visited test of the (mostly hub-bound) hits is served on-chip.
        const bool hubs = (MODE == 1) && p.hub_words && len >= p.dense_min;
        const uint32_t hub_n = hubs ? 32u * p.hub_words : 0u;
        if (hubs) {
            const uint4* src4 = reinterpret_cast<const uint4*>(Vc);
            uint4* dst4 = reinterpret_cast<uint4*>(hub);
            for (uint32_t i = threadIdx.x; i < p.hub_words / 4; i += THREADS) dst4[i] = src4[i];
            __syncthreads();
        }
        if (gw < NW) {
            for (uint64_t p0 = gw; p0 < len; p0 += (uint64_t)NW * kBatch) {
                unsigned long long e = kNoEntry;
                if (lane < kBatch) {
                    const uint64_t pos = p0 + (uint64_t)lane * NW;
                    if (pos < len) e = Qc[pos];
                }
                uint32_t alpha_l = 0;
                if (MODE == 0 && e != kNoEntry) {
                    const uint32_t ss = (uint32_t)(e >> 32);
                    alpha_l = reinterpret_cast<const uint8_t*>(Fc)[ss];  // frontier_byte :148-151
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
                    const uint32_t alpha = (MODE == 0) ? __shfl_sync(0xffffffffu, alpha_l, j)
                                                       : (uint32_t)((ej[j] >> 32) & 0xFFu);
                    uint32_t cnt[4];
                    column_counts<PULL>(mk[j], alpha, cnt);
                    const uint32_t u[4] = {rw[j].x, rw[j].y, rw[j].z, rw[j].w};
                    // All four dependent state loads of this VSS are issued before any of
                    // them is consumed (4 independent L1/L2 requests in flight per lane).
                    if (MODE == 1) {
                        // stage-1 sink (:286-289): relaxed OR into V_next unless the vertex
                        // was visited before this level or is already marked this level.
                        // visited before this level? (V_curr; hub prefix from shared memory)
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
                            if (!((vw[c] >> (u[c] & 31)) & 1u) && !(p.xflags & 2)) vw[c] = ld_relaxed_gpu(Vn + (u[c] >> 5));
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            if (!((vw[c] >> (u[c] & 31)) & 1u)) {
                                red_or(Vn + (u[c] >> 5), 1u << (u[c] & 31));
                                ++ctr[2];
                            }
                        }
                    } else {
                        // eager sink (:198-211)
                        uint32_t lv[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) lv[c] = cnt[c] ? p.L[u[c]] : 0u;
                        uint32_t old[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            old[c] = (lv[c] == kInf) ? atomicOr(Fn + (u[c] >> 5), 1u << (u[c] & 31))
                                                     : 0xFFFFFFFFu;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            bool push = false;
                            if (lv[c] == kInf) {
                                ++ctr[1];
                                if (!((old[c] >> (u[c] & 31)) & 1u)) {
                                    p.L[u[c]] = level;
                                    ++ctr[0];
                                    push = ((old[c] >> (8 * ((u[c] >> 3) & 3))) & 0xFFu) == 0;
                                }
                            }
                            push_column(p, push, (unsigned long long)(u[c] >> 3) << 32 | (u[c] >> 3), pbuf,
                                        pcount, Qn, qlen_next, ctr[3], ctr[1]);
                        }
                    }
                }
            }
        }

        if (MODE == 1) {
            level_barrier(p, sm, gen, level, ctr, 1);
            // ---- stage 2 (R:src/bfs_engine.cpp:296-338): chunked word sweep ----
            uint32_t* Fd = p.B2;  // this level's diff words (the reference's F_curr, :310-311)
            const uint64_t per = ((p.words + gridDim.x - 1) / gridDim.x + THREADS - 1) / THREADS * THREADS;
            const uint64_t w0 = (uint64_t)blockIdx.x * per;
            const uint64_t w1 = min(w0 + per, p.words);
            unsigned long long mine = 0;
            // pass A: diff, V_curr update, levels, VSS count of the sets to enqueue
            for (uint64_t wb = w0; wb < w1; wb += THREADS) {
                const uint64_t w = wb + threadIdx.x;
                uint32_t diff = 0;
                if (w < w1) {
                    const uint32_t nx = Vn[w];
                    diff = nx & ~Vc[w];
                    Fd[w] = diff;
                    if (diff) Vc[w] = nx;
                    for (uint32_t d = diff; d; ) {
                        const int bsel = (__ffs(d) - 1) >> 3;
                        d &= ~(0xFFu << (8 * bsel));
                        const uint64_t ss = 4 * w + bsel;
                        mine += p.rp[ss + 1] - p.rp[ss];
                    }
                }
                ctr[0] += __popc(diff);
                const uint64_t wwarp = wb + 32 * warp;  // this warp's 32 words
                unsigned ball = __ballot_sync(0xffffffffu, diff != 0);
                while (ball) {
                    const int k = __ffs(ball) - 1;
                    ball &= ball - 1;
                    const uint32_t dk = __shfl_sync(0xffffffffu, diff, k);
                    if ((dk >> lane) & 1u) p.L[32 * (wwarp + k) + lane] = level;
                }
            }
            unsigned long long cta_total = 0;
            block_excl_scan(sm, mine, &cta_total);
            // publish this CTA's count, then sum the predecessors' (level-tagged)
            if (threadIdx.x == 0) {
                const unsigned long long tag = ((unsigned long long)level << 40) | cta_total;
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.agg + blockIdx.x), "l"(tag) : "memory");
            }
            if (warp == 0) {
                unsigned long long before = 0;
                for (uint32_t c = lane; c < blockIdx.x; c += 32) {
                    unsigned long long x;
                    do {
                        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p.agg + c) : "memory");
                    } while ((x >> 40) != level);
                    before += x & ((1ull << 40) - 1);
                }
                before = warp_sum(before);
                if (lane == 0) {
                    sm.base = before;
                    if (blockIdx.x == gridDim.x - 1) *qlen_next = before + cta_total;
                }
            }
            __syncthreads();
            // pass B: expand the chunk's slice sets into the queue, in slice-set order
            unsigned long long running = sm.base;
            for (uint64_t wb = w0; wb < w1; wb += THREADS) {
                const uint64_t w = wb + threadIdx.x;
                const uint32_t diff = (w < w1) ? Fd[w] : 0u;
                uint32_t b[4], e[4];
                unsigned long long cnt = 0;
#pragma unroll
                for (int bsel = 0; bsel < 4; ++bsel) {
                    b[bsel] = e[bsel] = 0;
                    if ((diff >> (8 * bsel)) & 0xFFu) {
                        const uint64_t ss = 4 * w + bsel;
                        b[bsel] = p.rp[ss];
                        e[bsel] = p.rp[ss + 1];
                        cnt += e[bsel] - b[bsel];
                    }
                }
                unsigned long long it_total = 0;
                unsigned long long pos = running + block_excl_scan(sm, cnt, &it_total);
#pragma unroll
                for (int bsel = 0; bsel < 4; ++bsel) {
                    const unsigned long long aux = (unsigned long long)((diff >> (8 * bsel)) & 0xFFu) << 32;
                    for (uint32_t v = b[bsel]; v < e[bsel]; ++v) Qn[pos++] = aux | v;
                }
                running += it_total;
            }
            if (threadIdx.x == 0) ctr[3] += (uint32_t)cta_total;
        }
        if (MODE == 0 && pcount) {
            const uint32_t t = flush_pushes(p, pbuf, pcount, Qn, qlen_next);
            if (lane == 0) {
                ctr[3] += t;
                ctr[1] += 1;
            }
        }
        level_barrier(p, sm, gen, level, ctr, 2);
    }
    if (gtid == 0) p.ctl[4] = level - 1;
}

template <int MODE, int PULL>
void* pick_kernel(int threads) {
    switch (threads) {
        case 256: return (void*)k_bfs<MODE, PULL, 256>;
        case 512: return (void*)k_bfs<MODE, PULL, 512>;
        case 1024: return (void*)k_bfs<MODE, PULL, 1024>;
    }
    throw InvalidArgument("threads per CTA must be 256, 512 or 1024");
}

}  // namespace

BfsEngine::BfsEngine(const DeviceBvss& b) : b_(b) {
    words_ = ((uint64_t)b.n + 31) / 32;
    const uint64_t levels_bound = (uint64_t)b.n + 2;
    trace_cap_ = (uint32_t)std::min<uint64_t>(levels_bound, 1u << 20);
    levels_.alloc(b.n ? b.n : 1);
    bits_.alloc(3 * (words_ ? words_ : 1));
    q_.alloc(3 * (uint64_t)(b.num_vss ? b.num_vss : 1));
    ctl_.alloc(8);
    agg_.alloc(4096);
    aggS_.alloc(4096);
    sl_.alloc((uint64_t)b.num_sets + 1);
    CK(cudaMemset(agg_.p, 0, 4096 * 8));
    bar_.alloc(2);
    trace_.alloc(8ull * trace_cap_);
    tstamp_.alloc(3ull * trace_cap_);
    // hub prefix staged in shared memory on dense lazy levels (opt-in): at most what one
    // SM's shared memory holds, whole 16-byte granules inside the V_curr array
    hub_words_max_ = (uint32_t)std::min<uint64_t>(words_ / 4 * 4, 56u * 1024);
    CK(cudaMallocHost(&pinned_, 8 * sizeof(unsigned long long)));
}

BfsEngine::~BfsEngine() {
    if (pinned_) cudaFreeHost(pinned_);
}

void BfsEngine::launch(uint32_t src, const EngineOptions& opt) {
    if (src >= b_.n) throw InvalidArgument("bfs source out of range");
    const char* var_env = getenv("BLEST_LAZY_VARIANT");
    const bool lazy_tma = opt.mode == Mode::Lazy && (opt.lazy_tma || (var_env && std::string(var_env) == "tma"));
    const char* nc_env = getenv("BLEST_TMA_CONSUMERS");
    const int consumers = nc_env ? atoi(nc_env) : 8;
    const int threads = lazy_tma ? 32 * (consumers + 1) : (opt.threads ? (int)opt.threads : 512);
    void* kern = nullptr;
    if (opt.mode == Mode::Eager)
        kern = opt.pull == Pull::Mma ? pick_kernel<0, 1>(threads) : pick_kernel<0, 0>(threads);
    else
        kern = lazy_tma ? lazy_tma_kernel(opt.pull == Pull::Mma ? 1 : 0, consumers)
                        : lazy_kernel(opt.pull == Pull::Mma ? 1 : 0, threads);
    size_t dyn = 0;
    if (lazy_tma) {
        dyn = lazy_tma_smem(consumers);
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    }
    int per_sm = 0;
    if (!lazy_tma) {  // small shared footprint: give the rest of the SM's 256 KB to L1
        const char* co = getenv("BLEST_CARVEOUT");
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, co ? atoi(co) : 0));
    }
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, dyn));
    if (per_sm < 1) throw CudaError("BFS kernel cannot be resident");
    // Lazy: give each co-resident CTA an equal share of the SM's shared memory for the
    // hub prefix (minus the static part), rounded down to 16-byte granules.
    uint32_t hub_words = 0;
    const char* hub_env = getenv("BLEST_HUB_CACHE");
    const bool hub_cache = opt.hub_cache || (hub_env && atoi(hub_env) != 0);
    if (opt.mode == Mode::Lazy && !lazy_tma && hub_cache && hub_words_max_) {
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, kern));
        int dev = 0, smem_sm = 0, smem_blk = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
        CK(cudaDeviceGetAttribute(&smem_blk, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        const int64_t share = std::min<int64_t>(smem_sm / per_sm - 1024, smem_blk) - (int64_t)fa.sharedSizeBytes;
        if (share >= 1024) {
            hub_words = (uint32_t)std::min<uint64_t>(hub_words_max_, (uint64_t)share / 4 / 4 * 4);
            dyn = (size_t)hub_words * 4;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
            int check = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&check, kern, threads, dyn));
            if (check < per_sm) {  // keep the register-limited occupancy
                hub_words = 0;
                dyn = 0;
            }
        }
    }
    uint32_t ctas = (uint32_t)per_sm * (uint32_t)num_sms();
    if (opt.grid_ctas && opt.grid_ctas < ctas) ctas = opt.grid_ctas;
    if (ctas > agg_.count) ctas = (uint32_t)agg_.count;
    Params p{};
    p.n = b_.n;
    p.num_sets = b_.num_sets;
    p.words = words_;
    p.rp = b_.real_ptrs.p;
    p.masks = b_.masks.p;
    p.rows4 = reinterpret_cast<const uint4*>(b_.row_ids.p);
    p.L = levels_.p;
    p.B0 = bits_.p;
    p.B1 = bits_.p + words_;
    p.B2 = bits_.p + 2 * words_;
    const uint64_t qcap = b_.num_vss ? b_.num_vss : 1;
    p.Q0 = q_.p;
    p.Q1 = q_.p + qcap;
    p.Q2 = q_.p + 2 * qcap;
    p.ctl = ctl_.p;
    p.agg = agg_.p;
    p.aggS = aggS_.p;
    p.SL = sl_.p;
    p.bar = bar_.p;
    p.trace = trace_.p;
    p.tstamp = tstamp_.p;
    p.trace_cap = trace_cap_;
    p.src = src;
    p.cap = opt.max_levels ? opt.max_levels : b_.n + 1;
    p.num_warps = opt.num_warps;
    p.hub_words = hub_words;
    p.dense_min = (uint64_t)ctas * (threads / 32) * 8;
    if (const char* x = getenv("BLEST_XFLAGS")) p.xflags = (uint32_t)atoi(x);
    cudaStream_t st = stream();
    CK(cudaMemsetAsync(bar_.p, 0, 2 * sizeof(unsigned), st));
    void* args[] = {&p};
    CK(cudaLaunchCooperativeKernel(kern, dim3(ctas), dim3(threads), args, dyn, st));
    last_hub_words_ = hub_words;
    g_launches.fetch_add(1);
    last_ctas_ = ctas;
    last_threads_ = threads;
    last_src_ = src;
    last_mode_ = opt.mode;
    launched_ = true;
}

BfsOutcome BfsEngine::finish(uint32_t* levels_host) {
    if (!launched_) throw LogicError("finish() without launch()");
    cudaStream_t st = stream();
    CK(cudaMemcpyAsync(pinned_, ctl_.p, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (levels_host && b_.n)
        CK(cudaMemcpyAsync(levels_host, levels_.p, (size_t)b_.n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    BfsOutcome out;
    out.iterations = (uint32_t)pinned_[4];
    out.max_level = (uint32_t)pinned_[5];
    const bool runaway = pinned_[6] != 0;
    const uint32_t rows = std::min(out.iterations, trace_cap_);
    out.trace_truncated = out.iterations > trace_cap_;
    out.trace.resize(rows);
    if (rows)
        CK(cudaMemcpy(out.trace.data(), trace_.p, rows * sizeof(TraceRow), cudaMemcpyDeviceToHost));
    uint64_t visited = 1;
    for (uint32_t i = 0; i < rows; ++i) {
        TraceRow& r = out.trace[i];
        visited += r.discovered;
        r.frontier_population = (i == 0) ? 1 : out.trace[i - 1].discovered;
        r.stage1_full_atomics = (last_mode_ == Mode::Eager) ? r.full_atomics : 0;
    }
    out.visited = visited;
    out.phase_ns.resize(3ull * rows);
    if (rows)
        CK(cudaMemcpy(out.phase_ns.data(), tstamp_.p, 3ull * rows * 8, cudaMemcpyDeviceToHost));
    if (runaway)
        throw RuntimeError("BFS ran past the level safety cap at level " +
                           std::to_string(out.iterations + 1) + " — engine invariant broken");
    return out;
}

}  // namespace blestgpu
