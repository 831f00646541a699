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
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <string>

#include "bfs.cuh"
#include "bfs_device.cuh"
#include "sigma.cuh"

namespace blestgpu {

extern std::atomic<uint64_t> g_launches;

void* eager_kernel(int pull, int threads);       // bfs_eager.cu
void* lazy_kernel(int pull, int threads, bool sigma);  // bfs_lazy.cu
void* lazy_tma_kernel(int pull, int consumers);  // bfs_lazy_tma.cu (TMA producer/consumer)
size_t lazy_tma_smem(int consumers);

namespace {
using namespace bfsdev;

// Per-source summary of a finished launch (run_batch): [0] iterations, [1] max level,
// [2] runaway, [3] Σ queue, [4] Σ discovered, [5] Σ full, [6] Σ relaxed, [7] Σ pushes.
__global__ void k_summarise(const unsigned long long* __restrict__ ctl, const unsigned long long* __restrict__ trace,
                            uint32_t trace_cap, unsigned long long* __restrict__ out) {
    __shared__ unsigned long long acc[5];
    if (threadIdx.x < 5) acc[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t rows = ctl[4] < trace_cap ? ctl[4] : trace_cap;
    unsigned long long q = 0, d = 0, f = 0, r = 0, pu = 0;
    for (uint64_t i = threadIdx.x; i < rows; i += blockDim.x) {
        const unsigned long long* t = trace + 8 * i;
        q += t[1];
        d += t[3];
        f += t[4];
        r += t[6];
        pu += t[7];
    }
    atomicAdd(&acc[0], q);
    atomicAdd(&acc[1], d);
    atomicAdd(&acc[2], f);
    atomicAdd(&acc[3], r);
    atomicAdd(&acc[4], pu);
    __syncthreads();
    if (threadIdx.x == 0) {
        out[0] = ctl[4];
        out[1] = ctl[5];
        out[2] = ctl[6];
        for (int i = 0; i < 5; ++i) out[3 + i] = acc[i];
    }
}

// Rows present in the BVSS (a slot with a nonzero mask byte), as a bitmap over original
// ids: the vertices a BFS can discover (lazy exhaustion exit). Test-then-RED per slot.
__global__ void k_present(const uint32_t* __restrict__ masks, const uint4* __restrict__ rows4, uint64_t lanes,
                          uint32_t* present) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < lanes; i += stride) {
        const uint32_t mk = masks[i];
        if (!mk) continue;
        const uint4 r = rows4[i];
        const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if ((mk >> (8 * c)) & 0xFFu) {
                const uint32_t bit = 1u << (u[c] & 31);
                if (!(present[u[c] >> 5] & bit)) atomicOr(&present[u[c] >> 5], bit);
            }
    }
}

__global__ void k_popc_sum(const uint32_t* __restrict__ w, uint64_t words, unsigned long long* out) {
    unsigned long long c = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += stride) c += __popc(w[i]);
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

}  // namespace

void BfsEngine::ensure_present() {
    if (present_built_) return;
    present_.alloc(words_ ? words_ : 1);
    cudaStream_t st = stream();
    CK(cudaMemsetAsync(present_.p, 0, present_.bytes(), st));
    const uint64_t lanes = 32ull * b_.num_vss;
    if (lanes) {
        k_present<<<grid_for(lanes, 256), 256, 0, st>>>(b_.masks.p, reinterpret_cast<const uint4*>(b_.row_ids.p),
                                                        lanes, present_.p);
        CK(cudaGetLastError());
    }
    DevBuf<unsigned long long> cnt(1);
    CK(cudaMemsetAsync(cnt.p, 0, 8, st));
    k_popc_sum<<<grid_for(words_ ? words_ : 1, 256), 256, 0, st>>>(present_.p, words_, cnt.p);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    present_rows_ = h;
    present_built_ = true;
}

BfsEngine::BfsEngine(const DeviceBvss& b) : b_(b) {
    words_ = ((uint64_t)b.n + 31) / 32;
    const uint64_t levels_bound = (uint64_t)b.n + 2;
    trace_cap_ = (uint32_t)std::min<uint64_t>(levels_bound, 1u << 20);
    levels_.alloc(b.n ? b.n : 1);
    wstride_ = (words_ + 1 + 3) / 4 * 4;  // 16-byte aligned bitmaps (stage 2 reads uint4) + a sentinel word
    bits_.alloc(4 * (wstride_ ? wstride_ : 4));
    q_.alloc(3 * (uint64_t)(b.num_vss ? b.num_vss : 1));
    ctl_.alloc(16);
    agg_.alloc(4096);
    aggS_.alloc(4096);
    sl_.alloc((uint64_t)b.num_sets + 1);
    CK(cudaMemset(agg_.p, 0, 4096 * 8));
    bar_.alloc(4);  // count, pad, {payload | generation}
    trace_.alloc(8ull * trace_cap_);
    tstamp_.alloc(3ull * trace_cap_);
    CK(cudaMallocHost(&pinned_, 16 * sizeof(unsigned long long)));
}

BfsEngine::~BfsEngine() {
    pool_.reset();
    if (pinned_) cudaFreeHost(pinned_);
    if (stage_) cudaFreeHost(stage_);
    if (stage_max_) cudaFreeHost(stage_max_);
}

// Lazy exhaustion exit (bfs_lazy.cu), on unless BLEST_EXHAUST=0.
static bool exhaust_enabled() {
    const char* e = getenv("BLEST_EXHAUST");
    return !(e && atoi(e) == 0);
}

// Widening threads: the CPUs this process may run on (bench.py pins it to the GPU's NUMA
// node) minus the launching thread; BLEST_XFER_THREADS overrides.
static int xfer_threads() {
    if (const char* t = getenv("BLEST_XFER_THREADS")) return std::max(1, atoi(t));
    cpu_set_t set;
    int cpus = 8;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) cpus = CPU_COUNT(&set);
    return std::min(32, std::max(1, cpus - 1));
}

void BfsEngine::ensure_xfer() {
    if (!levels2_.p) levels2_.alloc(b_.n ? b_.n : 1);
    if (stage_ || !b_.n) return;
    const uint64_t slot = xfer_slot_bytes(b_.n);
    dpack_.alloc(2 * slot);
    CK(cudaHostAlloc(reinterpret_cast<void**>(&stage_), kStageRing * slot, cudaHostAllocDefault));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&stage_max_), kStageRing * sizeof(unsigned long long),
                     cudaHostAllocDefault));
    pool_.reset(new WidenPool(xfer_threads()));
}

void BfsEngine::ensure_sigma() {
    if (sigma_built_) return;
    const char* hot = getenv("BLEST_HOT");
    sigma_view_build(b_, sigma_, hot ? (uint32_t)atoll(hot) : 0u);
    sigma_built_ = true;
    // BLEST_SIGMA=1 forces the view; otherwise it is kept only where the hot rows hold a
    // large share of the slots (sigma.cuh kSigmaMinShare) — no engine copy otherwise
    const char* sig_env = getenv("BLEST_SIGMA");
    sigma_on_ = (sig_env && atoi(sig_env) == 1) || sigma_.hot_share >= kSigmaMinShare;
    if (!sigma_on_) {
        sigma_.rows.release();
        sigma_.sig.release();
        sigma_.inv.release();
        return;
    }
    const uint64_t stride = sigma_.hot_words + wstride_;  // both multiples of 4 words
    vext_.alloc(2 * stride);
}

uint64_t BfsEngine::prepare(const EngineOptions& opt) {
    const char* sig_env = getenv("BLEST_SIGMA");
    if (opt.mode == Mode::Lazy && opt.sigma && !(sig_env && atoi(sig_env) == 0)) ensure_sigma();
    if (exhaust_enabled()) ensure_present();
    ensure_xfer();
    CK(cudaStreamSynchronize(stream()));
    uint64_t bytes = levels_.count * 4 + levels2_.count * 4 + dpack_.count + bits_.count * 4 + q_.count * 8 + ctl_.count * 8 +
                     agg_.count * 8 + aggS_.count * 8 + sl_.count * 8 + bar_.count * 4 + trace_.count * 8 +
                     tstamp_.count * 8 + present_.count * 4;
    if (sigma_on_)
        bytes += sigma_.rows.count * 4 + sigma_.sig.count * 4 + sigma_.inv.count * 4 + vext_.count * 4;
    return bytes;
}

void BfsEngine::launch(uint32_t src, const EngineOptions& opt) {
    if (src >= b_.n) throw InvalidArgument("bfs source out of range");
    if (b_.num_sets >= (1u << 25)) throw InvalidArgument("the BFS engines support n < 2^28");
    const char* var_env = getenv("BLEST_LAZY_VARIANT");
    const bool lazy_tma = opt.mode == Mode::Lazy && (opt.lazy_tma || (var_env && std::string(var_env) == "tma"));
    const char* nc_env = getenv("BLEST_TMA_CONSUMERS");
    const int consumers = nc_env ? atoi(nc_env) : 8;
    const char* sig_env = getenv("BLEST_SIGMA");
    bool sigma = opt.mode == Mode::Lazy && !lazy_tma && opt.sigma && !(sig_env && atoi(sig_env) == 0);
    if (sigma) {
        ensure_sigma();
        sigma = sigma_on_;
    }
    const int threads = lazy_tma ? 32 * (consumers + 1) : (opt.threads ? (int)opt.threads : 512);
    void* kern = nullptr;
    if (opt.mode == Mode::Eager)
        kern = eager_kernel(opt.pull == Pull::Mma ? 1 : 0, threads);
    else
        kern = lazy_tma ? lazy_tma_kernel(opt.pull == Pull::Mma ? 1 : 0, consumers)
                        : lazy_kernel(opt.pull == Pull::Mma ? 1 : 0, threads, sigma);
    size_t dyn = 0;
    if (lazy_tma) {
        dyn = lazy_tma_smem(consumers);
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    } else {  // small shared footprint: give the rest of the SM's 256 KB to L1
        const char* co = getenv("BLEST_CARVEOUT");
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, co ? atoi(co) : 0));
    }
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, dyn));
    if (per_sm < 1) throw CudaError("BFS kernel cannot be resident");
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
    p.L = level_target_ ? level_target_ : levels_.p;
    p.B0 = bits_.p;
    p.B1 = bits_.p + wstride_;
    p.B2 = bits_.p + 2 * wstride_;
    p.B3 = bits_.p + 3 * wstride_;
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
    if (!lazy_tma && exhaust_enabled()) {  // both engines (the TMA ablation has no exit)
        ensure_present();
        p.present = present_.p;
        p.present_rows = present_rows_;
    }
    last_exhaust_ = p.present_rows != 0;
    if (sigma) {
        const uint64_t stride = sigma_.hot_words + wstride_;
        p.B0 = vext_.p;  // V_curr / V_next = [hot prefix | row words]
        p.B1 = vext_.p + stride;
        p.rows4 = reinterpret_cast<const uint4*>(sigma_.rows.p);
        p.inv = sigma_.inv.p;
        p.sig = sigma_.sig.p;
        p.hot_words = sigma_.hot_words;
    }
    // dense levels: eager from 8 VSSs per warp (re-check / prefetch mode); lazy from 96 per
    // warp — below that the contiguous-share pull without a materialised queue wins (C2
    // 1.574 -> 1.567 ms, C3 2.650 -> 2.628 ms against 8 per warp, same-box A/B)
    p.dense_min = (uint64_t)ctas * (threads / 32) * (opt.mode == Mode::Lazy ? 96 : 8);
    if (const char* d = getenv("BLEST_DENSE_MIN")) p.dense_min = (uint64_t)atoll(d);
    if (const char* x = getenv("BLEST_XFLAGS")) p.xflags = (uint32_t)atoi(x);
    p.tail_div = 8;  // dense lazy levels hand out their last eighth dynamically
    if (const char* t = getenv("BLEST_TAIL_DIV")) p.tail_div = (uint32_t)atoi(t);
    if (const char* rc = getenv("BLEST_LAZY_RECHECK")) p.lazy_recheck = (uint32_t)atoi(rc);
    // sparse lazy levels log their REDs' words (in Q0, unused then) so stage 2 visits those
    // words only; beyond words/8 log entries the Θ(n/32) sweep is cheaper
    p.log_cap = (uint32_t)std::min<uint64_t>(2 * qcap, std::max<uint64_t>(words_ / 8, 4096));
    if (const char* sm = getenv("BLEST_SMALL_S2"))  // the log lives in Q0: at most 2·qcap entries
        p.log_cap = (uint32_t)std::min<uint64_t>((uint64_t)std::max(0ll, atoll(sm)), 2 * qcap);
    cudaStream_t st = stream();
    CK(cudaMemsetAsync(bar_.p, 0, 4 * sizeof(unsigned), st));
    void* args[] = {&p};
    CK(cudaLaunchCooperativeKernel(kern, dim3(ctas), dim3(threads), args, dyn, st));
    g_launches.fetch_add(1);
    last_levels_ = p.L;
    last_ctas_ = ctas;
    last_threads_ = threads;
    last_src_ = src;
    last_mode_ = opt.mode;
    launched_ = true;
}

std::vector<BfsOutcome> BfsEngine::run_batch(const uint32_t* srcs, uint32_t count, const EngineOptions& opt,
                                             uint32_t* levels_host) {
    for (uint32_t k = 0; k < count; ++k)
        if (srcs[k] >= b_.n) throw InvalidArgument("bfs source out of range");
    std::vector<BfsOutcome> outs(count);
    if (!count) return outs;
    const uint64_t n = b_.n;
    // narrow transfers (xfer.cuh) unless BLEST_D2H_PACK=0: width 1, then 2, then plain u32
    // once a source's deepest level does not fit
    const char* pk = getenv("BLEST_D2H_PACK");
    const bool pack = levels_host && n && !(pk && atoi(pk) == 0);
    if (pack) ensure_xfer();
    if (!levels2_.p) levels2_.alloc(n ? n : 1);
    DevBuf<unsigned long long> summ(8ull * count);
    cudaStream_t st = stream(), cp = nullptr;
    cudaEvent_t kern_done[2] = {nullptr, nullptr}, copy_done[2] = {nullptr, nullptr};
    CK(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&kern_done[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&copy_done[i], cudaEventDisableTiming));
    }
    uint32_t* bufs[2] = {levels_.p, levels2_.p};
    const uint64_t slot = xfer_slot_bytes(n);
    int width = 1;
    std::vector<int> wk(count, 0);  // transfer width of source k (0 = u32 copy)
    std::vector<WidenPool::Job> jobs(count);
    std::vector<char> live(count, 0);
    auto drain = [&] {
        for (uint32_t j = 0; j < count; ++j)
            if (live[j]) {
                pool_->wait(&jobs[j]);
                live[j] = 0;
            }
    };
    // host side of source j once its copy has landed: widen it, or fetch the exact u32
    // array (still in its device buffer: the BFS two sources later waits for copy_done)
    auto finalize = [&](uint32_t j) {
        if (!wk[j]) return;
        const int s = j & 1;
        CK(cudaEventSynchronize(copy_done[s]));
        const unsigned long long deepest = stage_max_[j % kStageRing];
        const int w = wk[j];
        if (deepest < (w == 1 ? 255ull : 65535ull)) {
            WidenPool::Job& jb = jobs[j];
            jb.in = stage_ + (j % kStageRing) * slot;
            jb.width = w;
            jb.out = levels_host + (uint64_t)j * n;
            jb.n = n;
            pool_->submit(&jb);
            live[j] = 1;
        } else {
            CK(cudaMemcpyAsync(levels_host + (uint64_t)j * n, bufs[s], (size_t)n * 4, cudaMemcpyDeviceToHost, cp));
            CK(cudaEventRecord(copy_done[s], cp));
            if (width == w) width = (w == 1 && deepest < 65535ull) ? 2 : 0;
        }
    };
    try {
        for (uint32_t k = 0; k < count; ++k) {
            const int s = k & 1;
            if (k >= 2) {
                finalize(k - 2);
                CK(cudaStreamWaitEvent(st, copy_done[s], 0));  // buffer s free again
            }
            level_target_ = bufs[s];
            launch(srcs[k], opt);
            level_target_ = nullptr;
            k_summarise<<<1, 256, 0, st>>>(ctl_.p, trace_.p, trace_cap_, summ.p + 8ull * k);
            CK(cudaGetLastError());
            wk[k] = pack ? width : 0;
            if (wk[k]) pack_levels(bufs[s], n, wk[k], dpack_.p + s * slot, st);
            CK(cudaEventRecord(kern_done[s], st));
            if (levels_host && n) {
                CK(cudaStreamWaitEvent(cp, kern_done[s], 0));
                if (wk[k]) {
                    const uint32_t r = k % kStageRing;
                    if (k >= (uint32_t)kStageRing && live[k - kStageRing]) {  // staging slot r free
                        pool_->wait(&jobs[k - kStageRing]);
                        live[k - kStageRing] = 0;
                    }
                    CK(cudaMemcpyAsync(stage_ + r * slot, dpack_.p + s * slot, (size_t)n * wk[k],
                                       cudaMemcpyDeviceToHost, cp));
                    CK(cudaMemcpyAsync(stage_max_ + r, summ.p + 8ull * k + 1, 8, cudaMemcpyDeviceToHost, cp));
                } else {
                    CK(cudaMemcpyAsync(levels_host + (uint64_t)k * n, bufs[s], (size_t)n * 4,
                                       cudaMemcpyDeviceToHost, cp));
                }
            }
            CK(cudaEventRecord(copy_done[s], cp));
        }
        for (uint32_t j = count >= 2 ? count - 2 : 0; j < count; ++j) finalize(j);
        CK(cudaStreamSynchronize(st));
        CK(cudaStreamSynchronize(cp));
        drain();
    } catch (...) {
        level_target_ = nullptr;
        cudaStreamSynchronize(st);
        cudaStreamSynchronize(cp);
        drain();
        cudaStreamDestroy(cp);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(kern_done[i]);
            cudaEventDestroy(copy_done[i]);
        }
        throw;
    }
    CK(cudaStreamDestroy(cp));
    for (int i = 0; i < 2; ++i) {
        CK(cudaEventDestroy(kern_done[i]));
        CK(cudaEventDestroy(copy_done[i]));
    }
    std::vector<unsigned long long> h(8ull * count);
    CK(cudaMemcpy(h.data(), summ.p, h.size() * 8, cudaMemcpyDeviceToHost));
    for (uint32_t k = 0; k < count; ++k) {
        const unsigned long long* x = h.data() + 8ull * k;
        if (x[2])
            throw RuntimeError("BFS ran past the level safety cap at level " + std::to_string(x[0] + 1) +
                               " — engine invariant broken");
        BfsOutcome& o = outs[k];
        o.iterations = (uint32_t)x[0];
        o.max_level = (uint32_t)x[1];
        o.visited = 1 + x[4];
        o.trace_truncated = x[0] > trace_cap_;
        o.sum_queue = x[3];
        o.sum_full = x[5];
        o.sum_relaxed = x[6];
        o.sum_pushes = x[7];
    }
    launched_ = false;
    return outs;
}

BfsOutcome BfsEngine::finish(uint32_t* levels_host) {
    if (!launched_) throw LogicError("finish() without launch()");
    cudaStream_t st = stream();
    CK(cudaMemcpyAsync(pinned_, ctl_.p, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (levels_host && b_.n)
        CK(cudaMemcpyAsync(levels_host, levels_device(), (size_t)b_.n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    BfsOutcome out;
    out.iterations = (uint32_t)pinned_[4];
    out.max_level = (uint32_t)pinned_[5];
    out.unpulled_vss = last_exhaust_ ? pinned_[13] : 0;
    last_unpulled_ = out.unpulled_vss;
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
        out.sum_queue += r.queue_size;
        out.sum_full += r.full_atomics;
        out.sum_relaxed += r.relaxed_atomics;
        out.sum_pushes += r.queue_pushes;
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
