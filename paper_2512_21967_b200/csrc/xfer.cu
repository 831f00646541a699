// Narrow level-array transfers (xfer.cuh): the device pack kernel and the host widening pool.
#include "common.cuh"
#include "xfer.cuh"

#include <atomic>
#if defined(__x86_64__) || defined(__SSE2__)
#include <emmintrin.h>
#define BLEST_HAVE_SSE2 1
#endif

namespace blestgpu {

extern std::atomic<uint64_t> g_launches;

namespace {

// Four levels per thread: one 16 B load, one 4 B (u8) or 8 B (u16) store.
template <int W>
__global__ void k_pack_levels(const uint4* __restrict__ lv4, uint64_t n4, const uint32_t* __restrict__ lv, uint64_t n,
                              void* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 v = __ldcs(lv4 + i);  // read once: evict-first
        const uint32_t a = v.x + 1u, b = v.y + 1u, c = v.z + 1u, d = v.w + 1u;  // kInf -> 0
        if (W == 1)
            static_cast<uint32_t*>(out)[i] = (a & 0xFFu) | (b & 0xFFu) << 8 | (c & 0xFFu) << 16 | (d & 0xFFu) << 24;
        else
            static_cast<uint2*>(out)[i] = make_uint2((a & 0xFFFFu) | (b << 16), (c & 0xFFFFu) | (d << 16));
    }
    for (uint64_t i = 4 * n4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t a = lv[i] + 1u;
        if (W == 1)
            static_cast<uint8_t*>(out)[i] = (uint8_t)a;
        else
            static_cast<uint16_t*>(out)[i] = (uint16_t)a;
    }
}

}  // namespace

void pack_levels(const uint32_t* levels, uint64_t n, int width, void* out, cudaStream_t st) {
    if (!n) return;
    const uint64_t n4 = n / 4;  // levels come from cudaMalloc: 16 B aligned
    const unsigned blocks = grid_for(n4 ? n4 : 1, 256, (unsigned)num_sms() * 8);
    if (width == 1)
        k_pack_levels<1><<<blocks, 256, 0, st>>>(reinterpret_cast<const uint4*>(levels), n4, levels, n, out);
    else
        k_pack_levels<2><<<blocks, 256, 0, st>>>(reinterpret_cast<const uint4*>(levels), n4, levels, n, out);
    CK(cudaGetLastError());
    g_launches.fetch_add(1);
}

void widen_levels(const void* in, int width, uint32_t* out, uint64_t lo, uint64_t hi) {
    uint64_t i = lo;
    if (width == 1) {
        const uint8_t* p = static_cast<const uint8_t*>(in);
#ifdef BLEST_HAVE_SSE2
        for (; i < hi && (reinterpret_cast<uintptr_t>(out + i) & 15); ++i) out[i] = (uint32_t)p[i] - 1u;
        const __m128i zero = _mm_setzero_si128(), ones = _mm_set1_epi32(-1);
        for (; i + 16 <= hi; i += 16) {
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + i));
            const __m128i w0 = _mm_unpacklo_epi8(b, zero), w1 = _mm_unpackhi_epi8(b, zero);
            __m128i* o = reinterpret_cast<__m128i*>(out + i);
            _mm_stream_si128(o + 0, _mm_add_epi32(_mm_unpacklo_epi16(w0, zero), ones));
            _mm_stream_si128(o + 1, _mm_add_epi32(_mm_unpackhi_epi16(w0, zero), ones));
            _mm_stream_si128(o + 2, _mm_add_epi32(_mm_unpacklo_epi16(w1, zero), ones));
            _mm_stream_si128(o + 3, _mm_add_epi32(_mm_unpackhi_epi16(w1, zero), ones));
        }
        _mm_sfence();
#endif
        for (; i < hi; ++i) out[i] = (uint32_t)p[i] - 1u;
    } else {
        const uint16_t* p = static_cast<const uint16_t*>(in);
#ifdef BLEST_HAVE_SSE2
        for (; i < hi && (reinterpret_cast<uintptr_t>(out + i) & 15); ++i) out[i] = (uint32_t)p[i] - 1u;
        const __m128i zero = _mm_setzero_si128(), ones = _mm_set1_epi32(-1);
        for (; i + 8 <= hi; i += 8) {
            const __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + i));
            __m128i* o = reinterpret_cast<__m128i*>(out + i);
            _mm_stream_si128(o + 0, _mm_add_epi32(_mm_unpacklo_epi16(h, zero), ones));
            _mm_stream_si128(o + 1, _mm_add_epi32(_mm_unpackhi_epi16(h, zero), ones));
        }
        _mm_sfence();
#endif
        for (; i < hi; ++i) out[i] = (uint32_t)p[i] - 1u;
    }
}

WidenPool::WidenPool(int threads) {
    if (threads < 1) threads = 1;
    for (int t = 0; t < threads; ++t) workers_.emplace_back([this] { run(); });
}

WidenPool::~WidenPool() {
    {
        std::lock_guard<std::mutex> g(mu_);
        stop_ = true;
    }
    cv_work_.notify_all();
    for (auto& w : workers_) w.join();
}

void WidenPool::submit(Job* job) {
    // pieces of >= 1 M entries (4 MB of output), at most one per thread
    const uint64_t per = 1ull << 20;
    int parts = (int)std::min<uint64_t>((job->n + per - 1) / per, (uint64_t)workers_.size());
    if (parts < 1) parts = 1;
    {
        std::lock_guard<std::mutex> g(mu_);
        job->parts = parts;
        job->left = parts;
        for (int k = 0; k < parts; ++k) tasks_.emplace_back(job, k);
    }
    cv_work_.notify_all();
}

void WidenPool::wait(Job* job) {
    std::unique_lock<std::mutex> g(mu_);
    cv_done_.wait(g, [&] { return job->left == 0; });
}

void WidenPool::run() {
    for (;;) {
        std::pair<Job*, int> t;
        {
            std::unique_lock<std::mutex> g(mu_);
            cv_work_.wait(g, [&] { return stop_ || !tasks_.empty(); });
            if (tasks_.empty()) return;  // stop_ and drained
            t = tasks_.front();
            tasks_.pop_front();
        }
        Job* j = t.first;
        // 64-entry aligned piece bounds (whole 256 B of output per boundary)
        const uint64_t lo = (j->n * (uint64_t)t.second / j->parts) & ~63ull;
        const uint64_t hi = (t.second + 1 == j->parts) ? j->n : (j->n * (uint64_t)(t.second + 1) / j->parts) & ~63ull;
        widen_levels(j->in, j->width, j->out, lo, hi);
        bool done;
        {
            std::lock_guard<std::mutex> g(mu_);
            done = (--j->left == 0);
        }
        if (done) cv_done_.notify_all();
    }
}

}  // namespace blestgpu
