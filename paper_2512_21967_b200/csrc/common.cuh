// Shared device/host helpers for the BLEST B200 library (sm_100a only).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#if !defined(__CUDA_ARCH__) || __CUDA_ARCH__ >= 1000
#else
#error "libblest_b200 targets sm_100a only"
#endif

namespace blestgpu {

constexpr uint32_t kInf = 0xFFFFFFFFu;  // kUnreached (R:include/blest/graph.hpp:20)
constexpr uint32_t kSigma = 8;          // slice width (R:src/bvss.cpp:14-17)
constexpr uint32_t kTau = 128;          // slots per VSS (BvssConfig::tau, R:include/blest/bvss.hpp:19-21)

// Error classes mirror the reference's exception types (SURVEY §8(b) "Errors").
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct LogicError : std::logic_error {
    using std::logic_error::logic_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                        std::to_string(line) + ")");
}
#define CK(x) ::blestgpu::cuda_check((x), #x, __FILE__, __LINE__)

// The library-wide stream (set through blest_set_stream; default = legacy stream 0).
cudaStream_t stream();
void set_stream(cudaStream_t s);
int num_sms();

// RAII device buffer.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t count = 0;
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), count(o.count) { o.p = nullptr; o.count = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; count = o.count; o.p = nullptr; o.count = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t n) {
        release();
        count = n;
        if (n) CK(cudaMalloc(&p, n * sizeof(T)));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        count = 0;
    }
    size_t bytes() const { return count * sizeof(T); }
};

inline unsigned grid_for(uint64_t work, unsigned threads, unsigned cap_blocks = 0) {
    uint64_t b = (work + threads - 1) / threads;
    if (b == 0) b = 1;
    const uint64_t cap = cap_blocks ? cap_blocks : static_cast<uint64_t>(num_sms()) * 32;
    return static_cast<unsigned>(b < cap ? b : cap);
}

#ifdef __CUDACC__
// Streaming loads for the read-once BVSS arrays: non-coherent path, no L1 allocation,
// L2 evict-first policy so the hot state (levels / bitmaps / queues) keeps its lines.
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p, uint64_t pol) {
    uint4 v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}
// Predicated streaming row-id load: lanes whose pull found no candidate (every column's
// mask & α is 0) skip it and get zeros — pull_vss never dereferences their row ids
// (R:src/bfs_engine.cpp:131-146), so a 128 B line none of its 8 lanes needs is not fetched.
__device__ __forceinline__ uint4 ld_stream_u4_if(bool pred, const uint4* p, uint64_t pol) {
    uint4 v;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
        "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\tmov.b32 %2, 0;\n\tmov.b32 %3, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %6;\n\t}"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "r"((uint32_t)pred), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const unsigned* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Same load without the compiler barrier: for data whose ordering the caller does not
// need (e.g. a racy pre-check before an idempotent RED), so loads keep overlapping.
__device__ __forceinline__ uint32_t ld_l2_u32(const uint32_t* p) {
    uint32_t v;
    asm("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Grid-wide barrier of the cooperatively launched persistent grid. cooperative_groups'
// grid.sync() (one atomic per CTA on a flip-bit counter, no reset/release store) measured
// 1.2 µs on B200 vs 2.4-3.3 µs for a count-reset-generation barrier (tools/probes/
// barrier_probe.cu), so it is the primitive; `payload` (a value every CTA needs right after
// the barrier, e.g. the next queue length) is then read once per CTA and broadcast.
// payload2 (optional): a second word read with the first (same 128 B line in practice, so no
// extra latency), returned through out2.
// payload2 (optional): a second word read with the first (same 128 B line in practice, so no
// extra latency), returned through out2.
__device__ __forceinline__ uint32_t grid_barrier_pay(unsigned* bar, unsigned& gen, const unsigned long long* payload,
                                                     const unsigned long long* payload2 = nullptr,
                                                     unsigned long long* out2 = nullptr) {
    (void)bar;
    __shared__ uint32_t s_pay;
    __shared__ unsigned long long s_pay2;
    cooperative_groups::this_grid().sync();
    gen += 1;
    if (!payload && !payload2) return 0;
    if (threadIdx.x == 0) {
        if (payload) s_pay = (uint32_t)ld_relaxed_gpu_u64(payload);
        if (payload2) s_pay2 = ld_relaxed_gpu_u64(payload2);
    }
    __syncthreads();
    if (payload2) *out2 = s_pay2;
    return payload ? s_pay : 0u;
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) { grid_barrier_pay(bar, gen, nullptr); }

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
    const unsigned lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<unsigned>(o)) x += y;
    }
    return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
#endif

}  // namespace blestgpu
