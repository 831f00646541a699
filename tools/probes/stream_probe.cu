// Probe: how fast can warps stream BVSS-shaped data (per VSS: one 128 B mask line from one
// array + 512 B of row ids from another) in queue order with B VSSs in flight per warp?
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t pol_ef() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint32_t ldm(const uint32_t* p, uint64_t pol) { uint32_t v; asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol)); return v; }
__device__ __forceinline__ uint4 ldr(const uint4* p, uint64_t pol) { uint4 v; asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol)); return v; }
template <int B>
__global__ void __launch_bounds__(512) k_stream(const uint32_t* __restrict__ masks, const uint4* __restrict__ rows, uint32_t nv, uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31, gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, NW = (gridDim.x * blockDim.x) >> 5;
    const uint64_t pol = pol_ef();
    uint32_t acc = 0;
    for (uint64_t p0 = gw; p0 < nv; p0 += (uint64_t)NW * B) {
        uint32_t m[B]; uint4 r[B];
        #pragma unroll
        for (int j = 0; j < B; ++j) {
            const uint64_t v = p0 + (uint64_t)j * NW;
            if (v < nv) { m[j] = ldm(masks + 32 * v + lane, pol); r[j] = ldr(rows + 32 * v + lane, pol); }
            else { m[j] = 0; r[j] = make_uint4(0,0,0,0); }
        }
        #pragma unroll
        for (int j = 0; j < B; ++j) acc ^= m[j] ^ r[j].x ^ r[j].y ^ r[j].z ^ r[j].w;
    }
    if (acc == 0x9e3779b9u) out[0] = acc;
}
int main() {
    const uint32_t nv = 5285149;
    uint32_t *masks, *out; uint4* rows;
    cudaMalloc(&masks, (size_t)nv * 128); cudaMalloc(&rows, (size_t)nv * 512); cudaMalloc(&out, 4);
    cudaMemset(masks, 1, (size_t)nv * 128); cudaMemset(rows, 2, (size_t)nv * 512);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](auto kern, const char* name, int blocks_per_sm) {
        int nb = sms * blocks_per_sm;
        kern<<<nb, 512>>>(masks, rows, nv, out);
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) kern<<<nb, 512>>>(masks, rows, nv, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%s blocks/SM=%d: %.1f GB/s (%s)\n", name, blocks_per_sm, 5.0 * nv * 640 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    run(k_stream<4>, "B=4", 2); run(k_stream<4>, "B=4", 4);
    run(k_stream<8>, "B=8", 2); run(k_stream<8>, "B=8", 4);
    run(k_stream<2>, "B=2", 4);
    return 0;
}
