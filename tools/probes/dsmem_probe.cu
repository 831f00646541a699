// Probe: random 4-byte visited-bit lookups served from (a) L2 (2 MB array, L1 carveout max),
// (b) distributed shared memory of a 16-CTA cluster holding the 2 MB array in 128 KB slices,
// (c) distributed shared memory with 8-CTA clusters (portable size) holding 2 MB in 256 KB?
// (too big) -> 8 x 200 KB = 1.6 MB (index masked). Reports lookups/s. Also checks that a
// cooperative launch accepts a cluster dimension.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

__global__ void k_l2(const uint32_t* __restrict__ v, uint32_t words, uint32_t iters, uint32_t* out) {
    uint32_t acc = 0, s = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t i = 0; i < iters; i += 4) {
        uint32_t a0 = hash32(s + i) % words, a1 = hash32(s + i + 1) % words, a2 = hash32(s + i + 2) % words, a3 = hash32(s + i + 3) % words;
        acc += v[a0] + v[a1] + v[a2] + v[a3];
    }
    if (acc == 0x12345678) out[0] = acc;
}

template <int CL>
__global__ void k_dsmem(const uint32_t* __restrict__ v, uint32_t words, uint32_t slice_words, uint32_t iters, uint32_t* out) {
    extern __shared__ uint32_t sl[];
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t rank = cl.block_rank();
    for (uint32_t i = threadIdx.x; i < slice_words; i += blockDim.x) sl[i] = v[(rank * slice_words + i) % words];
    cl.sync();
    uint32_t acc = 0, s = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t total = slice_words * CL;
    for (uint32_t i = 0; i < iters; i += 4) {
        uint32_t a[4];
        #pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = hash32(s + i + k) % total;
        #pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t* remote = cl.map_shared_rank(sl, a[k] / slice_words);
            acc += remote[a[k] % slice_words];
        }
    }
    cl.sync();
    if (acc == 0x12345678) out[0] = acc;
}

int main() {
    const uint32_t words = 512 * 1024;  // 2 MB
    uint32_t *v, *out;
    cudaMalloc(&v, words * 4); cudaMalloc(&out, 4);
    cudaMemset(v, 1, words * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const uint32_t iters = 4096;
    // (a) L2
    {
        int bs = 512, nb = sms * 4;
        k_l2<<<nb, bs>>>(v, words, iters, out);
        cudaEventRecord(e0);
        k_l2<<<nb, bs>>>(v, words, iters, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("L2 random 4B loads: %.1f G/s (%s)\n", (double)nb * bs * iters / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    // (b) DSMEM cluster 16 (non-portable) and 8
    auto run = [&](auto kern, int CL, uint32_t slice_words) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, slice_words * 4);
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = slice_words * 4;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        int ncl = 0;
        cfg.gridDim = dim3(CL); cfg.attrs = at; cfg.numAttrs = 1;
        cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg);
        cfg.gridDim = dim3(CL * ncl);
        printf("cluster %d: max active clusters %d\n", CL, ncl);
        cudaLaunchKernelEx(&cfg, kern, (const uint32_t*)v, words, slice_words, iters, out);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, kern, (const uint32_t*)v, words, slice_words, iters, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("DSMEM cluster %d random 4B loads: %.1f G/s (%s)\n", CL, (double)CL * ncl * 1024 * iters / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        // cooperative + cluster
        at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
        cfg.numAttrs = 2;
        cudaError_t err = cudaLaunchKernelEx(&cfg, kern, (const uint32_t*)v, words, slice_words, iters, out);
        cudaDeviceSynchronize();
        printf("cooperative+cluster %d launch: %s / %s\n", CL, cudaGetErrorString(err), cudaGetErrorString(cudaGetLastError()));
    };
    run(k_dsmem<16>, 16, words / 16);
    run(k_dsmem<8>, 8, 48 * 1024);
    return 0;
}
