// Host widening throughput of the narrow batch transfers (xfer.cuh) on this box's CPUs:
// 1-byte (level + 1) -> u32 levels, n = 2^24 (C2) and 2^27 (C5), pool of T threads.
//   g++ -O2 -std=c++17 -I paper_2512_21967_b200/csrc -I /usr/local/cuda/include tools/probes/widen_probe.cpp \
//       -L paper_2512_21967_b200 -lblest_b200 -L /usr/local/cuda/lib64 -lcudart -pthread -o /tmp/widen_probe
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "xfer.cuh"

int main(int argc, char** argv) {
    for (uint64_t n : {1ull << 24, 1ull << 27}) {
        uint8_t* in = nullptr;
        uint32_t* out = nullptr;
        cudaHostAlloc((void**)&in, n, cudaHostAllocDefault);
        cudaHostAlloc((void**)&out, 4 * n, cudaHostAllocDefault);
        for (uint64_t i = 0; i < n; ++i) in[i] = (uint8_t)(i % 9);
        memset(out, 0, 4 * n);
        for (int t : {1, 4, 8, 16, 32}) {
            blestgpu::WidenPool pool(t);
            double best = 1e9;
            for (int r = 0; r < 5; ++r) {
                blestgpu::WidenPool::Job j;
                j.in = in; j.width = 1; j.out = out; j.n = n;
                auto t0 = std::chrono::steady_clock::now();
                pool.submit(&j);
                pool.wait(&j);
                best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
            }
            printf("n=%llu threads=%d widen %.3f ms  (%.1f GB/s of u32 output)\n", (unsigned long long)n, t,
                   1e3 * best, 4.0 * n / best / 1e9);
        }
        cudaFreeHost(in);
        cudaFreeHost(out);
    }
    return 0;
}
