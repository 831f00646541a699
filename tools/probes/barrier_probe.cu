// Probe: cost of one grid-wide barrier (the library's grid_barrier_pay) vs cooperative
// groups grid.sync(), for the persistent grid shapes the BFS uses.
#include <cooperative_groups.h>
#include <cstdio>
#include "../../paper_2512_21967_b200/csrc/common.cuh"
namespace cg = cooperative_groups;
using namespace blestgpu;
namespace blestgpu { cudaStream_t stream() { return 0; } void set_stream(cudaStream_t) {} int num_sms() { return 148; } }
__global__ void k_ours(unsigned* bar, int iters, unsigned long long* pay) {
    unsigned gen = 0;
    for (int i = 0; i < iters; ++i) grid_barrier_pay(bar, gen, pay);
}
__global__ void k_cg(int iters) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}
int main() {
    unsigned* bar; unsigned long long* pay;
    cudaMalloc(&bar, 16); cudaMalloc(&pay, 8); cudaMemset(pay, 0, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int threads : {256, 512, 1024}) for (int per_sm : {1, 2, 4}) {
        if (threads * per_sm > 2048) continue;
        int ctas = 148 * per_sm, iters = 2000;
        void* a1[] = {&bar, &iters, &pay};
        cudaMemset(bar, 0, 16);
        cudaLaunchCooperativeKernel((void*)k_ours, ctas, threads, a1, 0, 0);
        cudaMemset(bar, 0, 16);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_ours, ctas, threads, a1, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        void* a2[] = {&iters};
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_cg, ctas, threads, a2, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms2; cudaEventElapsedTime(&ms2, e0, e1);
        printf("%4d CTAs x %4d thr: ours %.2f us/barrier, cg::grid.sync %.2f us (%s)\n", ctas, threads,
               ms * 1e3 / iters, ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
}
