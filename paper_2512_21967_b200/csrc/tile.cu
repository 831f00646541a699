// Known-answer entry for the b1 tile (tc::mma_m8n8k128 + build_fragB + pack_fragA_round,
// R:src/tc_emu.cpp:9-45) on the device: one warp per tile runs the engine's own pull
// (column_counts<PULL = mma>, bfs_device.cuh — two mma.sync.m8n8k128.b1.and.popc per VSS)
// and writes the full 8x8 FragC of both rounds, lane t's pair at (t/4, 2(t%4)+{0,1})
// (the PTX fragment layout the reference's FragC follows, R:include/blest/tc_emu.hpp:67-75).
// Tests feed it the reference's tile KATs (R:tests/tc_emu_test.cpp:186-241).
#include "bfs_device.cuh"

namespace blestgpu {

extern std::atomic<uint64_t> g_launches;

namespace {

__global__ void k_tile_pull(const uint32_t* __restrict__ masks, const uint8_t* __restrict__ alpha, uint32_t count,
                            uint32_t* __restrict__ out) {
    const uint32_t tile = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (tile >= count) return;  // warp-uniform
    const unsigned lane = threadIdx.x & 31;
    uint32_t cnt[4];
    bfsdev::column_counts<1>(masks[32ull * tile + lane], alpha[tile], cnt);
    uint32_t* c = out + 128ull * tile;
    const uint32_t i = lane / 4, j = 2 * (lane % 4);
    for (int round = 0; round < 2; ++round) {
        c[64 * round + 8 * i + j] = cnt[2 * round];
        c[64 * round + 8 * i + j + 1] = cnt[2 * round + 1];
    }
}

}  // namespace

void tile_pull_device(const uint32_t* masks, const uint8_t* alpha, uint32_t count, uint32_t* counts) {
    if (!count) return;
    cudaStream_t st = stream();
    DevBuf<uint32_t> dm(32ull * count), dc(128ull * count);
    DevBuf<uint8_t> da(count);
    CK(cudaMemcpyAsync(dm.p, masks, 128ull * count, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(da.p, alpha, count, cudaMemcpyHostToDevice, st));
    k_tile_pull<<<(count + 3) / 4, 128, 0, st>>>(dm.p, da.p, count, dc.p);
    CK(cudaGetLastError());
    g_launches.fetch_add(1);
    CK(cudaMemcpyAsync(counts, dc.p, 512ull * count, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

}  // namespace blestgpu
