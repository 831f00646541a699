// Hub view builder (see hubs.cuh): slot histogram -> one 64-bit radix sort of
// (~count, row) -> hub tables -> engine copy of row_ids with virtual hub ids.
#include <cub/cub.cuh>

#include <cstdlib>

#include "hubs.cuh"

namespace blestgpu {

namespace {

// Slots per row (padding slots carry row n and are skipped).
__global__ void k_slot_hist(const uint32_t* __restrict__ rows, uint64_t slots, uint32_t n,
                            uint32_t* __restrict__ cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < slots;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = rows[i];
        if (r < n) atomicAdd(cnt + r, 1u);
    }
}

// key = (UINT32_MAX - count) << 32 | row: ascending order = most slots first, ties by id.
__global__ void k_hub_keys(const uint32_t* __restrict__ cnt, uint32_t n, uint64_t* __restrict__ keys,
                           unsigned long long* __restrict__ nonzero) {
    unsigned long long mine = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        keys[r] = ((uint64_t)(0xFFFFFFFFu - cnt[r]) << 32) | r;
        mine += cnt[r] != 0;
    }
    mine = warp_sum(mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(nonzero, mine);
}

__global__ void k_hub_tables(const uint64_t* __restrict__ keys, uint32_t K, uint32_t NL, bool spread,
                             uint32_t* __restrict__ hub_rows, uint32_t* __restrict__ hub_of) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < K;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)keys[q];
        const uint32_t line = (uint32_t)(q % NL), d = (uint32_t)(q / NL);
        const uint32_t h = spread ? line * 1024u + ((line + d) & 31u) * 32u + (d >> 5) : (uint32_t)q;
        hub_rows[h] = r;
        hub_of[r] = h;
    }
}

__global__ void k_flag_rows(const uint4* __restrict__ rows, uint64_t n4, const uint32_t* __restrict__ hub_of,
                            uint32_t hub_base, uint4* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = rows[i];
        uint32_t* e = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t h = hub_of[e[c]];  // hub_of has n + 1 entries (padding row n)
            if (h != kNoHub) e[c] = hub_base + h;
        }
        out[i] = v;
    }
}

__global__ void k_fill(uint32_t* __restrict__ p, uint64_t count, uint32_t val) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = val;
}

}  // namespace

void hub_view_build(const DeviceBvss& b, uint32_t max_hubs, uint32_t hub_base, HubView& out) {
    if (b.n >= kHubFlag || hub_base < b.n) throw InvalidArgument("hub view needs n < 2^31");
    cudaStream_t st = stream();
    const uint32_t n = b.n;
    const uint64_t slots = (uint64_t)b.num_vss * kTau;
    out.hub_of.alloc((uint64_t)n + 1);
    k_fill<<<grid_for(n + 1ull, 256), 256, 0, st>>>(out.hub_of.p, n + 1ull, kNoHub);
    out.K = 0;
    if (n && slots && max_hubs) {
        DevBuf<uint32_t> cnt(n);
        CK(cudaMemsetAsync(cnt.p, 0, (size_t)n * 4, st));
        k_slot_hist<<<grid_for(slots, 256), 256, 0, st>>>(b.row_ids.p, slots, n, cnt.p);
        DevBuf<uint64_t> keys(n), keys2(n);
        DevBuf<unsigned long long> nz(1);
        CK(cudaMemsetAsync(nz.p, 0, 8, st));
        k_hub_keys<<<grid_for(n, 256), 256, 0, st>>>(cnt.p, n, keys.p, nz.p);
        size_t temp = 0;
        CK(cub::DeviceRadixSort::SortKeys(nullptr, temp, keys.p, keys2.p, (int64_t)n, 0, 64, st));
        DevBuf<unsigned char> tmp(temp ? temp : 1);
        CK(cub::DeviceRadixSort::SortKeys(tmp.p, temp, keys.p, keys2.p, (int64_t)n, 0, 64, st));
        unsigned long long nonzero = 0;
        CK(cudaMemcpyAsync(&nonzero, nz.p, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        out.K = (uint32_t)std::min<unsigned long long>(nonzero, max_hubs / 1024 * 1024);
        out.bits = (out.K + 1023) / 1024 * 1024;
        const char* sp = getenv("BLEST_HUB_SPREAD");
        const bool spread = !(sp && atoi(sp) == 0);
        out.hub_rows.alloc(out.bits ? out.bits : 1);
        if (out.K)
            k_hub_tables<<<grid_for(out.K, 256), 256, 0, st>>>(keys2.p, out.K, out.bits / 1024, spread,
                                                              out.hub_rows.p, out.hub_of.p);
    }
    out.rows.alloc(slots ? slots : 1);
    if (slots)
        k_flag_rows<<<grid_for(slots / 4, 256), 256, 0, st>>>(reinterpret_cast<const uint4*>(b.row_ids.p),
                                                             slots / 4, out.hub_of.p, hub_base,
                                                             reinterpret_cast<uint4*>(out.rows.p));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
}

}  // namespace blestgpu
