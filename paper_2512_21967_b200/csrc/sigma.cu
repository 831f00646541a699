// Hot-row view builder (see sigma.cuh): slot histogram -> one 64-bit radix sort of
// (UINT32_MAX - count, row) -> engine ids (hot ranks, shifted rows) and σ⁻¹ of the hot
// ranks -> engine copy of row_ids.
#include <cub/cub.cuh>

#include <algorithm>

#include "sigma.cuh"

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
__global__ void k_rank_keys(const uint32_t* __restrict__ cnt, uint32_t n, uint64_t* __restrict__ keys) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x)
        keys[r] = ((uint64_t)(0xFFFFFFFFu - cnt[r]) << 32) | r;
}

// acc[0] = slots of the first K keys (the hot rows), acc[1] = all slots
__global__ void k_share(const uint64_t* __restrict__ keys, uint32_t n, uint32_t K, unsigned long long* acc) {
    unsigned long long hot = 0, all = 0;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n; q += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long c = 0xFFFFFFFFull - (keys[q] >> 32);
        all += c;
        if (q < K) hot += c;
    }
    for (int o = 16; o > 0; o >>= 1) {
        hot += __shfl_xor_sync(0xffffffffu, hot, o);
        all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (hot) atomicAdd(&acc[0], hot);
        if (all) atomicAdd(&acc[1], all);
    }
}

__global__ void k_engine_ids(uint32_t n, uint32_t base, uint32_t* __restrict__ sig) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x)
        sig[r] = base + (uint32_t)r;
}

__global__ void k_hot_tables(const uint64_t* __restrict__ keys, uint32_t K, uint32_t* __restrict__ sig,
                             uint32_t* __restrict__ inv) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < K;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)keys[q];
        inv[q] = r;
        sig[r] = (uint32_t)q;
    }
}

__global__ void k_sigma_rows(const uint4* __restrict__ rows, uint64_t n4, uint32_t n, const uint32_t* __restrict__ sig,
                             uint4* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = rows[i];
        v.x = v.x < n ? sig[v.x] : v.x;
        v.y = v.y < n ? sig[v.y] : v.y;
        v.z = v.z < n ? sig[v.z] : v.z;
        v.w = v.w < n ? sig[v.w] : v.w;
        out[i] = v;
    }
}

}  // namespace

void sigma_view_build(const DeviceBvss& b, SigmaView& out, uint32_t hot_cap) {
    cudaStream_t st = stream();
    const uint32_t n = b.n;
    const uint64_t slots = (uint64_t)b.num_vss * kTau;
    if (!hot_cap) hot_cap = 1u << 20;
    out.K = std::min(n, hot_cap);
    out.hot_words = ((uint64_t)out.K + 127) / 128 * 4;  // whole uint4 granules
    if (32 * out.hot_words + n >= (1ull << 32)) throw InvalidArgument("hot-row view needs n < 2^32 - K");
    out.sig.alloc(n ? n : 1);
    out.inv.alloc(out.K ? out.K : 1);
    if (n) {
        DevBuf<uint32_t> cnt(n);
        CK(cudaMemsetAsync(cnt.p, 0, (size_t)n * 4, st));
        if (slots) k_slot_hist<<<grid_for(slots, 256), 256, 0, st>>>(b.row_ids.p, slots, n, cnt.p);
        DevBuf<uint64_t> keys(n), keys2(n);
        k_rank_keys<<<grid_for(n, 256), 256, 0, st>>>(cnt.p, n, keys.p);
        size_t temp = 0;
        CK(cub::DeviceRadixSort::SortKeys(nullptr, temp, keys.p, keys2.p, (int64_t)n, 0, 64, st));
        DevBuf<unsigned char> tmp(temp ? temp : 1);
        CK(cub::DeviceRadixSort::SortKeys(tmp.p, temp, keys.p, keys2.p, (int64_t)n, 0, 64, st));
        // share of the slots held by the K hot rows (keys2 ascending = most slots first)
        {
            DevBuf<unsigned long long> acc(2);
            CK(cudaMemsetAsync(acc.p, 0, 16, st));
            k_share<<<grid_for(n, 256), 256, 0, st>>>(keys2.p, n, out.K, acc.p);
            CK(cudaGetLastError());
            unsigned long long h[2];
            CK(cudaMemcpyAsync(h, acc.p, 16, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            out.hot_share = h[1] ? (double)h[0] / (double)h[1] : 0.0;
        }
        k_engine_ids<<<grid_for(n, 256), 256, 0, st>>>(n, (uint32_t)(32 * out.hot_words), out.sig.p);
        if (out.K) k_hot_tables<<<grid_for(out.K, 256), 256, 0, st>>>(keys2.p, out.K, out.sig.p, out.inv.p);
    }
    out.rows.alloc(slots ? slots : 4);
    if (slots)
        k_sigma_rows<<<grid_for(slots / 4, 256), 256, 0, st>>>(reinterpret_cast<const uint4*>(b.row_ids.p),
                                                               slots / 4, n, out.sig.p,
                                                               reinterpret_cast<uint4*>(out.rows.p));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
}

}  // namespace blestgpu
