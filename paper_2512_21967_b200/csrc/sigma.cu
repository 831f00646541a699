// σ view builder (see sigma.cuh): slot histogram -> one 64-bit radix sort of
// (UINT32_MAX - count, row) -> σ / σ⁻¹ -> engine copy of row_ids.
#include <cub/cub.cuh>

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

// Rank q -> σ id: ranks stay contiguous within 128 B lines (1024 ids, the L1 unit), but the
// lines are dealt round-robin over kSpread stripes of σ space, so the hottest lines — the
// bulk of the early levels' discoveries — spread over all stage-2 chunks instead of one.
// Bijective: lines [0, B) with B = kSpread·⌊lines / kSpread⌋ are transposed, the rest kept.
constexpr uint32_t kSpread = 256;
__global__ void k_sigma_tables(const uint64_t* __restrict__ keys, uint32_t n, uint32_t* __restrict__ sig,
                               uint32_t* __restrict__ inv) {
    const uint64_t lines = ((uint64_t)n + 1023) / 1024;
    const uint64_t per = lines / kSpread, B = per * kSpread;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)keys[q];
        const uint64_t line = q >> 10;
        const uint64_t l2 = line < B ? (line % kSpread) * per + line / kSpread : line;
        const uint64_t id = (l2 << 10) | (q & 1023);
        // the last (partial) line keeps its ids < n; a full transposed line maps in range
        inv[id] = r;
        sig[r] = (uint32_t)id;
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

void sigma_view_build(const DeviceBvss& b, SigmaView& out) {
    cudaStream_t st = stream();
    const uint32_t n = b.n;
    const uint64_t slots = (uint64_t)b.num_vss * kTau;
    out.sig.alloc(n ? n : 1);
    out.inv.alloc(n ? n : 1);
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
        k_sigma_tables<<<grid_for(n, 256), 256, 0, st>>>(keys2.p, n, out.sig.p, out.inv.p);
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
