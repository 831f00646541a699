// GPU BVSS builder: arcs (u -> v) become (slice set u>>3, row v, bit u&7) pairs,
// radix-sorted by (set, row), OR-reduced by key into slices, counted per set, scanned
// into real_ptrs, and scattered column-major into the lane grid.
// Reference: build_bvss (R:src/bvss.cpp:19-101) — pass 1 count (:35-53), v2r (:55-58),
// sentinel fill (:60-61), pass 2 merge + placement (:65-98).
#include <cub/cub.cuh>

#include <vector>

#include "bvss.cuh"

namespace blestgpu {

namespace {

// Arcs whose target row lies outside [row_lo, row_hi) get the drop key (all ones, sorts
// last); `kept` counts the arcs inside (the structure's m).
__global__ void k_slice_pairs(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                              uint32_t n, uint32_t row_lo, uint32_t row_hi, uint64_t* __restrict__ keys,
                              uint8_t* __restrict__ bits, unsigned long long* __restrict__ kept) {
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long mine = 0;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n;
         u += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint64_t hi = (u >> 3) << 32;
        const uint8_t bit = (uint8_t)(1u << (u & 7));
        for (uint64_t i = off[u] + lane; i < off[u + 1]; i += 32) {
            const uint32_t v = tgt[i];
            const bool in = v >= row_lo && v < row_hi;
            keys[i] = in ? (hi | v) : ~0ull;
            bits[i] = in ? bit : (uint8_t)0;
            mine += in;
        }
    }
    mine = warp_sum(mine);
    if (lane == 0 && mine) atomicAdd(kept, mine);
}

// Row-range builds (one multi-GPU rank): only the arcs into [row_lo, row_hi) get a key, so
// the sort and the reduction run over this rank's share of m, not all of it. Pass 1
// (out == nullptr) counts them; pass 2 writes them (warp-aggregated slots, any order: the
// radix sort follows).
__global__ void k_slice_pairs_rows(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt, uint32_t n,
                                   uint32_t row_lo, uint32_t row_hi, uint64_t* __restrict__ keys,
                                   uint8_t* __restrict__ bits, unsigned long long* __restrict__ ctr) {
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long mine = 0;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n;
         u += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint64_t hi = (u >> 3) << 32;
        const uint8_t bit = (uint8_t)(1u << (u & 7));
        for (uint64_t i0 = off[u]; i0 < off[u + 1]; i0 += 32) {
            const uint64_t i = i0 + lane;
            const uint32_t v = i < off[u + 1] ? tgt[i] : row_hi;
            const bool in = v >= row_lo && v < row_hi;
            const unsigned ball = __ballot_sync(0xffffffffu, in);
            if (!keys) {
                mine += in;
                continue;
            }
            unsigned long long base = 0;
            if (lane == 0 && ball) base = atomicAdd(ctr, (unsigned long long)__popc(ball));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (in) {
                const uint64_t at = base + __popc(ball & ((1u << lane) - 1u));
                keys[at] = hi | v;
                bits[at] = bit;
            }
        }
    }
    if (!keys) {
        mine = warp_sum(mine);
        if (lane == 0 && mine) atomicAdd(ctr, mine);
    }
}

struct OrOp {
    __device__ __forceinline__ uint8_t operator()(uint8_t a, uint8_t b) const { return a | b; }
};

// set_start[s] = first slice index whose set >= s, s in [0, num_sets].
__global__ void k_set_starts(const uint64_t* __restrict__ skeys, uint64_t ns, uint32_t num_sets,
                             uint64_t* __restrict__ start) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= ns;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = (i < ns) ? (skeys[i] >> 32) : (uint64_t)num_sets;
        const uint64_t from = (i == 0) ? 0 : (skeys[i - 1] >> 32) + 1;
        for (uint64_t t = from; t <= s && t <= num_sets; ++t) start[t] = i;
    }
}

__global__ void k_vss_counts(const uint64_t* __restrict__ start, uint32_t num_sets,
                             uint32_t* __restrict__ cnt) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s <= num_sets;
         s += (uint64_t)gridDim.x * blockDim.x)
        cnt[s] = (s < num_sets) ? (uint32_t)((start[s + 1] - start[s] + kTau - 1) / kTau) : 0u;
}

__global__ void k_v2r(const uint32_t* __restrict__ rp, uint32_t num_sets, uint32_t* __restrict__ v2r) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < num_sets;
         s += (uint64_t)gridDim.x * blockDim.x)
        for (uint32_t v = rp[s]; v < rp[s + 1]; ++v) v2r[v] = (uint32_t)s;
}

__global__ void k_fill_u32(uint32_t* __restrict__ p, uint64_t count, uint32_t val) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = val;
}

__global__ void k_place(const uint64_t* __restrict__ skeys, const uint8_t* __restrict__ smask,
                        uint64_t ns, const uint64_t* __restrict__ start, const uint32_t* __restrict__ rp,
                        uint32_t* __restrict__ row_ids, uint8_t* __restrict__ mask_bytes) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ns;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = skeys[i];
        const uint32_t s = (uint32_t)(key >> 32);
        const uint64_t k = i - start[s];
        const uint64_t v = (uint64_t)rp[s] + k / kTau;
        const uint32_t slot = (uint32_t)(k % kTau), lane = slot & 31, col = slot >> 5;
        const uint64_t at = 4 * (32 * v + lane) + col;
        row_ids[at] = (uint32_t)key;
        mask_bytes[at] = smask[i];  // byte `col` of the little-endian word masks[32v+lane]
    }
}

template <typename T>
void radix_pairs(DevBuf<uint64_t>& k, DevBuf<T>& v, uint64_t count, int end_bit) {
    if (count <= 1) return;
    cudaStream_t st = stream();
    DevBuf<uint64_t> k2(count);
    DevBuf<T> v2(count);
    cub::DoubleBuffer<uint64_t> dk(k.p, k2.p);
    cub::DoubleBuffer<T> dv(v.p, v2.p);
    size_t temp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, temp, dk, dv, (int64_t)count, 0, end_bit, st));
    DevBuf<unsigned char> tmp(temp);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, temp, dk, dv, (int64_t)count, 0, end_bit, st));
    if (dk.Current() != k.p) std::swap(k, k2);
    if (dv.Current() != v.p) std::swap(v, v2);
}

int bits_of(uint64_t x) {
    int b = 0;
    while (b < 64 && (x >> b)) ++b;
    return b;
}

}  // namespace

DeviceBvss bvss_build(const DeviceGraph& g, uint32_t row_lo, uint32_t row_hi) {
    cudaStream_t st = stream();
    if (row_hi > g.n) row_hi = g.n;
    if (row_lo > row_hi) row_lo = row_hi;
    const bool all_rows = row_lo == 0 && row_hi == g.n;
    DeviceBvss b;
    b.n = g.n;
    b.m = g.m;
    b.row_lo = row_lo;
    b.row_hi = row_hi;
    b.num_sets = (uint32_t)(((uint64_t)g.n + kSigma - 1) / kSigma);
    b.real_ptrs.alloc((size_t)b.num_sets + 1);
    CK(cudaMemsetAsync(b.real_ptrs.p, 0, ((size_t)b.num_sets + 1) * 4, st));
    const uint64_t m = g.m;
    if (m == 0 || g.n == 0) {
        CK(cudaStreamSynchronize(st));
        return b;
    }
    // 1. (set, row) keys with the column bit, one per arc (row range: one per kept arc).
    uint64_t mk = m;
    DevBuf<uint64_t> keys;
    DevBuf<uint8_t> bits;
    if (all_rows) {
        keys.alloc(m);
        bits.alloc(m);
        DevBuf<unsigned long long> kept(1);
        CK(cudaMemsetAsync(kept.p, 0, 8, st));
        k_slice_pairs<<<grid_for((uint64_t)g.n * 32, 256), 256, 0, st>>>(g.off.p, g.tgt.p, g.n, row_lo, row_hi,
                                                                        keys.p, bits.p, kept.p);
        CK(cudaGetLastError());
    } else {
        DevBuf<unsigned long long> ctr(1);
        CK(cudaMemsetAsync(ctr.p, 0, 8, st));
        k_slice_pairs_rows<<<grid_for((uint64_t)g.n * 32, 256), 256, 0, st>>>(g.off.p, g.tgt.p, g.n, row_lo, row_hi,
                                                                             nullptr, nullptr, ctr.p);
        CK(cudaGetLastError());
        unsigned long long hk = 0;
        CK(cudaMemcpyAsync(&hk, ctr.p, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        mk = hk;
        b.m = hk;
        if (mk == 0) {
            CK(cudaStreamSynchronize(st));
            return b;
        }
        keys.alloc(mk);
        bits.alloc(mk);
        CK(cudaMemsetAsync(ctr.p, 0, 8, st));
        k_slice_pairs_rows<<<grid_for((uint64_t)g.n * 32, 256), 256, 0, st>>>(g.off.p, g.tgt.p, g.n, row_lo, row_hi,
                                                                             keys.p, bits.p, ctr.p);
        CK(cudaGetLastError());
    }
    radix_pairs(keys, bits, mk, 32 + bits_of(b.num_sets));
    // 2. OR-reduce by key -> unpadded slices, sorted by (set, row) (R:src/bvss.cpp:75-88).
    DevBuf<uint64_t> skeys(mk);
    DevBuf<uint8_t> smask(mk);
    DevBuf<unsigned long long> nsl(1);
    {
        size_t temp = 0;
        CK(cub::DeviceReduce::ReduceByKey(nullptr, temp, keys.p, skeys.p, bits.p, smask.p, nsl.p,
                                          OrOp(), (int64_t)mk, st));
        DevBuf<unsigned char> tmp(temp);
        CK(cub::DeviceReduce::ReduceByKey(tmp.p, temp, keys.p, skeys.p, bits.p, smask.p, nsl.p,
                                          OrOp(), (int64_t)mk, st));
    }
    unsigned long long ns = 0;
    CK(cudaMemcpyAsync(&ns, nsl.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    keys.release();
    bits.release();
    b.num_unpadded = ns;
    // 3. per-set slice ranges -> VSS counts -> real_ptrs (R:src/bvss.cpp:48-53).
    DevBuf<uint64_t> start((size_t)b.num_sets + 1);
    k_set_starts<<<grid_for(ns + 1, 256), 256, 0, st>>>(skeys.p, ns, b.num_sets, start.p);
    DevBuf<uint32_t> cnt((size_t)b.num_sets + 1);
    k_vss_counts<<<grid_for((uint64_t)b.num_sets + 1, 256), 256, 0, st>>>(start.p, b.num_sets, cnt.p);
    CK(cudaGetLastError());
    {
        size_t temp = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, temp, cnt.p, b.real_ptrs.p, (int64_t)b.num_sets + 1, st));
        DevBuf<unsigned char> tmp(temp);
        CK(cub::DeviceScan::ExclusiveSum(tmp.p, temp, cnt.p, b.real_ptrs.p, (int64_t)b.num_sets + 1, st));
    }
    uint32_t nv = 0;
    CK(cudaMemcpyAsync(&nv, b.real_ptrs.p + b.num_sets, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    b.num_vss = nv;
    // 4. v2r, sentinel/zero fill, placement (R:src/bvss.cpp:55-61, :89-97).
    b.v2r.alloc(nv ? nv : 1);
    b.masks.alloc((uint64_t)nv * 32 ? (uint64_t)nv * 32 : 1);
    b.row_ids.alloc((uint64_t)nv * kTau ? (uint64_t)nv * kTau : 1);
    k_v2r<<<grid_for(b.num_sets, 256), 256, 0, st>>>(b.real_ptrs.p, b.num_sets, b.v2r.p);
    k_fill_u32<<<grid_for((uint64_t)nv * kTau, 256), 256, 0, st>>>(b.row_ids.p, (uint64_t)nv * kTau, g.n);
    CK(cudaMemsetAsync(b.masks.p, 0, (uint64_t)nv * 32 * 4, st));
    k_place<<<grid_for(ns, 256), 256, 0, st>>>(skeys.p, smask.p, ns, start.p, b.real_ptrs.p, b.row_ids.p,
                                               reinterpret_cast<uint8_t*>(b.masks.p));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return b;
}

namespace {
__global__ void k_check_upload(const uint32_t* rp, uint32_t num_sets, const uint32_t* v2r, uint32_t nv,
                               const uint32_t* rows, const uint32_t* masks, uint32_t n,
                               unsigned long long* unpadded, unsigned* bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)nv * kTau;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = rows[i];
        const uint32_t mk = (masks[i >> 2] >> (8 * (i & 3))) & 0xFFu;
        if (r != n) {
            atomicAdd(unpadded, 1ull);
            if (r > n) atomicOr(bad, 1u);
        } else if (mk) {
            atomicOr(bad, 2u);  // padded slot with a nonzero mask would be dereferenced
        }
    }
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < num_sets;
         s += (uint64_t)gridDim.x * blockDim.x) {
        if (rp[s] > rp[s + 1]) atomicOr(bad, 4u);
        else
            for (uint32_t v = rp[s]; v < rp[s + 1] && v < nv; ++v)
                if (v2r[v] != s) atomicOr(bad, 8u);
    }
}
}  // namespace

DeviceBvss bvss_upload(uint32_t n, uint64_t m, uint32_t num_vss, const uint32_t* real_ptrs,
                       const uint32_t* v2r, const uint32_t* row_ids, const uint32_t* masks,
                       bool host_ptrs) {
    cudaStream_t st = stream();
    DeviceBvss b;
    b.n = n;
    b.m = m;
    b.num_sets = (uint32_t)(((uint64_t)n + kSigma - 1) / kSigma);
    b.num_vss = num_vss;
    const cudaMemcpyKind kind = host_ptrs ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    b.real_ptrs.alloc((size_t)b.num_sets + 1);
    b.v2r.alloc(num_vss ? num_vss : 1);
    b.masks.alloc((uint64_t)num_vss * 32 ? (uint64_t)num_vss * 32 : 1);
    b.row_ids.alloc((uint64_t)num_vss * kTau ? (uint64_t)num_vss * kTau : 1);
    CK(cudaMemcpyAsync(b.real_ptrs.p, real_ptrs, ((size_t)b.num_sets + 1) * 4, kind, st));
    if (num_vss) {
        CK(cudaMemcpyAsync(b.v2r.p, v2r, (size_t)num_vss * 4, kind, st));
        CK(cudaMemcpyAsync(b.masks.p, masks, (uint64_t)num_vss * 32 * 4, kind, st));
        CK(cudaMemcpyAsync(b.row_ids.p, row_ids, (uint64_t)num_vss * kTau * 4, kind, st));
    }
    uint32_t last = 0;
    CK(cudaMemcpyAsync(&last, b.real_ptrs.p + b.num_sets, 4, cudaMemcpyDeviceToHost, st));
    DevBuf<unsigned long long> unp(1);
    DevBuf<unsigned> bad(1);
    CK(cudaMemsetAsync(unp.p, 0, 8, st));
    CK(cudaMemsetAsync(bad.p, 0, 4, st));
    k_check_upload<<<grid_for((uint64_t)num_vss * kTau + b.num_sets, 256), 256, 0, st>>>(
        b.real_ptrs.p, b.num_sets, b.v2r.p, num_vss, b.row_ids.p, b.masks.p, n, unp.p, bad.p);
    CK(cudaGetLastError());
    unsigned long long hunp = 0;
    unsigned hbad = 0;
    CK(cudaMemcpyAsync(&hunp, unp.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (last != num_vss) throw InvalidArgument("real_ptrs back != numVSS");
    if (hbad) throw InvalidArgument("inconsistent BVSS arrays (code " + std::to_string(hbad) + ")");
    b.num_unpadded = hunp;
    return b;
}

namespace {
__global__ void k_divergence(const uint32_t* __restrict__ rows, uint32_t nv, uint32_t n,
                             double* __restrict__ out, uint8_t* __restrict__ counted) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
         v += (uint64_t)gridDim.x * blockDim.x) {
        double col_sum = 0;
        unsigned nonempty = 0;
        for (unsigned c = 0; c < 4; ++c) {
            double mean = 0;
            unsigned count = 0;
            for (unsigned lane = 0; lane < 32; ++lane) {
                const uint32_t r = rows[4 * (32 * v + lane) + c];
                if (r != n) { mean = __dadd_rn(mean, (double)r); ++count; }
            }
            if (count == 0) continue;
            mean = __ddiv_rn(mean, (double)count);
            double var = 0;
            for (unsigned lane = 0; lane < 32; ++lane) {
                const uint32_t r = rows[4 * (32 * v + lane) + c];
                if (r != n) {
                    const double d = __dsub_rn((double)r, mean);
                    var = __dadd_rn(var, __dmul_rn(d, d));
                }
            }
            col_sum = __dadd_rn(col_sum, __dsqrt_rn(__ddiv_rn(var, (double)count)));
            ++nonempty;
        }
        out[v] = nonempty ? __ddiv_rn(col_sum, (double)nonempty) : 0.0;
        counted[v] = nonempty ? 1 : 0;
    }
}

__global__ void k_hist(const uint32_t* __restrict__ rows, uint32_t nv, uint32_t n,
                       unsigned long long* __restrict__ hist) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
         v += (uint64_t)gridDim.x * blockDim.x) {
        unsigned c = 0;
        for (unsigned i = 0; i < kTau; ++i) c += rows[kTau * v + i] != n;
        atomicAdd(&hist[c], 1ull);
    }
}
}  // namespace

double bvss_update_divergence(const DeviceBvss& b) {
    if (b.num_vss == 0) return 0.0;
    cudaStream_t st = stream();
    DevBuf<double> d(b.num_vss);
    DevBuf<uint8_t> c(b.num_vss);
    k_divergence<<<grid_for(b.num_vss, 128), 128, 0, st>>>(b.row_ids.p, b.num_vss, b.n, d.p, c.p);
    CK(cudaGetLastError());
    std::vector<double> hd(b.num_vss);
    std::vector<uint8_t> hc(b.num_vss);
    CK(cudaMemcpyAsync(hd.data(), d.p, (size_t)b.num_vss * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hc.data(), c.p, b.num_vss, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double sum = 0;  // VSS order, as R:src/bvss.cpp:125-138
    uint64_t counted = 0;
    for (uint32_t v = 0; v < b.num_vss; ++v)
        if (hc[v]) { sum += hd[v]; ++counted; }
    return counted ? sum / (double)counted : 0.0;
}

double bvss_compression_ratio(const DeviceBvss& b) {
    if (b.num_unpadded == 0) return 0.0;
    return (double)b.m / ((double)b.num_unpadded * kSigma);
}

void bvss_slice_histogram(const DeviceBvss& b, uint64_t* hist129) {
    cudaStream_t st = stream();
    DevBuf<unsigned long long> h(129);
    CK(cudaMemsetAsync(h.p, 0, 129 * 8, st));
    if (b.num_vss) {
        k_hist<<<grid_for(b.num_vss, 128), 128, 0, st>>>(b.row_ids.p, b.num_vss, b.n, h.p);
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(hist129, h.p, 129 * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

}  // namespace blestgpu
