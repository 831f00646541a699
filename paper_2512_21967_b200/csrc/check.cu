// Device checkers the reference keeps next to its hot path:
//   * reference_bfs (R:src/graph.cpp:144-167) — the ground truth its CLI's --validate and
//     its tests compare the engines with. Here a level-synchronous top-down BFS straight
//     over the CSR out-view (no BVSS, no pull): one launch per level, a warp per frontier
//     vertex, lanes over its out-list, the first CAS on L[v] claims v and warp-aggregated
//     appends build the next frontier. Levels are unique, so the result is bit-identical
//     to the reference's FIFO order whatever the claim order;
//   * validate_roundtrip (R:src/bvss.cpp:143-188) — decode every BVSS slot, check the
//     padding rules, and compare the decoded arc set with the graph's incoming view row
//     by row (both as sorted (row << 32 | column) keys).
#include "io.cuh"

namespace blestgpu {

namespace {

__global__ void k_bfs_init(uint32_t* __restrict__ L, uint32_t n, uint32_t src) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        L[i] = i == src ? 0u : kInf;
}

__global__ void k_bfs_level(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                            uint32_t* __restrict__ L, const uint32_t* __restrict__ q, uint32_t qlen,
                            uint32_t* __restrict__ qn, unsigned* __restrict__ qn_len, uint32_t level) {
    const unsigned lane = threadIdx.x & 31;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < qlen;
         i += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t u = q[i];
        const uint64_t b = off[u], e = off[u + 1];
        for (uint64_t base = b; base < e; base += 32) {
            bool claim = false;
            uint32_t v = 0;
            if (base + lane < e) {
                v = tgt[base + lane];
                claim = L[v] == kInf && atomicCAS(&L[v], kInf, level) == kInf;
            }
            const unsigned ball = __ballot_sync(0xffffffffu, claim);
            if (!ball) continue;
            unsigned pos = 0;
            if (lane == 0) pos = atomicAdd(qn_len, (unsigned)__popc(ball));
            pos = __shfl_sync(0xffffffffu, pos, 0);
            if (claim) qn[pos + __popc(ball & ((1u << lane) - 1))] = v;
        }
    }
}

// Pass 1 / 2 over the slots: counts (and, with keys, the decoded (row << 32 | column) arcs).
__global__ void k_decode(const uint32_t* __restrict__ v2r, const uint32_t* __restrict__ rows,
                         const uint32_t* __restrict__ masks, uint64_t num_vss, uint32_t n,
                         unsigned long long* __restrict__ ctr, unsigned long long* __restrict__ first,
                         uint64_t* __restrict__ keys) {
    // ctr: [0] checked, [1] padded nonzero, [2] real zero mask, [3] beyond n, [4] key cursor
    for (uint64_t slot = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; slot < num_vss * 128;
         slot += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = slot >> 7;
        const uint32_t lane = (slot >> 2) & 31, c = slot & 3;  // row_ids[4(32v + lane) + c]
        const uint32_t r = rows[slot];
        const uint32_t mask = (masks[32 * v + lane] >> (8 * c)) & 0xFFu;
        if (r == n) {
            if (mask && !keys) {
                atomicAdd(&ctr[1], 1ull);
                atomicMin(&first[0], (unsigned long long)v);
            }
            continue;
        }
        if (!keys) {
            atomicAdd(&ctr[0], 1ull);
            if (!mask) {
                atomicAdd(&ctr[2], 1ull);
                atomicMin(&first[1], (unsigned long long)v);
            }
        }
        const uint32_t s = v2r[v];
        uint32_t bits = mask, cnt = 0;
        while (bits) {
            const uint32_t j = __ffs(bits) - 1;
            bits &= bits - 1;
            const uint64_t col = 8ull * s + j;
            if (col >= n) {
                if (!keys) {
                    atomicAdd(&ctr[3], 1ull);
                    atomicMin(&first[2], (unsigned long long)s);
                }
                continue;
            }
            if (keys) keys[atomicAdd(&ctr[4], 1ull)] = ((uint64_t)r << 32) | col;
            ++cnt;
        }
        if (!keys && cnt) atomicAdd(&ctr[4], (unsigned long long)cnt);
    }
}

__global__ void k_in_keys(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt, uint32_t n,
                          uint64_t* __restrict__ keys) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n;
         u += ((uint64_t)gridDim.x * blockDim.x) >> 5)
        for (uint64_t i = off[u] + lane; i < off[u + 1]; i += 32) keys[i] = ((uint64_t)tgt[i] << 32) | u;
}

__device__ __forceinline__ uint64_t lower_bound_key(const uint64_t* a, uint64_t len, uint64_t x) {
    uint64_t lo = 0, hi = len;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Row u's decoded list vs its incoming list (both sorted): mismatched rows counted.
__global__ void k_compare_rows(const uint64_t* __restrict__ dec, uint64_t nd, const uint64_t* __restrict__ ref,
                               uint64_t nr, uint32_t n, unsigned long long* __restrict__ ctr,
                               unsigned long long* __restrict__ first) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a0 = lower_bound_key(dec, nd, u << 32), a1 = lower_bound_key(dec, nd, (u + 1) << 32);
        const uint64_t b0 = lower_bound_key(ref, nr, u << 32), b1 = lower_bound_key(ref, nr, (u + 1) << 32);
        bool bad = a1 - a0 != b1 - b0;
        for (uint64_t k = 0; !bad && k < a1 - a0; ++k) bad = dec[a0 + k] != ref[b0 + k];
        if (bad) {
            atomicAdd(&ctr[5], 1ull);
            atomicMin(&first[3], (unsigned long long)u);
        }
    }
}

}  // namespace

uint32_t graph_bfs_levels(const DeviceGraph& g, uint32_t src, uint32_t* L, uint32_t* num_levels) {
    if (src >= g.n) throw InvalidArgument("bfs source out of range");
    cudaStream_t st = stream();
    DevBuf<uint32_t> q0(g.n), q1(g.n);
    DevBuf<unsigned> len(1);
    k_bfs_init<<<grid_for(g.n, 256), 256, 0, st>>>(L, g.n, src);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(q0.p, &src, 4, cudaMemcpyHostToDevice, st));
    uint32_t qlen = 1, visited = 1, level = 0;
    uint32_t *qc = q0.p, *qn = q1.p;
    while (qlen) {
        ++level;
        CK(cudaMemsetAsync(len.p, 0, 4, st));
        k_bfs_level<<<grid_for((uint64_t)qlen * 32, 256), 256, 0, st>>>(g.off.p, g.tgt.p, L, qc, qlen, qn, len.p,
                                                                         level);
        CK(cudaGetLastError());
        unsigned h = 0;
        CK(cudaMemcpyAsync(&h, len.p, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        qlen = h;
        visited += h;
        std::swap(qc, qn);
    }
    *num_levels = level;  // the last iteration discovered nothing: max level = level - 1
    return visited;
}

RoundtripCounts bvss_validate_roundtrip(const DeviceBvss& b, const DeviceGraph& g) {
    if (g.n != b.n) throw InvalidArgument("graph and structure sizes differ");
    cudaStream_t st = stream();
    DevBuf<unsigned long long> ctr(6), first(4);
    CK(cudaMemsetAsync(ctr.p, 0, 6 * 8, st));
    CK(cudaMemsetAsync(first.p, 0xFF, 4 * 8, st));
    const uint64_t slots = (uint64_t)b.num_vss * 128;
    RoundtripCounts out;
    unsigned long long h[6] = {0, 0, 0, 0, 0, 0}, f[4];
    if (slots) {
        k_decode<<<grid_for(slots, 256), 256, 0, st>>>(b.v2r.p, b.row_ids.p, b.masks.p, b.num_vss, b.n, ctr.p,
                                                        first.p, nullptr);
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(h, ctr.p, 6 * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint64_t nd = h[4];
    DevBuf<uint64_t> dec(nd ? nd : 1), ref(g.m ? g.m : 1);
    CK(cudaMemsetAsync(ctr.p + 4, 0, 8, st));
    if (slots && nd) {
        k_decode<<<grid_for(slots, 256), 256, 0, st>>>(b.v2r.p, b.row_ids.p, b.masks.p, b.num_vss, b.n, ctr.p,
                                                        first.p, dec.p);
        CK(cudaGetLastError());
    }
    if (g.n && g.m) {
        k_in_keys<<<grid_for((uint64_t)g.n * 32, 256), 256, 0, st>>>(g.off.p, g.tgt.p, g.n, ref.p);
        CK(cudaGetLastError());
    }
    sort_keys_u64(dec, nd, 64);
    sort_keys_u64(ref, g.m, 64);
    if (g.n) {
        k_compare_rows<<<grid_for(g.n, 256), 256, 0, st>>>(dec.p, nd, ref.p, g.m, g.n, ctr.p, first.p);
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(h, ctr.p, 6 * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(f, first.p, 4 * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out.checked_slices = h[0];
    out.padded_nonzero = h[1];
    out.real_zero_mask = h[2];
    out.beyond_n = h[3];
    out.rows_mismatched = h[5];
    out.first_padded_nonzero_vss = f[0];
    out.first_zero_mask_vss = f[1];
    out.first_beyond_set = f[2];
    out.first_mismatched_row = f[3];
    return out;
}

}  // namespace blestgpu
