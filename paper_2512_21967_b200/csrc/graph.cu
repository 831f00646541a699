// GPU graph ingestion: generators -> arc keys -> CUB radix sort -> unique -> CSR.
// Replaces the reference's single-threaded sort in Graph::from_edges
// (R:src/graph.cpp:33-55; 152 s at RMAT-24 on the survey host).
#include <cub/cub.cuh>

#include "graph.cuh"

namespace blestgpu {

namespace {

constexpr uint64_t kDrop = ~0ull;  // self-loop / invalid arc marker; sorts last

__global__ void k_keys_from_edges(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                  uint64_t k, uint32_t n, bool mirror, uint64_t* __restrict__ keys,
                                  unsigned* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = src[i], v = dst[i];
        if (u >= n || v >= n) {
            atomicOr(bad, 1u);
            keys[mirror ? 2 * i : i] = kDrop;
            if (mirror) keys[2 * i + 1] = kDrop;
            continue;
        }
        const bool loop = (u == v);
        if (mirror) {
            keys[2 * i] = loop ? kDrop : ((uint64_t)u << 32 | v);
            keys[2 * i + 1] = loop ? kDrop : ((uint64_t)v << 32 | u);
        } else {
            keys[i] = loop ? kDrop : ((uint64_t)u << 32 | v);
        }
    }
}

__global__ void k_mirror_inplace(uint64_t* keys, uint64_t k) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[i];
        const uint32_t u = key >> 32, v = (uint32_t)key;
        keys[k + i] = (key == kDrop || u == v) ? kDrop : ((uint64_t)v << 32 | u);
        if (u == v) keys[i] = kDrop;
    }
}

// offsets[v] = first arc index with source >= v, for v in [0, n]; arcs sorted.
__global__ void k_offsets(const uint64_t* __restrict__ keys, uint64_t m, uint32_t n,
                          uint64_t* __restrict__ off, uint32_t* __restrict__ tgt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = (i < m) ? (keys[i] >> 32) : (uint64_t)n;
        const uint64_t prev = (i == 0) ? 0 : (keys[i - 1] >> 32) + 1;
        for (uint64_t v = (i == 0 ? 0 : prev); v <= s && v <= n; ++v) off[v] = i;
        if (i < m) tgt[i] = (uint32_t)keys[i];
    }
}

void sort_keys(DevBuf<uint64_t>& keys, uint64_t k, int end_bit) {
    if (k <= 1) return;
    DevBuf<uint64_t> alt(k);
    cub::DoubleBuffer<uint64_t> db(keys.p, alt.p);
    size_t temp = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, temp, db, (int64_t)k, 0, end_bit, stream()));
    DevBuf<unsigned char> tmp(temp);
    CK(cub::DeviceRadixSort::SortKeys(tmp.p, temp, db, (int64_t)k, 0, end_bit, stream()));
    if (db.Current() != keys.p) std::swap(keys, alt);
}

}  // namespace

void sort_keys_u64(DevBuf<uint64_t>& keys, uint64_t k, int end_bit) { sort_keys(keys, k, end_bit); }

DeviceGraph graph_from_keys(uint32_t n, DevBuf<uint64_t>& keys, uint64_t k, bool directed) {
    cudaStream_t st = stream();
    uint64_t total = k;
    if (!directed && k) {
        if (keys.count < 2 * k) throw LogicError("graph_from_keys: key buffer too small to mirror");
        k_mirror_inplace<<<grid_for(k, 256), 256, 0, st>>>(keys.p, k);
        CK(cudaGetLastError());
        total = 2 * k;
    }
    // Sort on all 64 bits: kDrop (all ones) must land last.
    sort_keys(keys, total, 64);
    // Unique.
    uint64_t uniq = 0;
    if (total) {
        DevBuf<uint64_t> out(total);
        DevBuf<unsigned long long> nsel(1);
        size_t temp = 0;
        CK(cub::DeviceSelect::Unique(nullptr, temp, keys.p, out.p, nsel.p, (int64_t)total, st));
        DevBuf<unsigned char> tmp(temp);
        CK(cub::DeviceSelect::Unique(tmp.p, temp, keys.p, out.p, nsel.p, (int64_t)total, st));
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, nsel.p, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        uniq = h;
        std::swap(keys, out);
    }
    // Drop the trailing kDrop (at most one after unique).
    uint64_t m = uniq;
    if (uniq) {
        uint64_t last = 0;
        CK(cudaMemcpyAsync(&last, keys.p + uniq - 1, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (last == kDrop) m = uniq - 1;
    }
    DeviceGraph g;
    g.n = n;
    g.m = m;
    g.directed = directed;
    g.off.alloc((size_t)n + 1);
    g.tgt.alloc(m ? m : 1);
    k_offsets<<<grid_for(m + 1, 256), 256, 0, st>>>(keys.p, m, n, g.off.p, g.tgt.p);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return g;
}

DeviceGraph graph_from_edges(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t k,
                             bool directed, bool host_ptrs) {
    cudaStream_t st = stream();
    DevBuf<uint32_t> ds, dd;
    const uint32_t* s = src;
    const uint32_t* d = dst;
    if (host_ptrs && k) {
        ds.alloc(k);
        dd.alloc(k);
        CK(cudaMemcpyAsync(ds.p, src, k * 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dd.p, dst, k * 4, cudaMemcpyHostToDevice, st));
        s = ds.p;
        d = dd.p;
    }
    DevBuf<uint64_t> keys(directed ? (k ? k : 1) : (2 * k ? 2 * k : 1));
    DevBuf<unsigned> bad(1);
    CK(cudaMemsetAsync(bad.p, 0, 4, st));
    if (k) {
        k_keys_from_edges<<<grid_for(k, 256), 256, 0, st>>>(s, d, k, n, !directed, keys.p, bad.p);
        CK(cudaGetLastError());
    }
    unsigned hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hbad) throw InvalidArgument("edge endpoint out of range for n=" + std::to_string(n));
    // keys already mirrored when undirected: build as directed over the full arc list.
    DeviceGraph g = graph_from_keys(n, keys, directed ? k : 2 * k, true);
    g.directed = directed;
    return g;
}

namespace {
__global__ void k_keys_from_csr(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                                uint32_t n, uint64_t* __restrict__ keys, unsigned* __restrict__ bad) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = off[u], e = off[u + 1];
        if (e < b) { atomicOr(bad, 1u); continue; }
        for (uint64_t i = b; i < e; ++i) {
            const uint32_t v = tgt[i];
            if (v >= n) { atomicOr(bad, 1u); keys[i] = kDrop; continue; }
            keys[i] = (v == u) ? kDrop : ((uint64_t)u << 32 | v);
        }
    }
}

__global__ void k_permute_keys(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                               uint32_t n, const uint32_t* __restrict__ fwd, uint64_t* __restrict__ keys) {
    // one warp per source vertex keeps the target reads coalesced
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n;
         u += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint64_t pu = (uint64_t)fwd[u] << 32;
        for (uint64_t i = off[u] + lane; i < off[u + 1]; i += 32) keys[i] = pu | fwd[tgt[i]];
    }
}
}  // namespace

DeviceGraph graph_from_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt, bool directed,
                           bool host_ptrs) {
    cudaStream_t st = stream();
    uint64_t m = 0, first = 0;
    if (host_ptrs) {
        m = off[n];
        first = off[0];
    } else {
        CK(cudaMemcpy(&m, off + n, 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&first, off, 8, cudaMemcpyDeviceToHost));
    }
    // offsets[0] must be 0: otherwise keys[0, off[0]) would never be written
    if (first != 0) throw InvalidArgument("CSR offsets[0] must be 0");
    DevBuf<uint64_t> doff;
    DevBuf<uint32_t> dtgt;
    const uint64_t* o = off;
    const uint32_t* t = tgt;
    if (host_ptrs) {
        doff.alloc((size_t)n + 1);
        dtgt.alloc(m ? m : 1);
        CK(cudaMemcpyAsync(doff.p, off, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, st));
        if (m) CK(cudaMemcpyAsync(dtgt.p, tgt, m * 4, cudaMemcpyHostToDevice, st));
        o = doff.p;
        t = dtgt.p;
    }
    DevBuf<uint64_t> keys(m ? m : 1);
    DevBuf<unsigned> bad(1);
    CK(cudaMemsetAsync(bad.p, 0, 4, st));
    if (n) {
        k_keys_from_csr<<<grid_for(n, 256), 256, 0, st>>>(o, t, n, keys.p, bad.p);
        CK(cudaGetLastError());
    }
    unsigned hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hbad) throw InvalidArgument("CSR has a non-monotone offset or a target out of range");
    DeviceGraph g = graph_from_keys(n, keys, m, true);
    g.directed = directed;
    return g;
}

namespace {
__global__ void k_transpose_keys(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                                 uint32_t n, uint64_t* __restrict__ keys) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n;
         u += ((uint64_t)gridDim.x * blockDim.x) >> 5)
        for (uint64_t i = off[u] + lane; i < off[u + 1]; i += 32) keys[i] = (uint64_t)tgt[i] << 32 | u;
}
}  // namespace

// transpose (R:src/graph.cpp:136-142): the in-view as a CSR.
DeviceGraph graph_transpose(const DeviceGraph& g) {
    DevBuf<uint64_t> keys(g.m ? g.m : 1);
    if (g.n) {
        k_transpose_keys<<<grid_for((uint64_t)g.n * 32, 256), 256, 0, stream()>>>(g.off.p, g.tgt.p, g.n, keys.p);
        CK(cudaGetLastError());
    }
    DeviceGraph out = graph_from_keys(g.n, keys, g.m, true);
    out.directed = g.directed;
    return out;
}

DeviceGraph graph_permute(const DeviceGraph& g, const uint32_t* forward_dev) {
    cudaStream_t st = stream();
    DevBuf<uint64_t> keys(g.m ? g.m : 1);
    if (g.n) {
        k_permute_keys<<<grid_for((uint64_t)g.n * 32, 256), 256, 0, st>>>(g.off.p, g.tgt.p, g.n,
                                                                         forward_dev, keys.p);
        CK(cudaGetLastError());
    }
    DeviceGraph out = graph_from_keys(g.n, keys, g.m, true);
    out.directed = g.directed;
    return out;
}

// ---------------------------------------------------------------------------------------
// Generators (harness). Twin definitions: oracle/blest_oracle.c orc_gen_rmat / orc_gen_urand /
// orc_gen_grid / orc_random_relabel.
// ---------------------------------------------------------------------------------------
namespace {
__global__ void k_rmat(uint32_t scale, uint64_t num_edges, uint64_t seed, uint32_t a, uint32_t b,
                       uint32_t c, uint64_t* __restrict__ keys) {
    const uint64_t ab = (uint64_t)a + b, abc = ab + c;
    const uint64_t words = (scale + 1) / 2;
    const uint64_t s0 = mix64(seed);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < num_edges;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u = 0, v = 0;
        uint64_t w = 0;
        for (uint32_t k = 0; k < scale; ++k) {
            if ((k & 1) == 0) w = mix64(s0 ^ (e * words + k / 2));
            const uint64_t r = (k & 1) ? (w >> 32) : (w & 0xFFFFFFFFull);
            const uint32_t bu = r >= ab;
            const uint32_t bv = (r >= a && r < ab) || r >= abc;
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        keys[e] = (u == v) ? kDrop : ((uint64_t)u << 32 | v);
    }
}

__global__ void k_urand(uint32_t n, uint64_t num_edges, uint64_t seed, uint64_t* __restrict__ keys) {
    const uint64_t s0 = mix64(seed);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < num_edges;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = (uint32_t)__umul64hi(mix64(s0 ^ (2 * e)), n);
        const uint32_t v = (uint32_t)__umul64hi(mix64(s0 ^ (2 * e + 1)), n);
        keys[e] = (u == v) ? kDrop : ((uint64_t)u << 32 | v);
    }
}

__global__ void k_grid(uint32_t rows, uint32_t cols, uint64_t* __restrict__ keys) {
    // arc slots: 2 per vertex (right, down); missing ones dropped
    const uint64_t nv = (uint64_t)rows * cols;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)(v / cols), c = (uint32_t)(v % cols);
        keys[2 * v] = (c + 1 < cols) ? (v << 32 | (v + 1)) : kDrop;
        keys[2 * v + 1] = (r + 1 < rows) ? (v << 32 | (v + cols)) : kDrop;
    }
}

__global__ void k_hash_keys(uint32_t n, uint64_t seed, uint64_t* keys, uint32_t* idx) {
    const uint64_t s0 = mix64(seed);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        keys[i] = mix64(s0 ^ i);
        idx[i] = (uint32_t)i;
    }
}

__global__ void k_scatter_rank(const uint32_t* idx_sorted, uint32_t n, uint32_t* fwd) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
         p += (uint64_t)gridDim.x * blockDim.x)
        fwd[idx_sorted[p]] = (uint32_t)p;
}

__global__ void k_degrees(const uint64_t* off, uint32_t n, uint32_t* deg) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x)
        deg[u] = (uint32_t)(off[u + 1] - off[u]);
}
}  // namespace

DeviceGraph graph_generate_rmat(uint32_t scale, uint64_t num_edges, uint64_t seed, uint32_t a,
                                uint32_t b, uint32_t c) {
    if (scale == 0 || scale > 31) throw InvalidArgument("rmat scale must be in [1, 31]");
    const uint32_t n = 1u << scale;
    DevBuf<uint64_t> keys(2 * num_edges ? 2 * num_edges : 1);
    if (num_edges) {
        k_rmat<<<grid_for(num_edges, 256), 256, 0, stream()>>>(scale, num_edges, seed, a, b, c, keys.p);
        CK(cudaGetLastError());
    }
    DeviceGraph g = graph_from_keys(n, keys, num_edges, false);
    return g;
}

DeviceGraph graph_generate_urand(uint32_t n, uint64_t num_edges, uint64_t seed) {
    if (n == 0) throw InvalidArgument("urand needs n >= 1");
    DevBuf<uint64_t> keys(2 * num_edges ? 2 * num_edges : 1);
    if (num_edges) {
        k_urand<<<grid_for(num_edges, 256), 256, 0, stream()>>>(n, num_edges, seed, keys.p);
        CK(cudaGetLastError());
    }
    return graph_from_keys(n, keys, num_edges, false);
}

DeviceGraph graph_generate_grid(uint32_t rows, uint32_t cols) {
    const uint64_t nv = (uint64_t)rows * cols;
    if (nv >= 0xFFFFFFFFull) throw InvalidArgument("grid too large for 32-bit ids");
    DevBuf<uint64_t> keys(4 * nv ? 4 * nv : 1);
    if (nv) {
        k_grid<<<grid_for(nv, 256), 256, 0, stream()>>>(rows, cols, keys.p);
        CK(cudaGetLastError());
    }
    return graph_from_keys((uint32_t)nv, keys, 2 * nv, false);
}

void relabel_permutation(uint32_t n, uint64_t seed, uint32_t* forward_dev) {
    if (!n) return;
    cudaStream_t st = stream();
    DevBuf<uint64_t> k0(n), k1(n);
    DevBuf<uint32_t> i0(n), i1(n);
    k_hash_keys<<<grid_for(n, 256), 256, 0, st>>>(n, seed, k0.p, i0.p);
    CK(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> dk(k0.p, k1.p);
    cub::DoubleBuffer<uint32_t> dv(i0.p, i1.p);
    size_t temp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, temp, dk, dv, (int64_t)n, 0, 64, st));
    DevBuf<unsigned char> tmp(temp);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, temp, dk, dv, (int64_t)n, 0, 64, st));
    k_scatter_rank<<<grid_for(n, 256), 256, 0, st>>>(dv.Current(), n, forward_dev);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
}

void graph_out_degrees(const DeviceGraph& g, uint32_t* deg_dev) {
    if (!g.n) return;
    k_degrees<<<grid_for(g.n, 256), 256, 0, stream()>>>(g.off.p, g.n, deg_dev);
    CK(cudaGetLastError());
}

}  // namespace blestgpu

