// Reverse Cuthill-McKee on the GPU, permutation-identical to the reference's rcm
// (R:src/ordering.cpp:171-266):
//   * symmetrised adjacency (sorted-unique union of out- and in-neighbours, :171-182);
//   * components in ascending order of their smallest vertex (the loop at :255-263);
//   * start vertex by pseudo_peripheral (:220-242): repeated plain BFS, next start = the
//     smallest (degree, id) vertex of the last level, until the eccentricity stops growing;
//   * Cuthill-McKee visit order (sym_bfs with sorted children, :190-218): a FIFO queue
//     where each dequeued vertex appends its unvisited neighbours sorted by (degree, id).
//     Level by level that is: vertex w of level ℓ+1 belongs to the FIRST vertex of level ℓ
//     (in CM order) adjacent to it, so level ℓ+1 in CM order = its vertices sorted by
//     (position of that parent, degree, id) — one claim kernel (atomicMin of the parent
//     position) and two stable radix sorts per level instead of a sequential queue;
//   * reversed (:265).
// Isolated vertices are singleton components (pseudo_peripheral returns them at once).
// The plain BFSs run as one cooperative launch each (grid barrier per level).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "graph.cuh"
#include "ordering.cuh"

namespace blestgpu {
namespace {
namespace cg = cooperative_groups;

__global__ void k_arc_keys(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt, uint32_t n,
                           uint64_t* __restrict__ keys) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n;
         u += ((uint64_t)gridDim.x * blockDim.x) >> 5)
        for (uint64_t i = off[u] + lane; i < off[u + 1]; i += 32) keys[i] = (u << 32) | tgt[i];
}

__global__ void k_deg_init(const uint64_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ deg,
                           uint32_t* __restrict__ level, uint32_t* __restrict__ par) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        deg[v] = (uint32_t)(off[v + 1] - off[v]);
        level[v] = kInf;
        par[v] = kInf;
    }
}

// Smallest v in [from, n) with level[v] == kInf (not yet placed) and a neighbour.
__global__ void k_next_start(const uint32_t* __restrict__ level, const uint32_t* __restrict__ deg, uint32_t from,
                             uint32_t to, unsigned* __restrict__ best) {
    for (uint64_t v = from + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < to;
         v += (uint64_t)gridDim.x * blockDim.x)
        if (level[v] == kInf && deg[v] != 0) {
            atomicMin(best, (unsigned)v);
            return;
        }
}

// Plain level-synchronous BFS from start (sym_bfs without sorting, :190-218): vis gets the
// visited vertices level by level; ctl[0] = visited count, ctl[1] = eccentricity, ctl[2] =
// start of the last level in vis; key[0] = min (degree << 32 | id) over the last level.
__global__ void k_plain_bfs(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                            const uint32_t* __restrict__ deg, uint32_t start, uint32_t* __restrict__ level,
                            uint32_t* __restrict__ vis, unsigned long long* __restrict__ ctl,
                            unsigned long long* __restrict__ key) {
    cg::grid_group grid = cg::this_grid();
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t NW = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        level[start] = 0;
        vis[0] = start;
        ctl[0] = 1;
        ctl[1] = 0;
        ctl[2] = 0;
        key[0] = ~0ull;
    }
    grid.sync();
    uint64_t lo = 0, hi = 1;
    for (uint32_t l = 0;; ++l) {
        for (uint64_t i = lo + gw; i < hi; i += NW) {
            const uint32_t u = vis[i];
            for (uint64_t e0 = off[u]; e0 < off[u + 1]; e0 += 32) {
                const uint64_t e = e0 + lane;
                bool mine = false;
                uint32_t w = 0;
                if (e < off[u + 1]) {
                    w = tgt[e];
                    mine = level[w] == kInf && atomicCAS(level + w, kInf, l + 1) == kInf;
                }
                const unsigned ball = __ballot_sync(0xffffffffu, mine);
                unsigned long long base = 0;
                if (lane == 0 && ball) base = atomicAdd(&ctl[0], (unsigned long long)__popc(ball));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (mine) vis[base + __popc(ball & ((1u << lane) - 1u))] = w;
            }
        }
        grid.sync();
        const uint64_t nhi = *(volatile unsigned long long*)&ctl[0];
        if (nhi == hi) break;
        lo = hi;
        hi = nhi;
        grid.sync();  // everyone has read ctl[0] before the next level appends
    }
    // last non-empty level = [lo, hi): its smallest (degree, id)
    for (uint64_t i = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < hi;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = vis[i];
        atomicMin(key, ((unsigned long long)deg[v] << 32) | v);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl[1] = level[vis[hi - 1]];
        ctl[2] = lo;
    }
}

__global__ void k_reset_levels(const uint32_t* __restrict__ vis, uint64_t count, uint32_t* __restrict__ level) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        level[vis[i]] = kInf;
}


// Device-chained CM levels (no host round trip per level): ctl = {s, e, state, stopped
// level}; state 0 running, 1 done (an empty level), 2 stopped at a level too large for the
// one-CTA sort (the host sorts it with cub and resumes). Launches after a stop are no-ops.
enum { kS = 0, kE = 1, kState = 2, kStop = 3 };
__global__ void k_cm_claim_dev(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                               const uint32_t* __restrict__ ord, const unsigned long long* __restrict__ ctl,
                               uint32_t l, uint32_t* __restrict__ level, uint32_t* __restrict__ par,
                               uint32_t* __restrict__ nxt, unsigned long long* __restrict__ cnt) {
    if (ctl[kState] != 0) return;
    const uint64_t s = ctl[kS], e = ctl[kE];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t NW = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t p = s + gw; p < e; p += NW) {
        const uint32_t u = ord[p];
        for (uint64_t e0 = off[u]; e0 < off[u + 1]; e0 += 32) {
            const uint64_t i = e0 + lane;
            bool mine = false;
            uint32_t w = 0;
            if (i < off[u + 1]) {
                w = tgt[i];
                uint32_t lw = level[w];
                if (lw == kInf) {
                    lw = atomicCAS(level + w, kInf, l + 1);
                    mine = lw == kInf;
                    if (mine) lw = l + 1;
                }
                if (lw == l + 1) atomicMin(par + w, (uint32_t)p);
            }
            const unsigned ball = __ballot_sync(0xffffffffu, mine);
            unsigned long long base = 0;
            if (lane == 0 && ball) base = atomicAdd(cnt, (unsigned long long)__popc(ball));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (mine) nxt[base + __popc(ball & ((1u << lane) - 1u))] = w;
        }
    }
}

__global__ void k_cm_keys(const uint32_t* __restrict__ ids, uint64_t c, const uint32_t* __restrict__ par,
                          const uint32_t* __restrict__ deg, uint64_t* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < c; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t w = ids[i];
        keys[i] = ((uint64_t)par[w] << 32) | deg[w];
    }
}

// One CTA sorts a small level (c <= kSmallLevel) by (parent position, degree, id) and
// writes it to ord — the same order as the two stable radix sorts of a large level.
constexpr uint32_t kSmallLevel = 8192;
__global__ void __launch_bounds__(1024) k_cm_sort_small(const uint32_t* __restrict__ nxt, unsigned long long* cnt,
                                                        const uint32_t* __restrict__ par,
                                                        const uint32_t* __restrict__ deg, uint32_t* __restrict__ ord,
                                                        unsigned long long* ctl, uint32_t l) {
    extern __shared__ unsigned long long sk[];  // [kSmallLevel] (par << 32 | deg)
    uint32_t* sid = reinterpret_cast<uint32_t*>(sk + kSmallLevel);
    if (ctl[kState] != 0) return;
    const uint64_t c = *cnt;
    if (c == 0 || c > kSmallLevel) {  // done, or too large for one CTA: the host takes over
        __syncthreads();
        if (threadIdx.x == 0) {
            ctl[kState] = c == 0 ? 1 : 2;
            ctl[kStop] = l;
        }
        return;
    }
    uint32_t* out = ord + ctl[kE];
    uint32_t P = 1;
    while (P < c) P <<= 1;
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        if (i < c) {
            const uint32_t w = nxt[i];
            sk[i] = ((unsigned long long)par[w] << 32) | deg[w];
            sid[i] = w;
        } else {
            sk[i] = ~0ull;
            sid[i] = 0xFFFFFFFFu;
        }
    }
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const unsigned long long a = sk[i], b = sk[l];
                    const uint32_t ia = sid[i], ib = sid[l];
                    const bool gt = a > b || (a == b && ia > ib);
                    if (gt == up) {
                        sk[i] = b;
                        sk[l] = a;
                        sid[i] = ib;
                        sid[l] = ia;
                    }
                }
            }
            __syncthreads();
        }
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) out[i] = sid[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        ctl[kS] = ctl[kE];
        ctl[kE] += c;
        *cnt = 0;
    }
}



struct Plain {
    uint32_t ecc;
    uint32_t next;    // smallest (degree, id) vertex of the last level
    uint64_t visited;
};

}  // namespace

std::vector<uint32_t> rcm_forward(const DeviceGraph& g) {
    cudaStream_t st = stream();
    const bool trace = getenv("BLEST_RCM_TRACE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!trace) return;
        CK(cudaStreamSynchronize(st));
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[rcm] %s %.3f s\n", what, std::chrono::duration<double>(t1 - t0).count());
        t0 = t1;
    };
    const uint32_t n = g.n;
    std::vector<uint32_t> forward(n);
    if (!n) return forward;
    // symmetrised adjacency (:171-182): the out-view itself when undirected
    DeviceGraph sym;
    const uint64_t* off = g.off.p;
    const uint32_t* tgt = g.tgt.p;
    if (g.directed && g.m) {
        DevBuf<uint64_t> keys(2 * g.m);
        k_arc_keys<<<grid_for((uint64_t)n * 32, 256), 256, 0, st>>>(g.off.p, g.tgt.p, n, keys.p);
        CK(cudaGetLastError());
        sym = graph_from_keys(n, keys, g.m, false);
        off = sym.off.p;
        tgt = sym.tgt.p;
    }
    DevBuf<uint32_t> deg(n), level(n), par(n), vis(n), ord(n), nxt(n), ids2(n), forward_dev(n);
    DevBuf<uint64_t> keys(n), keys2(n);
    DevBuf<unsigned long long> ctl(4), key(1), cnt(1), cml(4);
    const uint32_t claim_ctas = 8u * (uint32_t)num_sms();
    DevBuf<unsigned> best(1);
    k_deg_init<<<grid_for(n, 256), 256, 0, st>>>(off, n, deg.p, level.p, par.p);
    CK(cudaGetLastError());
    lap("symmetrise + init");
    // cub scratch for the per-level sorts, sized once for n items
    size_t t1 = 0, t2 = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, t1, nxt.p, ids2.p, (int64_t)n, 0, 32, st));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, keys.p, keys2.p, ids2.p, nxt.p, (int64_t)n, 0, 64, st));
    DevBuf<unsigned char> tmp(std::max<size_t>({t1, t2, 1}));
    CK(cudaFuncSetAttribute(k_cm_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSmallLevel * 12)));
    // plain BFS: one cooperative launch
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_plain_bfs, 256, 0));
    const uint32_t bfs_ctas = (uint32_t)std::max(1, per_sm) * (uint32_t)num_sms();
    auto plain_bfs = [&](uint32_t start) -> Plain {
        void* args[] = {(void*)&off, (void*)&tgt, (void*)&deg.p, (void*)&start, (void*)&level.p, (void*)&vis.p,
                        (void*)&ctl.p, (void*)&key.p};
        CK(cudaLaunchCooperativeKernel((void*)k_plain_bfs, dim3(bfs_ctas), dim3(256), args, 0, st));
        unsigned long long h[3], k = 0;
        CK(cudaMemcpyAsync(h, ctl.p, 24, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&k, key.p, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        k_reset_levels<<<grid_for(h[0], 256), 256, 0, st>>>(vis.p, h[0], level.p);
        CK(cudaGetLastError());
        Plain r;
        r.visited = h[0];
        r.ecc = (uint32_t)h[1];
        r.next = (uint32_t)k;
        return r;
    };
    // components, smallest vertex first; order[] collects the CM orders, isolated vertices
    // are merged in by id at the end
    std::vector<std::pair<uint32_t, uint64_t>> comps;  // (smallest vertex, CM offset)
    uint64_t placed = 0;
    uint32_t cursor = 0;
    for (;;) {
        // next unplaced non-isolated vertex >= cursor (scanned in 1 M windows)
        uint32_t v = kInf;
        while (cursor < n) {
            const uint32_t to = (uint32_t)std::min<uint64_t>((uint64_t)cursor + (1u << 20), n);
            CK(cudaMemsetAsync(best.p, 0xFF, 4, st));
            k_next_start<<<grid_for(to - cursor, 256), 256, 0, st>>>(level.p, deg.p, cursor, to, best.p);
            CK(cudaGetLastError());
            unsigned h = 0;
            CK(cudaMemcpyAsync(&h, best.p, 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (h != 0xFFFFFFFFu) {
                v = h;
                break;
            }
            cursor = to;
        }
        if (v == kInf) break;
        cursor = v + 1;
        // pseudo_peripheral (:220-242)
        uint32_t current = v, best_ecc = 0;
        for (;;) {
            const Plain r = plain_bfs(current);
            if (r.ecc <= best_ecc && current != v) break;
            if (r.ecc == 0) break;
            if (r.ecc <= best_ecc) break;
            best_ecc = r.ecc;
            current = r.next;
        }
        lap("pseudo_peripheral");
        // Cuthill-McKee order of the component from `current`, level by level
        comps.emplace_back(v, placed);
        const uint32_t one_level = 0;
        CK(cudaMemcpyAsync(ord.p + placed, &current, 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(level.p + current, &one_level, 4, cudaMemcpyHostToDevice, st));
        uint64_t s = placed, e = placed + 1;
        {
            const unsigned long long init[4] = {s, e, 0, 0};
            CK(cudaMemcpyAsync(cml.p, init, 32, cudaMemcpyHostToDevice, st));
            CK(cudaMemsetAsync(cnt.p, 0, 8, st));
        }
        uint32_t l = 0;
        constexpr uint32_t kBatchLevels = 64;
        for (;;) {
            for (uint32_t k = 0; k < kBatchLevels; ++k) {
                k_cm_claim_dev<<<claim_ctas, 256, 0, st>>>(off, tgt, ord.p, cml.p, l + k, level.p, par.p, nxt.p,
                                                           cnt.p);
                k_cm_sort_small<<<1, 1024, kSmallLevel * 12, st>>>(nxt.p, cnt.p, par.p, deg.p, ord.p, cml.p, l + k);
            }
            CK(cudaGetLastError());
            unsigned long long h[4];
            CK(cudaMemcpyAsync(h, cml.p, 32, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            s = h[kS];
            e = h[kE];
            if (h[kState] == 1) break;
            if (h[kState] == 0) {
                l += kBatchLevels;
                continue;
            }
            // a large level: ascending id, then a stable sort by (parent position, degree)
            unsigned long long c = 0;
            CK(cudaMemcpyAsync(&c, cnt.p, 8, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            size_t a = tmp.count;
            CK(cub::DeviceRadixSort::SortKeys(tmp.p, a, nxt.p, ids2.p, (int64_t)c, 0, 32, st));
            k_cm_keys<<<grid_for(c, 256), 256, 0, st>>>(ids2.p, c, par.p, deg.p, keys.p);
            CK(cudaGetLastError());
            a = tmp.count;
            CK(cub::DeviceRadixSort::SortPairs(tmp.p, a, keys.p, keys2.p, ids2.p, ord.p + e, (int64_t)c, 0, 64, st));
            s = e;
            e += c;
            const unsigned long long resume[4] = {s, e, 0, 0};
            CK(cudaMemcpyAsync(cml.p, resume, 32, cudaMemcpyHostToDevice, st));
            CK(cudaMemsetAsync(cnt.p, 0, 8, st));
            l = (uint32_t)h[kStop] + 1;
        }
        placed = e;
        lap("cuthill_mckee");
    }
    lap("component search");
    // merge the isolated vertices (singleton components) in by id, then reverse
    std::vector<uint32_t> deg_h(n), ord_h(placed);
    CK(cudaMemcpyAsync(deg_h.data(), deg.p, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    if (placed) CK(cudaMemcpyAsync(ord_h.data(), ord.p, placed * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<uint32_t> order;
    order.reserve(n);
    size_t ci = 0;
    for (uint32_t v = 0; v < n; ++v) {
        if (ci < comps.size() && comps[ci].first == v) {
            const uint64_t b = comps[ci].second, en = ci + 1 < comps.size() ? comps[ci + 1].second : placed;
            order.insert(order.end(), ord_h.begin() + b, ord_h.begin() + en);
            ++ci;
        } else if (deg_h[v] == 0) {
            order.push_back(v);
        }
    }
    if (order.size() != n) throw LogicError("rcm: order does not cover every vertex");
    lap("merge");
    for (uint32_t i = 0; i < n; ++i) forward[order[i]] = n - 1 - i;
    return forward;
}

}  // namespace blestgpu
