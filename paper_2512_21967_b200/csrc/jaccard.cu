// Jaccard-window clustering (BLEST Alg. 1; jaccard_with_windows, R:src/ordering.cpp:139-166,
// WindowClusterer :65-135) on the GPU: one CTA per window, windows handed out dynamically.
//
// Per cluster: seed = smallest unpicked id; then sigma-1 greedy picks maximising
// J(j, U) = |N(j) ∩ U| / (deg(j) + |U| - |N(j) ∩ U|) in double precision, strict '>' in
// ascending id order (ties to the smallest id), where U is the union of the members'
// out-lists. As in the reference, |N(j) ∩ U| is maintained incrementally: when x newly
// enters U, every unpicked in-window in-neighbour j of x gains one (:92-109).
//
// GPU specifics (same permutation, different data structures):
//  * "x is new to U" is tested by binary search in the (sorted) out-lists of the ≤7
//    earlier members instead of an n-sized epoch array per worker (:97-99);
//  * inter counts and their epoch stamps live in one 64-bit word per vertex (the
//    window-owned slice of an n-sized array), bumped with CAS so concurrent updates
//    are exact; the first bump of a cluster appends j to a candidate list;
//  * argmax (:111-126) only scans candidates: any j with inter > 0 scores > 0 and beats
//    every non-candidate (score 0); with no unpicked candidate the smallest unpicked id
//    wins, exactly as the reference's strict-'>' scan starting at -1.0 resolves it.
#include <cub/cub.cuh>

#include "ordering.cuh"

namespace blestgpu {

DeviceGraph graph_transpose(const DeviceGraph& g);

namespace {

constexpr int kJT = 256;

struct JP {
    const uint64_t* __restrict__ off;
    const uint32_t* __restrict__ tgt;
    const uint64_t* __restrict__ ioff;
    const uint32_t* __restrict__ isrc;
    uint32_t n, sigma, w, num_windows;
    unsigned long long* word;  // (epoch << 32) | inter, per vertex
    uint32_t* cand;            // gridDim.x * w
    uint32_t* forward;
    unsigned* next_window;
};

__device__ __forceinline__ bool bsearch_u32(const uint32_t* a, uint64_t lo, uint64_t hi, uint32_t x) {
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        const uint32_t v = a[mid];
        if (v == x) return true;
        if (v < x) lo = mid + 1;
        else hi = mid;
    }
    return false;
}

__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* a, uint64_t lo, uint64_t hi, uint32_t x) {
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

struct JS {
    uint32_t members[8];
    uint32_t nmem;
    uint32_t union_size;
    uint32_t cand_count;
    uint32_t pos;
    uint32_t first_unpicked;
    uint32_t epoch;
    uint32_t best;
    uint32_t window;
    double red_score[kJT / 32];
    uint32_t red_j[kJT / 32];
};

__global__ void __launch_bounds__(kJT) k_jaccard(JP p) {
    extern __shared__ uint32_t picked[];  // (w + 31) / 32 words
    __shared__ JS s;
    const uint32_t tid = threadIdx.x;
    const uint32_t pw = (p.w + 31) / 32;
    uint32_t* cand = p.cand + (uint64_t)blockIdx.x * p.w;
    if (tid == 0) s.epoch = 0;
    for (;;) {
        __syncthreads();
        if (tid == 0) s.window = atomicAdd(p.next_window, 1u);
        __syncthreads();
        const uint32_t win = s.window;
        if (win >= p.num_windows) break;
        const uint32_t begin = win * p.w;
        const uint32_t end = ((uint64_t)begin + p.w < p.n) ? begin + p.w : p.n;
        const uint32_t len = end - begin;
        for (uint32_t i = tid; i < pw; i += kJT) picked[i] = 0;
        if (tid == 0) {
            s.pos = 0;
            s.first_unpicked = 0;
        }
        __syncthreads();

        while (s.pos < len) {
            if (tid == 0) {
                ++s.epoch;
                s.union_size = 0;
                s.cand_count = 0;
                s.nmem = 0;
                uint32_t f = s.first_unpicked;  // seed: smallest unpicked id (:79-80)
                while ((picked[f >> 5] >> (f & 31)) & 1u) ++f;
                s.first_unpicked = f;
                s.best = begin + f;
            }
            __syncthreads();
            for (uint32_t r = 0; r < p.sigma; ++r) {
                if (r > 0) {
                    if (s.pos >= len) break;  // uniform: read after a barrier
                    // ---- argmax over candidates (:111-126) ----
                    double bs = -1.0;
                    uint32_t bj = 0xFFFFFFFFu;
                    const uint32_t cc = s.cand_count;
                    const double us = (double)s.union_size;
                    for (uint32_t i = tid; i < cc; i += kJT) {
                        const uint32_t j = cand[i];
                        const uint32_t lj = j - begin;
                        if ((picked[lj >> 5] >> (lj & 31)) & 1u) continue;
                        const uint32_t inter = (uint32_t)p.word[j];
                        const double denom = ((double)(p.off[j + 1] - p.off[j]) + us) - (double)inter;
                        const double score = denom > 0 ? (double)inter / denom : 0.0;
                        if (score > bs || (score == bs && j < bj)) {
                            bs = score;
                            bj = j;
                        }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
                        const uint32_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
                        if (os > bs || (os == bs && oj < bj)) {
                            bs = os;
                            bj = oj;
                        }
                    }
                    if ((tid & 31) == 0) {
                        s.red_score[tid >> 5] = bs;
                        s.red_j[tid >> 5] = bj;
                    }
                    __syncthreads();
                    if (tid == 0) {
                        double b = -1.0;
                        uint32_t j = 0xFFFFFFFFu;
                        for (int k = 0; k < kJT / 32; ++k)
                            if (s.red_score[k] > b || (s.red_score[k] == b && s.red_j[k] < j)) {
                                b = s.red_score[k];
                                j = s.red_j[k];
                            }
                        if (j == 0xFFFFFFFFu) {  // no unpicked candidate: smallest unpicked id
                            uint32_t f = s.first_unpicked;
                            while ((picked[f >> 5] >> (f & 31)) & 1u) ++f;
                            s.first_unpicked = f;
                            j = begin + f;
                        }
                        s.best = j;
                    }
                    __syncthreads();
                }
                // ---- take(best) (:92-109) ----
                const uint32_t v = s.best;
                const uint32_t nprior = s.nmem;
                __syncthreads();
                if (tid == 0) {
                    const uint32_t lv = v - begin;
                    picked[lv >> 5] |= 1u << (lv & 31);
                    p.forward[v] = begin + s.pos;
                    s.pos += 1;
                    s.members[s.nmem] = v;
                    s.nmem += 1;
                }
                __syncthreads();
                const uint64_t vb = p.off[v], ve = p.off[v + 1];
                const uint32_t ep = s.epoch;
                for (uint64_t i = vb + tid; i < ve; i += kJT) {
                    const uint32_t x = p.tgt[i];
                    bool fresh = true;
                    for (uint32_t k = 0; k < nprior && fresh; ++k) {
                        const uint32_t c = s.members[k];
                        if (bsearch_u32(p.tgt, p.off[c], p.off[c + 1], x)) fresh = false;
                    }
                    if (!fresh) continue;
                    atomicAdd(&s.union_size, 1u);
                    const uint64_t ib = p.ioff[x], ie = p.ioff[x + 1];
                    for (uint64_t t = lower_bound_u32(p.isrc, ib, ie, begin); t < ie; ++t) {
                        const uint32_t j = p.isrc[t];
                        if (j >= end) break;
                        const uint32_t lj = j - begin;
                        if ((picked[lj >> 5] >> (lj & 31)) & 1u) continue;
                        unsigned long long old = p.word[j], nw;
                        bool first;
                        do {
                            first = (uint32_t)(old >> 32) != ep;
                            nw = first ? (((unsigned long long)ep << 32) | 1ull) : old + 1;
                            const unsigned long long seen = atomicCAS(&p.word[j], old, nw);
                            if (seen == old) break;
                            old = seen;
                        } while (true);
                        if (first) cand[atomicAdd(&s.cand_count, 1u)] = j;
                    }
                }
                __syncthreads();
            }
        }
    }
}

}  // namespace

void jaccard_windows_forward(const DeviceGraph& g, uint32_t sigma, uint32_t w, uint32_t* forward_host) {
    if (sigma == 0 || w == 0 || w % sigma != 0)
        throw InvalidArgument("window size must be a positive multiple of sigma");
    if (sigma > 8) throw InvalidArgument("sigma > 8 is not supported by the GPU clusterer");
    const uint32_t n = g.n;
    if (n == 0) return;
    cudaStream_t st = stream();
    DeviceGraph gt;
    const DeviceGraph* in = &g;
    if (g.directed) {
        gt = graph_transpose(g);
        in = &gt;
    }
    const uint32_t num_windows = (uint32_t)(((uint64_t)n + w - 1) / w);
    const size_t smem = (size_t)((w + 31) / 32) * 4;
    if (smem > 200 * 1024) throw InvalidArgument("window too large for the GPU clusterer");
    CK(cudaFuncSetAttribute(k_jaccard, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jaccard, kJT, smem));
    uint32_t ctas = std::max(1, per_sm) * (uint32_t)num_sms();
    if (ctas > num_windows) ctas = num_windows;
    DevBuf<unsigned long long> word(n);
    DevBuf<uint32_t> cand((uint64_t)ctas * w);
    DevBuf<uint32_t> fwd(n);
    DevBuf<unsigned> next(1);
    CK(cudaMemsetAsync(word.p, 0, (size_t)n * 8, st));
    CK(cudaMemsetAsync(next.p, 0, 4, st));
    JP p{g.off.p, g.tgt.p, in->off.p, in->tgt.p, n, sigma, w, num_windows, word.p, cand.p, fwd.p, next.p};
    k_jaccard<<<ctas, kJT, smem, st>>>(p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(forward_host, fwd.p, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

}  // namespace blestgpu
