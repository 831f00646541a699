// Row-partitioned multi-GPU BFS: rank g owns destination rows
// [row_lo, row_hi) (32-aligned) and a BVSS of A[rows_g, all columns] (bvss_build with a
// row range: every column slice set, only this rank's rows). One level, lazy-style:
//   pull    — stage 1 over the local queue: visited tests on owned rows, REDs into V_next;
//   sweep   — stage 2 over the owned words: diff = V_next & ~V_curr, levels, V_curr |= diff,
//             diff words written to the rank's slot of the exchange buffer;
//   (host)  — all-gather of the diff words over NCCL (every rank gets the n/8-byte frontier);
//   enqueue — every rank scans the gathered diff and queues its local VSSs of each active set.
// No OR-reduction is ever needed (NCCL has none): row ownership makes each diff word
// single-writer. Termination is consistent because every rank sees the same gathered diff.
#include <memory>

#include "bvss.cuh"
#include "common.cuh"

namespace blestgpu {

struct PartEngine {
    const DeviceBvss& b;
    uint64_t words = 0, w_lo = 0, w_hi = 0;
    DevBuf<uint32_t> L, Vc, Vn;
    DevBuf<unsigned long long> Q, ctr;  // ctr: [0] queue len, [1] discovered, [2] REDs, [3] total diff bits
    explicit PartEngine(const DeviceBvss& bb) : b(bb) {
        words = ((uint64_t)b.n + 31) / 32;
        const uint32_t hi = b.row_hi > b.n ? b.n : b.row_hi;
        w_lo = b.row_lo / 32;
        w_hi = ((uint64_t)hi + 31) / 32;
        L.alloc(b.n ? b.n : 1);
        Vc.alloc(words ? words : 1);
        Vn.alloc(words ? words : 1);
        Q.alloc(b.num_vss ? b.num_vss : 1);
        ctr.alloc(4);
    }
};

namespace {

__global__ void k_part_begin(uint32_t n, uint32_t row_lo, uint32_t row_hi, uint64_t w_lo, uint64_t w_hi,
                             uint32_t src, const uint32_t* __restrict__ rp, uint32_t* L, uint32_t* Vc,
                             uint32_t* Vn, unsigned long long* Q, unsigned long long* ctr) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = row_lo + t; i < row_hi; i += T) L[i] = (i == src) ? 0u : kInf;
    for (uint64_t w = w_lo + t; w < w_hi; w += T) {
        const uint32_t seed = (w == (src >> 5) && src >= row_lo && src < row_hi) ? 1u << (src & 31) : 0u;
        Vc[w] = seed;
        Vn[w] = seed;
    }
    const uint32_t ss = src >> 3, b = rp[ss], e = rp[ss + 1];
    const unsigned long long aux = (unsigned long long)(1u << (src & 7)) << 32;
    for (uint64_t i = t; i < e - b; i += T) Q[i] = aux | (b + i);
    if (t == 0) {
        ctr[0] = e - b;
        ctr[1] = ctr[2] = ctr[3] = 0;
    }
}

__global__ void k_part_pull(const unsigned long long* __restrict__ Q, unsigned long long len,
                            const uint32_t* __restrict__ masks, const uint4* __restrict__ rows4,
                            const uint32_t* __restrict__ Vc, uint32_t* Vn, unsigned long long* ctr) {
    constexpr int B = 4;  // VSSs in flight per warp (as the fused lazy kernel's stage 1)
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t NW = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t pol = evict_first_policy();
    uint32_t reds = 0;
    for (uint64_t p0 = gw; p0 < len; p0 += NW * B) {
        unsigned long long e = ~0ull;
        if (lane < B && p0 + lane * NW < len) e = Q[p0 + lane * NW];
        uint32_t m[B], alpha[B];
        uint4 r[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
            const unsigned long long ej = __shfl_sync(0xffffffffu, e, j);
            alpha[j] = ej == ~0ull ? 0u : (uint32_t)(ej >> 32) & 0xFFu;
            m[j] = 0;
            r[j] = make_uint4(0, 0, 0, 0);
            if (ej != ~0ull) {
                const uint64_t v = (uint32_t)ej;
                m[j] = ld_stream_u32(masks + 32 * v + lane, pol);
                r[j] = ld_stream_u4(rows4 + 32 * v + lane, pol);
            }
        }
#pragma unroll
        for (int j = 0; j < B; ++j) {
            const uint32_t x = m[j] & (alpha[j] * 0x01010101u);
            const uint32_t u[4] = {r[j].x, r[j].y, r[j].z, r[j].w};
            uint32_t vw[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) vw[c] = ((x >> (8 * c)) & 0xFFu) ? Vc[u[c] >> 5] : ~0u;  // before ℓ?
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (!((vw[c] >> (u[c] & 31)) & 1u)) vw[c] = ld_l2_u32(Vn + (u[c] >> 5));  // marked at ℓ?
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (!((vw[c] >> (u[c] & 31)) & 1u)) {
                    atomicOr(Vn + (u[c] >> 5), 1u << (u[c] & 31));
                    ++reds;
                }
        }
    }
    reds = warp_sum(reds);
    if (lane == 0 && reds) atomicAdd(&ctr[2], (unsigned long long)reds);
}

__global__ void k_part_sweep(uint64_t w_lo, uint64_t w_hi, uint32_t level, uint32_t* Vc, const uint32_t* Vn,
                             uint32_t* L, uint32_t* diff_out, unsigned long long* ctr) {
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long disc = 0;
    for (uint64_t wb = w_lo + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull); wb < w_hi;
         wb += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = wb + lane;
        uint32_t diff = 0;
        if (w < w_hi) {
            const uint32_t nx = Vn[w];
            diff = nx & ~Vc[w];
            if (diff) Vc[w] = nx;
            diff_out[w - w_lo] = diff;
        }
        disc += __popc(diff);
        unsigned ball = __ballot_sync(0xffffffffu, diff != 0);
        while (ball) {
            const int k = __ffs(ball) - 1;
            ball &= ball - 1;
            const uint32_t dk = __shfl_sync(0xffffffffu, diff, k);
            if ((dk >> lane) & 1u) L[32 * (wb + k) + lane] = level;
        }
    }
    disc = warp_sum(disc);
    if (lane == 0 && disc) atomicAdd(&ctr[1], disc);
}

__global__ void k_part_enqueue(const uint32_t* __restrict__ diff, uint64_t words, const uint32_t* __restrict__ rp,
                               unsigned long long* Q, unsigned long long* ctr) {
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long bits = 0;
    for (uint64_t wb = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull; wb < words;
         wb += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = wb + lane;
        const uint32_t d = (w < words) ? diff[w] : 0u;
        bits += __popc(d);
        uint32_t b[4] = {0, 0, 0, 0}, c[4] = {0, 0, 0, 0};
        uint32_t cnt = 0;
#pragma unroll
        for (int s = 0; s < 4; ++s)
            if ((d >> (8 * s)) & 0xFFu) {
                b[s] = rp[4 * w + s];
                c[s] = rp[4 * w + s + 1] - b[s];
                cnt += c[s];
            }
        const uint32_t incl = warp_incl_scan(cnt);
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long base = 0;
        if (lane == 31 && tot) base = atomicAdd(&ctr[0], (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 31);
        unsigned long long pos = base + incl - cnt;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const unsigned long long aux = (unsigned long long)((d >> (8 * s)) & 0xFFu) << 32;
            for (uint32_t i = 0; i < c[s]; ++i) Q[pos++] = aux | (b[s] + i);
        }
    }
    bits = warp_sum(bits);
    if (lane == 0 && bits) atomicAdd(&ctr[3], bits);
}

}  // namespace

PartEngine* part_create(const DeviceBvss& b) { return new PartEngine(b); }
void part_destroy(PartEngine* e) { delete e; }

void part_range(const PartEngine& e, uint32_t* row_lo, uint32_t* row_hi, uint64_t* w_lo, uint64_t* w_hi) {
    if (row_lo) *row_lo = e.b.row_lo;
    if (row_hi) *row_hi = e.b.row_hi > e.b.n ? e.b.n : e.b.row_hi;
    if (w_lo) *w_lo = e.w_lo;
    if (w_hi) *w_hi = e.w_hi;
}

uint64_t part_begin(PartEngine& e, uint32_t src) {
    if (src >= e.b.n) throw InvalidArgument("bfs source out of range");
    const uint32_t hi = e.b.row_hi > e.b.n ? e.b.n : e.b.row_hi;
    k_part_begin<<<grid_for(hi - e.b.row_lo + 1, 256), 256, 0, stream()>>>(
        e.b.n, e.b.row_lo, hi, e.w_lo, e.w_hi, src, e.b.real_ptrs.p, e.L.p, e.Vc.p, e.Vn.p, e.Q.p, e.ctr.p);
    CK(cudaGetLastError());
    unsigned long long len = 0;
    CK(cudaMemcpyAsync(&len, e.ctr.p, 8, cudaMemcpyDeviceToHost, stream()));
    CK(cudaStreamSynchronize(stream()));
    return len;
}

void part_pull(PartEngine& e, uint64_t len) {
    if (!len) return;
    k_part_pull<<<grid_for(len * 8, 256), 256, 0, stream()>>>(e.Q.p, len, e.b.masks.p,
                                                               reinterpret_cast<const uint4*>(e.b.row_ids.p), e.Vc.p,
                                                               e.Vn.p, e.ctr.p);
    CK(cudaGetLastError());
}

uint64_t part_sweep(PartEngine& e, uint32_t level, uint32_t* diff_out_dev) {
    CK(cudaMemsetAsync(e.ctr.p + 1, 0, 8, stream()));
    if (e.w_hi > e.w_lo) {
        k_part_sweep<<<grid_for(e.w_hi - e.w_lo, 256), 256, 0, stream()>>>(e.w_lo, e.w_hi, level, e.Vc.p, e.Vn.p,
                                                                           e.L.p, diff_out_dev, e.ctr.p);
        CK(cudaGetLastError());
    }
    unsigned long long d = 0;
    CK(cudaMemcpyAsync(&d, e.ctr.p + 1, 8, cudaMemcpyDeviceToHost, stream()));
    CK(cudaStreamSynchronize(stream()));
    return d;
}

uint64_t part_enqueue(PartEngine& e, const uint32_t* full_diff_dev, uint64_t* total_bits) {
    CK(cudaMemsetAsync(e.ctr.p, 0, 8, stream()));
    CK(cudaMemsetAsync(e.ctr.p + 3, 0, 8, stream()));
    if (e.words) {
        k_part_enqueue<<<grid_for(e.words, 256), 256, 0, stream()>>>(full_diff_dev, e.words, e.b.real_ptrs.p, e.Q.p,
                                                                     e.ctr.p);
        CK(cudaGetLastError());
    }
    unsigned long long h[4];
    CK(cudaMemcpyAsync(h, e.ctr.p, 32, cudaMemcpyDeviceToHost, stream()));
    CK(cudaStreamSynchronize(stream()));
    if (total_bits) *total_bits = h[3];
    return h[0];
}

void part_levels(const PartEngine& e, uint32_t* levels_host) {
    const uint32_t hi = e.b.row_hi > e.b.n ? e.b.n : e.b.row_hi;
    if (hi > e.b.row_lo)
        CK(cudaMemcpy(levels_host, e.L.p + e.b.row_lo, (size_t)(hi - e.b.row_lo) * 4, cudaMemcpyDeviceToHost));
}

}  // namespace blestgpu
