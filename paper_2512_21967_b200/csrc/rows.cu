// Row-partitioned multi-GPU BFS engine: see rows.cuh for the protocol. Stage 1 is the
// single-GPU lazy pull (lazy_pull.cuh) over the rank's local VSSs; stage 2 is split into
// the owned-word sweep (2a) and the whole-frontier sweep (2b) around the exchange.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cstring>

#include "bfs_device.cuh"
#include "lazy_pull.cuh"
#include "rows.cuh"

namespace blestgpu {

extern std::atomic<uint64_t> g_launches;

// ctl slots
enum : int {
    kT = 0,        // VSSs queued for the level (local)
    kS = 1,        // sets queued (local)
    kBits = 2,     // discovered bits in the last exchanged frontier (global: same on every rank)
    kTail = 3,     // stage-1 tail chunk counter
    kIters = 4,    // level iterations of the last BFS (including the barren last one)
    kStatus = 6,   // 0 ok, 1 runaway, 2 cross-rank barrier timeout
    kXBar = 7,     // fused: cross-rank barriers passed (persistent across BFSs)
    kDone = 8,     // stepped: BFS finished (later launches are no-ops)
    kVis = 9,      // stepped: vertices visited through the previous level (9 | 10 by level parity)
    kUnpulled = 11,  // local VSSs of a barren last level accounted without a pull (exhaustion exit)
    kCtl = 16
};

struct RowsParams {
    uint32_t n, rank, world, src, level, cap, trace_cap, tail_div;
    uint64_t words, w_lo, w_hi, xstride, per, dense_min;
    const uint32_t* rp;
    const uint32_t* masks;
    const uint4* rows4;
    uint32_t* L;
    uint32_t* Vc;
    uint32_t* Vn;
    uint32_t* X;               // own exchange buffer: X0 | X1 | arrival counter
    const uintptr_t* peers;    // [world] exchange bases (own included)
    uint32_t* send;            // stepped: owned diff words
    const uint32_t* recv;      // stepped: gathered (world × per, rank-major)
    const uint64_t* bounds;    // [world + 1] owned word bounds of every rank
    unsigned long long* Q;
    unsigned long long* SL;
    unsigned long long* ctl;
    unsigned long long* agg;   // 3 × 4096: per-CTA (level << 40 | VSS), (… | sets), (… | bits)
    unsigned long long* trace;
    unsigned long long* tstamp;  // 4 per level (timeline), may be null
    uint32_t sys_scope;          // fused exchange with peers on other GPUs (IPC): system-scope sync
    uint32_t xstamp;             // timing study (BLEST_XSTAMP): exchange-phase stamp point, 0 = default
    // hot-row view of the rank's rows (sigma.cuh; hot_words = 0: plain row ids): V words =
    // [hot prefix | row words]; inv: hot rank -> row; sig: row -> engine id; H: staging
    // words (row space) for the hot discoveries of the level
    uint64_t hot_words;
    const uint32_t* inv;
    const uint32_t* sig;
    uint32_t* H;
    unsigned* hflags;          // mapped host flags
    // exhaustion exit (as in the lazy kernel): global bitmap of the rows present in the BVSS
    // (every vertex with an in-arc) and their count; 0 = off
    const uint32_t* present;
    uint64_t present_rows;
};

// Every rank's parameters of one launch, passed by value (kernel parameter space: constant
// bank loads, no per-thread copy of a global struct). One entry per rank of the launch.
constexpr uint32_t kMaxLaunchRanks = 12;
struct RowsLaunch {
    RowsParams r[kMaxLaunchRanks];
};
static_assert(sizeof(RowsLaunch) <= 4096, "kernel parameter block");

namespace {
using namespace bfsdev;
namespace cg = cooperative_groups;

constexpr unsigned long long kTagMask = (1ull << 40) - 1;
constexpr uint32_t kAggStride = 4096;
constexpr unsigned long long kTimeoutNs = 30ull * 1000 * 1000 * 1000;

__device__ __forceinline__ void red_release_sys_add(unsigned* p, unsigned v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Cross-rank arrival barrier (fused mode). Callers: every thread, after a grid barrier that
// follows their (system-fenced) peer stores. Thread 0 of the rank's first CTA adds 1 to every
// rank's arrival counter (X word 2·xstride; release, system scope) and waits for its own to
// reach world × (barriers passed + 1) (acquire); then a grid barrier spreads it. A wait
// past kTimeoutNs (a peer is not running) raises the abort word (X word 2·xstride + 1) of
// every rank and returns false everywhere — virtual ranks sharing one grid all see it
// after the same grid barrier, so they leave the level loop together.
__device__ bool cross_rank_barrier(const RowsParams& p, uint32_t vb) {
    volatile unsigned* abort_word = p.X + 2 * p.xstride + 1;
    if (vb == 0 && threadIdx.x == 0) {
        // peers on other GPUs (IPC mappings): system scope; virtual ranks of one device share
        // its L2, so device scope suffices (a system-scope release costs ~0.3 ms per level here)
        if (p.sys_scope) {
            __threadfence_system();  // cumulative: every CTA's stores ordered before it by the grid barrier
            for (uint32_t r = 0; r < p.world; ++r)
                red_release_sys_add(reinterpret_cast<unsigned*>(p.peers[r]) + 2 * p.xstride, 1u);
        } else {
            for (uint32_t r = 0; r < p.world; ++r)
                red_release_gpu_add(reinterpret_cast<unsigned*>(p.peers[r]) + 2 * p.xstride, 1u);
        }
        const unsigned* mine = p.X + 2 * p.xstride;
        const unsigned long long passed = p.ctl[kXBar];
        const unsigned want = (unsigned)(p.world * (passed + 1));
        const unsigned long long t0 = globaltimer();
        while (!*abort_word &&
               (int)((p.sys_scope ? ld_acquire_sys(mine) : ld_acquire_gpu_u32(mine)) - want) < 0) {
            if (globaltimer() - t0 > kTimeoutNs) {
                p.ctl[kStatus] = 2;
                for (uint32_t r = 0; r < p.world; ++r)
                    reinterpret_cast<volatile unsigned*>(p.peers[r])[2 * p.xstride + 1] = 1u;
                __threadfence_system();
                break;
            }
        }
        p.ctl[kXBar] = passed + 1;
    }
    __syncwarp();
    cg::this_grid().sync();
    if (*abort_word) {
        if (vb == 0 && threadIdx.x == 0) p.ctl[kStatus] = 2;
        return false;
    }
    return true;
}

// word w of the gathered frontier (stepped mode): rank-major chunks of `per` words
__device__ __forceinline__ uint32_t gathered_word(const RowsParams& p, uint64_t w) {
    uint32_t r = 0;
    while (r + 1 < p.world && w >= p.bounds[r + 1]) ++r;
    return p.recv[(uint64_t)r * p.per + (w - p.bounds[r])];
}

// Stage 2b: sweep the whole frontier (Xsrc; stepped mode unpacks it from recv into X0
// first), count its bits, and queue the active sets that have local VSSs as SL entries
// (set | first position << 32) in ascending order: per-CTA counts published with a level
// tag, predecessors summed, no contended atomics. The rank's last CTA stores the totals.
template <int THREADS, bool STEPPED>
__device__ unsigned long long stage2b(const RowsParams& p, Smem<THREADS, 1>& sm, uint32_t level, uint32_t vb,
                                      uint32_t vG, const uint32_t* Xsrc, uint32_t (&ctr)[4]) {
    constexpr uint64_t CH = 4ull * THREADS;
    const uint64_t chunks = (p.words + CH - 1) / CH;
    const uint64_t k0 = (uint64_t)vb * chunks / vG, k1 = (uint64_t)(vb + 1) * chunks / vG;
    uint32_t* X0 = p.X;
    auto load4 = [&](uint64_t w0, uint32_t (&d)[4], bool unpack) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint64_t w = w0 + k;
            uint32_t v = 0;
            if (w < p.words) {
                if (STEPPED && unpack) {
                    v = gathered_word(p, w);
                    X0[w] = v;  // α of this launch's stage 1
                } else {
                    v = __ldcg(Xsrc + w);
                }
            }
            d[k] = v;
        }
    };
    const uint64_t num_sets = (p.n + 7ull) / 8;
    auto counts = [&](uint64_t w0, const uint32_t (&d)[4], unsigned long long& nv, unsigned long long& ns) {
        if (!(d[0] | d[1] | d[2] | d[3])) return;
        uint32_t r[17];  // the 16 sets' real_ptrs bounds, loaded together (bfs_device.cuh s2_rp)
        s2_rp(p.rp, num_sets, w0, r);
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const uint32_t c = ((d[k] >> (8 * b)) & 0xFFu) ? r[4 * k + b + 1] - r[4 * k + b] : 0u;
                nv += c;
                ns += c != 0;
            }
    };
    unsigned long long my_v = 0, my_s = 0, my_b = 0, nzm = 0;
    if (threadIdx.x == 0) sm.nz = 0;
    if (STEPPED) {
        for (uint64_t ch = k0; ch < k1; ++ch) {
            const uint64_t w0 = ch * CH + 4ull * threadIdx.x;
            uint32_t d[4];
            load4(w0, d, true);
#pragma unroll
            for (int k = 0; k < 4; ++k) my_b += __popc(d[k]);
            if (d[0] | d[1] | d[2] | d[3]) nzm |= chunk_bit(ch - k0);
            counts(w0, d, my_v, my_s);
        }
    } else {
        // fused: 4 chunks per round, their uint4 loads issued together (X is 16-byte aligned)
        constexpr int U = 4;
        for (uint64_t c0 = k0; c0 < k1; c0 += U) {
            uint32_t d[U][4];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t w0 = (c0 + u) * CH + 4ull * threadIdx.x;
                if (c0 + u < k1 && w0 + 4 <= p.words) {
                    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(Xsrc + w0));
                    d[u][0] = v.x; d[u][1] = v.y; d[u][2] = v.z; d[u][3] = v.w;
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) d[u][k] = (c0 + u < k1 && w0 + k < p.words) ? __ldcg(Xsrc + w0 + k) : 0u;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (c0 + u >= k1) break;
                const uint64_t w0 = (c0 + u) * CH + 4ull * threadIdx.x;
#pragma unroll
                for (int k = 0; k < 4; ++k) my_b += __popc(d[u][k]);
                if (d[u][0] | d[u][1] | d[u][2] | d[u][3]) nzm |= chunk_bit(c0 + u - k0);
                counts(w0, d[u], my_v, my_s);
            }
        }
    }
    unsigned long long cta_v = 0, cta_s = 0, cta_b = 0;
    block_excl_scan(sm, my_v, &cta_v);
    block_or_nz(sm, nzm);
    block_excl_scan(sm, my_s, &cta_s);
    block_excl_scan(sm, my_b, &cta_b);
    unsigned long long* aggV = p.agg;
    unsigned long long* aggS = p.agg + kAggStride;
    unsigned long long* aggB = p.agg + 2 * kAggStride;
    if (threadIdx.x == 0) {
        const unsigned long long tag = (unsigned long long)level << 40;
        aggS[vb] = tag | cta_s;
        aggB[vb] = tag | cta_b;
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(aggV + vb), "l"(tag | cta_v) : "memory");
    }
    if (STEPPED) __syncthreads();  // the unpacked X0 words are re-read below by other threads
    unsigned long long bv = 0, bs = 0, bb = 0;
    for (uint32_t c = threadIdx.x; c < vb; c += THREADS) {
        unsigned long long x;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(aggV + c) : "memory");
        } while ((x >> 40) != level);
        bv += x & kTagMask;
        bs += ld_relaxed_gpu_u64(aggS + c) & kTagMask;
    }
    // grid totals of the bits come from the last CTA summing everyone
    if (vb == vG - 1)
        for (uint32_t c = threadIdx.x; c < vG; c += THREADS) {
            unsigned long long x;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(aggV + c) : "memory");
            } while ((x >> 40) != level);
            bb += ld_relaxed_gpu_u64(aggB + c) & kTagMask;
        }
    unsigned long long run_v = 0, run_s = 0, all_b = 0;
    block_excl_scan(sm, bv, &run_v);
    block_excl_scan(sm, bs, &run_s);
    block_excl_scan(sm, bb, &all_b);
    if (threadIdx.x == 0) {
        ctr[3] += (uint32_t)cta_v;
        if (vb == vG - 1) {
            p.ctl[kT] = run_v + cta_v;
            p.ctl[kS] = run_s + cta_s;
            p.ctl[kBits] = all_b;
        }
    }
    const uint32_t* Xs = STEPPED ? X0 : Xsrc;
    const unsigned long long nz = sm.nz;  // after the scans' __syncthreads
    for (uint64_t ch = k0; ch < k1; ++ch) {
        if (!(nz & chunk_bit(ch - k0))) continue;  // no frontier word: nothing to queue
        const uint64_t w0 = ch * CH + 4ull * threadIdx.x;
        uint32_t d[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) d[k] = (w0 + k < p.words) ? __ldcg(Xs + w0 + k) : 0u;
        unsigned long long nv = 0, ns = 0;
        counts(w0, d, nv, ns);
        unsigned long long it_v = 0, it_s = 0;
        unsigned long long pv = run_v + block_excl_scan(sm, nv, &it_v);
        unsigned long long ps = run_s + block_excl_scan(sm, ns, &it_s);
        if (ns) {
            uint32_t r[17];
            s2_rp(p.rp, num_sets, w0, r);
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const uint32_t c = ((d[k] >> (8 * b)) & 0xFFu) ? r[4 * k + b + 1] - r[4 * k + b] : 0u;
                    if (c) {
                        p.SL[ps++] = (pv << 32) | (4 * (w0 + k) + b);
                        pv += c;
                    }
                }
        }
        run_v += it_v;
        run_s += it_s;
    }
    return nz;  // the CTA's chunks holding a frontier word (clear list of the next level)
}

// Stage 2a: the owned V words — diff = V_next & ~V_curr, V_curr = V_next, levels (one
// coalesced 128 B store per changed word); each diff word goes to `emit(w, d)`.
template <typename Emit>
__device__ __forceinline__ void stage2a(const RowsParams& p, uint32_t level, uint64_t gtid, uint64_t gthreads,
                                        uint32_t (&ctr)[4], Emit emit) {
    constexpr int U = 4;  // words per thread per round, their loads issued together
    const unsigned lane = lane_id();
    const uint64_t span = p.w_hi - p.w_lo;
    uint32_t* Vc = p.Vc + p.hot_words;  // row words (after the hot prefix)
    const uint32_t* Vn = p.Vn + p.hot_words;
    const bool hot = p.hot_words != 0;
    for (uint64_t i0 = gtid - lane; i0 < span; i0 += U * gthreads) {
        uint32_t nx[U], cu[U], h[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + u * gthreads + lane;
            const uint64_t w = p.w_lo + i;
            const bool ok = i < span;
            nx[u] = ok ? __ldcg(Vn + w) : 0u;
            cu[u] = ok ? Vc[w] : 0u;
            h[u] = (ok && hot) ? __ldcg(p.H + w) : 0u;  // the hot rows' discoveries (levels stored)
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t iw = i0 + u * gthreads;  // the warp's first word of this round
            const uint64_t w = p.w_lo + iw + lane;
            const uint32_t d = nx[u] & ~cu[u];
            if (iw + lane < span) {
                if (d) Vc[w] = nx[u];
                if (hot && h[u]) p.H[w] = 0u;
                emit(w, d | h[u]);
            }
            ctr[0] += __popc(d);
            unsigned ball = __ballot_sync(0xffffffffu, d != 0);
            while (ball) {
                const int k = __ffs(ball) - 1;
                ball &= ball - 1;
                const uint32_t dk = __shfl_sync(0xffffffffu, d, k);
                const uint64_t wk = p.w_lo + iw + k;
                if ((dk >> lane) & 1u) p.L[32 * wk + lane] = level;
            }
        }
    }
}

// Hot pass of stage 2a: the hot prefix of V (word w handled by CTA w mod G): each hot
// discovery mapped back by σ⁻¹ to store its level and RED its bit into H (row space); the
// owned-word sweep merges H after a grid barrier.
__device__ __forceinline__ void stage2a_hot(const RowsParams& p, uint32_t level, uint32_t vb, uint32_t vG,
                                            uint32_t (&ctr)[4]) {
    for (uint64_t w = vb + (uint64_t)threadIdx.x * vG; w < p.hot_words; w += (uint64_t)blockDim.x * vG) {
        const uint32_t nx = __ldcg(p.Vn + w), d = nx & ~p.Vc[w];
        if (!d) continue;
        p.Vc[w] = nx;
        ctr[0] += __popc(d);
        for (uint32_t rest = d; rest; rest &= rest - 1) {
            const uint32_t r = __ldg(p.inv + 32 * w + (__ffs(rest) - 1));
            p.L[r] = level;
            red_or(p.H + (r >> 5), 1u << (r & 31));
        }
    }
}

// Per-level counters into the trace row: warp sums, then one shared-memory sum per CTA, then
// one atomic per CTA and counter (not per warp: 4.7 K same-address atomics per level cost
// tens of µs).
template <int THREADS>
__device__ __forceinline__ void trace_add(const RowsParams& p, Smem<THREADS, 1>& sm, uint32_t level, uint32_t (&ctr)[4]) {
    if (threadIdx.x < 4) sm.ctr[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t s = warp_sum(ctr[i]);
        if (lane_id() == 0 && s) atomicAdd(&sm.ctr[i], (unsigned long long)s);
        ctr[i] = 0;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        const unsigned long long s = sm.ctr[threadIdx.x];
        const uint32_t row = min(level - 1, p.trace_cap - 1);
        constexpr int slot[4] = {3, 4, 6, 7};  // discovered, full, relaxed, pushes
        if (s) atomicAdd(&p.trace[8ull * row + slot[threadIdx.x]], s);
    }
    __syncwarp();
}

// Level timeline (rank 0's first CTA, %globaltimer): [start, stage-1 end, exchange end, level end].
__device__ __forceinline__ void stamp(const RowsParams& p, uint32_t vb, uint32_t level, int slot) {
    if (vb == 0 && threadIdx.x == 0 && p.tstamp && level - 1 < p.trace_cap)
        p.tstamp[4ull * (level - 1) + slot] = globaltimer();
}

template <int PULL, int THREADS, bool STEPPED>
__global__ void __launch_bounds__(THREADS, 1024 / THREADS) k_bfs_rows(const __grid_constant__ RowsLaunch P, uint32_t cpr) {
    constexpr int WPC = THREADS / 32;
    __shared__ Smem<THREADS, 1> sm;
    const RowsParams& p = P.r[blockIdx.x / cpr];
    // the parameters come from global memory, so their pointers would otherwise be generic
    // (LD/ST instead of LDG/STG/RED everywhere)
    __builtin_assume(__isGlobal(p.rp) && __isGlobal(p.masks) && __isGlobal(p.rows4) && __isGlobal(p.L));
    __builtin_assume(__isGlobal(p.Vc) && __isGlobal(p.Vn) && __isGlobal(p.X) && __isGlobal(p.peers));
    __builtin_assume(__isGlobal(p.Q) && __isGlobal(p.SL) && __isGlobal(p.ctl) && __isGlobal(p.agg));
    __builtin_assume(__isGlobal(p.trace) && __isGlobal(p.bounds));
    if (p.hot_words) __builtin_assume(__isGlobal(p.inv) && __isGlobal(p.sig) && __isGlobal(p.H));
    if (STEPPED) __builtin_assume(__isGlobal(p.send) && __isGlobal(p.recv) && __isGlobal(p.hflags));
    const uint32_t vb = blockIdx.x % cpr, vG = cpr;
    const unsigned lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t gtid = vb * (uint64_t)THREADS + threadIdx.x;
    const uint64_t gthreads = (uint64_t)vG * THREADS;
    const uint32_t gw = vb * WPC + warp, all_warps = vG * WPC;
    const uint32_t sent = (uint32_t)(p.hot_words + p.words);  // sentinel word index of V (all ones)
    uint32_t ctr[4] = {0, 0, 0, 0};           // discovered, -, relaxed, pushes
    auto grid_sync = [] { cg::this_grid().sync(); };

    uint32_t level = STEPPED ? p.level : 1;
    if (STEPPED && level > 1 && ld_relaxed_gpu_u64(&p.ctl[kDone])) return;  // BFS over: no-op launch
    if (STEPPED && gtid == 0) p.hflags[0] = level;  // progress (host run-ahead limit)

    if (level == 1) {
        // ---- init_state (R:src/bfs_engine.cpp:30-49) restricted to the owned rows ----
        const uint32_t src = p.src, sset = src / kSigma;
        for (uint64_t i = 32 * p.w_lo + gtid; i < 32 * p.w_hi && i < p.n; i += gthreads) p.L[i] = (i == src) ? 0u : kInf;
        // V: the hot prefix and the owned row words; the source's engine id if it is ours
        const bool own_src = src >= 32 * p.w_lo && src < 32 * p.w_hi;
        const uint32_t vsrc = own_src ? (p.hot_words ? p.sig[src] : src) : 0xFFFFFFFFu;
        for (uint64_t w = gtid; w < p.hot_words; w += gthreads) {
            const uint32_t seed = (own_src && w == (vsrc >> 5)) ? 1u << (vsrc & 31) : 0u;
            p.Vc[w] = seed;
            p.Vn[w] = seed;
        }
        for (uint64_t w = p.w_lo + gtid; w < p.w_hi; w += gthreads) {
            const uint64_t ew = p.hot_words + w;
            const uint32_t seed = (own_src && ew == (vsrc >> 5)) ? 1u << (vsrc & 31) : 0u;
            p.Vc[ew] = seed;
            p.Vn[ew] = seed;
            if (p.hot_words) p.H[w] = 0u;
        }
        // α of level 1: the source's bit in X0 (every rank); fused: X1 cleared for the peers
        for (uint64_t w = gtid; w < p.words; w += gthreads) {
            p.X[w] = (w == (src >> 5)) ? 1u << (src & 31) : 0u;
            if (!STEPPED) p.X[p.xstride + w] = 0;
        }
        if (threadIdx.x == 0) {
            p.agg[vb] = 0;
            p.agg[kAggStride + vb] = 0;
            p.agg[2 * kAggStride + vb] = 0;
        }
        if (gtid == 0) {
            p.Vc[sent] = ~0u;
            p.Vn[sent] = ~0u;
            const uint32_t b = p.rp[sset], e = p.rp[sset + 1];
            p.SL[0] = sset;
            p.ctl[kT] = e - b;
            p.ctl[kS] = (e > b) ? 1 : 0;
            p.ctl[kBits] = 1;
            p.ctl[kIters] = 0;
            p.ctl[kStatus] = 0;
            p.ctl[kDone] = 0;
            p.ctl[kUnpulled] = 0;
            for (int i = 0; i < 8; ++i) p.trace[i] = 0;
        }
        grid_sync();
        if (!STEPPED) {
            __threadfence_system();
            grid_sync();
            if (!cross_rank_barrier(p, vb)) return;  // every rank initialised before any peer store
        }
    } else {
        // ---- stepped, level > 1: unpack the gathered frontier, 2b ----
        stage2b<THREADS, STEPPED>(p, sm, level - 1, vb, vG, nullptr, ctr);
        grid_sync();
        trace_add<THREADS>(p, sm, level - 1, ctr);
        if (ld_relaxed_gpu_u64(&p.ctl[kBits]) == 0) {  // level - 1 discovered nothing anywhere
            if (gtid == 0) {
                p.ctl[kIters] = level - 1;
                p.ctl[kDone] = 1;
                __threadfence_system();
                p.hflags[1] = level - 1;
            }
            return;
        }
    }

    // fused: the CTA's 2b chunks holding the last frontier's words (level 1: the source's)
    unsigned long long prev_nz = 0;
    {
        constexpr uint64_t CH = 4ull * THREADS;
        const uint64_t chunks = (p.words + CH - 1) / CH;
        const uint64_t k0 = (uint64_t)vb * chunks / vG, k1 = (uint64_t)(vb + 1) * chunks / vG;
        const uint64_t cs = (uint64_t)(p.src >> 5) / CH;
        if (cs >= k0 && cs < k1) prev_nz = chunk_bit(cs - k0);
    }
    // exhaustion exit: every rank sees the same exchanged frontiers, so every rank keeps the
    // same visited count (1 + Σ kBits) and stops at the same level once it covers every row
    // present anywhere (plus the source if it is not one): that level is barren
    const uint64_t reach = p.present_rows
                               ? p.present_rows + (((p.present[p.src >> 5] >> (p.src & 31)) & 1u) ? 0u : 1u)
                               : ~0ull;
    unsigned long long visited = 0;  // fused: running sum of kBits (level 1: the source)
    for (;; ++level) {
        const unsigned long long len = ld_relaxed_gpu_u64(&p.ctl[kT]);
        const uint32_t S = (uint32_t)ld_relaxed_gpu_u64(&p.ctl[kS]);
        const unsigned long long bits = ld_relaxed_gpu_u64(&p.ctl[kBits]);
        if (!STEPPED && bits == 0) break;
        if (STEPPED) {  // one launch per level: the count travels in ctl (two slots by parity)
            visited = (level == 1 ? 0ull : ld_relaxed_gpu_u64(&p.ctl[kVis + (level & 1)])) + bits;
            if (gtid == 0) p.ctl[kVis + ((level + 1) & 1)] = visited;
        } else {
            visited += bits;
        }
        if (level > p.cap) {  // runaway (R:src/bfs_engine.cpp:72-75)
            if (gtid == 0) {
                p.ctl[kStatus] = 1;
                if (STEPPED) {
                    p.ctl[kDone] = 1;
                    p.ctl[kIters] = level - 1;
                    __threadfence_system();
                    p.hflags[2] = 1;
                    p.hflags[1] = level - 1;
                }
            }
            break;
        }
        const uint32_t* Fd = p.X + (STEPPED ? 0 : ((level - 1) & 1) * p.xstride);  // α words
        stamp(p, vb, level, 0);
        if (gtid == 0) {
            p.ctl[kTail] = 0;
            if (level - 1 < p.trace_cap) {
                p.trace[8ull * (level - 1) + 0] = level;
                p.trace[8ull * (level - 1) + 1] = len;
            }
            if (level < p.trace_cap)
                for (int i = 0; i < 8; ++i) p.trace[8ull * level + i] = 0;
        }
        if (visited >= reach) {  // barren by exhaustion: its trace row is (level, len, 0, …)
            if (gtid == 0) {
                p.ctl[kUnpulled] = len;
                if (STEPPED) {
                    p.ctl[kIters] = level;
                    p.ctl[kDone] = 1;
                    __threadfence_system();
                    p.hflags[1] = level;
                }
            }
            if (STEPPED) return;
            ++level;  // the barren level counts as an iteration
            break;
        }
        // ---- stage 1: pull of the local VSSs (lazy_pull.cuh) ----
        // reconverge warp 0 after the single-thread blocks above: a diverged warp would run
        // the whole pull through the shuffles' divergent fallback (measured: 2x stage 1)
        __syncwarp();
        PullCtx pc;
        pc.rp = p.rp;
        pc.masks = p.masks;
        pc.rows4 = p.rows4;
        pc.Fd8 = reinterpret_cast<const uint8_t*>(Fd);
        pc.SL = p.SL;
        pc.Q = p.Q;
        pc.tail_ctr = &p.ctl[kTail];
        pc.W = p.Vn;
        pc.Vn = p.Vn;
        pc.len = len;
        pc.S = S;
        pc.sent = sent;
        pc.recheck = false;
        pc.tail_div = p.tail_div;
        pc.gw = gw;
        pc.NW = all_warps;
        pc.all_warps = all_warps;
        pc.pol = evict_first_policy();
        if (len < p.dense_min) {
            ctr[2] += pull_sparse<PULL>(pc);
            if (cpr != gridDim.x) grid_sync();  // virtual ranks: same barrier count on every rank
        } else {
            expand_queue(pc);
            grid_sync();
            ctr[2] += pull_dense<PULL>(pc);
        }
        grid_sync();
        stamp(p, vb, level, 1);

        // ---- stage 2a: owned words; diffs to the exchange ----
        if (p.hot_words) {  // same on every rank of a launch: the barrier counts match
            stage2a_hot(p, level, vb, vG, ctr);
            grid_sync();
            if (p.xstamp == 1) stamp(p, vb, level, 2);
        }
        if (STEPPED) {
            stage2a(p, level, gtid, gthreads, ctr, [&](uint64_t w, uint32_t d) { p.send[w - p.w_lo] = d; });
            trace_add<THREADS>(p, sm, level, ctr);
            return;  // host: all-gather, then the next level's launch
        }
        const uint64_t xo = (uint64_t)(level & 1) * p.xstride;
        stage2a(p, level, gtid, gthreads, ctr, [&](uint64_t w, uint32_t d) {
            if (d)
                for (uint32_t r = 0; r < p.world; ++r) reinterpret_cast<uint32_t*>(p.peers[r])[xo + w] = d;
        });
        if (p.xstamp == 2) stamp(p, vb, level, 2);
        // this level's α words (read by stage 1 only) are cleared for the level after next:
        // only the CTA's 2b chunks that held a frontier word (prev_nz, from the last 2b)
        {
            uint32_t* Fold = p.X + ((level - 1) & 1) * p.xstride;
            constexpr uint64_t CH = 4ull * THREADS;
            const uint64_t chunks = (p.words + CH - 1) / CH;
            const uint64_t k0 = (uint64_t)vb * chunks / vG, k1 = (uint64_t)(vb + 1) * chunks / vG;
            for (uint64_t ch = k0; ch < k1; ++ch) {
                if (!(prev_nz & chunk_bit(ch - k0))) continue;
                const uint64_t w0 = ch * CH + 4ull * threadIdx.x;
                if (w0 + 4 <= p.words) {
                    *reinterpret_cast<uint4*>(Fold + w0) = make_uint4(0, 0, 0, 0);
                } else {
                    for (uint64_t w = w0; w < p.words && w < w0 + 4; ++w) Fold[w] = 0;
                }
            }
        }
        // the peer stores are ordered before the arrival by this grid barrier (gpu scope) and
        // the cumulative system-scope fence + release of cross_rank_barrier's thread
        grid_sync();
        if (p.xstamp == 3) stamp(p, vb, level, 2);
        if (!cross_rank_barrier(p, vb)) break;
        if (p.xstamp == 0) stamp(p, vb, level, 2);

        // ---- stage 2b: the whole exchanged frontier → termination, next SL ----
        prev_nz = stage2b<THREADS, false>(p, sm, level, vb, vG, p.X + xo, ctr);
        grid_sync();
        trace_add<THREADS>(p, sm, level, ctr);
        stamp(p, vb, level, 3);
    }
    if (!STEPPED && gtid == 0) p.ctl[kIters] = level - 1;
}

template <int PULL, bool STEPPED>
void* rows_kernel(int threads) {
    switch (threads) {
        case 256: return (void*)k_bfs_rows<PULL, 256, STEPPED>;
        case 512: return (void*)k_bfs_rows<PULL, 512, STEPPED>;
    }
    throw InvalidArgument("rows engine: threads per CTA must be 256 or 512");
}

// ---- slice-balanced partition ----
__global__ void k_set_row_keys(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt, uint32_t n,
                               uint64_t* __restrict__ keys) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t u = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; u < n;
         u += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint64_t hi = (u >> 3) << 32;
        for (uint64_t i = off[u] + lane; i < off[u + 1]; i += 32) keys[i] = hi | tgt[i];
    }
}

__global__ void k_row_slices(const uint64_t* __restrict__ keys, uint64_t m, uint32_t* __restrict__ cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        if (i == 0 || keys[i] != keys[i - 1]) atomicAdd(&cnt[(uint32_t)keys[i]], 1u);
}

// words[w] = slices of rows 32w .. 32w+31
__global__ void k_word_slices(const uint32_t* __restrict__ cnt, uint32_t n, uint64_t words, uint64_t* __restrict__ ws) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t s = 0;
        for (uint32_t k = 0; k < 32; ++k) {
            const uint64_t r = 32 * w + k;
            if (r < n) s += cnt[r];
        }
        ws[w] = s;
    }
}

}  // namespace

namespace {
__global__ void k_arc_targets(const uint32_t* __restrict__ tgt, uint64_t m, uint32_t* present) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = tgt[i], bit = 1u << (r & 31);
        if (!(present[r >> 5] & bit)) atomicOr(&present[r >> 5], bit);
    }
}
__global__ void k_popc_words(const uint32_t* __restrict__ w, uint64_t words, unsigned long long* out) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x)
        c += __popc(w[i]);
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
}  // namespace

uint64_t graph_present_rows(const DeviceGraph& g, DevBuf<uint32_t>& bits) {
    const uint64_t words = ((uint64_t)g.n + 31) / 32;
    bits.alloc(words ? words : 1);
    cudaStream_t st = stream();
    CK(cudaMemsetAsync(bits.p, 0, bits.bytes(), st));
    if (g.m) {
        k_arc_targets<<<grid_for(g.m, 256), 256, 0, st>>>(g.tgt.p, g.m, bits.p);
        CK(cudaGetLastError());
    }
    DevBuf<unsigned long long> cnt(1);
    CK(cudaMemsetAsync(cnt.p, 0, 8, st));
    k_popc_words<<<grid_for(words ? words : 1, 256), 256, 0, st>>>(bits.p, words, cnt.p);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return h;
}

std::vector<uint64_t> partition_rows_by_slices(const DeviceGraph& g, uint32_t world, std::vector<uint64_t>* slices_out) {
    if (world == 0) throw InvalidArgument("world size must be positive");
    const uint64_t words = ((uint64_t)g.n + 31) / 32;
    std::vector<uint64_t> bounds(world + 1, 0);
    bounds[world] = words;
    cudaStream_t st = stream();
    std::vector<uint64_t> prefix(words + 1, 0);
    if (g.m && words) {
        DevBuf<uint64_t> keys(g.m), keys2(g.m);
        k_set_row_keys<<<grid_for((uint64_t)g.n * 32, 256), 256, 0, st>>>(g.off.p, g.tgt.p, g.n, keys.p);
        CK(cudaGetLastError());
        cub::DoubleBuffer<uint64_t> dk(keys.p, keys2.p);
        size_t temp = 0;
        CK(cub::DeviceRadixSort::SortKeys(nullptr, temp, dk, (int64_t)g.m, 0, 64, st));
        DevBuf<unsigned char> tmp(temp);
        CK(cub::DeviceRadixSort::SortKeys(tmp.p, temp, dk, (int64_t)g.m, 0, 64, st));
        DevBuf<uint32_t> cnt(g.n);
        CK(cudaMemsetAsync(cnt.p, 0, (size_t)g.n * 4, st));
        k_row_slices<<<grid_for(g.m, 256), 256, 0, st>>>(dk.Current(), g.m, cnt.p);
        CK(cudaGetLastError());
        DevBuf<uint64_t> ws(words), incl(words);
        k_word_slices<<<grid_for(words, 256), 256, 0, st>>>(cnt.p, g.n, words, ws.p);
        CK(cudaGetLastError());
        size_t t2 = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, t2, ws.p, incl.p, (int64_t)words, st));
        DevBuf<unsigned char> tmp2(t2);
        CK(cub::DeviceScan::InclusiveSum(tmp2.p, t2, ws.p, incl.p, (int64_t)words, st));
        CK(cudaMemcpyAsync(prefix.data() + 1, incl.p, words * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    const uint64_t total = prefix[words];
    for (uint32_t r = 1; r < world; ++r) {
        // first word boundary whose prefix reaches r/world of the slices (and keeps order)
        const uint64_t target = (total * r + world - 1) / world;
        uint64_t w = std::lower_bound(prefix.begin(), prefix.end(), target) - prefix.begin();
        if (w > words) w = words;
        bounds[r] = std::max(bounds[r - 1], w);
    }
    if (slices_out) {
        slices_out->assign(world, 0);
        for (uint32_t r = 0; r < world; ++r) (*slices_out)[r] = prefix[bounds[r + 1]] - prefix[bounds[r]];
    }
    return bounds;
}

RowsEngine::RowsEngine(const DeviceBvss& b, uint32_t rank, uint32_t world, const std::vector<uint64_t>& word_bounds)
    : b_(b), rank_(rank), world_(world), bounds_(word_bounds) {
    if (world == 0 || rank >= world) throw InvalidArgument("rank out of range");
    if (bounds_.size() != world + 1) throw InvalidArgument("word bounds must have world + 1 entries");
    words_ = ((uint64_t)b.n + 31) / 32;
    if (bounds_[0] != 0 || bounds_[world] != words_) throw InvalidArgument("word bounds must span [0, ceil(n/32)]");
    for (uint32_t r = 0; r < world; ++r)
        if (bounds_[r] > bounds_[r + 1]) throw InvalidArgument("word bounds must be ascending");
    w_lo_ = bounds_[rank];
    w_hi_ = bounds_[rank + 1];
    row_lo_ = (uint32_t)std::min<uint64_t>(32 * w_lo_, b.n);
    row_hi_ = (uint32_t)std::min<uint64_t>(32 * w_hi_, b.n);
    const uint32_t bhi = b.row_hi > b.n ? b.n : b.row_hi;
    if (b.row_lo != row_lo_ || bhi != row_hi_)
        throw InvalidArgument("the BVSS row range does not match this rank's word bounds");
    per_ = 1;
    for (uint32_t r = 0; r < world; ++r) per_ = std::max<uint64_t>(per_, bounds_[r + 1] - bounds_[r]);
    xstride_ = (words_ + 3) / 4 * 4;
    dbounds_.alloc(world + 1);
    CK(cudaMemcpy(dbounds_.p, bounds_.data(), (world + 1) * 8, cudaMemcpyHostToDevice));
    L_.alloc(b.n ? b.n : 1);
    // hot-row view of this rank's rows (BLEST_SIGMA=0: plain row ids)
    const char* sig_env = getenv("BLEST_SIGMA");
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t sigma_bytes = (uint64_t)b.num_vss * kTau * 4 + 8ull * b.n;  // engine row ids + tables
    if (b.num_vss && !(sig_env && atoi(sig_env) == 0) && sigma_bytes + (4ull << 30) < free_b) {
        const char* hot = getenv("BLEST_HOT");
        sigma_view_build(b, sigma_, hot ? (uint32_t)atoll(hot) : 0u);
        sigma_built_ = (sig_env && atoi(sig_env) == 1) || sigma_.hot_share >= kSigmaMinShare;
        if (sigma_built_) {
            H_.alloc(words_ + 4);
            CK(cudaMemset(H_.p, 0, H_.bytes()));
        } else {
            sigma_.rows.release();
            sigma_.sig.release();
            sigma_.inv.release();
        }
    }
    vstride_ = (sigma_built_ ? sigma_.hot_words : 0) + (words_ + 4) / 4 * 4 + 4;  // + sentinel, 16 B aligned
    V_.alloc(2 * vstride_);
    xbuf_.alloc(2 * xstride_ + 4);
    CK(cudaMemset(xbuf_.p, 0, xbuf_.bytes()));
    send_.alloc(per_);
    CK(cudaMemset(send_.p, 0, send_.bytes()));
    q_.alloc(b.num_vss ? b.num_vss : 1);
    sl_.alloc((uint64_t)b.num_sets + 1);
    ctl_.alloc(kCtl);
    CK(cudaMemset(ctl_.p, 0, kCtl * 8));
    agg_.alloc(3 * kAggStride);
    CK(cudaMemset(agg_.p, 0, agg_.bytes()));
    trace_cap_ = (uint32_t)std::min<uint64_t>((uint64_t)b.n + 2, 1u << 20);
    trace_.alloc(8ull * trace_cap_);
    tstamp_.alloc(4ull * trace_cap_);
    peers_.alloc(world);
    std::vector<uintptr_t> self(world, 0);
    self[rank] = reinterpret_cast<uintptr_t>(xbuf_.p);
    CK(cudaMemcpy(peers_.p, self.data(), world * sizeof(uintptr_t), cudaMemcpyHostToDevice));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&hflags_), 4 * sizeof(unsigned), cudaHostAllocMapped));
    std::memset(hflags_, 0, 4 * sizeof(unsigned));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hflags_dev_), hflags_, 0));
}

RowsEngine::~RowsEngine() {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    if (hflags_) cudaFreeHost(hflags_);
}

void RowsEngine::ipc_handle(void* out64) const {
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, xbuf_.p));
    static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
    std::memcpy(out64, &h, 64);
}

void RowsEngine::open_peers(const void* handles) {
    std::vector<uintptr_t> bases(world_, 0);
    for (uint32_t r = 0; r < world_; ++r) {
        if (r == rank_) {
            bases[r] = reinterpret_cast<uintptr_t>(xbuf_.p);
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char*>(handles) + 64ull * r, 64);
        void* p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        opened_.push_back(p);
        bases[r] = reinterpret_cast<uintptr_t>(p);
    }
    CK(cudaMemcpy(peers_.p, bases.data(), world_ * sizeof(uintptr_t), cudaMemcpyHostToDevice));
}

void RowsEngine::set_local_peers(const std::vector<RowsEngine*>& ranks) {
    if (ranks.size() != world_) throw InvalidArgument("one engine per rank expected");
    std::vector<uintptr_t> bases(world_, 0);
    for (uint32_t r = 0; r < world_; ++r) bases[r] = reinterpret_cast<uintptr_t>(ranks[r]->xbuf_.p);
    CK(cudaMemcpy(peers_.p, bases.data(), world_ * sizeof(uintptr_t), cudaMemcpyHostToDevice));
}

void RowsEngine::fill_params(RowsParams& p, uint32_t src, uint32_t level, const uint32_t* recv, bool allow_sigma) const {
    std::memset(&p, 0, sizeof(p));
    p.n = b_.n;
    p.rank = rank_;
    p.world = world_;
    p.src = src;
    p.level = level;
    p.cap = b_.n + 1;
    p.trace_cap = trace_cap_;
    p.tail_div = 8;
    if (const char* t = getenv("BLEST_TAIL_DIV")) p.tail_div = (uint32_t)atoi(t);
    p.words = words_;
    p.w_lo = w_lo_;
    p.w_hi = w_hi_;
    p.xstride = xstride_;
    p.per = per_;
    p.rp = b_.real_ptrs.p;
    p.masks = b_.masks.p;
    p.rows4 = reinterpret_cast<const uint4*>(b_.row_ids.p);
    p.L = L_.p;
    p.Vc = V_.p;
    p.Vn = V_.p + vstride_;
    if (sigma_built_ && allow_sigma) {
        p.rows4 = reinterpret_cast<const uint4*>(sigma_.rows.p);
        p.hot_words = sigma_.hot_words;
        p.inv = sigma_.inv.p;
        p.sig = sigma_.sig.p;
        p.H = H_.p;
    }
    p.X = xbuf_.p;
    p.peers = peers_.p;
    p.send = send_.p;
    p.recv = recv;
    p.bounds = dbounds_.p;
    p.Q = q_.p;
    p.SL = sl_.p;
    p.ctl = ctl_.p;
    p.agg = agg_.p;
    p.trace = trace_.p;
    p.tstamp = tstamp_.p;
    p.hflags = hflags_dev_;
    p.sys_scope = opened_.empty() ? 0u : 1u;
    const char* ex = getenv("BLEST_EXHAUST");
    if (present_ && !(ex && atoi(ex) == 0)) {
        p.present = present_;
        p.present_rows = present_rows_;
    }
    if (const char* x = getenv("BLEST_XSTAMP")) p.xstamp = (uint32_t)atoi(x);
}

namespace {
struct Geometry {
    void* kern;
    int threads;
    uint32_t ctas;
};
// Stage 1 of every level pulls contiguous equal shares of the queue (the sparse-level path
// of lazy_pull.cuh). The dense-level path (materialised queue, round-robin + dynamic tail)
// measured 1.8x slower in this kernel on C2 (3.7 vs 2.07 ms per BFS at one rank; ncu:
// identical instruction, L1/L2 and DRAM counts, the difference is warps waiting at the
// grid barrier after stage 1), so it is only used when BLEST_DENSE_MIN asks for it.
uint64_t rows_dense_min() {
    if (const char* d = getenv("BLEST_DENSE_MIN")) return (uint64_t)atoll(d);
    return ~0ull;
}

Geometry rows_geometry(bool stepped, int threads) {
    Geometry g;
    g.threads = threads;
    g.kern = stepped ? rows_kernel<0, true>(threads) : rows_kernel<0, false>(threads);
    CK(cudaFuncSetAttribute(g.kern, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, g.kern, threads, 0));
    if (per_sm < 1) throw CudaError("rows kernel cannot be resident");
    g.ctas = (uint32_t)per_sm * (uint32_t)num_sms();
    return g;
}
}  // namespace

void rows_launch(RowsEngine& e, const RowsParams& hp, bool fused) {
    const Geometry g = rows_geometry(!fused, 512);
    const uint32_t ctas = std::min<uint32_t>(g.ctas, kAggStride);
    RowsParams p = hp;
    p.dense_min = rows_dense_min();
    RowsLaunch L;
    std::memset(&L, 0, sizeof(L));
    L.r[0] = p;
    uint32_t cpr = ctas;
    void* args[] = {&L, &cpr};
    CK(cudaLaunchCooperativeKernel(g.kern, dim3(ctas), dim3(g.threads), args, 0, stream()));
    g_launches.fetch_add(1);
    e.ctas_ = ctas;
}

void RowsEngine::launch_fused(uint32_t src) {
    if (src >= b_.n) throw InvalidArgument("bfs source out of range");
    RowsParams p;
    fill_params(p, src, 1, nullptr);
    rows_launch(*this, p, true);
}

void RowsEngine::step(uint32_t level, uint32_t src, const uint32_t* recv) {
    if (src >= b_.n) throw InvalidArgument("bfs source out of range");
    if (level == 0) throw InvalidArgument("levels start at 1");
    if (level > 1 && !recv) throw InvalidArgument("level > 1 needs the gathered frontier");
    if (level == 1) {
        hflags_[0] = 0;
        hflags_[1] = 0;
        hflags_[2] = 0;
    }
    RowsParams p;
    fill_params(p, src, level, recv);
    rows_launch(*this, p, false);
}

void rows_group_launch(const std::vector<RowsEngine*>& ranks, uint32_t src) {
    const uint32_t G = (uint32_t)ranks.size();
    if (!G) throw InvalidArgument("empty rank group");
    if (G > kMaxLaunchRanks) throw InvalidArgument("at most 12 virtual ranks per launch");
    for (uint32_t r = 0; r < G; ++r)
        if (ranks[r]->rank_ != r || ranks[r]->world_ != G) throw InvalidArgument("rank group out of order");
    if (src >= ranks[0]->b_.n) throw InvalidArgument("bfs source out of range");
    const Geometry g = rows_geometry(false, 512);
    const uint32_t cpr = std::min<uint32_t>(g.ctas / G, kAggStride);
    if (cpr < 1) throw InvalidArgument("more virtual ranks than co-resident CTAs");
    std::vector<RowsParams> hp(G);
    // one grid: every rank must run the same barrier sequence, so the hot-row view (an
    // extra barrier per level) is used only if every rank has it
    bool all_sigma = true;
    for (uint32_t r = 0; r < G; ++r) all_sigma = all_sigma && ranks[r]->sigma_built_;
    for (uint32_t r = 0; r < G; ++r) {
        ranks[r]->fill_params(hp[r], src, 1, nullptr, all_sigma);
        hp[r].dense_min = rows_dense_min();
        ranks[r]->ctas_ = cpr;
    }
    RowsLaunch L;
    std::memset(&L, 0, sizeof(L));
    for (uint32_t r = 0; r < G; ++r) L.r[r] = hp[r];
    uint32_t c = cpr;
    void* args[] = {&L, &c};
    CK(cudaLaunchCooperativeKernel(g.kern, dim3(cpr * G), dim3(g.threads), args, 0, stream()));
    g_launches.fetch_add(1);
}

std::vector<uint64_t> RowsEngine::phase_times(uint32_t cap) {
    unsigned long long it = 0;
    CK(cudaMemcpy(&it, ctl_.p + kIters, 8, cudaMemcpyDeviceToHost));
    const uint32_t rows = (uint32_t)std::min<uint64_t>({it, (uint64_t)cap, (uint64_t)trace_cap_});
    std::vector<uint64_t> out(4ull * rows);
    if (rows) CK(cudaMemcpy(out.data(), tstamp_.p, out.size() * 8, cudaMemcpyDeviceToHost));
    return out;
}

RowsEngine::Stats RowsEngine::finish(uint32_t* levels_owned_host) {
    cudaStream_t st = stream();
    unsigned long long c[kCtl];
    CK(cudaMemcpyAsync(c, ctl_.p, sizeof(c), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    Stats s;
    s.iterations = (uint32_t)c[kIters];
    s.unpulled = c[kUnpulled];
    if (c[kStatus] == 1) throw RuntimeError("BFS ran past the level safety cap — engine invariant broken");
    if (c[kStatus] == 2) throw RuntimeError("rows engine: cross-rank barrier timed out (a peer is not running)");
    const uint32_t rows = std::min(s.iterations, trace_cap_);
    std::vector<unsigned long long> t(8ull * std::max<uint32_t>(rows, 1));
    if (rows) CK(cudaMemcpy(t.data(), trace_.p, 8ull * rows * 8, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < rows; ++i) {
        s.queue += t[8ull * i + 1];
        s.discovered += t[8ull * i + 3];
        s.relaxed += t[8ull * i + 6];
        s.pushes += t[8ull * i + 7];
        if (t[8ull * i + 3]) s.max_level = i + 1;
    }
    if (levels_owned_host && row_hi_ > row_lo_)
        CK(cudaMemcpy(levels_owned_host, L_.p + row_lo_, (size_t)(row_hi_ - row_lo_) * 4, cudaMemcpyDeviceToHost));
    return s;
}

}  // namespace blestgpu
