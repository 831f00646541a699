// Eager engine (BLEST Alg. 2; run_eager, R:src/bfs_engine.cpp:155-236) as one fused
// persistent cooperative kernel: init_state and every level in one launch, one grid
// barrier per level (it also broadcasts the next queue length).
//
// Work unit = one VSS handled by one warp (lane t: its mask word, one coalesced 128 B line
// per VSS, and its 4 row ids, one 16 B load; streaming loads). Warps take queue positions
// round-robin exactly like the reference (p ≡ warp mod #warps, :190), kBatch at a time.
// Queue entries are 64-bit: low = VSS id, high = slice set (saves virtual_to_real, :192);
// α is the set's byte of F_curr (frontier_byte :148-151), loaded beside the mask/row loads.
//
// Sink (:198-211): the reference's levels[u] test becomes "VIS | F_curr" — two plain
// 4-byte bitmap loads (2 × n/8 bytes, L1/L2-resident, unlike the 4n-byte level array):
// VIS holds every discovery up to level ℓ-2 (level ℓ-1's discoveries are F_curr, frozen;
// they are ORed into VIS during this level's pull with a RED per dequeued VSS — adding
// bits that F_curr already has, so concurrent readers' union never changes). A clear test elects the discoverer with
// one atomicOr into F_next (old bit clear), which stores levels[u] = ℓ; the first bit of
// a slice set in F_next this level (old byte zero, :204-205) pushes the set's VSS range. Pushes gather in a per-warp shared
// buffer; a flush reserves queue space with ONE atomicAdd per buffer (warp-aggregated
// reservation) and expands [real_ptrs[s], real_ptrs[s+1]).
//
// Frontier bitmaps are triple-buffered: level ℓ reads F[ℓ%3], ORs into F[(ℓ+1)%3], and
// zeroes the bytes of F[(ℓ+2)%3] that level ℓ-1 read (set ids fetched from queue ℓ-1 at
// the level's start, stores issued after the pull), so no Θ(n) clear is ever needed
// (the reference clears every word, :227-228) and nothing sits on the level's critical path.
#include <atomic>

#include "bfs.cuh"
#include "bfs_device.cuh"

namespace blestgpu {

namespace {
using namespace bfsdev;

template <int PULL, int THREADS>
#ifndef BLEST_EAGER_MINB
#define BLEST_EAGER_MINB 1
#endif
__global__ void __launch_bounds__(THREADS, BLEST_EAGER_MINB) k_bfs_eager(Params p) {
    constexpr int WPC = THREADS / 32;
    __shared__ Smem<THREADS, 0> sm;
    const unsigned lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t gtid = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    const uint64_t gthreads = (uint64_t)gridDim.x * THREADS;
    const uint32_t gw = blockIdx.x * WPC + warp;
    const uint32_t all_warps = gridDim.x * WPC;
    const uint32_t NW = (p.num_warps && p.num_warps < all_warps) ? p.num_warps : all_warps;
    unsigned gen = 0;
    const uint64_t pol = evict_first_policy();
    if (threadIdx.x < 4) sm.ctr[threadIdx.x] = 0;
    uint32_t* VIS = p.B3;

    // ---- init_state (R:src/bfs_engine.cpp:30-49), fused ----
    const uint32_t src = p.src;
    const uint32_t sset = src / kSigma;
    const uint32_t seed_b = p.rp[sset], seed_e = p.rp[sset + 1];
    for (uint64_t i = gtid; i < p.n; i += gthreads) p.L[i] = (i == src) ? 0u : kInf;
    const uint32_t src_word = src >> 5, src_bit = 1u << (src & 31);
    for (uint64_t w = gtid; w < p.words; w += gthreads) {
        const uint32_t seed = (w == src_word) ? src_bit : 0u;
        p.B0[w] = 0;
        p.B1[w] = seed;  // F[1] = F_curr of level 1
        p.B2[w] = 0;
        VIS[w] = 0;  // the source is in F_curr of level 1
    }
    {
        const unsigned long long aux = (unsigned long long)sset << 32;
        for (uint64_t i = gtid; i < seed_e - seed_b; i += gthreads) p.Q1[i] = aux | (seed_b + i);
    }
    if (gtid == 0) {
        p.ctl[0] = 0;
        p.ctl[1] = seed_e - seed_b;
        for (int i = 2; i < 8; ++i) p.ctl[i] = 0;
        for (int i = 0; i < 8; ++i) p.trace[i] = 0;
    }
    uint32_t next_len = grid_barrier_pay(p.bar, gen, &p.ctl[1]);

    unsigned long long* pbuf = sm.push[warp];
    uint32_t pcount = 0;
    uint32_t ctr[4] = {0, 0, 0, 0};  // discovered, full, relaxed, pushes
    unsigned long long prev_len = 0;  // length of queue ℓ-1 (its sets' F bytes get zeroed)
    uint32_t level = 1;
    for (;; ++level) {
        const unsigned long long len = next_len;
        if (len == 0) break;
        if (level > p.cap) {  // runaway (R:src/bfs_engine.cpp:72-75)
            if (gtid == 0) p.ctl[6] = 1;
            break;
        }
        if (gtid == 0) {
            p.ctl[(level + 2) & 3] = 0;
            if (level - 1 < p.trace_cap) {
                p.trace[8ull * (level - 1) + 0] = level;
                p.trace[8ull * (level - 1) + 1] = len;
                p.tstamp[3ull * (level - 1)] = globaltimer();
            } else {
                atomicAdd(&p.trace[8ull * (p.trace_cap - 1) + 1], len);
            }
            if (level < p.trace_cap)
                for (int i = 0; i < 8; ++i) p.trace[8ull * level + i] = 0;
        }
        // triple buffers by select (a runtime-indexed array would live in local memory)
        auto qsel = [&](uint32_t k) { return k == 0 ? p.Q0 : (k == 1 ? p.Q1 : p.Q2); };
        auto fsel = [&](uint32_t k) { return k == 0 ? p.B0 : (k == 1 ? p.B1 : p.B2); };
        const uint32_t k0 = level % 3, k1 = (level + 1) % 3, k2 = (level + 2) % 3;
        const unsigned long long* Qc = qsel(k0);
        unsigned long long* Qn = qsel(k1);
        const uint8_t* Fc8 = reinterpret_cast<const uint8_t*>(fsel(k0));
        uint32_t* Fn = fsel(k1);
        unsigned long long* qlen_next = &p.ctl[(level + 1) & 3];
        // Frontier bytes level ℓ-1 read (sets of queue ℓ-1) become F_next at ℓ+1: fetch this
        // thread's set id now, store the zero after the pull (latency hidden by the pull).
        uint8_t* Fz = reinterpret_cast<uint8_t*>(fsel(k2));
        const unsigned long long* Qz = qsel(k2);
        const uint32_t zss = (gtid < prev_len) ? (uint32_t)(Qz[gtid] >> 32) : 0xFFFFFFFFu;

        // ---- pull over the queue (pull_vss, R:src/bfs_engine.cpp:131-146) ----
        if (gw < NW) {
            unsigned long long e_next = kNoEntry;
            if (lane < kBatch && gw + (uint64_t)lane * NW < len) e_next = Qc[gw + (uint64_t)lane * NW];
            for (uint64_t p0 = gw; p0 < len; p0 += (uint64_t)NW * kBatch) {
                const unsigned long long e = e_next;
                e_next = kNoEntry;
                if (lane < kBatch) {
                    const uint64_t pos = p0 + (uint64_t)NW * kBatch + (uint64_t)lane * NW;
                    if (pos < len) e_next = Qc[pos];
                }
                const uint32_t alpha_l = (e != kNoEntry) ? Fc8[e >> 32] : 0u;  // frontier_byte
                if (e != kNoEntry) {  // fold level ℓ-1's discoveries of this set into VIS
                    const uint32_t ss = (uint32_t)(e >> 32);
                    red_or(VIS + (ss >> 2), alpha_l << (8 * (ss & 3)));
                }
                uint32_t mk[kBatch];
                uint4 rw[kBatch];
                unsigned long long ej[kBatch];
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    ej[j] = __shfl_sync(0xffffffffu, e, j);
                    mk[j] = 0;
                    rw[j] = make_uint4(0, 0, 0, 0);
                    if (ej[j] != kNoEntry) {
                        const uint64_t v = (uint32_t)ej[j];
                        mk[j] = ld_stream_u32(p.masks + 32 * v + lane, pol);
                        rw[j] = ld_stream_u4(p.rows4 + 32 * v + lane, pol);
                    }
                }
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    if (ej[j] == kNoEntry) continue;  // warp-uniform
                    const uint32_t alpha = __shfl_sync(0xffffffffu, alpha_l, j);
                    uint32_t cnt[4];
                    column_counts<PULL>(mk[j], alpha, cnt);
                    const uint32_t u[4] = {rw[j].x, rw[j].y, rw[j].z, rw[j].w};
                    uint32_t vw[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        vw[c] = cnt[c] ? (VIS[u[c] >> 5] | reinterpret_cast<const uint32_t*>(Fc8)[u[c] >> 5]) : ~0u;
                    // not visited before: already claimed this level? (F_next at L2; a stale
                    // miss only costs the atomic) — spares the returned atomic on dense levels
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (!((vw[c] >> (u[c] & 31)) & 1u) && ((ld_l2_u32(Fn + (u[c] >> 5)) >> (u[c] & 31)) & 1u))
                            vw[c] |= 1u << (u[c] & 31);
                    uint32_t old[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        old[c] = ((vw[c] >> (u[c] & 31)) & 1u) ? ~0u : atomicOr(Fn + (u[c] >> 5), 1u << (u[c] & 31));
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        bool push = false;
                        if (!((vw[c] >> (u[c] & 31)) & 1u)) {
                            ++ctr[1];
                            if (!((old[c] >> (u[c] & 31)) & 1u)) {  // this lane discovered u
                                p.L[u[c]] = level;
                                ++ctr[0];
                                push = ((old[c] >> (8 * ((u[c] >> 3) & 3))) & 0xFFu) == 0;
                            }
                        }
                        push_column(p, push, (unsigned long long)(u[c] >> 3) << 32 | (u[c] >> 3), pbuf, pcount,
                                    Qn, qlen_next, ctr[3], ctr[1]);
                    }
                }
            }
        }
        if (pcount) {
            const uint32_t t = flush_pushes(p, pbuf, pcount, Qn, qlen_next);
            if (lane == 0) {
                ctr[3] += t;
                ctr[1] += 1;
            }
        }
        if (zss != 0xFFFFFFFFu) Fz[zss] = 0;
        for (uint64_t i = gtid + gthreads; i < prev_len; i += gthreads) Fz[Qz[i] >> 32] = 0;
        prev_len = len;
        next_len = level_barrier(p, sm, gen, level, ctr, 2, qlen_next);
    }
    if (gtid == 0) p.ctl[4] = level - 1;
}

}  // namespace

void* eager_kernel(int pull, int threads) {
    if (pull == 1) {
        switch (threads) {
            case 256: return (void*)k_bfs_eager<1, 256>;
            case 512: return (void*)k_bfs_eager<1, 512>;
            case 1024: return (void*)k_bfs_eager<1, 1024>;
        }
    } else {
        switch (threads) {
            case 256: return (void*)k_bfs_eager<0, 256>;
            case 512: return (void*)k_bfs_eager<0, 512>;
            case 1024: return (void*)k_bfs_eager<0, 1024>;
        }
    }
    throw InvalidArgument("threads per CTA must be 256, 512 or 1024");
}

}  // namespace blestgpu
