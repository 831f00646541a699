// Cluster engine: the eager algorithm (BLEST Alg. 2; run_eager, R:src/bfs_engine.cpp:155-236)
// run by ONE thread-block cluster (16 CTAs, one per SM), for high-diameter graphs whose
// levels are short (grids / meshes after RCM: C4 has ~8 K levels of <= 8 K VSSs). The grid
// engine pays a grid barrier (~1.2 µs + the queue-length read) and a global queue (tail
// atomic at L2, entry load at L2) on every level; here the level barrier is the hardware
// cluster barrier (barrier.cluster arrive.release / wait.acquire) and the queue lives in
// shared memory:
//   - the queue is one cluster-wide index space spread over the CTAs' shared memory:
//     position i of a queue lives in CTA i % C, slot i / C (ring lq[3][kLqCap], level ℓ
//     pulls lq[ℓ%3] and pushes into lq[(ℓ+1)%3]); a warp's flush reserves positions with
//     ONE atomic on CTA 0's counter through distributed shared memory and stores the
//     entries into their owners' slots (st.shared::cluster); positions past C·kLqCap go
//     to the global spill queue Q[(ℓ+1)%3] at index i - C·kLqCap (no second atomic);
//   - every CTA pulls its own slots (balanced by construction), the spill queue is shared
//     by all the cluster's warps; the next length is one DSMEM load after the barrier.
// Per VSS the pull, the visited test (VIS word, then atomicOr on F_next electing the
// discoverer), levels[u] = ℓ and the push of the set's VSS range are bfs_eager.cu's; the
// frontier bitmaps stay triple-buffered with the bytes of queue ℓ-1's sets zeroed during ℓ.
// init_state (R:src/bfs_engine.cpp:30-49) is a separate whole-GPU kernel (k_cluster_init)
// so the Θ(n) fills do not run on 16 SMs. Same outputs (levels, ctl, trace rows) as the
// grid engine.
#include <cooperative_groups.h>

#include "bfs.cuh"
#include "bfs_device.cuh"

namespace blestgpu {

namespace {
using namespace bfsdev;
namespace cg = cooperative_groups;

constexpr uint32_t kLqCap = 4096;  // local queue entries per ring slot (3 × 32 KB)

template <int THREADS>
struct ClusterSmem {
    unsigned long long lq[3][kLqCap];                  // set << 32 | VSS
    unsigned long long push[THREADS / 32][kPushCap];   // per-warp pushed sets
    unsigned long long ctr[2][4];                      // per level parity: discovered, full, relaxed, pushes
    uint32_t lqn[3];                                   // CTA 0: queue lengths (cluster-wide positions)
};

// Distributed shared memory (PTX mapa + shared::cluster accesses): `local` is this CTA's
// address of the variable; `rank` selects which CTA's copy.
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, uint32_t rank) {
    const uint32_t la = (uint32_t)__cvta_generic_to_shared(local);
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
    return ra;
}
__device__ __forceinline__ uint32_t dsmem_atomic_add(const uint32_t* local, uint32_t rank, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(dsmem_addr(local, rank)), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint32_t dsmem_load(const uint32_t* local, uint32_t rank) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(dsmem_addr(local, rank)) : "memory");
    return v;
}
__device__ __forceinline__ void dsmem_store(const unsigned long long* local, uint32_t rank, unsigned long long v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(dsmem_addr(local, rank)), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t row_of(const uint4 (&rw)[kBatch], int k) {
    const uint4& r = rw[k >> 2];
    return (k & 3) == 0 ? r.x : (k & 3) == 1 ? r.y : (k & 3) == 2 ? r.z : r.w;
}

__global__ void k_cluster_init(Params p) {
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gthreads = (uint64_t)gridDim.x * blockDim.x;
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
        p.B3[w] = seed;  // VIS
    }
    const unsigned long long aux = (unsigned long long)sset << 32;
    for (uint64_t i = gtid; i < seed_e - seed_b; i += gthreads) p.Q1[i] = aux | (seed_b + i);
    if (gtid == 0) {
        p.ctl[0] = 0;
        p.ctl[1] = seed_e - seed_b;  // level 1 = the source set's VSSs, in the spill queue
        for (int i = 2; i < 8; ++i) p.ctl[i] = 0;
        for (int i = 0; i < 8; ++i) p.trace[i] = 0;
    }
}

// Expand the warp's buffered sets into the next queue: ONE reservation (atomic on CTA 0's
// counter through DSMEM), entries stored into their owner CTAs' slots; positions past
// C·kLqCap go to the spill queue.
template <int THREADS>
__device__ __forceinline__ void flush_local(const Params& p, unsigned long long* buf, uint32_t& count,
                                            unsigned long long* lq_next, const uint32_t* q_count, uint32_t C,
                                            unsigned long long* Qspill, uint32_t (&ctr)[4]) {
    const unsigned lane = lane_id();
    uint32_t my_off[kPushCap / 32], my_b[kPushCap / 32], my_len[kPushCap / 32];
    uint32_t total = 0;
#pragma unroll
    for (int k = 0; k < kPushCap / 32; ++k) {
        const uint32_t i = k * 32 + lane;
        uint32_t b = 0, len = 0;
        if (i < count) {
            const uint32_t ss = (uint32_t)buf[i];
            b = p.rp[ss];
            len = p.rp[ss + 1] - b;
        }
        const uint32_t incl = warp_incl_scan(len);
        my_off[k] = total + incl - len;
        my_b[k] = b;
        my_len[k] = len;
        total += __shfl_sync(0xffffffffu, incl, 31);
    }
    uint32_t base = 0;
    if (lane == 0 && total) base = dsmem_atomic_add(q_count, 0, total);
    base = __shfl_sync(0xffffffffu, base, 0);
    const uint32_t local_cap = C * kLqCap;
    for (uint32_t i = 0; i < count; ++i) {
        const int k = i >> 5;
        const uint32_t src_lane = i & 31;
        uint32_t off = 0, b = 0, len = 0;
#pragma unroll
        for (int kk = 0; kk < kPushCap / 32; ++kk)
            if (kk == k) {
                off = __shfl_sync(0xffffffffu, my_off[kk], src_lane);
                b = __shfl_sync(0xffffffffu, my_b[kk], src_lane);
                len = __shfl_sync(0xffffffffu, my_len[kk], src_lane);
            }
        const unsigned long long aux = buf[i] & 0xFFFFFFFF00000000ull;
        for (uint32_t t = lane; t < len; t += 32) {
            const uint32_t pos = base + off + t;
            const unsigned long long e = aux | (unsigned long long)(b + t);
            if (pos < local_cap)
                dsmem_store(lq_next + pos / C, pos % C, e);
            else
                Qspill[pos - local_cap] = e;
            // the next level pulls these lines: start them towards L2 now
            const uint64_t v = b + t;
            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p.masks + 32 * v));
#pragma unroll
            for (int l = 0; l < 4; ++l) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p.rows4 + 32 * v + 8 * l));
        }
    }
    __syncwarp();
    count = 0;
    if (lane == 0) {
        ctr[3] += total;
        ctr[1] += 1;  // queue-size reservation (R:src/bfs_engine.cpp:206)
    }
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k_bfs_cluster(Params p) {
    constexpr int WPC = THREADS / 32;
    extern __shared__ __align__(16) unsigned char dsm[];
    ClusterSmem<THREADS>& sm = *reinterpret_cast<ClusterSmem<THREADS>*>(dsm);
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t C = cl.num_blocks();
    const uint32_t rank = cl.block_rank();
    const unsigned lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t cw = rank * WPC + warp, CW = C * WPC;
    const uint64_t pol = evict_first_policy();
    uint32_t* VIS = p.B3;
    if (threadIdx.x < 3) sm.lqn[threadIdx.x] = 0;
    if (threadIdx.x < 8) (&sm.ctr[0][0])[threadIdx.x] = 0;
    cl.sync();

    unsigned long long* pbuf = sm.push[warp];
    uint32_t pcount = 0;
    uint32_t ctr[4] = {0, 0, 0, 0};  // discovered, full, relaxed, pushes
    const uint32_t local_cap = C * kLqCap;
    uint32_t len_l = 0, prev_l = 0;  // this CTA's slots of queue ℓ / ℓ-1
    uint64_t len_g = p.ctl[1], prev_g = 0;  // spill queue ℓ / ℓ-1 (level 1: the source set)
    uint64_t total = len_g;         // queue ℓ over the cluster
    uint32_t level = 1;
    for (;; ++level) {
        if (total == 0) break;
        if (level > p.cap) {  // runaway (R:src/bfs_engine.cpp:72-75)
            if (rank == 0 && threadIdx.x == 0) p.ctl[6] = 1;
            break;
        }
        const uint32_t k0 = level % 3, k1 = (level + 1) % 3, k2 = (level + 2) % 3;
        if (threadIdx.x == 0) {
            if (rank == 0) {
                sm.lqn[k2] = 0;  // queue ℓ-1's length: becomes queue ℓ+2's (filled after the barrier)
                if (level - 1 < p.trace_cap) {
                    p.trace[8ull * (level - 1) + 0] = level;
                    p.trace[8ull * (level - 1) + 1] = total;
                    p.tstamp[3ull * (level - 1)] = globaltimer();
                } else {
                    atomicAdd(&p.trace[8ull * (p.trace_cap - 1) + 1], total);
                }
                if (level < p.trace_cap)
                    for (int i = 0; i < 8; ++i) p.trace[8ull * level + i] = 0;
            }
        }
        auto qsel = [&](uint32_t k) { return k == 0 ? p.Q0 : (k == 1 ? p.Q1 : p.Q2); };
        auto fsel = [&](uint32_t k) { return k == 0 ? p.B0 : (k == 1 ? p.B1 : p.B2); };
        const uint8_t* Fc8 = reinterpret_cast<const uint8_t*>(fsel(k0));
        uint32_t* Fn = fsel(k1);
        unsigned long long* Qspill = qsel(k1);
        unsigned long long* lq_next = sm.lq[k1];
        const uint32_t* q_count = &sm.lqn[k1];

        // ---- pull (pull_vss, R:src/bfs_engine.cpp:131-146) + sink (:198-211) ----
        auto pull = [&](const unsigned long long* Q, uint64_t len, uint32_t w0, uint32_t nw) {
            const uint64_t step = (uint64_t)nw * kBatch;
            for (uint64_t b0 = w0; b0 < len; b0 += step) {
                const uint64_t pos = b0 + (uint64_t)lane * nw;
                const unsigned long long e = (lane < kBatch && pos < len) ? Q[pos] : kNoEntry;
                const uint32_t alpha_l = (e != kNoEntry) ? Fc8[e >> 32] : 0u;  // frontier_byte
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
                const bool first = b0 == w0 && Q == sm.lq[k0];
                probe(p, level, 4096, mk[0] ^ rw[0].x ^ alpha_l, first);
                uint32_t vw[4 * kBatch];
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    const uint32_t a = ej[j] != kNoEntry ? __shfl_sync(0xffffffffu, alpha_l, j) : 0u;
                    const uint32_t m = mk[j] & (a * 0x01010101u);
#pragma unroll
                    for (int c = 0; c < 4; ++c) vw[4 * j + c] = cand_word(VIS, row_of(rw, 4 * j + c), m, 0xFFu << (8 * c));
                }
                probe(p, level, 8192, vw[0] ^ vw[1] ^ vw[2] ^ vw[3], first);
#pragma unroll
                for (int k = 0; k < 4 * kBatch; ++k) {
                    const uint32_t x = row_of(rw, k);
                    ctr[1] += ((vw[k] >> (x & 31)) & 1u) ^ 1u;  // full atomics (R:src/bfs_engine.cpp:203)
                    vw[k] = atom_if_clear(Fn, x, vw[k]);
                }
                probe(p, level, 16384, vw[0] ^ vw[1] ^ vw[2] ^ vw[3], first);
                uint32_t disc = 0;
#pragma unroll
                for (int k = 0; k < 4 * kBatch; ++k) {
                    const uint32_t x = row_of(rw, k);
                    if (!((vw[k] >> (x & 31)) & 1u)) {  // this lane discovered x
                        disc |= 1u << k;
                        p.L[x] = level;
                        red_or(VIS + (x >> 5), 1u << (x & 31));
                    }
                }
                ctr[0] += __popc(disc);
                if (__any_sync(0xffffffffu, disc != 0)) {
#pragma unroll
                    for (int k = 0; k < 4 * kBatch; ++k) {
                        const uint32_t x = row_of(rw, k);
                        const bool push = ((disc >> k) & 1u) && ((vw[k] >> (8 * ((x >> 3) & 3))) & 0xFFu) == 0;
                        const unsigned ball = __ballot_sync(0xffffffffu, push);
                        if (!ball) continue;
                        const uint32_t nk = __popc(ball);
                        if (pcount + nk > kPushCap)
                            flush_local<THREADS>(p, pbuf, pcount, lq_next, q_count, C, Qspill, ctr);
                        if (push) pbuf[pcount + __popc(ball & ((1u << lane) - 1))] = (unsigned long long)(x >> 3) << 32 | (x >> 3);
                        __syncwarp();
                        pcount += nk;
                    }
                }
            }
        };
        pull(sm.lq[k0], len_l, warp, WPC);
        pull(qsel(k0), len_g, cw, CW);
        if (pcount) flush_local<THREADS>(p, pbuf, pcount, lq_next, q_count, C, Qspill, ctr);
        probe(p, level, 32768, pcount, true);

        // F bytes queue ℓ-1 read become F_next at ℓ+1: zero them (local ring slot + spill)
        {
            uint8_t* Fz = reinterpret_cast<uint8_t*>(fsel(k2));
            const unsigned long long* lz = sm.lq[k2];
            for (uint32_t i = threadIdx.x; i < prev_l; i += THREADS) Fz[lz[i] >> 32] = 0;
            const unsigned long long* Qz = qsel(k2);
            for (uint64_t i = (uint64_t)rank * THREADS + threadIdx.x; i < prev_g; i += (uint64_t)C * THREADS)
                Fz[Qz[i] >> 32] = 0;
        }
        if ((p.xflags & 64) && threadIdx.x == 0 && level - 1 < p.trace_cap)  // timing study
            atomicMax(&p.tstamp[3ull * (level - 1) + 1], globaltimer());
        unsigned long long* sc = sm.ctr[level & 1];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t s = warp_sum(ctr[i]);
            if (lane == 0 && s) atomicAdd(&sc[i], (unsigned long long)s);
            ctr[i] = 0;
        }
        probe(p, level, 65536, ctr[0], true);
        cl.sync();  // level barrier (release/acquire at cluster scope)

        // queue ℓ+1: its length from CTA 0 (DSMEM); this CTA holds positions ≡ rank (mod C)
        prev_l = len_l;
        prev_g = len_g;
        uint32_t t32 = 0;
        if (lane == 0) t32 = dsmem_load(q_count, 0);
        total = __shfl_sync(0xffffffffu, t32, 0);
        const uint32_t m = min((uint32_t)total, local_cap);
        len_l = (m + C - 1 - rank) / C;
        len_g = total - m;
        if (threadIdx.x == 0) {
            const uint32_t row = min(level - 1, p.trace_cap - 1);
            unsigned long long* t = p.trace + 8ull * row;
            if (sc[0]) {
                atomicAdd(&t[3], sc[0]);
                atomicMax(&p.ctl[5], (unsigned long long)level);
            }
            if (sc[1]) atomicAdd(&t[4], sc[1]);
            if (sc[2]) atomicAdd(&t[6], sc[2]);
            if (sc[3]) atomicAdd(&t[7], sc[3]);
            for (int i = 0; i < 4; ++i) sc[i] = 0;
            if (rank == 0 && level - 1 < p.trace_cap) p.tstamp[3ull * (level - 1) + 2] = globaltimer();
        }
    }
    if (rank == 0 && threadIdx.x == 0) p.ctl[4] = level - 1;
    cl.sync();  // no CTA exits while a peer may still read its shared memory
}

}  // namespace

void* cluster_kernel(int threads) {
    switch (threads) {
        case 512: return (void*)k_bfs_cluster<512>;
        case 1024: return (void*)k_bfs_cluster<1024>;
    }
    throw InvalidArgument("cluster engine: threads per CTA must be 512 or 1024");
}

size_t cluster_smem(int threads) {
    return threads == 1024 ? sizeof(ClusterSmem<1024>) : sizeof(ClusterSmem<512>);
}

void cluster_init_launch(const Params& p, int ctas, cudaStream_t st) {
    k_cluster_init<<<ctas, 512, 0, st>>>(p);
}

}  // namespace blestgpu
