// Row-partitioned multi-GPU BFS engine (the reference has no multi-GPU mode,
// PAPER.md:668 lists it as future work). Rank g of G owns destination rows
// [32·w_lo_g, 32·w_hi_g) — ranges balanced by BVSS slice count (partition_rows_by_slices) —
// and a BVSS of A[rows_g, all columns]; row ids stay global. One BFS per rank is the lazy
// algorithm (run_lazy, R:src/bfs_engine.cpp:238-350) split at the frontier:
//   stage 1  pull of the rank's local VSSs of the active column sets (lazy_pull.cuh);
//   stage 2a sweep of the owned V words: diff, V_curr, levels; the diff words are the
//            rank's share of the next frontier;
//   exchange every rank gets the whole n/8-byte frontier (each word has one writer, its
//            row owner, so no OR-reduction is needed — NCCL has none);
//   stage 2b every rank sweeps the whole frontier: termination (total discovered bits, the
//            same on every rank) and the next level's active sets with local VSSs (SL).
// Exchange modes:
//   fused (P2P) — one cooperative launch per BFS per rank; 2a stores its nonzero diff words
//            straight into every peer's frontier buffer (NVLink stores through CUDA IPC
//            mappings), then a cross-rank arrival barrier (system-scope release/acquire);
//            no host involvement between levels. G virtual ranks on one GPU run the same
//            kernel in ONE launch (CTA range per rank) — the test/bench stand-in for G GPUs.
//   stepped (NCCL) — one cooperative launch per level per rank: [unpack the gathered
//            frontier, 2b] stage 1, 2a → send buffer; the host enqueues ncclAllGather
//            (torch.distributed) on the same stream and the next level's launch without
//            waiting: termination is read from a mapped host flag the kernels set, the host
//            running at most `ahead` levels in front (extra launches are no-ops).
#pragma once

#include <vector>

#include "bvss.cuh"
#include "common.cuh"
#include "sigma.cuh"

namespace blestgpu {

struct RowsParams;

class RowsEngine {
public:
    // b: this rank's BVSS (bvss_build with the row range of word_bounds[rank] .. [rank+1]).
    RowsEngine(const DeviceBvss& b, uint32_t rank, uint32_t world, const std::vector<uint64_t>& word_bounds);
    ~RowsEngine();
    RowsEngine(const RowsEngine&) = delete;
    RowsEngine& operator=(const RowsEngine&) = delete;

    // CUDA IPC handle (64 bytes) of the exchange buffer (frontier words + arrival counter).
    void ipc_handle(void* out64) const;
    // Map every peer's exchange buffer (handles: world × 64 bytes, rank-major; own slot ignored).
    void open_peers(const void* handles);
    // Peers on this device (virtual ranks): siblings' buffers directly.
    void set_local_peers(const std::vector<RowsEngine*>& ranks);

    // fused: one BFS from src (global id), async on stream(); peers must run it too.
    void launch_fused(uint32_t src);
    // stepped: level 1 initialises from src; level > 1 reads recv (world × per words,
    // rank-major, the all-gather of every rank's send buffer). Async; no-op once done.
    void step(uint32_t level, uint32_t src, const uint32_t* recv);
    uint32_t* send_buffer() const { return send_.p; }
    uint64_t per_words() const { return per_; }
    // mapped host flags written by the kernels: [0] last level launched to completion,
    // [1] level at which the BFS terminated (0 = running), [2] status (0 ok, 1 runaway, 2 timeout)
    const volatile unsigned* host_flags() const { return hflags_; }

    // after the BFS: owned rows' levels (host, row_hi - row_lo entries), per-level trace sums
    struct Stats {
        uint32_t iterations = 0, max_level = 0;
        uint64_t queue = 0, discovered = 0, relaxed = 0, pushes = 0;
        uint64_t unpulled = 0;  // local VSSs of a barren last level not pulled (exhaustion exit)
    };
    Stats finish(uint32_t* levels_owned_host);
    // per level of the last BFS (rank 0's timeline in a group launch, %globaltimer ns):
    // start, stage-1 end, exchange end (fused), level end
    std::vector<uint64_t> phase_times(uint32_t cap);
    uint32_t row_lo() const { return row_lo_; }
    uint32_t row_hi() const { return row_hi_; }
    uint32_t rank() const { return rank_; }
    uint32_t world() const { return world_; }
    const DeviceBvss& bvss() const { return b_; }
    // exhaustion exit: global bitmap of the rows present in the whole BVSS (device, n bits,
    // owned by the caller) and their count (graph_present_rows); unset = off
    void set_present(const uint32_t* bits, uint64_t count) { present_ = bits; present_rows_ = count; }
    // device copy of this rank's kernel parameters (group launch)
    void fill_params(RowsParams& p, uint32_t src, uint32_t level, const uint32_t* recv, bool allow_sigma = true) const;

private:
    const DeviceBvss& b_;
    const uint32_t* present_ = nullptr;
    uint64_t present_rows_ = 0;
    uint32_t rank_, world_;
    uint32_t row_lo_, row_hi_;
    uint64_t words_, w_lo_, w_hi_, per_, xstride_;
    std::vector<uint64_t> bounds_;
    DevBuf<uint64_t> dbounds_;
    DevBuf<uint32_t> L_, V_;             // levels (global size), V_curr | V_next ([hot prefix] + global words + sentinel)
    uint64_t vstride_ = 0;
    SigmaView sigma_;                    // hot-row view of the rank's rows (sigma.cuh)
    bool sigma_built_ = false;
    DevBuf<uint32_t> H_;                 // hot discoveries of the level, row-space words
    DevBuf<uint32_t> xbuf_;              // exchange: X0 | X1 (xstride each) | arrival counter
    DevBuf<uint32_t> send_;              // stepped: owned diff words (per)
    DevBuf<unsigned long long> q_, sl_, ctl_, agg_, trace_, tstamp_;
    DevBuf<uintptr_t> peers_;            // [world] peer exchange bases
    std::vector<void*> opened_;          // IPC mappings to close
    unsigned* hflags_ = nullptr;         // mapped host memory
    unsigned* hflags_dev_ = nullptr;
    uint32_t trace_cap_ = 0;
    uint32_t ctas_ = 0;
    friend void rows_group_launch(const std::vector<RowsEngine*>& ranks, uint32_t src);
    friend void rows_launch(RowsEngine& e, const RowsParams& p, bool fused);
};

// Virtual ranks: every engine on this device, one cooperative launch (CTA range per rank).
void rows_group_launch(const std::vector<RowsEngine*>& ranks, uint32_t src);

// Row ranges balanced by BVSS slice count: bounds[0..world] in frontier words (32 rows),
// bounds[0] = 0, bounds[world] = ⌈n/32⌉. slices_out (optional, host) gets each rank's count.
std::vector<uint64_t> partition_rows_by_slices(const DeviceGraph& g, uint32_t world, std::vector<uint64_t>* slices_out);
// Rows present in the BVSS of g (every vertex with an in-arc) as a bitmap (n bits) + count.
uint64_t graph_present_rows(const DeviceGraph& g, DevBuf<uint32_t>& bits);

}  // namespace blestgpu
