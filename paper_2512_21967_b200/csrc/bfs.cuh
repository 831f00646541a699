// The fused persistent BFS engine (eager = Alg. 2, lazy = Alg. 3) over a DeviceBvss.
// Reference: run_eager / run_lazy (R:src/bfs_engine.cpp:155-350), pull_vss (:131-146),
// init_state (:30-49), counters (R:include/blest/bfs_engine.hpp:27-50).
#pragma once

#include <vector>
#include <cstdint>

#include "bvss.cuh"
#include "sigma.cuh"
#include "xfer.cuh"

#include <memory>

namespace blestgpu {

enum class Mode : int { Eager = 0, Lazy = 1 };
enum class Pull : int { Popc = 0, Mma = 1 };  // CUDA-core popcount vs b1 mma.sync tile

// Tile known-answer entry (tile.cu): `count` tiles, host arrays (blest_tile_pull).
void tile_pull_device(const uint32_t* masks, const uint8_t* alpha, uint32_t count, uint32_t* counts);

struct EngineOptions {
    Mode mode = Mode::Eager;
    Pull pull = Pull::Popc;
    uint32_t max_levels = 0;  // 0 = n + 1 (R:src/bfs_engine.cpp:68-70)
    uint32_t num_warps = 0;   // logical warps for the round-robin VSS split; 0 = whole grid
    uint32_t grid_ctas = 0;   // 0 = every co-resident CTA (persistent grid)
    uint32_t threads = 0;     // threads per CTA (256 / 512 / 1024); 0 = default
    bool sigma = true;        // lazy: hot-row view of the visited bitmaps (sigma.cuh)
    bool lazy_tma = false;    // lazy: TMA producer/consumer pipeline (measured slower on C2)
};

// One row per level, same fields as LevelTrace (R:include/blest/bfs_engine.hpp:27-37).
struct TraceRow {
    uint64_t level, queue_size, frontier_population, discovered, full_atomics,
        stage1_full_atomics, relaxed_atomics, queue_pushes;
};

struct BfsOutcome {
    uint32_t iterations = 0;  // trace length (includes the barren final level)
    uint32_t max_level = 0;   // levels_processed
    uint64_t visited = 0;
    bool trace_truncated = false;
    std::vector<TraceRow> trace;
    std::vector<uint64_t> phase_ns;  // per level: start, stage-1 end (lazy), level end
    // totals over the levels (run_batch fills these instead of `trace`)
    uint64_t sum_queue = 0, sum_full = 0, sum_relaxed = 0, sum_pushes = 0;
    // lazy: VSSs of a barren last level accounted without a pull (exhaustion exit), else 0
    uint64_t unpulled_vss = 0;
};

// Per-structure device workspace; sized once, reused across sources.
class BfsEngine {
public:
    explicit BfsEngine(const DeviceBvss& b);
    ~BfsEngine();
    BfsEngine(const BfsEngine&) = delete;
    BfsEngine& operator=(const BfsEngine&) = delete;

    // Build what launches of `opt` need up front (lazy: the hot-row view) and return the
    // engine's device bytes (workspace + view), so a caller can time and size it apart
    // from the BFS itself.
    uint64_t prepare(const EngineOptions& opt);
    // Enqueue init + the fused level loop on stream() (no host sync). Throws on bad args.
    void launch(uint32_t src, const EngineOptions& opt);
    // Wait for the last launch, read back trace/counters, check status (throws
    // RuntimeError past the level cap). Copies levels to host when levels_host != null.
    BfsOutcome finish(uint32_t* levels_host);
    // BFS from each of `count` sources back to back, pipelined: source k's level array is
    // copied to levels_host + k·n (when non-null) on a copy stream while source k+1 runs
    // (two device level buffers) — narrowed to 1 or 2 bytes per vertex on the device and
    // widened back to u32 by host threads (xfer.cuh; BLEST_D2H_PACK=0: plain u32 copies);
    // each kernel's trace is folded on the device into a per-source summary. Returns
    // per-source outcomes without per-level rows (trace empty).
    std::vector<BfsOutcome> run_batch(const uint32_t* srcs, uint32_t count, const EngineOptions& opt,
                                      uint32_t* levels_host);
    // level array written by the last launch (run_batch alternates two buffers)
    const uint32_t* levels_device() const { return last_levels_ ? last_levels_ : levels_.p; }
    uint32_t trace_capacity() const { return trace_cap_; }
    uint32_t last_grid_ctas() const { return last_ctas_; }
    uint32_t last_threads() const { return last_threads_; }
    uint32_t last_src() const { return last_src_; }
    // VSSs of the last finished run's barren level accounted without a pull (lazy exhaustion exit)
    uint64_t last_unpulled() const { return last_unpulled_; }
    const DeviceBvss& bvss() const { return b_; }

private:
    void ensure_sigma();
    void ensure_xfer();
    void ensure_present();  // lazy exhaustion exit: BVSS row bitmap + count  // run_batch's narrow level transfers: device pack buffers, pinned ring, pool
    const DeviceBvss& b_;
    uint64_t words_ = 0, wstride_ = 0;
    uint32_t trace_cap_ = 0;
    DevBuf<uint32_t> levels_;
    DevBuf<uint32_t> levels2_;           // run_batch: second level buffer
    uint32_t* level_target_ = nullptr;   // launch(): level array written (null = levels_)
    const uint32_t* last_levels_ = nullptr;  // level array of the last launch
    DevBuf<uint32_t> bits_;              // 3 * words_
    DevBuf<unsigned long long> q_;       // 3 * max(num_vss, 1) entries
    DevBuf<unsigned long long> ctl_;     // qlen[4], result[4]
    DevBuf<unsigned long long> agg_;     // lazy stage-2 per-CTA VSS counts
    DevBuf<unsigned long long> aggS_;    // lazy stage-2 per-CTA slice-set counts
    DevBuf<unsigned long long> sl_;      // lazy queue: active slice sets
    SigmaView sigma_;                    // lazy: hot-row view, built on the first lazy launch
    DevBuf<uint32_t> vext_;              // lazy hot-row view: V_curr, V_next with the hot prefix
    bool sigma_built_ = false;
    bool sigma_on_ = false;              // view built and worth using (hot share, BLEST_SIGMA)
    DevBuf<unsigned> bar_;               // grid barrier [2]
    DevBuf<unsigned long long> trace_;   // trace_cap_ * 8
    DevBuf<unsigned long long> tstamp_;  // trace_cap_ * 3
    unsigned long long* pinned_ = nullptr;  // host mirror for ctl_ readback
    // run_batch narrow transfers (xfer.cuh): packed levels on the device (2 buffers of up to
    // 2 bytes per vertex), a pinned staging ring, per-slot max levels, host widening threads
    static constexpr int kStageRing = 3;
    DevBuf<uint8_t> dpack_;
    uint8_t* stage_ = nullptr;
    unsigned long long* stage_max_ = nullptr;
    std::unique_ptr<WidenPool> pool_;
    DevBuf<uint32_t> present_;  // rows present in the BVSS (original ids)
    uint64_t present_rows_ = 0;
    bool present_built_ = false;
    bool last_exhaust_ = false;   // the last launch had the exhaustion exit armed
    uint64_t last_unpulled_ = 0;
    uint32_t last_ctas_ = 0, last_threads_ = 0, last_src_ = 0;
    Mode last_mode_ = Mode::Eager;
    bool launched_ = false;
};

}  // namespace blestgpu
