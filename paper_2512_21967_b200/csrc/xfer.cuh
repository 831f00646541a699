// Narrow level-array transfers for the batch path (BfsEngine::run_batch).
//
// A level array is n u32 words, but a BFS of a social or random graph ends after a handful
// of levels: C2 (Kron-24) copies 67 MB per source over PCIe for values below 16. The device
// packs each level as (level + 1) in 1 or 2 bytes (0 = unreached, so the host's widening
// is a plain zero-extend minus one: kInf = 0xFFFFFFFF falls out of 0 - 1), the narrow array
// crosses PCIe, and host threads widen it into the caller's u32 buffer while the next
// source runs. A source whose deepest level does not fit the width is copied as u32
// instead (and later sources of the batch move to the next width), so the caller's array
// is always the exact level array.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

namespace blestgpu {

// Bytes per packed buffer (2 per vertex at most), rounded to 16 so every buffer of a
// back-to-back pair keeps the pack kernel's 4 B / 8 B vector stores aligned (odd n).
inline uint64_t xfer_slot_bytes(uint64_t n) { return (2 * n + 15) & ~15ull; }

// levels (u32, n) -> out (width 1 or 2 bytes per vertex): (level + 1) truncated, 0 for kInf.
void pack_levels(const uint32_t* levels, uint64_t n, int width, void* out, cudaStream_t st);

// Host-side widening pool: a job widens n packed entries into u32 levels, split over the
// pool's threads (non-temporal 16 B stores; the buffer is the caller's output).
class WidenPool {
public:
    explicit WidenPool(int threads);
    ~WidenPool();
    WidenPool(const WidenPool&) = delete;
    WidenPool& operator=(const WidenPool&) = delete;

    struct Job {
        const void* in = nullptr;
        int width = 1;
        uint32_t* out = nullptr;
        uint64_t n = 0;
        int parts = 0;
        int left = 0;  // parts not finished (guarded by the pool mutex)
    };
    void submit(Job* job);  // job must outlive its wait()
    void wait(Job* job);
    int threads() const { return (int)workers_.size(); }

private:
    void run();
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_work_, cv_done_;
    std::deque<std::pair<Job*, int>> tasks_;
    bool stop_ = false;
};

// Widen entries [lo, hi) of a packed array (exposed for the CPU tests).
void widen_levels(const void* in, int width, uint32_t* out, uint64_t lo, uint64_t hi);

}  // namespace blestgpu
