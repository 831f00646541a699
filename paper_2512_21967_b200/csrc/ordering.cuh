// Orderings for the BVSS builder (R:include/blest/ordering.hpp, R:src/ordering.cpp).
#pragma once

#include <string>
#include <vector>

#include "graph.cuh"

namespace blestgpu {

struct SocialReport {
    double top1_share = 0, top10_share = 0, power_law_slope = 0, power_law_fit_r2 = 0;
    bool is_social_like = false, heavy_tail = false, power_law = false;
};

// classify_social_like(g, DegreeSide::Out) (R:src/ordering.cpp:346-387); degree histogram
// from device out-degrees, floating-point steps in the reference's order (bit-exact).
SocialReport classify_social_like(const DeviceGraph& g);

// rcm (R:src/ordering.cpp:171-266) on the GPU (rcm.cu): identical permutation; plain BFSs
// as cooperative launches, the Cuthill-McKee order level by level (parent position,
// degree, id) with radix sorts instead of the sequential queue.
std::vector<uint32_t> rcm_forward(const DeviceGraph& g);

// jaccard_with_windows(g, sigma, w, nullptr) (R:src/ordering.cpp:139-166) on the GPU:
// one CTA per window, greedy argmax with ties to the smallest id and the reference's
// double-precision score, so the permutation is identical.
void jaccard_windows_forward(const DeviceGraph& g, uint32_t sigma, uint32_t w, uint32_t* forward_host);

// random_order(n, seed) (R:src/ordering.cpp:268-275) with the reference's Rng.
std::vector<uint32_t> random_order_forward(uint32_t n, uint64_t seed);

// Rng(seed).next_below(n) draws (R:include/blest/rng.hpp:18-25, R:tools/blest.cpp:201-203).
std::vector<uint32_t> pick_sources(const DeviceGraph& g, uint32_t count, uint64_t seed, bool skip_isolated);

}  // namespace blestgpu
