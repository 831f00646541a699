// Hub view of a BVSS for the lazy engine's visited tests (B200 layout choice, no
// reference counterpart: the reference tests V_curr/V_next for every nonzero pull,
// R:src/bfs_engine.cpp:286-289).
//
// Stage 1's cost on social graphs is the visited test, a random 4-byte load per candidate
// row that mostly misses L1. The tests concentrate on few rows — on Kron-20 (Jaccard
// order) the 10% most frequent rows take 86% of them. The hub view renumbers the K most
// frequent rows (K = what a CTA's share of shared memory holds as a bitmap) as hubs, and an
// engine copy of row_ids names hub h by the virtual row id hub_base + h, hub_base = 32 ×
// the V_next stride: the hubs' V_next bits (HN) simply extend V_next, so re-checks and REDs
// treat hubs like rows, and on dense levels a snapshot of HN (= the hubs' V_curr) sits in
// every CTA's shared memory for the visited-before test. A hub's first discoverers also
// set its real row's V_next bit, so stage 2 is unchanged.
//
// The canonical BVSS arrays are untouched (API, parity, eager engine); the view is an
// extra copy of row_ids (4 B per slot) built once per structure on the first lazy BFS.
#pragma once

#include "bvss.cuh"

namespace blestgpu {

constexpr uint32_t kHubFlag = 0x80000000u;  // n must stay below (virtual hub ids follow)
constexpr uint32_t kNoHub = 0xFFFFFFFFu;

struct HubView {
    uint32_t K = 0;              // number of hubs
    uint32_t bits = 0;           // hub-space size: ceil(K / 1024) * 1024 (whole 128 B lines)
    DevBuf<uint32_t> rows;       // engine row_ids: hub_base + h for hubs, else the row id
    DevBuf<uint32_t> hub_rows;   // h -> row id
    DevBuf<uint32_t> hub_of;     // row id -> h or kNoHub (n + 1 entries, padding row n too)
};

// Hubs = the max_hubs rows with the most BVSS slots (ties: smaller id first). Requires
// n < 2^31 and hub_base >= n. Hub-space position of the q-th most frequent row: with NL =
// bits / 1024 lines of 32 words, line q mod NL, word (q mod NL + q / NL) mod 32, bit
// q / (32 NL) — consecutive hot hubs land in different 128 B lines (no hot L2 line for
// the REDs of a level that discovers the hubs) and in different shared-memory banks.
void hub_view_build(const DeviceBvss& b, uint32_t max_hubs, uint32_t hub_base, HubView& out);

}  // namespace blestgpu
