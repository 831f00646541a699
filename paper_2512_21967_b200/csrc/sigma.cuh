// Hot-row view for the lazy engine's visited bitmaps (a B200 layout choice; the reference
// tests V_curr/V_next by plain row id, R:src/bfs_engine.cpp:286-289).
//
// Stage 1 is bound by its visited tests: one random 4-byte load per candidate row into a
// 2 MB bitmap (C2), served from L1 or L2. The tests concentrate on few rows — on Kron-20
// (Jaccard order) the 10 % most frequent rows take 86 % of them — but those rows are
// scattered over the id space, so every hot bit drags a 128 B L1 line of cold neighbours.
// The view ranks the rows by BVSS slot count and gives the K most frequent (K ≈ 1 M: 128 KB
// of bits) engine ids 0..K-1 — a dense hot prefix of the visited bitmaps that L1 keeps —
// while every other row r keeps its place at engine id 32·hot_words + r. An engine copy
// of row_ids holds the engine ids. Stage 2 sweeps the hot prefix first (each discovery
// mapped back by σ⁻¹ to store its level and RED its bit into the original-space frontier
// Fd), then the row words exactly like the plain engine, merging Fd — so only hot
// discoveries (≤ K per BFS) pay a scattered update.
//
// The canonical BVSS arrays are untouched (API, parity, eager engine).
#pragma once

#include "bvss.cuh"

namespace blestgpu {

struct SigmaView {
    uint32_t K = 0;          // hot rows
    uint64_t hot_words = 0;  // hot prefix of the visited bitmaps, words (multiple of 4)
    DevBuf<uint32_t> rows;   // engine row_ids (hot rank, or 32·hot_words + row); padding kept
    DevBuf<uint32_t> sig;    // row -> engine id
    DevBuf<uint32_t> inv;    // hot rank -> row
    double hot_share = 0;    // share of the (non-padding) BVSS slots held by the K hot rows
};

// The view pays off when the hot rows take a large share of the visited tests (Kron-24:
// ~0.8 of the slots; C2 1.93 -> 1.55 ms); on graphs without hubs (urand-24: ~0.07) its hot
// pass is pure overhead (C3 2.56 -> 2.60 ms). Engines use it from this share up.
constexpr double kSigmaMinShare = 0.3;

// hot_cap: most hot rows (0 = default 2^20).
void sigma_view_build(const DeviceBvss& b, SigmaView& out, uint32_t hot_cap = 0);

}  // namespace blestgpu
