// Frequency-ranked row space for the lazy engine's visited bitmaps (a B200 layout choice;
// the reference tests V_curr/V_next by plain row id, R:src/bfs_engine.cpp:286-289).
//
// Stage 1 is bound by its visited tests: one random 4-byte load per candidate row into a
// 2 MB bitmap (C2), served from L1 or L2. The tests concentrate on few rows — on Kron-20
// (Jaccard order) the 10 % most frequent rows take 86 % of them — but those rows are
// scattered over the id space, so every hot bit drags a 128 B L1 line of cold neighbours.
// σ ranks the rows by their BVSS slot count (most frequent first, ties by id): in σ space
// the hot rows' bits are contiguous, the hottest ~2 M of them in the first ~256 KB — what
// one SM's L1 holds. The lazy kernel keeps V_curr / V_next in σ space and reads an engine
// copy of row_ids holding σ(row); stage 2 maps each discovery back (σ⁻¹) to store its
// level and set its bit in the original-space frontier bitmap (α of the slice sets, the
// next queue).
//
// The canonical BVSS arrays are untouched (API, parity, eager engine).
#pragma once

#include "bvss.cuh"

namespace blestgpu {

struct SigmaView {
    DevBuf<uint32_t> rows;  // engine row_ids: σ(row); padding slots keep row n
    DevBuf<uint32_t> sig;   // row -> σ(row)
    DevBuf<uint32_t> inv;   // σ -> row
};

void sigma_view_build(const DeviceBvss& b, SigmaView& out);

}  // namespace blestgpu
