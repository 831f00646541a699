// Device-resident BVSS (R:include/blest/bvss.hpp:34-63) and its GPU builder.
//
// HBM layout is the reference's, byte for byte (so a host blest::Bvss uploads as-is):
//   real_ptrs[num_sets+1]  u32   VSS range of each slice set
//   v2r[num_vss]           u32   slice set of each VSS
//   masks[num_vss*32]      u32   lane t's word packs its 4 column masks (column c = byte c)
//   row_ids[num_vss*128]   u32   lane t's 4 row ids contiguous at 4*(32v+t)+c (one 16 B load)
// One VSS = one 128 B mask line + four 128 B row-id lines; a warp reads both coalesced.
// All slot arithmetic is 64-bit (the reference's u32 row_id() index wraps at 2^25 VSS).
#pragma once

#include "common.cuh"
#include "graph.cuh"

namespace blestgpu {

struct DeviceBvss {
    uint32_t n = 0;
    uint64_t m = 0;
    uint32_t num_sets = 0;
    uint32_t num_vss = 0;
    uint64_t num_unpadded = 0;
    uint32_t row_lo = 0, row_hi = 0xFFFFFFFFu;  // rows packed (multi-GPU partition), else all
    DevBuf<uint32_t> real_ptrs;
    DevBuf<uint32_t> v2r;
    DevBuf<uint32_t> masks;
    DevBuf<uint32_t> row_ids;
};

// build_bvss (R:src/bvss.cpp:19-101) on the GPU from the (permuted) out-view. With a row
// range, only arcs into rows [row_lo, row_hi) are packed (the multi-GPU row partition:
// all n/8 column slice sets, this rank's destination rows; row ids stay global).
DeviceBvss bvss_build(const DeviceGraph& g, uint32_t row_lo = 0, uint32_t row_hi = 0xFFFFFFFFu);

// Upload a host structure (R:include/blest/bvss.hpp:34-50 public fields), validated.
DeviceBvss bvss_upload(uint32_t n, uint64_t m, uint32_t num_vss, const uint32_t* real_ptrs,
                       const uint32_t* v2r, const uint32_t* row_ids, const uint32_t* masks,
                       bool host_ptrs);

// update_divergence (R:src/bvss.cpp:109-141): per-VSS values on device with the
// reference's IEEE operation order, summed in VSS order on the host (bit-exact).
double bvss_update_divergence(const DeviceBvss& b);

// compression_ratio (R:src/bvss.cpp:103-107)
double bvss_compression_ratio(const DeviceBvss& b);

// bvss_stats histogram (R:src/bvss.cpp:190-216): per_vss_slice_histogram[k] for k in 0..128.
void bvss_slice_histogram(const DeviceBvss& b, uint64_t* hist129);

}  // namespace blestgpu
