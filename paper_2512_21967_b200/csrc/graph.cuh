// Device-resident graph (CSR out-view) and its construction on the GPU.
// Mirrors blest::Graph (R:include/blest/graph.hpp:38-79) for the hot path: the BVSS
// builder consumes the out-view (R:src/bvss.cpp:35-46, :71-88).
#pragma once

#include "common.cuh"

namespace blestgpu {

struct DeviceGraph {
    uint32_t n = 0;
    uint64_t m = 0;
    bool directed = true;
    DevBuf<uint64_t> off;  // n + 1
    DevBuf<uint32_t> tgt;  // m, sorted ascending per source, duplicate-free, no self-loops
};

// Graph::from_edges (R:src/graph.cpp:33-55) over an arc-key array (u << 32 | v) already in
// device memory. Consumes `keys` (k valid entries; capacity must allow 2k when undirected).
// Self-loops are dropped, duplicates removed, CSR built with sorted targets.
DeviceGraph graph_from_keys(uint32_t n, DevBuf<uint64_t>& keys, uint64_t k, bool directed);

// Host (or device) src/dst arrays -> DeviceGraph, with the reference's range check (:40-43).
DeviceGraph graph_from_edges(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t k,
                             bool directed, bool host_ptrs);

// Host (or device) CSR -> DeviceGraph (validated: monotone offsets, ids < n; rebuilt
// through graph_from_keys so targets are sorted/deduplicated as the reference stores them).
DeviceGraph graph_from_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt, bool directed,
                           bool host_ptrs);

// apply_permutation (R:src/graph.cpp:126-134): relabel u -> forward[u] and rebuild.
DeviceGraph graph_permute(const DeviceGraph& g, const uint32_t* forward_dev);

// Harness generators (definitions shared bit-for-bit with oracle/blest_oracle.c).
DeviceGraph graph_generate_rmat(uint32_t scale, uint64_t num_edges, uint64_t seed, uint32_t a,
                                uint32_t b, uint32_t c);
DeviceGraph graph_generate_urand(uint32_t n, uint64_t num_edges, uint64_t seed);
DeviceGraph graph_generate_grid(uint32_t rows, uint32_t cols);

// CUB radix sort of k u64 keys on bits [0, end_bit) (keys may be swapped with a new buffer).
void sort_keys_u64(DevBuf<uint64_t>& keys, uint64_t k, int end_bit);

// transpose (R:src/graph.cpp:136-142)
DeviceGraph graph_transpose(const DeviceGraph& g);

// Seeded relabel permutation: forward[i] = rank of (hash64(seed, i), i).
void relabel_permutation(uint32_t n, uint64_t seed, uint32_t* forward_dev);

// Out-degree array (uint32, n entries) on device.
void graph_out_degrees(const DeviceGraph& g, uint32_t* deg_dev);

__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t hash64(uint64_t seed, uint64_t i) { return mix64(mix64(seed) ^ i); }

}  // namespace blestgpu
