// Host file formats of the reference (io.cu): BVSS binary cache, permutation files, graph
// files, and the graph digest that keys the cache.
#pragma once

#include <string>
#include <vector>

#include "bvss.cuh"
#include "graph.cuh"

namespace blestgpu {

// ParseError (R:include/blest/graph.hpp:23-32): a runtime_error carrying the line number.
struct ParseError : RuntimeError {
    size_t line;
    explicit ParseError(const std::string& what, size_t l = 0)
        : RuntimeError(l ? what + " (line " + std::to_string(l) + ")" : what), line(l) {}
};

// save_bvss / load_bvss (R:src/bvss.cpp:250-295), 'BVSS' v1.
void bvss_save(const DeviceBvss& b, const std::string& path);
DeviceBvss bvss_load(const std::string& path);

// save_permutation / load_permutation (R:src/graph.cpp:396-417): forward maps in and out.
void permutation_save(const uint32_t* forward, uint32_t n, const std::string& path);
std::vector<uint32_t> permutation_load(const std::string& path);

// load_matrix_market / load_edge_list (R:src/graph.cpp:233-394), parsed to an arc list.
struct LoadedEdges {
    uint32_t n = 0;
    bool directed = true;
    std::vector<uint32_t> src, dst;
};
LoadedEdges load_matrix_market(const std::string& path);
LoadedEdges load_edge_list(const std::string& path);

// Graph::digest (R:src/graph.cpp:62-75).
uint64_t graph_digest(const DeviceGraph& g);

// reference_bfs (R:src/graph.cpp:144-167) on the device: level-synchronous top-down BFS
// over the CSR out-view (no BVSS). levels_dev: n entries. Returns visited; *num_levels =
// max level + 1.
uint32_t graph_bfs_levels(const DeviceGraph& g, uint32_t src, uint32_t* levels_dev, uint32_t* num_levels);

// validate_roundtrip (R:src/bvss.cpp:143-188) on the device: decodes every slot, checks
// the padding rules, and compares the decoded arcs with g's incoming view row by row.
struct RoundtripCounts {
    uint64_t checked_slices = 0;
    uint64_t padded_nonzero = 0, real_zero_mask = 0, beyond_n = 0, rows_mismatched = 0;
    uint64_t first_padded_nonzero_vss = ~0ull, first_zero_mask_vss = ~0ull, first_beyond_set = ~0ull,
             first_mismatched_row = ~0ull;
};
RoundtripCounts bvss_validate_roundtrip(const DeviceBvss& b, const DeviceGraph& g);

}  // namespace blestgpu
