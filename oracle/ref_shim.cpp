// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference implementation (/root/reference/proj),
// compiled from its own sources by oracle/Makefile into oracle/_ref/libblest_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs
// load it; it is the checker, never the thing measured as our product.
//
// Every entry point forwards to the reference symbol named in its comment.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <utility>
#include <vector>

#include "blest/bfs_engine.hpp"
#include "blest/bvss.hpp"
#include "blest/graph.hpp"
#include "blest/ordering.hpp"
#include "blest/rng.hpp"
#include "blest/tc_emu.hpp"
#include "generators.hpp"
#include "oracles.hpp"
#include "bvss_check.hpp"

using namespace blest;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::invalid_argument*>(&e)) return -1;
    if (dynamic_cast<const std::logic_error*>(&e)) return -3;
    if (dynamic_cast<const std::runtime_error*>(&e)) return -2;
    return -4;
}
}  // namespace

#define GUARD(...)                          \
    try {                                   \
        __VA_ARGS__;                        \
        return 0;                           \
    } catch (const std::exception& e) {     \
        return fail(e);                     \
    }

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- graph (R:src/graph.cpp) -------------------------------------------------
void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

// Graph::from_edges (R:src/graph.cpp:33-55)
int ref_graph_from_edges(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t k,
                         int directed, void** out) {
    GUARD({
        std::vector<std::pair<VertexId, VertexId>> e(k);
        for (uint64_t i = 0; i < k; ++i) e[i] = {src[i], dst[i]};
        *out = new Graph(Graph::from_edges(n, std::move(e), directed != 0));
    })
}

// Builds a reference Graph from a CSR out-view by replaying its arcs through from_edges.
int ref_graph_from_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt, int directed,
                       void** out) {
    GUARD({
        std::vector<std::pair<VertexId, VertexId>> e;
        e.reserve(off[n]);
        for (uint32_t u = 0; u < n; ++u)
            for (uint64_t i = off[u]; i < off[u + 1]; ++i) e.emplace_back(u, tgt[i]);
        *out = new Graph(Graph::from_edges(n, std::move(e), directed != 0));
    })
}

uint32_t ref_graph_n(const void* g) { return static_cast<const Graph*>(g)->num_vertices(); }
uint64_t ref_graph_m(const void* g) { return static_cast<const Graph*>(g)->num_edges(); }
uint64_t ref_graph_digest(const void* g) { return static_cast<const Graph*>(g)->digest(); }

// out_offsets()/out_targets() (R:include/blest/graph.hpp:63-66); in_* when incoming != 0
void ref_graph_csr(const void* gp, int incoming, uint64_t* off, uint32_t* tgt) {
    const Graph& g = *static_cast<const Graph*>(gp);
    const auto& o = incoming ? g.in_offsets() : g.out_offsets();
    const auto& t = incoming ? g.in_sources() : g.out_targets();
    std::memcpy(off, o.data(), o.size() * sizeof(uint64_t));
    if (!t.empty()) std::memcpy(tgt, t.data(), t.size() * sizeof(uint32_t));
}

// reference_bfs (R:src/graph.cpp:144-167)
int ref_reference_bfs(const void* g, uint32_t src, uint32_t* levels, uint32_t* visited,
                      uint32_t* num_levels) {
    GUARD({
        BfsResult r = reference_bfs(*static_cast<const Graph*>(g), src);
        std::copy(r.levels.begin(), r.levels.end(), levels);
        *visited = r.visited_count;
        *num_levels = r.num_levels;
    })
}

// testing::matrix_bfs_levels (R:tests/support/oracles.cpp:10-36)
int ref_matrix_bfs(const void* g, uint32_t src, uint32_t* levels) {
    GUARD({
        auto l = testing::matrix_bfs_levels(*static_cast<const Graph*>(g), src);
        std::copy(l.begin(), l.end(), levels);
    })
}

// apply_permutation (R:src/graph.cpp:126-134)
int ref_apply_permutation(const void* g, const uint32_t* forward, void** out) {
    GUARD({
        const Graph& gg = *static_cast<const Graph*>(g);
        std::vector<VertexId> f(forward, forward + gg.num_vertices());
        *out = new Graph(apply_permutation(gg, Permutation::from_forward(std::move(f))));
    })
}

// ---- corpus generators (R:tests/support/generators.cpp) ----------------------
// kind: 0 path,1 ring,2 star,3 tree,4 grid(a=rows,b=cols),5 gnp(a=n,p,seed,directed=b),
//       6 pa(a=n,b=attach,seed),7 rgg(a=n,p=radius,seed),8 planted(a=n,b=communities,
//       c=intra,d=global,seed),9 two_components(seed)
int ref_generate(int kind, uint32_t a, uint32_t b, uint32_t c, uint32_t d, double p,
                 uint64_t seed, void** out) {
    GUARD({
        Graph g;
        switch (kind) {
            case 0: g = testing::path_graph(a); break;
            case 1: g = testing::ring_graph(a); break;
            case 2: g = testing::star_graph(a); break;
            case 3: g = testing::binary_tree(a); break;
            case 4: g = testing::grid_graph(a, b); break;
            case 5: g = testing::gnp_graph(a, p, seed, b != 0); break;
            case 6: g = testing::preferential_attachment(a, b, seed); break;
            case 7: g = testing::random_geometric(a, p, seed); break;
            case 8: g = testing::planted_communities(a, b, c, d, seed); break;
            case 9: g = testing::two_components(seed); break;
            default: throw std::invalid_argument("unknown generator kind");
        }
        *out = new Graph(std::move(g));
    })
}

// testing::scrambled (R:tests/support/generators.cpp:160-162)
int ref_scrambled(const void* g, uint64_t seed, void** out) {
    GUARD({ *out = new Graph(testing::scrambled(*static_cast<const Graph*>(g), seed)); })
}

// ---- orderings (R:src/ordering.cpp) -------------------------------------------
int ref_rcm(const void* g, uint32_t* forward) {
    GUARD({
        Permutation p = rcm(*static_cast<const Graph*>(g));
        std::copy(p.forward_map().begin(), p.forward_map().end(), forward);
    })
}
int ref_jaccard_windows(const void* g, uint32_t sigma, uint32_t w, unsigned workers,
                        uint32_t* forward) {
    GUARD({
        Permutation p =
            jaccard_with_windows(*static_cast<const Graph*>(g), sigma, w, nullptr, workers);
        std::copy(p.forward_map().begin(), p.forward_map().end(), forward);
    })
}
int ref_naive_window_order(const void* g, uint32_t sigma, uint32_t w, uint32_t* forward) {
    GUARD({
        Permutation p = testing::naive_window_order(*static_cast<const Graph*>(g), sigma, w);
        std::copy(p.forward_map().begin(), p.forward_map().end(), forward);
    })
}
int ref_random_order(uint32_t n, uint64_t seed, uint32_t* forward) {
    GUARD({
        Permutation p = random_order(n, seed);
        std::copy(p.forward_map().begin(), p.forward_map().end(), forward);
    })
}
int ref_bfs_locality_prepass(const void* g, uint32_t* forward) {
    GUARD({
        Permutation p = bfs_locality_prepass(*static_cast<const Graph*>(g));
        std::copy(p.forward_map().begin(), p.forward_map().end(), forward);
    })
}
int ref_is_cuthill_mckee_order(const void* g, const uint32_t* order, uint32_t n) {
    return testing::is_cuthill_mckee_order(*static_cast<const Graph*>(g),
                                           std::vector<VertexId>(order, order + n))
               ? 1
               : 0;
}

// classify_social_like (R:src/ordering.cpp:346-387): out[0..3] = top1, top10, slope, r2
int ref_classify(const void* g, double* out, int* social) {
    GUARD({
        SocialLikeReport r = classify_social_like(*static_cast<const Graph*>(g));
        out[0] = r.top1_share;
        out[1] = r.top10_share;
        out[2] = r.power_law_slope;
        out[3] = r.power_law_fit_r2;
        *social = r.is_social_like ? 1 : 0;
    })
}

// ---- BVSS (R:src/bvss.cpp) -----------------------------------------------------
void ref_bvss_free(void* b) { delete static_cast<Bvss*>(b); }

// build_bvss (R:src/bvss.cpp:19-101)
int ref_build_bvss(const void* g, unsigned workers, void** out) {
    GUARD({ *out = new Bvss(build_bvss(*static_cast<const Graph*>(g), {}, workers)); })
}

// Bvss from raw arrays (public fields, R:include/blest/bvss.hpp:34-50).
int ref_bvss_from_arrays(uint32_t n, uint64_t m, uint32_t num_vss, const uint32_t* real_ptrs,
                         const uint32_t* v2r, const uint32_t* row_ids, const uint32_t* masks,
                         void** out) {
    GUARD({
        auto* b = new Bvss();
        b->n = n;
        b->m = m;
        b->num_slice_sets = static_cast<uint32_t>((uint64_t(n) + 7) / 8);
        b->num_vss = num_vss;
        b->real_ptrs.assign(real_ptrs, real_ptrs + b->num_slice_sets + 1);
        b->virtual_to_real.assign(v2r, v2r + num_vss);
        b->row_ids.assign(row_ids, row_ids + uint64_t(num_vss) * 128);
        b->masks.assign(masks, masks + uint64_t(num_vss) * 32);
        for (uint32_t r : b->row_ids)
            if (r != n) ++b->num_unpadded_slices;
        *out = b;
    })
}

// sizes[0..3] = num_slice_sets, num_vss, num_unpadded_slices, m
void ref_bvss_sizes(const void* bp, uint64_t* sizes) {
    const Bvss& b = *static_cast<const Bvss*>(bp);
    sizes[0] = b.num_slice_sets;
    sizes[1] = b.num_vss;
    sizes[2] = b.num_unpadded_slices;
    sizes[3] = b.m;
}
void ref_bvss_arrays(const void* bp, uint32_t* real_ptrs, uint32_t* v2r, uint32_t* row_ids,
                     uint32_t* masks) {
    const Bvss& b = *static_cast<const Bvss*>(bp);
    std::copy(b.real_ptrs.begin(), b.real_ptrs.end(), real_ptrs);
    std::copy(b.virtual_to_real.begin(), b.virtual_to_real.end(), v2r);
    std::copy(b.row_ids.begin(), b.row_ids.end(), row_ids);
    std::copy(b.masks.begin(), b.masks.end(), masks);
}
double ref_compression_ratio(const void* b) { return compression_ratio(*static_cast<const Bvss*>(b)); }
double ref_update_divergence(const void* b) { return update_divergence(*static_cast<const Bvss*>(b)); }

// testing::check_bvss_invariants (R:tests/support/bvss_check.cpp:8-87): returns #violations
int ref_check_bvss_invariants(const void* b, const void* g) {
    return static_cast<int>(
        testing::check_bvss_invariants(*static_cast<const Bvss*>(b), *static_cast<const Graph*>(g))
            .size());
}

// save_bvss / load_bvss (R:src/bvss.cpp:250-295)
int ref_save_bvss(const void* b, const char* path) {
    GUARD({ save_bvss(*static_cast<const Bvss*>(b), path); })
}
int ref_load_bvss(const char* path, void** out) {
    GUARD({ *out = new Bvss(load_bvss(path)); })
}

// save_permutation / load_permutation (R:src/graph.cpp:396-417): forward maps
int ref_save_permutation(const uint32_t* forward, uint32_t n, const char* path) {
    GUARD({ save_permutation(Permutation::from_forward(std::vector<VertexId>(forward, forward + n)), path); })
}
int ref_load_permutation(const char* path, uint32_t* forward, uint32_t cap, uint32_t* n) {
    GUARD({
        const Permutation p = load_permutation(path);
        *n = p.size();
        for (uint32_t i = 0; i < p.size() && i < cap; ++i) forward[i] = p.forward(i);
    })
}

// load_graph (R:src/graph.cpp:390-394)
int ref_load_graph(const char* path, void** out) {
    GUARD({ *out = new Graph(load_graph(path)); })
}

// validate_roundtrip (R:src/bvss.cpp:143-188): number of discrepancies
int ref_validate_roundtrip(const void* b, const void* g, uint64_t* checked) {
    try {
        const RoundtripReport r = validate_roundtrip(*static_cast<const Bvss*>(b), *static_cast<const Graph*>(g));
        *checked = r.checked_slices;
        return static_cast<int>(r.discrepancies.size());
    } catch (const std::exception& e) {
        return -fail(e) - 100;
    }
}

// ---- engines (R:src/bfs_engine.cpp) ---------------------------------------------
// trace_out rows (8 u64 per level): level, queue_size, frontier_population, discovered,
// full_atomics, stage1_full_atomics, relaxed_atomics, queue_pushes.
// counters_out: mma_calls, full_atomics, relaxed_atomics, queue_pushes, vss_dequeues,
// brs_baseline_mma_calls, levels_processed, visited_count, num_levels, trace_len.
int ref_run_engine(const void* bp, uint32_t src, int lazy, unsigned warps, unsigned workers,
                   uint32_t max_levels, uint32_t* levels, uint64_t* counters_out,
                   uint64_t* trace_out, uint64_t trace_cap, uint64_t* per_warp_max_spread) {
    GUARD({
        const Bvss& b = *static_cast<const Bvss*>(bp);
        EngineConfig cfg;
        cfg.num_warps = warps;
        cfg.workers = workers;
        cfg.max_levels = max_levels;
        cfg.mode = lazy ? EngineMode::Lazy : EngineMode::Eager;
        auto [r, c] = lazy ? run_lazy(b, src, cfg) : run_eager(b, src, cfg);
        if (levels) std::copy(r.levels.begin(), r.levels.end(), levels);
        counters_out[0] = c.mma_calls;
        counters_out[1] = c.full_atomics;
        counters_out[2] = c.relaxed_atomics;
        counters_out[3] = c.queue_pushes;
        counters_out[4] = c.vss_dequeues;
        counters_out[5] = c.brs_baseline_mma_calls;
        counters_out[6] = c.levels_processed;
        counters_out[7] = r.visited_count;
        counters_out[8] = r.num_levels;
        counters_out[9] = c.trace.size();
        uint64_t spread = 0;
        for (std::size_t i = 0; i < c.trace.size(); ++i) {
            const LevelTrace& t = c.trace[i];
            if (i < trace_cap && trace_out) {
                uint64_t* row = trace_out + 8 * i;
                row[0] = t.level;
                row[1] = t.queue_size;
                row[2] = t.frontier_population;
                row[3] = t.discovered;
                row[4] = t.full_atomics;
                row[5] = t.stage1_full_atomics;
                row[6] = t.relaxed_atomics;
                row[7] = t.queue_pushes;
            }
            if (!t.per_warp_mma.empty()) {
                auto [lo, hi] = std::minmax_element(t.per_warp_mma.begin(), t.per_warp_mma.end());
                spread = std::max<uint64_t>(spread, *hi - *lo);
            }
        }
        if (per_warp_max_spread) *per_warp_max_spread = spread;
    })
}

// init_state (R:src/bfs_engine.cpp:30-49): returns q_curr length, writes q (cap entries)
int ref_init_state_queue(const void* bp, uint32_t src, uint32_t* q, uint32_t cap, uint32_t* len) {
    GUARD({
        FrontierState st = init_state(*static_cast<const Bvss*>(bp), src, EngineMode::Eager);
        *len = static_cast<uint32_t>(st.q_curr.size());
        for (uint32_t i = 0; i < st.q_curr.size() && i < cap; ++i) q[i] = st.q_curr[i];
    })
}

// ---- tile emulator (R:src/tc_emu.cpp) ---------------------------------------------
// One pull round of a VSS: mask words (32) + alpha + round -> 64 popcounts of FragC.
int ref_tile_pull(const uint32_t* mask_words, uint8_t alpha, unsigned round, uint32_t* c64) {
    GUARD({
        std::array<uint32_t, 32> m{};
        std::copy(mask_words, mask_words + 32, m.begin());
        tc::FragA a = tc::pack_fragA_round(m, round);
        tc::FragC c = tc::mma_m8n8k128(a, tc::build_fragB(alpha));
        std::copy(c.counts.begin(), c.counts.end(), c64);
    })
}

// Rng::next_below stream (R:include/blest/rng.hpp:18-25), as the CLI samples sources.
void ref_rng_next_below(uint64_t seed, uint64_t bound, uint64_t count, uint64_t* out) {
    Rng rng(seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = rng.next_below(bound);
}

}  // extern "C"
