// blest_b200.hpp — C++ drop-in façade for the reference's hot-path API, over the C-ABI in
// blest_b200.h (libblest_b200.so). A program written against R:include/blest/{graph,bvss,
// ordering,bfs_engine}.hpp keeps its calls — same names, value types, arguments and
// exception classes — and runs graph build, reordering, BVSS construction and every BFS on
// the B200:
//
//   blest::Graph::from_edges      R:include/blest/graph.hpp:43-44    (GPU sort/unique/CSR)
//   blest::load_graph / transpose / reference_bfs / Graph::digest / in-views
//                                 R:include/blest/graph.hpp:54-71, :109, :119, :150
//   blest::save_bvss / load_bvss / validate_roundtrip / save_permutation / load_permutation
//                                 R:include/blest/bvss.hpp:80-111, R:src/graph.cpp:396-417
//   blest::apply_permutation      R:include/blest/graph.hpp:106
//   blest::classify_social_like / select_plan / make_permutation / rcm / jaccard_with_windows
//   / random_order                R:include/blest/ordering.hpp:44-81
//   blest::build_bvss             R:include/blest/bvss.hpp:65       (GPU builder)
//   blest::compression_ratio / update_divergence / bvss_stats       R:include/blest/bvss.hpp:68-97
//   blest::init_state / run_eager / run_lazy / run_auto_prebuilt / run_auto
//                                 R:include/blest/bfs_engine.hpp:63-101 (fused sm_100a kernel)
//
// Differences a caller can observe: EngineConfig::workers is accepted and ignored (the GPU
// grid replaces CPU workers), num_warps = 0 means "whole persistent grid", per-warp MMA
// counts are not recorded (LevelTrace::per_warp_mma stays empty), and Bvss additionally
// owns a device handle (its public host arrays are filled as in the reference).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <functional>
#include <thread>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "blest_b200.h"

namespace blest {

using VertexId = std::uint32_t;
using EdgeId = std::uint64_t;
using Level = std::uint32_t;
inline constexpr Level kUnreached = std::numeric_limits<Level>::max();

// ParseError (R:include/blest/graph.hpp:23-32)
class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& what, std::size_t line = 0)
        : std::runtime_error(what), line_(line) {}
    std::size_t line() const { return line_; }

private:
    std::size_t line_;
};

namespace detail {
inline std::size_t parse_line(const std::string& msg) {  // "... (line N)"
    const auto p = msg.rfind("(line ");
    return p == std::string::npos ? 0 : (std::size_t)std::stoull(msg.substr(p + 6));
}
inline void check(int rc) {
    if (rc == BLEST_OK) return;
    const std::string msg = blest_last_error();
    switch (rc) {
        case BLEST_EPARSE: throw ParseError(msg, parse_line(msg));
        case BLEST_EINVAL: throw std::invalid_argument(msg);
        case BLEST_ELOGIC: throw std::logic_error(msg);
        case BLEST_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}
struct GraphDel {
    void operator()(blest_graph_s* g) const { blest_graph_free(g); }
};
struct BvssDel {
    void operator()(blest_bvss_s* b) const { blest_bvss_free(b); }
};
}  // namespace detail

// ---- graph (R:include/blest/graph.hpp) -----------------------------------------------
class Graph {
public:
    Graph() = default;

    static Graph from_edges(VertexId n, std::vector<std::pair<VertexId, VertexId>> edges, bool directed = true) {
        std::vector<VertexId> s(edges.size()), d(edges.size());
        for (std::size_t i = 0; i < edges.size(); ++i) {
            s[i] = edges[i].first;
            d[i] = edges[i].second;
        }
        blest_graph h = nullptr;
        detail::check(blest_graph_from_edges(n, s.data(), d.data(), edges.size(), directed ? 1 : 0, 1, &h));
        return Graph(h);
    }

    VertexId num_vertices() const { return n_; }
    EdgeId num_edges() const { return m_; }
    bool directed() const { return directed_; }
    std::span<const VertexId> out_neighbors(VertexId u) const {
        return {out_targets_.data() + out_offsets_[u], out_targets_.data() + out_offsets_[u + 1]};
    }
    std::span<const VertexId> in_neighbors(VertexId v) const {
        return {in_sources_.data() + in_offsets_[v], in_sources_.data() + in_offsets_[v + 1]};
    }
    EdgeId out_degree(VertexId u) const { return out_offsets_[u + 1] - out_offsets_[u]; }
    EdgeId in_degree(VertexId v) const { return in_offsets_[v + 1] - in_offsets_[v]; }
    bool has_edge(VertexId u, VertexId v) const {
        const auto nb = out_neighbors(u);
        return std::binary_search(nb.begin(), nb.end(), v);
    }
    const std::vector<EdgeId>& out_offsets() const { return out_offsets_; }
    const std::vector<VertexId>& out_targets() const { return out_targets_; }
    const std::vector<EdgeId>& in_offsets() const { return in_offsets_; }
    const std::vector<VertexId>& in_sources() const { return in_sources_; }
    // FNV-1a over (n, m, arc list); keys the on-disk caches (R:src/graph.cpp:62-75).
    std::uint64_t digest() const {
        std::uint64_t d = 0;
        detail::check(blest_graph_digest(h_.get(), &d));
        return d;
    }
    blest_graph handle() const { return h_.get(); }

private:
    explicit Graph(blest_graph h) : h_(h, detail::GraphDel{}) {
        uint32_t n = 0;
        uint64_t m = 0;
        int dir = 1;
        detail::check(blest_graph_info(h, &n, &m, &dir));
        n_ = n;
        m_ = m;
        directed_ = dir != 0;
        out_offsets_.resize((std::size_t)n + 1);
        out_targets_.resize(m);
        detail::check(blest_graph_copy_csr(h, out_offsets_.data(), out_targets_.data()));
        in_offsets_.resize((std::size_t)n + 1);  // both views materialised, as the reference does
        in_sources_.resize(m);
        detail::check(blest_graph_copy_in_csr(h, in_offsets_.data(), in_sources_.data()));
    }
    friend Graph apply_permutation(const Graph&, const class Permutation&);
    friend Graph transpose(const Graph&);
    friend Graph load_graph(const std::string&);
    std::shared_ptr<blest_graph_s> h_;
    VertexId n_ = 0;
    EdgeId m_ = 0;
    bool directed_ = true;
    std::vector<EdgeId> out_offsets_{0};
    std::vector<VertexId> out_targets_;
    std::vector<EdgeId> in_offsets_{0};
    std::vector<VertexId> in_sources_;
};

class Permutation {
public:
    Permutation() = default;
    static Permutation identity(VertexId n) {
        std::vector<VertexId> f(n);
        for (VertexId i = 0; i < n; ++i) f[i] = i;
        return from_forward(std::move(f));
    }
    static Permutation from_forward(std::vector<VertexId> forward) {
        const auto n = static_cast<VertexId>(forward.size());
        std::vector<VertexId> inverse(n, n);
        for (VertexId i = 0; i < n; ++i) {
            if (forward[i] >= n || inverse[forward[i]] != n)
                throw std::invalid_argument("permutation is not a bijection on [0, n)");
            inverse[forward[i]] = i;
        }
        Permutation p;
        p.forward_ = std::move(forward);
        p.inverse_ = std::move(inverse);
        return p;
    }
    static Permutation from_inverse(std::vector<VertexId> inverse) { return from_forward(std::move(inverse)).inverted(); }
    VertexId size() const { return static_cast<VertexId>(forward_.size()); }
    VertexId forward(VertexId old_id) const { return forward_[old_id]; }
    VertexId inverse(VertexId new_id) const { return inverse_[new_id]; }
    const std::vector<VertexId>& forward_map() const { return forward_; }
    const std::vector<VertexId>& inverse_map() const { return inverse_; }
    Permutation inverted() const {
        Permutation p;
        p.forward_ = inverse_;
        p.inverse_ = forward_;
        return p;
    }
    static Permutation composed(const Permutation& first, const Permutation& second) {
        if (first.size() != second.size()) throw std::invalid_argument("cannot compose permutations of different sizes");
        std::vector<VertexId> f(first.size());
        for (VertexId i = 0; i < first.size(); ++i) f[i] = second.forward(first.forward(i));
        return from_forward(std::move(f));
    }
    bool is_identity() const {
        for (VertexId i = 0; i < size(); ++i)
            if (forward_[i] != i) return false;
        return true;
    }

private:
    std::vector<VertexId> forward_, inverse_;
};

// save_permutation / load_permutation (R:src/graph.cpp:396-417): one inverse id per line.
inline void save_permutation(const Permutation& p, const std::string& path) {
    detail::check(blest_permutation_save(p.forward_map().data(), p.size(), path.c_str()));
}

inline Permutation load_permutation(const std::string& path) {
    std::uint32_t n = 0;
    detail::check(blest_permutation_load(path.c_str(), nullptr, &n));
    std::vector<VertexId> f(n);
    detail::check(blest_permutation_load(path.c_str(), f.data(), &n));
    return Permutation::from_forward(std::move(f));
}

inline Graph apply_permutation(const Graph& g, const Permutation& perm) {
    if (perm.size() != g.num_vertices()) throw std::invalid_argument("permutation size does not match vertex count");
    blest_graph h = nullptr;
    detail::check(blest_graph_apply_permutation(g.handle(), perm.forward_map().data(), 1, &h));
    return Graph(h);
}

// transpose (R:include/blest/graph.hpp:109, R:src/graph.cpp:136-142), on the device.
inline Graph transpose(const Graph& g) {
    blest_graph h = nullptr;
    detail::check(blest_graph_transpose(g.handle(), &h));
    return Graph(h);
}

// load_graph (R:include/blest/graph.hpp:150): ".mtx" Matrix Market, else an edge list.
inline Graph load_graph(const std::string& path) {
    blest_graph h = nullptr;
    detail::check(blest_graph_load(path.c_str(), &h));
    return Graph(h);
}

struct BfsResult {
    VertexId source = 0;
    std::vector<Level> levels;
    VertexId visited_count = 0;
    Level num_levels = 0;
};

// reference_bfs (R:include/blest/graph.hpp:119): the ground truth the engines are checked
// against — here a top-down BFS straight over the CSR on the device (no BVSS).
inline BfsResult reference_bfs(const Graph& g, VertexId source) {
    BfsResult r;
    r.source = source;
    r.levels.resize(g.num_vertices());
    std::uint32_t vis = 0, nl = 0;
    detail::check(blest_graph_bfs(g.handle(), source, r.levels.data(), &vis, &nl));
    r.visited_count = vis;
    r.num_levels = nl;
    return r;
}


// ---- ordering (R:include/blest/ordering.hpp) ------------------------------------------
enum class OrderingStrategy { JaccardWindows, Rcm, Random, Identity };
enum class PrePass { None, BfsLocality };
enum class DegreeSide { Out, In, Total };

struct SocialLikeReport {
    double top1_share = 0, top10_share = 0, power_law_slope = 0, power_law_fit_r2 = 0;
    bool is_social_like = false;
    std::vector<std::string> triggered_rules;
};
struct OrderingPlan {
    OrderingStrategy strategy = OrderingStrategy::Identity;
    std::uint32_t window_size = 0;
    PrePass pre_pass = PrePass::None;
    SocialLikeReport classification;
};
struct SelectDefaults {
    std::uint32_t window_size = 1u << 16;
    PrePass pre_pass = PrePass::None;
    std::optional<OrderingStrategy> force;
};

inline SocialLikeReport classify_social_like(const Graph& g, DegreeSide side = DegreeSide::Out) {
    if (side != DegreeSide::Out) throw std::invalid_argument("only DegreeSide::Out is on the hot path");
    blest_social_report r{};
    detail::check(blest_classify_social_like(g.handle(), &r));
    SocialLikeReport out{r.top1_share, r.top10_share, r.power_law_slope, r.power_law_fit_r2, r.is_social_like != 0, {}};
    if (r.heavy_tail_fired) out.triggered_rules.emplace_back("heavy-tail");
    if (r.power_law_fired) out.triggered_rules.emplace_back("power-law");
    return out;
}

inline OrderingPlan select_plan(const Graph& g, std::uint32_t sigma, const SelectDefaults& defaults) {
    OrderingPlan plan;
    plan.classification = classify_social_like(g);
    plan.pre_pass = defaults.pre_pass;
    plan.strategy = defaults.force ? *defaults.force
                                   : (plan.classification.is_social_like ? OrderingStrategy::JaccardWindows
                                                                         : OrderingStrategy::Rcm);
    if (plan.strategy == OrderingStrategy::JaccardWindows) {
        plan.window_size = defaults.window_size;
        if (plan.window_size == 0 || plan.window_size % sigma != 0)
            throw std::invalid_argument("window size must be a positive multiple of sigma");
    }
    return plan;
}

inline Permutation rcm(const Graph& g) {
    std::vector<VertexId> f(g.num_vertices());
    detail::check(blest_order_rcm(g.handle(), f.data()));
    return Permutation::from_forward(std::move(f));
}

inline Permutation jaccard_with_windows(const Graph& g, std::uint32_t sigma, std::uint32_t w,
                                        const Permutation* pre_pass = nullptr, unsigned workers = 1) {
    (void)workers;
    if (pre_pass && !pre_pass->is_identity()) {
        const Graph h = apply_permutation(g, *pre_pass);
        return Permutation::composed(*pre_pass, jaccard_with_windows(h, sigma, w));
    }
    std::vector<VertexId> f(g.num_vertices());
    detail::check(blest_order_jaccard_windows(g.handle(), sigma, w, f.data()));
    return Permutation::from_forward(std::move(f));
}

inline Permutation random_order(VertexId n, std::uint64_t seed) {
    std::vector<VertexId> f(n);
    detail::check(blest_order_random(n, seed, f.data()));
    return Permutation::from_forward(std::move(f));
}

inline Permutation make_permutation(const Graph& g, const OrderingPlan& plan, std::uint32_t sigma,
                                    std::uint64_t seed = 0, unsigned workers = 1) {
    switch (plan.strategy) {
        case OrderingStrategy::Identity: return Permutation::identity(g.num_vertices());
        case OrderingStrategy::Random: return random_order(g.num_vertices(), seed);
        case OrderingStrategy::Rcm: return rcm(g);
        case OrderingStrategy::JaccardWindows:
            if (plan.pre_pass == PrePass::BfsLocality)
                throw std::invalid_argument("bfs-locality pre-pass is not on the GPU path");
            return jaccard_with_windows(g, sigma, plan.window_size, nullptr, workers);
    }
    throw std::logic_error("unhandled ordering strategy");
}

// ---- BVSS (R:include/blest/bvss.hpp) --------------------------------------------------
struct BvssConfig {
    std::uint32_t sigma = 8;
    std::uint32_t warp_size = 32;
    std::uint32_t slices_per_thread() const { return warp_size / sigma; }
    std::uint32_t tau() const { return warp_size * slices_per_thread(); }
    void validate() const {
        if (sigma != 8 || warp_size != 32)
            throw std::invalid_argument("unsupported tile geometry: sigma must be 8, warp size 32");
    }
};

class Bvss {
public:
    BvssConfig config;
    VertexId n = 0;
    EdgeId m = 0;
    std::uint32_t num_slice_sets = 0;
    std::uint32_t num_vss = 0;
    std::uint64_t num_unpadded_slices = 0;
    std::vector<std::uint32_t> real_ptrs, virtual_to_real, row_ids, masks;
    std::optional<Permutation> producing_permutation;
    std::string ordering_tag;

    VertexId sentinel() const { return n; }
    std::uint8_t slice_mask(std::uint32_t vss, unsigned lane, unsigned column) const {
        return static_cast<std::uint8_t>(masks[32ull * vss + lane] >> (8 * column));
    }
    std::uint32_t row_id(std::uint32_t vss, unsigned lane, unsigned column) const {
        return row_ids[4ull * (32ull * vss + lane) + column];  // 64-bit slot math
    }
    blest_bvss handle() const { return h_.get(); }

    // Adopt a device structure; fills the public host arrays unless host_mirror is false.
    static Bvss adopt(blest_bvss h, bool host_mirror = true) {
        Bvss b;
        b.h_.reset(h, detail::BvssDel{});
        blest_bvss_info info{};
        detail::check(blest_bvss_get_info(h, &info));
        b.n = info.n;
        b.m = info.m;
        b.num_slice_sets = info.num_slice_sets;
        b.num_vss = info.num_vss;
        b.num_unpadded_slices = info.num_unpadded_slices;
        if (host_mirror) {
            b.real_ptrs.resize((std::size_t)info.num_slice_sets + 1);
            b.virtual_to_real.resize(info.num_vss);
            b.row_ids.resize((std::size_t)info.num_vss * 128);
            b.masks.resize((std::size_t)info.num_vss * 32);
            detail::check(blest_bvss_download(h, b.real_ptrs.data(), b.virtual_to_real.data(), b.row_ids.data(),
                                              b.masks.data()));
        }
        return b;
    }

private:
    std::shared_ptr<blest_bvss_s> h_;
};

inline Bvss build_bvss(const Graph& g, const BvssConfig& cfg = {}, unsigned workers = 1) {
    (void)workers;
    cfg.validate();
    blest_bvss h = nullptr;
    detail::check(blest_bvss_build(g.handle(), &h));
    return Bvss::adopt(h);
}

// save_bvss / load_bvss (R:include/blest/bvss.hpp:106-111): the reference's 'BVSS' v1 file.
inline void save_bvss(const Bvss& b, const std::string& path) {
    detail::check(blest_bvss_save(b.handle(), path.c_str()));
}
inline Bvss load_bvss(const std::string& path) {
    blest_bvss h = nullptr;
    detail::check(blest_bvss_load(path.c_str(), &h));
    return Bvss::adopt(h);
}

// validate_roundtrip (R:include/blest/bvss.hpp:75-82), decoded and compared on the device;
// one discrepancy entry per violation class, naming its first offender and count.
struct RoundtripReport {
    std::uint64_t checked_slices = 0;
    std::vector<std::string> discrepancies;
    bool ok() const { return discrepancies.empty(); }
};
inline RoundtripReport validate_roundtrip(const Bvss& b, const Graph& g) {
    blest_roundtrip_report r{};
    detail::check(blest_bvss_validate_roundtrip(b.handle(), g.handle(), &r));
    RoundtripReport out;
    out.checked_slices = r.checked_slices;
    auto add = [&](std::uint64_t count, const char* what, std::uint64_t first) {
        if (count)
            out.discrepancies.push_back(std::string(what) + std::to_string(first) + " (" + std::to_string(count) +
                                        " in total)");
    };
    add(r.padded_nonzero_mask, "padded slot with nonzero mask at vss ", r.first_padded_nonzero_vss);
    add(r.real_zero_mask, "real slot with zero mask at vss ", r.first_zero_mask_vss);
    add(r.mask_bit_beyond_n, "mask bit beyond n at slice set ", r.first_beyond_set);
    add(r.rows_mismatched, "incoming list mismatch at row ", r.first_mismatched_row);
    return out;
}

inline double compression_ratio(const Bvss& b) {
    return b.num_unpadded_slices ? (double)b.m / ((double)b.num_unpadded_slices * b.config.sigma) : 0.0;
}

inline double update_divergence(const Bvss& b) {
    double d = 0;
    detail::check(blest_bvss_update_divergence(b.handle(), &d));
    return d;
}

struct BvssStats {
    double compression_ratio = 0, update_divergence = 0;
    std::uint32_t num_slice_sets = 0, num_vss = 0;
    std::uint64_t num_slices_padded = 0, num_unpadded_slices = 0, connectivity_bits = 0;
    std::map<std::uint32_t, std::uint32_t> per_vss_slice_histogram;
    std::uint64_t bytes_real_ptrs = 0, bytes_virtual_to_real = 0, bytes_row_ids = 0, bytes_masks = 0;
    std::uint64_t bytes_static() const { return bytes_real_ptrs + bytes_virtual_to_real + bytes_row_ids + bytes_masks; }
    std::uint64_t bytes_dynamic = 0, bytes_levels = 0;
};

inline BvssStats bvss_stats(const Bvss& b) {
    blest_bvss_stats_t s{};
    detail::check(blest_bvss_stats(b.handle(), &s));
    BvssStats out;
    out.compression_ratio = s.compression_ratio;
    out.update_divergence = s.update_divergence;
    out.num_slice_sets = s.num_slice_sets;
    out.num_vss = s.num_vss;
    out.num_slices_padded = s.num_slices_padded;
    out.num_unpadded_slices = s.num_unpadded_slices;
    out.connectivity_bits = s.connectivity_bits;
    for (int k = 0; k <= 128; ++k)
        if (s.per_vss_slice_histogram[k]) out.per_vss_slice_histogram[k] = (std::uint32_t)s.per_vss_slice_histogram[k];
    out.bytes_real_ptrs = s.bytes_real_ptrs;
    out.bytes_virtual_to_real = s.bytes_virtual_to_real;
    out.bytes_row_ids = s.bytes_row_ids;
    out.bytes_masks = s.bytes_masks;
    out.bytes_dynamic = s.bytes_dynamic;
    out.bytes_levels = s.bytes_levels;
    return out;
}

// ---- engines (R:include/blest/bfs_engine.hpp) ------------------------------------------
enum class EngineMode { Eager, Lazy, Auto };

inline std::string to_string(EngineMode m) {
    return m == EngineMode::Eager ? "eager" : (m == EngineMode::Lazy ? "lazy" : "auto");
}
inline EngineMode engine_mode_from_string(const std::string& s) {
    if (s == "eager") return EngineMode::Eager;
    if (s == "lazy") return EngineMode::Lazy;
    if (s == "auto") return EngineMode::Auto;
    throw std::invalid_argument("unknown engine mode: " + s);
}

struct EngineConfig {
    unsigned num_warps = 0;  // 0 = the whole persistent grid (reference default: 1 simulated warp)
    EngineMode mode = EngineMode::Auto;
    double lazy_divergence_threshold = 25000.0;
    Level max_levels = 0;
    unsigned workers = 1;  // accepted, unused: the GPU grid replaces CPU workers
    bool mma_tiles = false;  // b1 m8n8k128 mma.sync pull (ablation) instead of CUDA-core popcount
};

struct LevelTrace {
    Level level = 0;
    std::uint64_t queue_size = 0, frontier_population = 0, discovered = 0, full_atomics = 0,
                  stage1_full_atomics = 0, relaxed_atomics = 0, queue_pushes = 0;
    std::vector<std::uint64_t> per_warp_mma;  // not recorded on the GPU
};

struct EngineCounters {
    std::uint64_t mma_calls = 0, full_atomics = 0, relaxed_atomics = 0, queue_pushes = 0, vss_dequeues = 0,
                  brs_baseline_mma_calls = 0;
    Level levels_processed = 0;
    std::vector<std::vector<std::uint64_t>> per_warp_mma_calls;
    std::vector<LevelTrace> trace;
};

struct FrontierState {
    std::vector<std::uint32_t> f_curr, f_next, v_curr, v_next;
    std::vector<Level> levels;
    std::vector<std::uint32_t> q_curr, q_next;
    Level current_level = 0;
};

// init_state (R:src/bfs_engine.cpp:30-49): the state the fused kernel seeds on the device.
inline FrontierState init_state(const Bvss& b, VertexId src, EngineMode mode) {
    if (src >= b.n) throw std::invalid_argument("bfs source out of range");
    FrontierState st;
    const std::size_t words = ((std::size_t)b.n + 31) / 32;
    st.f_curr.assign(words, 0);
    st.f_next.assign(words, 0);
    st.levels.assign(b.n, kUnreached);
    st.levels[src] = 0;
    st.f_curr[src / 32] |= 1u << (src % 32);
    if (mode == EngineMode::Lazy) {
        st.v_curr = st.f_curr;
        st.v_next = st.f_curr;
    }
    for (std::uint32_t v = b.real_ptrs[src / 8]; v < b.real_ptrs[src / 8 + 1]; ++v) st.q_curr.push_back(v);
    return st;
}

namespace detail {
inline std::pair<BfsResult, EngineCounters> run(const Bvss& b, VertexId src, const EngineConfig& cfg, bool lazy) {
    blest_engine_config c{lazy ? BLEST_MODE_LAZY : BLEST_MODE_EAGER, cfg.mma_tiles ? BLEST_PULL_MMA : BLEST_PULL_POPC,
                          cfg.max_levels, cfg.num_warps, 0, 0};
    BfsResult r;
    r.source = src;
    r.levels.resize(b.n);
    blest_counters k{};
    std::vector<blest_level_trace> tr(1u << 16);
    check(blest_bfs(b.handle(), src, &c, r.levels.data(), &k, tr.data(), (uint32_t)tr.size()));
    r.visited_count = (VertexId)k.visited_count;
    r.num_levels = k.num_levels;
    EngineCounters out;
    out.mma_calls = k.mma_calls;
    out.full_atomics = k.full_atomics;
    out.relaxed_atomics = k.relaxed_atomics;
    out.queue_pushes = k.queue_pushes;
    out.vss_dequeues = k.vss_dequeues;
    out.brs_baseline_mma_calls = k.brs_baseline_mma_calls;
    out.levels_processed = k.levels_processed;
    for (uint32_t i = 0; i < k.trace_len && i < tr.size(); ++i) {
        const blest_level_trace& t = tr[i];
        out.trace.push_back(LevelTrace{(Level)t.level, t.queue_size, t.frontier_population, t.discovered,
                                       t.full_atomics, t.stage1_full_atomics, t.relaxed_atomics, t.queue_pushes, {}});
    }
    return {std::move(r), std::move(out)};
}
}  // namespace detail

inline std::pair<BfsResult, EngineCounters> run_eager(const Bvss& b, VertexId src, const EngineConfig& cfg) {
    return detail::run(b, src, cfg, false);
}
inline std::pair<BfsResult, EngineCounters> run_lazy(const Bvss& b, VertexId src, const EngineConfig& cfg) {
    return detail::run(b, src, cfg, true);
}

struct AutoConfig {
    EngineConfig engine;
    SelectDefaults ordering;
    std::uint64_t seed = 0;
};
struct AutoResult {
    BfsResult bfs;
    EngineCounters counters;
    OrderingPlan plan;
    BvssStats stats;
    EngineMode chosen_mode = EngineMode::Eager;
};

// run_auto_prebuilt (R:src/bfs_engine.cpp:352-386).
inline AutoResult run_auto_prebuilt(const Bvss& b, const OrderingPlan& plan, VertexId src, const AutoConfig& cfg) {
    AutoResult out;
    out.plan = plan;
    out.stats = bvss_stats(b);
    EngineConfig engine = cfg.engine;
    out.chosen_mode = engine.mode != EngineMode::Auto
                          ? engine.mode
                          : ((plan.classification.is_social_like &&
                              out.stats.update_divergence >= engine.lazy_divergence_threshold)
                                 ? EngineMode::Lazy
                                 : EngineMode::Eager);
    const bool mapped = b.producing_permutation.has_value() && !b.producing_permutation->is_identity();
    if (src >= b.n) throw std::invalid_argument("bfs source out of range");
    const VertexId run_src = mapped ? b.producing_permutation->forward(src) : src;
    auto [bfs, counters] = detail::run(b, run_src, engine, out.chosen_mode == EngineMode::Lazy);
    out.counters = std::move(counters);
    if (mapped) {
        out.bfs.source = src;
        out.bfs.visited_count = bfs.visited_count;
        out.bfs.num_levels = bfs.num_levels;
        out.bfs.levels.resize(bfs.levels.size());
        for (VertexId v = 0; v < bfs.levels.size(); ++v) out.bfs.levels[v] = bfs.levels[b.producing_permutation->forward(v)];
    } else {
        out.bfs = std::move(bfs);
    }
    return out;
}

// run_auto (R:src/bfs_engine.cpp:388-402).
inline AutoResult run_auto(const Graph& g, VertexId src, const AutoConfig& cfg) {
    const OrderingPlan plan = select_plan(g, 8, cfg.ordering);
    Permutation perm = make_permutation(g, plan, 8, cfg.seed);
    Bvss b = perm.is_identity() ? build_bvss(g) : build_bvss(apply_permutation(g, perm));
    b.ordering_tag = plan.strategy == OrderingStrategy::JaccardWindows ? "jaccard-windows"
                     : plan.strategy == OrderingStrategy::Rcm          ? "rcm"
                     : plan.strategy == OrderingStrategy::Random       ? "random"
                                                                       : "identity";
    b.producing_permutation = std::move(perm);
    return run_auto_prebuilt(b, plan, src, cfg);
}

// ---- row-partitioned multi-GPU BFS (no reference counterpart: SURVEY §8(e); the C-ABI
// blest_partition_rows / blest_rows_*, paper_2512_21967_b200/multigpu.py is the Python twin)
class RowsEngine {
public:
    // Slice-balanced frontier-word bounds (world + 1 entries); slices per rank optional.
    static std::vector<std::uint64_t> partition(const Graph& g, std::uint32_t world,
                                                std::vector<std::uint64_t>* slices = nullptr) {
        std::vector<std::uint64_t> b(world + 1), sl(world);
        detail::check(blest_partition_rows(g.handle(), world, b.data(), sl.data()));
        if (slices) *slices = sl;
        return b;
    }
    RowsEngine(const Graph& g, std::uint32_t rank, std::uint32_t world, const std::vector<std::uint64_t>& bounds)
        : world_(world) {
        if (bounds.size() != (std::size_t)world + 1) throw std::invalid_argument("world + 1 word bounds expected");
        blest_rows h = nullptr;
        detail::check(blest_rows_create(g.handle(), rank, world, bounds.data(), &h));
        h_.reset(h);
        std::uint32_t lo = 0, hi = 0, nv = 0;
        std::uint64_t per = 0;
        detail::check(blest_rows_info(h, &lo, &hi, &nv, &per));
        row_lo_ = lo;
        row_hi_ = hi;
        num_vss_ = nv;
        per_ = per;
    }
    VertexId row_lo() const { return row_lo_; }
    VertexId row_hi() const { return row_hi_; }
    std::uint32_t num_vss() const { return num_vss_; }
    std::uint64_t per_words() const { return per_; }
    std::uint32_t world() const { return world_; }
    blest_rows handle() const { return h_.get(); }

    // fused (P2P) mode: CUDA IPC handle of the frontier buffer; every rank's, rank-major
    std::array<char, 64> ipc_handle() const {
        std::array<char, 64> a{};
        detail::check(blest_rows_ipc_handle(h_.get(), a.data()));
        return a;
    }
    void open_peers(const std::vector<std::array<char, 64>>& handles) {
        std::vector<char> blob;
        for (const auto& a : handles) blob.insert(blob.end(), a.begin(), a.end());
        detail::check(blest_rows_open_peers(h_.get(), blob.data()));
    }
    void bfs(VertexId src) { detail::check(blest_rows_bfs(h_.get(), src)); }

    // stepped (NCCL) mode
    std::uint32_t* send_buffer() const {
        std::uint32_t* p = nullptr;
        detail::check(blest_rows_send_buffer(h_.get(), &p));
        return p;
    }
    void step(std::uint32_t level, VertexId src, const std::uint32_t* recv_device) {
        detail::check(blest_rows_step(h_.get(), level, src, recv_device));
    }
    void flags(std::uint32_t& progress, std::uint32_t& done, std::uint32_t& status) const {
        detail::check(blest_rows_flags(h_.get(), &progress, &done, &status));
    }

    // the owned rows' levels [row_lo, row_hi) and the per-BFS counters
    std::vector<Level> finish(blest_rows_stats* stats = nullptr) {
        std::vector<Level> lv(row_hi_ - row_lo_);
        blest_rows_stats st{};
        detail::check(blest_rows_finish(h_.get(), lv.data(), &st));
        if (stats) *stats = st;
        return lv;
    }

private:
    struct Del {
        void operator()(blest_rows_s* r) const { blest_rows_free(r); }
    };
    std::unique_ptr<blest_rows_s, Del> h_;
    std::uint32_t world_ = 0, num_vss_ = 0;
    VertexId row_lo_ = 0, row_hi_ = 0;
    std::uint64_t per_ = 0;
};

// The stepped-mode host protocol (one rank; multigpu.SteppedBfs): level 1 from src, then per
// level the caller's all-gather of send_buffer() (per_words u32 per rank) into recv_device
// (world × per_words u32, rank-major) — e.g. ncclAllGather on the library's stream — and the
// next launch, never waiting for a level: the kernels' mapped flags give termination, the
// host runs at most `ahead` levels in front, and every rank issues iterations + 1 + ahead
// all-gathers (so collectives match across ranks). max_levels > 0 caps the launches.
struct RowsOutcome {
    std::vector<Level> levels;  // owned rows [row_lo, row_hi)
    blest_rows_stats stats{};
    std::uint32_t collectives = 0;
};
inline RowsOutcome rows_bfs_stepped(RowsEngine& e, VertexId src, std::uint32_t* recv_device,
                                    const std::function<void(const std::uint32_t*, std::uint32_t*, std::uint64_t)>& allgather,
                                    std::uint32_t ahead = 2, std::uint32_t max_levels = 0) {
    e.step(1, src, nullptr);
    std::uint32_t issued = 0, done = 0;
    std::int64_t target = -1;
    while (target < 0 || (std::int64_t)issued < target) {
        for (;;) {  // run-ahead limit: the launch issued + 1 - ahead has started
            std::uint32_t prog = 0, d = 0, status = 0;
            e.flags(prog, d, status);
            if (d && target < 0) {
                done = d;
                target = (std::int64_t)done + 1 + ahead;  // identical on every rank
            }
            if ((std::int64_t)prog + ahead >= (std::int64_t)issued + 1 || target >= 0) break;
            std::this_thread::yield();
        }
        if (target >= 0 && (std::int64_t)issued >= target) break;
        if (max_levels && issued >= max_levels)
            throw std::runtime_error("BFS ran past the level safety cap at level " + std::to_string(issued + 1));
        allgather(e.send_buffer(), recv_device, e.per_words());
        ++issued;
        e.step(issued + 1, src, recv_device);
    }
    RowsOutcome out;
    out.levels = e.finish(&out.stats);
    out.collectives = issued;
    if (out.stats.iterations != done) throw std::logic_error("ranks' termination level disagrees with the engine");
    return out;
}

// Virtual ranks: every engine of this device in one fused launch (peers = the siblings).
inline void rows_set_local_peers(const std::vector<RowsEngine*>& ranks) {
    std::vector<blest_rows> h;
    for (auto* r : ranks) h.push_back(r->handle());
    detail::check(blest_rows_set_local_peers(h.data(), (std::uint32_t)h.size()));
}
inline void rows_group_bfs(const std::vector<RowsEngine*>& ranks, VertexId src) {
    std::vector<blest_rows> h;
    for (auto* r : ranks) h.push_back(r->handle());
    detail::check(blest_rows_group_bfs(h.data(), (std::uint32_t)h.size(), src));
}

}  // namespace blest
