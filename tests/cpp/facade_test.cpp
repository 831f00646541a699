// C++ drop-in test: reference-style code against include/blest_b200.hpp (every call runs on
// the B200 through the C-ABI). Re-expresses known answers of R:tests/bfs_engine_test.cpp and
// R:tests/bvss_test.cpp; levels are checked against a queue BFS written here (test oracle).
#include <cstdio>
#include <deque>
#include <random>
#include <stdexcept>
#include <string>

#include "blest_b200.hpp"

using namespace blest;

static int failures = 0;
#define CHECK(c)                                                             \
    do {                                                                     \
        if (!(c)) {                                                          \
            ++failures;                                                      \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
        }                                                                    \
    } while (0)

static std::vector<Level> queue_bfs(const Graph& g, VertexId s) {
    std::vector<Level> L(g.num_vertices(), kUnreached);
    std::deque<VertexId> q{s};
    L[s] = 0;
    while (!q.empty()) {
        const VertexId u = q.front();
        q.pop_front();
        for (VertexId v : g.out_neighbors(u))
            if (L[v] == kUnreached) {
                L[v] = L[u] + 1;
                q.push_back(v);
            }
    }
    return L;
}

int main() {
    EngineConfig cfg;
    // worked example: incoming {17,19,22} -> 3 packs mask 0x4A (R:tests/bvss_test.cpp:39-57)
    {
        const Graph g = Graph::from_edges(24, {{17, 3}, {19, 3}, {22, 3}});
        const Bvss b = build_bvss(g);
        CHECK(b.num_vss == 1 && b.num_slice_sets == 3);
        CHECK((b.real_ptrs == std::vector<std::uint32_t>{0, 0, 0, 1}));
        CHECK(b.slice_mask(0, 0, 0) == 0x4A && b.row_id(0, 0, 0) == 3);
        CHECK(b.row_id(0, 1, 0) == b.sentinel());
    }
    // worked pull (R:tests/bfs_engine_test.cpp:116-144)
    {
        std::vector<std::pair<VertexId, VertexId>> e = {{17, 3}, {19, 3}, {22, 3}};
        for (VertexId r = 64; r < 322; ++r) e.emplace_back(0, r);
        const Bvss b = build_bvss(Graph::from_edges(384, e));
        for (bool lazy : {false, true}) {
            auto [r, c] = lazy ? run_lazy(b, 17, cfg) : run_eager(b, 17, cfg);
            CHECK(r.levels[17] == 0 && r.levels[3] == 1 && r.visited_count == 2);
            CHECK(c.trace.size() == 2 && c.trace[0].queue_pushes == 3 && c.trace[1].queue_size == 3);
            CHECK(c.mma_calls == 8 && c.vss_dequeues == 4 && c.brs_baseline_mma_calls == 64);
        }
        const FrontierState st = init_state(b, 17, EngineMode::Eager);
        CHECK(st.levels[17] == 0 && st.q_curr.size() == 1);
    }
    // diamond: one push per slice set per level (R:tests/bfs_engine_test.cpp:146-161)
    {
        const Bvss b = build_bvss(Graph::from_edges(5, {{0, 1}, {0, 2}, {1, 3}, {2, 3}, {3, 4}}));
        for (bool lazy : {false, true}) {
            auto [r, c] = lazy ? run_lazy(b, 0, cfg) : run_eager(b, 0, cfg);
            CHECK((r.levels == std::vector<Level>{0, 1, 1, 2, 3}));
            CHECK(c.trace.size() == 4 && c.trace[0].queue_pushes == 1 && c.trace[3].queue_pushes == 0);
        }
    }
    // random directed + undirected graphs vs a queue BFS, both engines, both pulls
    {
        std::mt19937_64 rng(7);
        for (int t = 0; t < 4; ++t) {
            const VertexId n = 500 + 137 * t;
            std::vector<std::pair<VertexId, VertexId>> e;
            for (int i = 0; i < 6 * (int)n; ++i) e.emplace_back(rng() % n, rng() % n);
            const Graph g = Graph::from_edges(n, e, t % 2 == 0);
            const Bvss b = build_bvss(g);
            for (VertexId s : {VertexId(0), VertexId(n / 2), VertexId(n - 1)}) {
                const auto want = queue_bfs(g, s);
                for (bool lazy : {false, true})
                    for (bool mma : {false, true}) {
                        EngineConfig c2 = cfg;
                        c2.mma_tiles = mma;
                        auto [r, c] = lazy ? run_lazy(b, s, c2) : run_eager(b, s, c2);
                        CHECK(r.levels == want);
                        CHECK(c.mma_calls == 2 * c.vss_dequeues);
                    }
            }
        }
    }
    // errors keep the reference's exception classes
    {
        std::vector<std::pair<VertexId, VertexId>> e;
        for (VertexId v = 1; v < 16; ++v) e.emplace_back(v - 1, v);
        const Bvss b = build_bvss(Graph::from_edges(16, e, false));
        bool threw = false;
        try {
            run_eager(b, 16, cfg);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        EngineConfig capped = cfg;
        capped.max_levels = 2;
        threw = false;
        try {
            run_lazy(b, 0, capped);
        } catch (const std::runtime_error&) {
            threw = true;
        }
        CHECK(threw);
        threw = false;
        try {
            Graph::from_edges(3, {{0, 7}});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // run_auto on a star: social-like -> Jaccard windows + eager (R:tests/bfs_engine_test.cpp:324-334)
    {
        std::vector<std::pair<VertexId, VertexId>> e;
        for (VertexId v = 1; v < 900; ++v) e.emplace_back(0, v);
        const Graph g = Graph::from_edges(900, e, false);
        AutoConfig ac;
        ac.ordering.window_size = 1u << 10;
        const AutoResult a = run_auto(g, 3, ac);
        CHECK(a.plan.strategy == OrderingStrategy::JaccardWindows && a.chosen_mode == EngineMode::Eager);
        CHECK(a.bfs.levels == queue_bfs(g, 3));
    }
    std::printf("facade_test: %s (%d failures)\n", failures ? "FAIL" : "ok", failures);
    return failures ? 1 : 0;
}
