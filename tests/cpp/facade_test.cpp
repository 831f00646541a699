// C++ drop-in test: reference-style code against include/blest_b200.hpp (every call runs on
// the B200 through the C-ABI). Re-expresses known answers of R:tests/bfs_engine_test.cpp and
// R:tests/bvss_test.cpp; expected levels, digests and structure files come from the
// UNMODIFIED reference itself (oracle/_ref/libblest_ref.so, through its C forwarder
// oracle/ref_shim.cpp — test infrastructure, linked only into this test program).
#include <cstdio>
#include <unistd.h>
#include <barrier>
#include <fstream>
#include <random>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "blest_b200.hpp"

extern "C" {  // oracle/ref_shim.cpp (the reference, R = /root/reference/proj)
int ref_graph_from_edges(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t k, int directed, void** out);
void ref_graph_free(void* g);
uint64_t ref_graph_digest(const void* g);
int ref_reference_bfs(const void* g, uint32_t src, uint32_t* levels, uint32_t* visited, uint32_t* num_levels);
int ref_build_bvss(const void* g, unsigned workers, void** out);
void ref_bvss_free(void* b);
int ref_save_bvss(const void* b, const char* path);
int ref_load_permutation(const char* path, uint32_t* forward, uint32_t cap, uint32_t* n);
}

using namespace blest;

static int failures = 0;
#define CHECK(c)                                                             \
    do {                                                                     \
        if (!(c)) {                                                          \
            ++failures;                                                      \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
        }                                                                    \
    } while (0)

// The reference's own graph over the same arc list (RAII handle on blest::Graph).
struct RefGraph {
    void* g = nullptr;
    RefGraph(VertexId n, const std::vector<std::pair<VertexId, VertexId>>& e, bool directed) {
        std::vector<uint32_t> s, d;
        for (auto [u, v] : e) {
            s.push_back(u);
            d.push_back(v);
        }
        if (ref_graph_from_edges(n, s.data(), d.data(), e.size(), directed, &g) != 0) throw std::runtime_error("ref");
    }
    ~RefGraph() { ref_graph_free(g); }
    std::vector<Level> bfs(VertexId src, VertexId n) const {  // reference_bfs (R:src/graph.cpp:144-167)
        std::vector<Level> L(n);
        uint32_t vis = 0, nl = 0;
        ref_reference_bfs(g, src, L.data(), &vis, &nl);
        return L;
    }
};

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
    // random directed + undirected graphs vs the reference's reference_bfs, both engines,
    // both pulls; digest, in-views and the device reference_bfs vs the reference's
    {
        std::mt19937_64 rng(7);
        for (int t = 0; t < 4; ++t) {
            const VertexId n = 500 + 137 * t;
            std::vector<std::pair<VertexId, VertexId>> e;
            for (int i = 0; i < 6 * (int)n; ++i) e.emplace_back(rng() % n, rng() % n);
            const bool directed = t % 2 == 0;
            const Graph g = Graph::from_edges(n, e, directed);
            const RefGraph rg(n, e, directed);
            CHECK(g.digest() == ref_graph_digest(rg.g));
            const Graph gt = transpose(g);
            CHECK(gt.out_offsets() == g.in_offsets() && gt.out_targets() == g.in_sources());
            for (VertexId u = 0; u < n; u += 97)
                for (VertexId v : g.in_neighbors(u)) CHECK(g.has_edge(v, u));
            const Bvss b = build_bvss(g);
            CHECK(validate_roundtrip(b, g).ok());
            for (VertexId s : {VertexId(0), VertexId(n / 2), VertexId(n - 1)}) {
                const auto want = rg.bfs(s, n);
                CHECK(reference_bfs(g, s).levels == want);
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
    // row-partitioned engine (blest_rows_*, include/blest_b200.hpp RowsEngine): the assembled
    // owned levels equal the reference's reference_bfs — virtual ranks in one fused launch,
    // and the stepped host protocol (rows_bfs_stepped) on one rank per host thread with a
    // device all-gather standing in for ncclAllGather
    for (bool directed : {false, true}) {
        std::mt19937_64 rng(23 + directed);
        const VertexId n = 7000;
        std::vector<std::pair<VertexId, VertexId>> e;
        for (int i = 0; i < 8 * (int)n; ++i) e.emplace_back(rng() % n, rng() % n);
        const Graph g = Graph::from_edges(n, e, directed);
        const RefGraph rg(n, e, directed);
        const VertexId srcs[] = {0, n / 3, n - 1};
        for (std::uint32_t world : {1u, 2u, 3u}) {
            std::vector<std::uint64_t> slices;
            const auto bounds = RowsEngine::partition(g, world, &slices);
            CHECK(bounds.size() == world + 1 && bounds.front() == 0 && bounds.back() == (n + 31) / 32);
            auto make = [&] {
                std::vector<std::unique_ptr<RowsEngine>> r;
                for (std::uint32_t k = 0; k < world; ++k) r.push_back(std::make_unique<RowsEngine>(g, k, world, bounds));
                return r;
            };
            // fused: G virtual ranks of this device, one launch per BFS
            auto ranks = make();
            std::vector<RowsEngine*> ptrs;
            for (auto& r : ranks) ptrs.push_back(r.get());
            rows_set_local_peers(ptrs);
            for (VertexId s : srcs) {
                rows_group_bfs(ptrs, s);
                std::vector<Level> L(n, 0);
                for (std::uint32_t k = 0; k < world; ++k) {
                    RowsEngine* r = ptrs[k];
                    CHECK(r->row_lo() == bounds[k] * 32);
                    const auto lv = r->finish();
                    std::copy(lv.begin(), lv.end(), L.begin() + r->row_lo());
                }
                CHECK(L == rg.bfs(s, n));
            }
            // stepped: one host thread per rank, all-gather = device copies between barriers
            auto st = make();
            const std::uint64_t per = st[0]->per_words();
            std::vector<std::uint32_t*> recv(world, nullptr);
            for (auto& p : recv) CHECK(cudaMalloc(&p, world * per * 4) == cudaSuccess);
            std::barrier sync(world);
            auto gather = [&](const std::uint32_t*, std::uint32_t* out, std::uint64_t w) {
                sync.arrive_and_wait();  // every rank's step of this level is enqueued
                cudaDeviceSynchronize();
                for (std::uint32_t k = 0; k < world; ++k)
                    cudaMemcpy(out + k * w, st[k]->send_buffer(), w * 4, cudaMemcpyDeviceToDevice);
                cudaDeviceSynchronize();
                sync.arrive_and_wait();  // no rank overwrites its send buffer before all copied
            };
            for (VertexId s : srcs) {
                std::vector<RowsOutcome> out(world);
                std::vector<std::thread> th;
                for (std::uint32_t k = 0; k < world; ++k)
                    th.emplace_back([&, k] { out[k] = rows_bfs_stepped(*st[k], s, recv[k], gather); });
                for (auto& t : th) t.join();
                std::vector<Level> L(n, 0);
                for (std::uint32_t k = 0; k < world; ++k) {
                    CHECK(out[k].collectives == out[0].collectives && out[k].stats.iterations == out[0].stats.iterations);
                    CHECK(out[k].collectives == out[k].stats.iterations + 1 + 2);
                    std::copy(out[k].levels.begin(), out[k].levels.end(), L.begin() + st[k]->row_lo());
                }
                CHECK(L == rg.bfs(s, n));
            }
            for (auto p : recv) cudaFree(p);
        }
    }
    // BVSS cache + permutation files are the reference's: a file written by the reference's
    // save_bvss loads here; our permutation file loads in the reference's load_permutation
    {
        std::vector<std::pair<VertexId, VertexId>> e;
        std::mt19937_64 rng(11);
        for (int i = 0; i < 4000; ++i) e.emplace_back(rng() % 700, rng() % 700);
        const Graph g = Graph::from_edges(700, e, false);
        const RefGraph rg(700, e, false);
        void* rb = nullptr;
        CHECK(ref_build_bvss(rg.g, 1, &rb) == 0);
        const std::string path = "/tmp/facade_test_" + std::to_string(::getpid()) + ".bvss";
        CHECK(ref_save_bvss(rb, path.c_str()) == 0);
        ref_bvss_free(rb);
        const Bvss loaded = load_bvss(path);
        const Bvss built = build_bvss(g);
        CHECK(loaded.row_ids == built.row_ids && loaded.masks == built.masks && loaded.real_ptrs == built.real_ptrs);
        CHECK(run_lazy(loaded, 5, cfg).first.levels == rg.bfs(5, 700));
        const Permutation p = random_order(700, 3);
        save_permutation(p, path + ".perm");
        std::vector<uint32_t> f(700);
        uint32_t pn = 0;
        CHECK(ref_load_permutation((path + ".perm").c_str(), f.data(), 700, &pn) == 0);
        CHECK(pn == 700 && f == p.forward_map());
        CHECK(load_permutation(path + ".perm").forward_map() == p.forward_map());
        std::remove(path.c_str());
        std::remove((path + ".perm").c_str());
        std::ofstream(path + ".mtx") << "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n4 1\n";
        bool threw = false;
        try {
            load_graph(path + ".mtx");
        } catch (const ParseError& pe) {
            threw = pe.line() == 4;
        }
        CHECK(threw);
        std::remove((path + ".mtx").c_str());
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
        CHECK(a.bfs.levels == RefGraph(900, e, false).bfs(3, 900));
    }
    std::printf("facade_test: %s (%d failures)\n", failures ? "FAIL" : "ok", failures);
    return failures ? 1 : 0;
}
