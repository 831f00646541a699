/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product library.
 *
 * Plain-C restatement of the reference algorithms on the BLEST hot path
 * (/root/reference/proj, "R:" below), used only by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the checker. Pinned against the compiled
 * reference (oracle/_ref) and the committed golden fixtures in tests/golden/.
 *
 * Differences from the reference that do not change any output: 64-bit slot
 * indexing (the reference's u32 row_id() index wraps at >= 2^25 VSS,
 * R:include/blest/bvss.hpp:60-62), single-threaded execution.
 */
#ifndef BLEST_ORACLE_H
#define BLEST_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- synthetic inputs (harness twins of the product's device generators) ---- */
uint64_t orc_hash64(uint64_t seed, uint64_t i);
void orc_gen_rmat(uint32_t scale, uint64_t num_edges, uint64_t seed, uint32_t a, uint32_t b,
                  uint32_t c, uint32_t* src, uint32_t* dst);
void orc_gen_urand(uint32_t n, uint64_t num_edges, uint64_t seed, uint32_t* src, uint32_t* dst);
uint64_t orc_gen_grid(uint32_t rows, uint32_t cols, uint32_t* src, uint32_t* dst);
void orc_random_relabel(uint32_t n, uint64_t seed, uint32_t* forward);

/* ---- graph (R:src/graph.cpp) ---- */
/* Graph::from_edges (R:src/graph.cpp:33-55). Writes the out-view CSR; offsets has n+1
 * entries; targets must hold 2k (undirected) or k arcs. Returns m, or UINT64_MAX when an
 * endpoint is out of range. */
uint64_t orc_from_edges(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t k,
                        int directed, uint64_t* offsets, uint32_t* targets);
/* apply_permutation (R:src/graph.cpp:126-134) on a CSR out-view. */
uint64_t orc_apply_permutation(uint32_t n, const uint64_t* off, const uint32_t* tgt,
                               const uint32_t* forward, uint64_t* off_out, uint32_t* tgt_out);
/* reference_bfs (R:src/graph.cpp:144-167). Returns visited_count; *num_levels = max+1. */
uint32_t orc_reference_bfs(uint32_t n, const uint64_t* off, const uint32_t* tgt, uint32_t src,
                           uint32_t* levels, uint32_t* num_levels);
/* Many sources in parallel (OpenMP), one levels row of n per source. */
void orc_reference_bfs_many(uint32_t n, const uint64_t* off, const uint32_t* tgt,
                            const uint32_t* srcs, uint32_t count, uint32_t* levels,
                            uint32_t* visited, int threads);
/* Graph500-style validity of a level array: every reached u and arc u->v has
 * L[v] <= L[u]+1; every reached v != src has an in-arc from level L[v]-1; src is 0.
 * Returns 0 when valid, else 1 + index of the first offending vertex. */
uint64_t orc_validate_levels(uint32_t n, const uint64_t* off, const uint32_t* tgt, uint32_t src,
                             const uint32_t* levels);

/* ---- BVSS (R:src/bvss.cpp) ---- */
/* Pass 1 of build_bvss (R:src/bvss.cpp:35-53): real_ptrs (num_sets+1) and slice count.
 * Returns num_vss. */
uint64_t orc_bvss_count(uint32_t n, const uint64_t* off, const uint32_t* tgt, uint32_t* real_ptrs,
                        uint64_t* num_unpadded);
/* Pass 2 (R:src/bvss.cpp:55-101): v2r (num_vss), row_ids (num_vss*128), masks (num_vss*32). */
void orc_bvss_fill(uint32_t n, const uint64_t* off, const uint32_t* tgt, const uint32_t* real_ptrs,
                   uint64_t num_vss, uint32_t* v2r, uint32_t* row_ids, uint32_t* masks);
/* compression_ratio (R:src/bvss.cpp:103-107) */
double orc_compression_ratio(uint64_t m, uint64_t num_unpadded);
/* update_divergence (R:src/bvss.cpp:109-141) */
double orc_update_divergence(uint32_t n, uint64_t num_vss, const uint32_t* row_ids);

/* ---- engines (R:src/bfs_engine.cpp:155-350), single worker ----
 * trace rows of 8 u64: level, queue_size, frontier_population, discovered,
 * full_atomics, stage1_full_atomics, relaxed_atomics, queue_pushes — the eager rows
 * carry the reference's single-worker atomic counts; lazy rows count relaxed atomics
 * per nonzero pull and one full atomic per 32-thread warp batch with pending pushes for
 * num_warps warps (R:src/bfs_engine.cpp:296-336).
 * Returns the number of levels iterated, or -1 past the level cap (R:src/bfs_engine.cpp:68-75),
 * -2 when more than trace_cap levels would be written. */
int64_t orc_run_engine(uint32_t n, const uint32_t* real_ptrs, uint64_t num_vss, const uint32_t* v2r,
                       const uint32_t* row_ids, const uint32_t* masks, uint32_t src, int lazy,
                       uint32_t num_warps, uint32_t max_levels, uint32_t* levels,
                       uint64_t* trace, uint64_t trace_cap);

/* ---- full scale (blest_oracle_scale.c): multi-threaded, same results ---- */
void orc_free(void* p);
/* Generator twin (kind 0 RMAT(scale=a, k edges, seed, thresholds t0..t2), 1 urand(n=a, k
 * edges, seed), 2 grid(rows=a, cols=b)) -> optional relabel (forward map, may be NULL) ->
 * Graph::from_edges(undirected). *off / *tgt are malloc'd (orc_free). Returns m. */
uint64_t orc_gen_csr(int kind, uint32_t a, uint32_t b, uint64_t k, uint64_t seed, uint32_t t0,
                     uint32_t t1, uint32_t t2, const uint32_t* forward, int threads,
                     uint64_t** off, uint32_t** tgt);
void orc_random_relabel_mt(uint32_t n, uint64_t seed, int threads, uint32_t* forward);
uint64_t orc_permute_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt, const uint32_t* forward,
                         int threads, uint64_t* off_out, uint32_t* tgt_out);
uint64_t orc_transpose_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt, uint64_t* ioff,
                           uint32_t* isrc);
uint64_t orc_symmetrise_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt, const uint64_t* ioff,
                            const uint32_t* isrc, uint64_t* aoff, uint32_t* atgt);
int orc_jaccard_windows(uint32_t n, const uint64_t* off, const uint32_t* tgt, const uint64_t* ioff,
                        const uint32_t* isrc, uint32_t sigma, uint32_t w, int threads, uint32_t* forward);
void orc_rcm(uint32_t n, const uint64_t* aoff, const uint32_t* atgt, uint32_t* forward);
uint64_t orc_bvss_count_mt(uint32_t n, const uint64_t* off, const uint32_t* tgt, int threads,
                           uint32_t* real_ptrs, uint64_t* num_unpadded);
void orc_bvss_fill_mt(uint32_t n, const uint64_t* off, const uint32_t* tgt, const uint32_t* real_ptrs,
                      int threads, uint32_t* v2r, uint32_t* row_ids, uint32_t* masks);
uint64_t orc_traversed_edges(uint32_t n, const uint64_t* off, const uint32_t* levels);

/* Tile semantics of one pull round (R:src/tc_emu.cpp:9-45): c64 = FragC counts. */
void orc_tile_pull(const uint32_t* mask_words, uint8_t alpha, unsigned round, uint32_t* c64);

#ifdef __cplusplus
}
#endif
#endif
