/*
 * blest_b200.h — C-ABI of the B200-native BLEST pull-BFS library (libblest_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path (graph load -> reorder ->
 * BVSS build -> bfs(source) -> level array). The reference is a C++ library with no
 * FFI (R = /root/reference/proj); each entry point below names the reference
 * declaration it replaces. The C++ façade include/blest_b200.hpp re-exposes these
 * with the reference's own names, types and exception classes.
 *
 * Conventions
 *   - Plain pointers and sizes only. `host` flags say whether array arguments live in
 *     host memory (1) or device memory (0).
 *   - Every call returns BLEST_OK (0) or a negative status; blest_last_error() returns the
 *     message of the calling thread's last failure. Status classes map 1:1 onto the
 *     reference's exceptions: BLEST_EINVAL = std::invalid_argument, BLEST_ERUNTIME =
 *     std::runtime_error, BLEST_ELOGIC = std::logic_error.
 *   - All device work is ordered on one CUDA stream (blest_set_stream; default: the
 *     legacy default stream). There is no CPU fallback: without a usable sm_100 device
 *     every compute entry point fails with BLEST_ECUDA.
 */
#ifndef BLEST_B200_H
#define BLEST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLEST_OK 0
#define BLEST_EINVAL (-1)
#define BLEST_ERUNTIME (-2)
#define BLEST_ELOGIC (-3)
#define BLEST_ECUDA (-4)
#define BLEST_ENOMEM (-5)
#define BLEST_EPARSE (-6) /* blest::ParseError (R:include/blest/graph.hpp:23-32), a runtime_error */

typedef struct blest_graph_s* blest_graph; /* device CSR out-view (blest::Graph, R:include/blest/graph.hpp:38-79) */
typedef struct blest_bvss_s* blest_bvss;   /* device BVSS + BFS workspace (blest::Bvss, R:include/blest/bvss.hpp:34-63) */

/* EngineMode (R:include/blest/bfs_engine.hpp:14) */
#define BLEST_MODE_EAGER 0
#define BLEST_MODE_LAZY 1
#define BLEST_MODE_AUTO 2
/* Pull variants: CUDA-core AND+popcount, or the b1 m8n8k128 mma.sync tile (BLEST §4.1). */
#define BLEST_PULL_POPC 0
#define BLEST_PULL_MMA 1

/* ---- library ---------------------------------------------------------------------- */
const char* blest_last_error(void);
const char* blest_version(void);
/* Order all subsequent device work on `cuda_stream` (a cudaStream_t; NULL = default). */
int blest_set_stream(void* cuda_stream);
/* Device name, SM count, compute capability; fails with BLEST_ECUDA without a device. */
int blest_device_info(char* name, int name_len, int* sm_count, int* cc_major, int* cc_minor);
/* Number of library kernels launched so far (process-wide counter; bench evidence). */
uint64_t blest_kernel_launches(void);

/* ---- graph (R:include/blest/graph.hpp) ----------------------------------------------- */
/* Graph::from_edges(n, edges, directed) (R:include/blest/graph.hpp:43-44, R:src/graph.cpp:33-55):
 * mirrors when undirected, range-checks (BLEST_EINVAL), drops self-loops, sorts+dedups. */
int blest_graph_from_edges(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t num_edges,
                           int directed, int host, blest_graph* out);
/* CSR out-view (offsets[n+1], targets[m]) -> graph; normalised like from_edges. */
int blest_graph_from_csr(uint32_t n, const uint64_t* offsets, const uint32_t* targets, int directed,
                         int host, blest_graph* out);
/* Harness generators (no reference counterpart): kind 0 = RMAT(scale=a,
 * edges=k, seed, thresholds t0..t2 as 2^32-scaled probabilities), 1 = urand(n=a, edges=k,
 * seed), 2 = grid(rows=a, cols=b; R:tests/support/generators.cpp:41-50 semantics). */
int blest_graph_generate(int kind, uint32_t a, uint32_t b, uint64_t k, uint64_t seed, uint32_t t0,
                         uint32_t t1, uint32_t t2, blest_graph* out);
int blest_graph_info(blest_graph g, uint32_t* n, uint64_t* m, int* directed);
/* Device pointers of the CSR (valid until blest_graph_free). */
int blest_graph_device_csr(blest_graph g, const uint64_t** offsets, const uint32_t** targets);
/* out_offsets()/out_targets() copies (R:include/blest/graph.hpp:63-66) into host arrays. */
int blest_graph_copy_csr(blest_graph g, uint64_t* offsets, uint32_t* targets);
/* apply_permutation (R:include/blest/graph.hpp:106, R:src/graph.cpp:126-134). forward[old]=new. */
int blest_graph_apply_permutation(blest_graph g, const uint32_t* forward, int host, blest_graph* out);
/* Out-degrees (uint32[n]) into host or device memory. */
int blest_graph_out_degrees(blest_graph g, uint32_t* deg, int host);
/* Undirected edges in the component reached by a level array: ½·Σ_{L[v]≠∞} outdeg(v)
 * (the GTEPS numerator); levels in device memory. */
int blest_graph_traversed_edges(blest_graph g, const uint32_t* levels_dev, uint64_t* edges);
int blest_graph_free(blest_graph g);
/* transpose (R:include/blest/graph.hpp:109, R:src/graph.cpp:136-142): every arc reversed. */
int blest_graph_transpose(blest_graph g, blest_graph* out);
/* in_offsets()/in_sources() (R:include/blest/graph.hpp:58-68): the incoming view (transpose on
 * the device) copied into host arrays (offsets[n+1], sources[m]). */
int blest_graph_copy_in_csr(blest_graph g, uint64_t* offsets, uint32_t* sources);
/* Graph::digest (R:include/blest/graph.hpp:70-71, R:src/graph.cpp:62-75): FNV-1a over
 * (n, m, arc list) — the BVSS cache key. */
int blest_graph_digest(blest_graph g, uint64_t* digest);
/* reference_bfs (R:include/blest/graph.hpp:119, R:src/graph.cpp:144-167) on the device: a
 * top-down BFS straight over the CSR (no BVSS) — the validation oracle the CLI's --validate
 * uses. levels_out: host, n entries. */
int blest_graph_bfs(blest_graph g, uint32_t src, uint32_t* levels_out, uint32_t* visited_count,
                    uint32_t* num_levels);
/* load_graph (R:include/blest/graph.hpp:150, R:src/graph.cpp:390-394): ".mtx" -> Matrix Market
 * coordinate (pattern/real/integer, general/symmetric), else a SNAP-style edge list ("# Nodes:"
 * directive honoured). Parse failures: BLEST_EPARSE (message carries the line number). */
int blest_graph_load(const char* path, blest_graph* out);

/* ---- ordering (R:include/blest/ordering.hpp) --------------------------------------------- */
typedef struct {
    double top1_share, top10_share, power_law_slope, power_law_fit_r2;
    int is_social_like;
    int heavy_tail_fired, power_law_fired;
} blest_social_report;
/* classify_social_like(g, DegreeSide::Out) (R:include/blest/ordering.hpp:75, R:src/ordering.cpp:346-387) */
int blest_classify_social_like(blest_graph g, blest_social_report* out);
/* rcm (R:include/blest/ordering.hpp:56, R:src/ordering.cpp:246-266). forward map into host array. */
int blest_order_rcm(blest_graph g, uint32_t* forward);
/* jaccard_with_windows(g, sigma, w, nullptr) (R:include/blest/ordering.hpp:52-53,
 * R:src/ordering.cpp:139-166) — one CTA per window on the GPU. */
int blest_order_jaccard_windows(blest_graph g, uint32_t sigma, uint32_t w, uint32_t* forward);
/* random_order(n, seed) (R:include/blest/ordering.hpp:58, R:src/ordering.cpp:268-275). */
int blest_order_random(uint32_t n, uint64_t seed, uint32_t* forward);
/* Harness relabel: forward[i] = rank of (splitmix64(seed, i), i); host or device output. */
int blest_relabel_permutation(uint32_t n, uint64_t seed, uint32_t* forward, int host);
/* Seeded sources as the CLI samples them (Rng(seed).next_below(n), R:tools/blest.cpp:201-203),
 * skipping zero-out-degree vertices when skip_isolated != 0. */
int blest_pick_sources(blest_graph g, uint32_t count, uint64_t seed, int skip_isolated, uint32_t* out);

/* ---- BVSS (R:include/blest/bvss.hpp) ---------------------------------------------------- */
typedef struct {
    uint32_t n, num_slice_sets, num_vss, sigma, tau;
    uint64_t m, num_unpadded_slices;
} blest_bvss_info;
typedef struct {
    double compression_ratio, update_divergence;
    uint32_t num_slice_sets, num_vss;
    uint64_t num_slices_padded, num_unpadded_slices, connectivity_bits;
    uint64_t bytes_real_ptrs, bytes_virtual_to_real, bytes_row_ids, bytes_masks, bytes_dynamic,
        bytes_levels;
    uint64_t per_vss_slice_histogram[129]; /* [k] = #VSS with k real slices */
} blest_bvss_stats_t;
/* build_bvss(g) (R:include/blest/bvss.hpp:65, R:src/bvss.cpp:19-101) on the GPU. */
int blest_bvss_build(blest_graph g, blest_bvss* out);
/* Adopt a host (or device) structure laid out as blest::Bvss's public arrays. */
int blest_bvss_upload(uint32_t n, uint64_t m, uint32_t num_vss, const uint32_t* real_ptrs,
                      const uint32_t* virtual_to_real, const uint32_t* row_ids, const uint32_t* masks,
                      int host, blest_bvss* out);
int blest_bvss_get_info(blest_bvss b, blest_bvss_info* out);
/* Copy the four arrays back (host arrays sized per blest_bvss_info). */
int blest_bvss_download(blest_bvss b, uint32_t* real_ptrs, uint32_t* virtual_to_real, uint32_t* row_ids,
                        uint32_t* masks);
/* bvss_stats (R:include/blest/bvss.hpp:97, R:src/bvss.cpp:190-216). */
int blest_bvss_stats(blest_bvss b, blest_bvss_stats_t* out);
/* update_divergence alone (R:src/bvss.cpp:109-141), bit-exact with the reference. */
int blest_bvss_update_divergence(blest_bvss b, double* out);
int blest_bvss_free(blest_bvss b);
/* save_bvss / load_bvss (R:include/blest/bvss.hpp:106-111, R:src/bvss.cpp:250-295): the
 * reference's binary cache ('BVSS' magic, version 1, little-endian u32 words: sigma, tau, n,
 * m lo/hi, numVSS, realPtrs, virtualToReal, rowIds, masks) — files are interchangeable with
 * the reference's. Errors: BLEST_ERUNTIME (cannot open, bad magic/version, truncated,
 * corrupt realPtrs), BLEST_EINVAL (sigma != 8). */
int blest_bvss_save(blest_bvss b, const char* path);
int blest_bvss_load(const char* path, blest_bvss* out);
/* save_permutation / load_permutation (R:src/graph.cpp:396-417): one inverse id per line.
 * load: call with forward == NULL to get *n, then with a forward[*n] array. */
int blest_permutation_save(const uint32_t* forward, uint32_t n, const char* path);
int blest_permutation_load(const char* path, uint32_t* forward, uint32_t* n);
/* validate_roundtrip (R:include/blest/bvss.hpp:80-82, R:src/bvss.cpp:143-188) on the device. */
typedef struct {
    uint64_t checked_slices;
    uint64_t padded_nonzero_mask, real_zero_mask, mask_bit_beyond_n, rows_mismatched;
    uint64_t first_padded_nonzero_vss, first_zero_mask_vss, first_beyond_set, first_mismatched_row;
} blest_roundtrip_report;
int blest_bvss_validate_roundtrip(blest_bvss b, blest_graph g, blest_roundtrip_report* out);

/* ---- BFS (R:include/blest/bfs_engine.hpp) --------------------------------------------- */
/* EngineConfig (R:include/blest/bfs_engine.hpp:19-25) plus device knobs. */
typedef struct {
    int mode;              /* BLEST_MODE_EAGER / BLEST_MODE_LAZY (AUTO is resolved by the caller) */
    int pull;              /* BLEST_PULL_POPC / BLEST_PULL_MMA */
    uint32_t max_levels;   /* 0 = n + 1 */
    uint32_t num_warps;    /* logical warps for the round-robin VSS split; 0 = whole grid */
    uint32_t grid_ctas;    /* 0 = persistent grid (all co-resident CTAs) */
    uint32_t threads_per_cta; /* 256, 512 or 1024; 0 = default (512) */
} blest_engine_config;
/* EngineCounters (R:include/blest/bfs_engine.hpp:39-50) + BfsResult scalars (graph.hpp:111-116). */
typedef struct {
    uint64_t mma_calls, full_atomics, relaxed_atomics, queue_pushes, vss_dequeues,
        brs_baseline_mma_calls;
    uint32_t levels_processed;
    uint32_t num_levels;
    uint64_t visited_count;
    uint32_t trace_len;       /* level iterations (including the barren last one) */
    uint32_t trace_truncated; /* trace rows beyond the device capacity were folded */
} blest_counters;
/* LevelTrace (R:include/blest/bfs_engine.hpp:27-37), per_warp_mma omitted. */
typedef struct {
    uint64_t level, queue_size, frontier_population, discovered, full_atomics, stage1_full_atomics,
        relaxed_atomics, queue_pushes;
} blest_level_trace;

/* run_eager / run_lazy (R:include/blest/bfs_engine.hpp:70-78, R:src/bfs_engine.cpp:155-350):
 * synchronous. levels_out (host, n entries) may be NULL; trace_out may be NULL. Throws-
 * equivalents: BLEST_EINVAL (src >= n), BLEST_ERUNTIME (level cap exceeded). */
int blest_bfs(blest_bvss b, uint32_t src, const blest_engine_config* cfg, uint32_t* levels_out,
              blest_counters* counters, blest_level_trace* trace_out, uint32_t trace_cap);
/* Many sources back to back (the CLI's / acceptance loop over sources, R:tools/blest.cpp:283,
 * R:tests/acceptance_main.cpp:246-263, as one call): source k's levels land in
 * levels_out + k*n (host, may be NULL), counters in counters[k] (may be NULL). The device
 * pipelines it: the level array of source k is copied to the host while source k+1 runs.
 * Errors as blest_bfs (checked for every source before any work). */
int blest_bfs_batch(blest_bvss b, const uint32_t* srcs, uint32_t count, const blest_engine_config* cfg,
                    uint32_t* levels_out, blest_counters* counters);
/* Asynchronous split of blest_bfs for stream-ordered timing: launch enqueues the fused
 * kernel (init + all levels) on the library stream; finish waits and reads back. */
int blest_bfs_launch(blest_bvss b, uint32_t src, const blest_engine_config* cfg);
int blest_bfs_finish(blest_bvss b, uint32_t* levels_out, blest_counters* counters,
                     blest_level_trace* trace_out, uint32_t trace_cap);
/* Per-level device timestamps of the last finished run (%globaltimer ns, 3 per level:
 * level start, lazy stage-1 end, level end); *rows = levels recorded. */
int blest_bfs_phase_times(blest_bvss b, uint64_t* out, uint32_t cap, uint32_t* rows);
/* Build what runs of `cfg` need before the first BFS (lazy: the hot-row view of the visited
 * bitmaps and the present-row bitmap of the exhaustion exit; every mode: the second level
 * buffer, the packed-level buffers, the pinned staging ring (3 × 2n bytes) and the widening
 * threads of blest_bfs_batch) and report the engine's device bytes; optional — the first
 * BFS / batch builds them otherwise. No reference counterpart (device workspace). */
int blest_bfs_prepare(blest_bvss b, const blest_engine_config* cfg, uint64_t* engine_bytes);
/* Device pointer to the level array of the last run on b (n entries). */
int blest_bfs_levels_device(blest_bvss b, const uint32_t** levels);
/* Launch geometry of the last run (CTAs, threads per CTA). */
int blest_bfs_last_geometry(blest_bvss b, uint32_t* ctas, uint32_t* threads);
/* VSSs of the last finished blest_bfs / blest_bfs_finish run that the counters include but
 * the kernel did not pull: the engines stop pulling once every vertex with an in-edge
 * is visited (eager: detected after dense levels) (the remaining level is provably barren; its trace row is written as the
 * reference's would be). Measurement only (bytes actually streamed); no reference counterpart. */
int blest_bfs_last_unpulled(blest_bvss b, uint64_t* vss);

/* ---- tile known-answer entry (R:src/tc_emu.cpp:9-45) -------------------------------- */
/* One warp per tile runs the engines' b1 pull (2 x mma.sync.m8n8k128.b1.and.popc with
 * BLEST's fragB broadcast of alpha, build_fragB / pack_fragA_round) on the device:
 * masks[32*t + lane] and alpha[t] in, counts[128*t + 64*round + 8*i + j] = FragC(i, j) of
 * round 0/1 out (host arrays) — tc::mma_m8n8k128(pack_fragA_round(masks, round),
 * build_fragB(alpha)). For the reference's tile KATs (R:tests/tc_emu_test.cpp:186-241). */
int blest_tile_pull(const uint32_t* masks, const uint8_t* alpha, uint32_t count, uint32_t* counts);

/* ---- row-partitioned multi-GPU mode (no reference counterpart: the paper
 * lists multi-GPU as future work) -------------------------------------------
 * Rank g of `world` owns destination rows [32*word_bounds[g], 32*word_bounds[g+1]) and a
 * BVSS of A[those rows, all columns] (row ids stay global). Per level: lazy stage 1 over
 * the local VSSs, the owned V words swept (levels, diff), the n/8-byte frontier exchanged
 * (each word has one writer, so no OR-reduction), the whole frontier swept by every rank
 * (termination, next queue). Two exchange modes, one kernel:
 *   fused   — blest_rows_bfs: one cooperative launch per BFS per rank; diff words stored
 *             into every peer's frontier buffer over CUDA IPC (NVLink), cross-rank
 *             arrival barrier in the kernel; blest_rows_group_bfs runs G virtual ranks of
 *             one device in one launch;
 *   stepped — blest_rows_step: one launch per level; the caller all-gathers every rank's
 *             send buffer (ncclAllGather / torch.distributed) on the same stream into recv.
 * Everything is ordered on the library stream; nothing here synchronises the host. */
typedef struct blest_rows_s* blest_rows;
typedef struct {
    uint32_t iterations;  /* level iterations (including the final barren one) */
    uint32_t max_level;   /* deepest level with a discovery in the owned rows */
    uint64_t queue;       /* sum over levels of the local VSS queue */
    uint64_t discovered;  /* owned rows discovered (source excluded) */
    uint64_t relaxed;     /* stage-1 REDs issued */
    uint64_t pushes;      /* local VSSs queued for next levels */
    uint64_t unpulled;    /* local VSSs of a barren last level counted in queue but not pulled:
                             every rank stops pulling once every vertex with an in-arc is
                             visited (exhaustion exit; BLEST_EXHAUST=0 pulls it) */
} blest_rows_stats;
/* Row ranges balanced by BVSS slice count (one slice = a (column slice set, row) pair, the
 * unit of pull work): word_bounds[0..world], slices[0..world-1] (optional) per rank. */
int blest_partition_rows(blest_graph g, uint32_t world, uint64_t* word_bounds, uint64_t* slices);
/* BVSS of A[rows [row_lo, row_hi), all columns] (row_lo 32-aligned, row_hi 32-aligned or n):
 * every column slice set keeps its VSS range, row ids stay global (one rank's slice). */
int blest_bvss_build_rows(blest_graph g, uint32_t row_lo, uint32_t row_hi, blest_bvss* out);
/* This rank's engine: builds its BVSS slice from g (device) with the given bounds. */
int blest_rows_create(blest_graph g, uint32_t rank, uint32_t world, const uint64_t* word_bounds, blest_rows* out);
int blest_rows_info(blest_rows r, uint32_t* row_lo, uint32_t* row_hi, uint32_t* num_vss, uint64_t* per_words);
/* fused mode plumbing: this rank's IPC handle (64 bytes); every rank's (world x 64 bytes,
 * rank-major) to map the peers; or the sibling engines of one device (virtual ranks). */
int blest_rows_ipc_handle(blest_rows r, void* handle64);
int blest_rows_open_peers(blest_rows r, const void* handles);
int blest_rows_set_local_peers(blest_rows* ranks, uint32_t world);
int blest_rows_bfs(blest_rows r, uint32_t src);
int blest_rows_group_bfs(blest_rows* ranks, uint32_t world, uint32_t src);
/* stepped mode: level 1 starts a BFS from src; level > 1 reads recv (device, world x
 * per_words u32, rank-major: the all-gather of every rank's send buffer). send: device,
 * per_words u32 (the rank's owned diff words, zero-padded). flags (mapped host memory,
 * no sync): progress = last level launched, done = iterations once finished (else 0). */
int blest_rows_step(blest_rows r, uint32_t level, uint32_t src, const uint32_t* recv);
int blest_rows_send_buffer(blest_rows r, uint32_t** send);
int blest_rows_flags(blest_rows r, uint32_t* progress, uint32_t* done, uint32_t* status);
/* Waits for the stream; owned rows' levels (host, row_hi-row_lo entries; may be NULL). */
int blest_rows_finish(blest_rows r, uint32_t* levels_owned, blest_rows_stats* out);
/* Level timeline of the last fused BFS (%globaltimer ns; 4 per level: start, stage-1 end,
 * exchange end, level end); *rows = levels recorded. */
int blest_rows_phase_times(blest_rows r, uint64_t* out, uint32_t cap, uint32_t* rows);
int blest_rows_free(blest_rows r);

#ifdef __cplusplus
}
#endif
#endif /* BLEST_B200_H */
