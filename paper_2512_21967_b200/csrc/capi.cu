// extern "C" boundary (include/blest_b200.h). Every entry point catches C++ exceptions
// and maps them onto status codes with the reference's exception classes.
#include <atomic>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/blest_b200.h"
#include "bfs.cuh"
#include "bvss.cuh"
#include "graph.cuh"
#include "io.cuh"
#include "ordering.cuh"
#include "rows.cuh"

using namespace blestgpu;

struct blest_graph_s {
    DeviceGraph g;
};
struct blest_bvss_s {
    DeviceBvss b;
    std::unique_ptr<BfsEngine> engine;
    std::vector<uint64_t> last_phase_ns;
    BfsEngine& eng() {
        if (!engine) engine = std::make_unique<BfsEngine>(b);
        return *engine;
    }
};

namespace blestgpu {
namespace {
cudaStream_t g_stream = nullptr;
int g_sms = 0;
}  // namespace
cudaStream_t stream() { return g_stream; }
void set_stream(cudaStream_t s) { g_stream = s; }
int num_sms() {
    if (!g_sms) {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return g_sms;
}
std::atomic<uint64_t> g_launches{0};
}  // namespace blestgpu

namespace {
thread_local std::string t_err;

int fail_with(int code, const char* what) {
    t_err = what;
    return code;
}

void require_device() {
    static int ok = -1;
    if (ok < 0) {
        int count = 0;
        const cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0) {
            ok = 0;
        } else {
            int dev = 0, major = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
            ok = major >= 10 ? 1 : 0;
        }
    }
    if (!ok) throw CudaError("no sm_100 CUDA device available (libblest_b200 has no CPU fallback)");
}
}  // namespace

#define API_BEGIN try {
#define API_END                                                              \
    return BLEST_OK;                                                         \
    }                                                                        \
    catch (const InvalidArgument& e) { return fail_with(BLEST_EINVAL, e.what()); } \
    catch (const ParseError& e) { return fail_with(BLEST_EPARSE, e.what()); }      \
    catch (const RuntimeError& e) { return fail_with(BLEST_ERUNTIME, e.what()); }  \
    catch (const LogicError& e) { return fail_with(BLEST_ELOGIC, e.what()); }      \
    catch (const CudaError& e) { return fail_with(BLEST_ECUDA, e.what()); }        \
    catch (const std::bad_alloc& e) { return fail_with(BLEST_ENOMEM, e.what()); }  \
    catch (const std::invalid_argument& e) { return fail_with(BLEST_EINVAL, e.what()); } \
    catch (const std::exception& e) { return fail_with(BLEST_ERUNTIME, e.what()); }

#define NEED(p, msg) \
    if (!(p)) throw InvalidArgument(msg)

extern "C" {

const char* blest_last_error(void) { return t_err.c_str(); }
const char* blest_version(void) { return "blest_b200 0.1 (sm_100a)"; }
uint64_t blest_kernel_launches(void) { return g_launches.load(); }

int blest_set_stream(void* s) {
    API_BEGIN
    set_stream(reinterpret_cast<cudaStream_t>(s));
    API_END
}

int blest_device_info(char* name, int name_len, int* sm_count, int* cc_major, int* cc_minor) {
    API_BEGIN
    require_device();
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    if (name && name_len > 0) {
        std::strncpy(name, prop.name, name_len - 1);
        name[name_len - 1] = 0;
    }
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (cc_major) *cc_major = prop.major;
    if (cc_minor) *cc_minor = prop.minor;
    API_END
}

// ---- graph ------------------------------------------------------------------------------
int blest_graph_from_edges(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t k,
                           int directed, int host, blest_graph* out) {
    API_BEGIN
    NEED(out, "out is null");
    NEED(k == 0 || (src && dst), "edge arrays are null");
    require_device();
    auto h = std::make_unique<blest_graph_s>();
    h->g = graph_from_edges(n, src, dst, k, directed != 0, host != 0);
    *out = h.release();
    API_END
}

int blest_graph_from_csr(uint32_t n, const uint64_t* off, const uint32_t* tgt, int directed, int host,
                         blest_graph* out) {
    API_BEGIN
    NEED(out && off, "null argument");
    require_device();
    auto h = std::make_unique<blest_graph_s>();
    h->g = graph_from_csr(n, off, tgt, directed != 0, host != 0);
    *out = h.release();
    API_END
}

int blest_graph_generate(int kind, uint32_t a, uint32_t b, uint64_t k, uint64_t seed, uint32_t t0,
                         uint32_t t1, uint32_t t2, blest_graph* out) {
    API_BEGIN
    NEED(out, "out is null");
    require_device();
    auto h = std::make_unique<blest_graph_s>();
    switch (kind) {
        case 0: h->g = graph_generate_rmat(a, k, seed, t0, t1, t2); break;
        case 1: h->g = graph_generate_urand(a, k, seed); break;
        case 2: h->g = graph_generate_grid(a, b); break;
        default: throw InvalidArgument("unknown generator kind");
    }
    *out = h.release();
    API_END
}

int blest_graph_info(blest_graph g, uint32_t* n, uint64_t* m, int* directed) {
    API_BEGIN
    NEED(g, "null graph");
    if (n) *n = g->g.n;
    if (m) *m = g->g.m;
    if (directed) *directed = g->g.directed ? 1 : 0;
    API_END
}

int blest_graph_device_csr(blest_graph g, const uint64_t** off, const uint32_t** tgt) {
    API_BEGIN
    NEED(g, "null graph");
    if (off) *off = g->g.off.p;
    if (tgt) *tgt = g->g.tgt.p;
    API_END
}

int blest_graph_copy_csr(blest_graph g, uint64_t* off, uint32_t* tgt) {
    API_BEGIN
    NEED(g, "null graph");
    if (off) CK(cudaMemcpyAsync(off, g->g.off.p, ((size_t)g->g.n + 1) * 8, cudaMemcpyDeviceToHost, stream()));
    if (tgt && g->g.m) CK(cudaMemcpyAsync(tgt, g->g.tgt.p, g->g.m * 4, cudaMemcpyDeviceToHost, stream()));
    CK(cudaStreamSynchronize(stream()));
    API_END
}

int blest_graph_apply_permutation(blest_graph g, const uint32_t* forward, int host, blest_graph* out) {
    API_BEGIN
    NEED(g && forward && out, "null argument");
    const uint32_t n = g->g.n;
    DevBuf<uint32_t> f(n ? n : 1);
    std::vector<uint32_t> hf(n);
    if (host) std::memcpy(hf.data(), forward, (size_t)n * 4);
    else CK(cudaMemcpy(hf.data(), forward, (size_t)n * 4, cudaMemcpyDeviceToHost));
    // Permutation::from_forward bijection check (R:src/graph.cpp:86-99)
    std::vector<char> seen(n, 0);
    for (uint32_t i = 0; i < n; ++i) {
        if (hf[i] >= n || seen[hf[i]]) throw InvalidArgument("permutation is not a bijection on [0, n)");
        seen[hf[i]] = 1;
    }
    if (n) CK(cudaMemcpyAsync(f.p, hf.data(), (size_t)n * 4, cudaMemcpyHostToDevice, stream()));
    auto h = std::make_unique<blest_graph_s>();
    h->g = graph_permute(g->g, f.p);
    *out = h.release();
    API_END
}

int blest_graph_out_degrees(blest_graph g, uint32_t* deg, int host) {
    API_BEGIN
    NEED(g && deg, "null argument");
    const uint32_t n = g->g.n;
    if (!n) return BLEST_OK;
    if (host) {
        DevBuf<uint32_t> d(n);
        graph_out_degrees(g->g, d.p);
        CK(cudaMemcpyAsync(deg, d.p, (size_t)n * 4, cudaMemcpyDeviceToHost, stream()));
        CK(cudaStreamSynchronize(stream()));
    } else {
        graph_out_degrees(g->g, deg);
    }
    API_END
}

namespace blestgpu {
__global__ void k_traversed(const uint64_t* off, const uint32_t* L, uint32_t n, unsigned long long* out) {
    unsigned long long acc = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
        if (L[v] != kInf) acc += off[v + 1] - off[v];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}
}  // namespace blestgpu

int blest_graph_traversed_edges(blest_graph g, const uint32_t* levels_dev, uint64_t* edges) {
    API_BEGIN
    NEED(g && levels_dev && edges, "null argument");
    DevBuf<unsigned long long> acc(1);
    CK(cudaMemsetAsync(acc.p, 0, 8, stream()));
    if (g->g.n) {
        k_traversed<<<grid_for(g->g.n, 256), 256, 0, stream()>>>(g->g.off.p, levels_dev, g->g.n, acc.p);
        CK(cudaGetLastError());
    }
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, acc.p, 8, cudaMemcpyDeviceToHost, stream()));
    CK(cudaStreamSynchronize(stream()));
    *edges = h / 2;
    API_END
}

int blest_graph_free(blest_graph g) {
    API_BEGIN
    delete g;
    API_END
}

int blest_graph_transpose(blest_graph g, blest_graph* out) {
    API_BEGIN
    NEED(g && out, "null argument");
    auto h = std::make_unique<blest_graph_s>();
    h->g = graph_transpose(g->g);
    *out = h.release();
    API_END
}

int blest_graph_copy_in_csr(blest_graph g, uint64_t* offsets, uint32_t* sources) {
    API_BEGIN
    NEED(g && offsets && (sources || g->g.m == 0), "null argument");
    const DeviceGraph t = graph_transpose(g->g);
    CK(cudaMemcpy(offsets, t.off.p, ((size_t)t.n + 1) * 8, cudaMemcpyDeviceToHost));
    if (t.m) CK(cudaMemcpy(sources, t.tgt.p, t.m * 4, cudaMemcpyDeviceToHost));
    API_END
}

int blest_graph_digest(blest_graph g, uint64_t* digest) {
    API_BEGIN
    NEED(g && digest, "null argument");
    *digest = graph_digest(g->g);
    API_END
}

int blest_graph_bfs(blest_graph g, uint32_t src, uint32_t* levels_out, uint32_t* visited_count,
                    uint32_t* num_levels) {
    API_BEGIN
    NEED(g, "null graph");
    DevBuf<uint32_t> L(g->g.n ? g->g.n : 1);
    uint32_t nl = 0;
    const uint32_t vis = graph_bfs_levels(g->g, src, L.p, &nl);
    if (levels_out && g->g.n) CK(cudaMemcpy(levels_out, L.p, (size_t)g->g.n * 4, cudaMemcpyDeviceToHost));
    if (visited_count) *visited_count = vis;
    if (num_levels) *num_levels = nl;
    API_END
}

int blest_graph_load(const char* path, blest_graph* out) {
    API_BEGIN
    NEED(path && out, "null argument");
    const std::string p(path);
    require_device();
    const LoadedEdges e = (p.size() >= 4 && p.compare(p.size() - 4, 4, ".mtx") == 0) ? load_matrix_market(p)
                                                                                    : load_edge_list(p);
    auto h = std::make_unique<blest_graph_s>();
    h->g = graph_from_edges(e.n, e.src.data(), e.dst.data(), e.src.size(), e.directed, true);
    *out = h.release();
    API_END
}

// ---- ordering ---------------------------------------------------------------------------
int blest_classify_social_like(blest_graph g, blest_social_report* out) {
    API_BEGIN
    NEED(g && out, "null argument");
    const SocialReport r = classify_social_like(g->g);
    out->top1_share = r.top1_share;
    out->top10_share = r.top10_share;
    out->power_law_slope = r.power_law_slope;
    out->power_law_fit_r2 = r.power_law_fit_r2;
    out->is_social_like = r.is_social_like;
    out->heavy_tail_fired = r.heavy_tail;
    out->power_law_fired = r.power_law;
    API_END
}

int blest_order_rcm(blest_graph g, uint32_t* forward) {
    API_BEGIN
    NEED(g && (forward || g->g.n == 0), "null argument");
    const auto f = rcm_forward(g->g);
    std::memcpy(forward, f.data(), f.size() * 4);
    API_END
}

int blest_order_jaccard_windows(blest_graph g, uint32_t sigma, uint32_t w, uint32_t* forward) {
    API_BEGIN
    NEED(g && (forward || g->g.n == 0), "null argument");
    if (sigma == 0 || w == 0 || w % sigma != 0)
        throw InvalidArgument("window size must be a positive multiple of sigma");
    jaccard_windows_forward(g->g, sigma, w, forward);
    API_END
}

int blest_order_random(uint32_t n, uint64_t seed, uint32_t* forward) {
    API_BEGIN
    NEED(forward || n == 0, "null argument");
    const auto f = random_order_forward(n, seed);
    std::memcpy(forward, f.data(), f.size() * 4);
    API_END
}

int blest_relabel_permutation(uint32_t n, uint64_t seed, uint32_t* forward, int host) {
    API_BEGIN
    NEED(forward || n == 0, "null argument");
    require_device();
    if (host) {
        DevBuf<uint32_t> f(n ? n : 1);
        relabel_permutation(n, seed, f.p);
        if (n) CK(cudaMemcpy(forward, f.p, (size_t)n * 4, cudaMemcpyDeviceToHost));
    } else {
        relabel_permutation(n, seed, forward);
    }
    API_END
}

int blest_pick_sources(blest_graph g, uint32_t count, uint64_t seed, int skip_isolated, uint32_t* out) {
    API_BEGIN
    NEED(g && (out || count == 0), "null argument");
    const auto s = pick_sources(g->g, count, seed, skip_isolated != 0);
    std::memcpy(out, s.data(), s.size() * 4);
    API_END
}

// ---- BVSS -------------------------------------------------------------------------------
int blest_bvss_build(blest_graph g, blest_bvss* out) {
    API_BEGIN
    NEED(g && out, "null argument");
    auto h = std::make_unique<blest_bvss_s>();
    h->b = bvss_build(g->g);
    *out = h.release();
    API_END
}

int blest_bvss_save(blest_bvss b, const char* path) {
    API_BEGIN
    NEED(b && path, "null argument");
    bvss_save(b->b, path);
    API_END
}

int blest_bvss_load(const char* path, blest_bvss* out) {
    API_BEGIN
    NEED(path && out, "null argument");
    require_device();
    auto h = std::make_unique<blest_bvss_s>();
    h->b = bvss_load(path);
    *out = h.release();
    API_END
}

int blest_permutation_save(const uint32_t* forward, uint32_t n, const char* path) {
    API_BEGIN
    NEED((forward || n == 0) && path, "null argument");
    permutation_save(forward, n, path);
    API_END
}

int blest_permutation_load(const char* path, uint32_t* forward, uint32_t* n) {
    API_BEGIN
    NEED(path && n, "null argument");
    const std::vector<uint32_t> f = permutation_load(path);
    if (forward) {
        NEED(*n >= f.size(), "forward array too small");
        std::memcpy(forward, f.data(), f.size() * 4);
    }
    *n = (uint32_t)f.size();
    API_END
}

int blest_bvss_validate_roundtrip(blest_bvss b, blest_graph g, blest_roundtrip_report* out) {
    API_BEGIN
    NEED(b && g && out, "null argument");
    const RoundtripCounts r = bvss_validate_roundtrip(b->b, g->g);
    out->checked_slices = r.checked_slices;
    out->padded_nonzero_mask = r.padded_nonzero;
    out->real_zero_mask = r.real_zero_mask;
    out->mask_bit_beyond_n = r.beyond_n;
    out->rows_mismatched = r.rows_mismatched;
    out->first_padded_nonzero_vss = r.first_padded_nonzero_vss;
    out->first_zero_mask_vss = r.first_zero_mask_vss;
    out->first_beyond_set = r.first_beyond_set;
    out->first_mismatched_row = r.first_mismatched_row;
    API_END
}

int blest_bvss_build_rows(blest_graph g, uint32_t row_lo, uint32_t row_hi, blest_bvss* out) {
    API_BEGIN
    NEED(g && out, "null argument");
    NEED((row_lo % 32 == 0 || row_lo >= g->g.n) && (row_hi % 32 == 0 || row_hi >= g->g.n),
         "row range must be 32-aligned");
    NEED(row_lo <= row_hi, "empty row range");
    auto h = std::make_unique<blest_bvss_s>();
    h->b = bvss_build(g->g, row_lo, row_hi);
    *out = h.release();
    API_END
}

struct blest_rows_s {
    DeviceBvss b;
    DevBuf<uint32_t> present;  // rows present in the whole BVSS (exhaustion exit)
    std::unique_ptr<RowsEngine> e;
};

int blest_partition_rows(blest_graph g, uint32_t world, uint64_t* word_bounds, uint64_t* slices) {
    API_BEGIN
    NEED(g && word_bounds, "null argument");
    NEED(world >= 1, "world size must be positive");
    std::vector<uint64_t> sl;
    const auto bounds = partition_rows_by_slices(g->g, world, slices ? &sl : nullptr);
    std::memcpy(word_bounds, bounds.data(), (world + 1) * 8);
    if (slices) std::memcpy(slices, sl.data(), world * 8);
    API_END
}

int blest_rows_create(blest_graph g, uint32_t rank, uint32_t world, const uint64_t* word_bounds, blest_rows* out) {
    API_BEGIN
    NEED(g && word_bounds && out, "null argument");
    NEED(world >= 1 && rank < world, "rank out of range");
    require_device();
    std::vector<uint64_t> bounds(word_bounds, word_bounds + world + 1);
    const uint64_t words = ((uint64_t)g->g.n + 31) / 32;
    NEED(bounds[0] == 0 && bounds[world] == words, "word bounds must span [0, ceil(n/32)]");
    for (uint32_t r = 0; r < world; ++r) NEED(bounds[r] <= bounds[r + 1], "word bounds must be ascending");
    auto h = std::make_unique<blest_rows_s>();
    const uint64_t lo = std::min<uint64_t>(32 * bounds[rank], g->g.n), hi = std::min<uint64_t>(32 * bounds[rank + 1], g->g.n);
    h->b = bvss_build(g->g, (uint32_t)lo, (uint32_t)hi);
    h->e = std::make_unique<RowsEngine>(h->b, rank, world, bounds);
    const uint64_t present_rows = graph_present_rows(g->g, h->present);
    h->e->set_present(h->present.p, present_rows);
    *out = h.release();
    API_END
}

int blest_rows_info(blest_rows r, uint32_t* row_lo, uint32_t* row_hi, uint32_t* num_vss, uint64_t* per_words) {
    API_BEGIN
    NEED(r, "null engine");
    if (row_lo) *row_lo = r->e->row_lo();
    if (row_hi) *row_hi = r->e->row_hi();
    if (num_vss) *num_vss = r->b.num_vss;
    if (per_words) *per_words = r->e->per_words();
    API_END
}

int blest_rows_ipc_handle(blest_rows r, void* handle64) {
    API_BEGIN
    NEED(r && handle64, "null argument");
    r->e->ipc_handle(handle64);
    API_END
}

int blest_rows_open_peers(blest_rows r, const void* handles) {
    API_BEGIN
    NEED(r && handles, "null argument");
    r->e->open_peers(handles);
    API_END
}

namespace {
std::vector<RowsEngine*> rank_group(blest_rows* ranks, uint32_t world) {
    std::vector<RowsEngine*> v(world);
    for (uint32_t i = 0; i < world; ++i) {
        if (!ranks[i]) throw InvalidArgument("null engine in the rank group");
        v[i] = ranks[i]->e.get();
    }
    return v;
}
}  // namespace

int blest_rows_set_local_peers(blest_rows* ranks, uint32_t world) {
    API_BEGIN
    NEED(ranks && world, "null argument");
    const auto v = rank_group(ranks, world);
    for (auto* e : v) e->set_local_peers(v);
    API_END
}

int blest_rows_bfs(blest_rows r, uint32_t src) {
    API_BEGIN
    NEED(r, "null engine");
    r->e->launch_fused(src);
    API_END
}

int blest_rows_group_bfs(blest_rows* ranks, uint32_t world, uint32_t src) {
    API_BEGIN
    NEED(ranks && world, "null argument");
    rows_group_launch(rank_group(ranks, world), src);
    API_END
}

int blest_rows_step(blest_rows r, uint32_t level, uint32_t src, const uint32_t* recv) {
    API_BEGIN
    NEED(r, "null engine");
    r->e->step(level, src, recv);
    API_END
}

int blest_rows_send_buffer(blest_rows r, uint32_t** send) {
    API_BEGIN
    NEED(r && send, "null argument");
    *send = r->e->send_buffer();
    API_END
}

int blest_rows_flags(blest_rows r, uint32_t* progress, uint32_t* done, uint32_t* status) {
    API_BEGIN
    NEED(r, "null engine");
    const volatile unsigned* f = r->e->host_flags();
    if (progress) *progress = f[0];
    if (done) *done = f[1];
    if (status) *status = f[2];
    API_END
}

int blest_rows_finish(blest_rows r, uint32_t* levels_owned, blest_rows_stats* out) {
    API_BEGIN
    NEED(r, "null engine");
    const RowsEngine::Stats s = r->e->finish(levels_owned);
    if (out) {
        out->iterations = s.iterations;
        out->max_level = s.max_level;
        out->queue = s.queue;
        out->discovered = s.discovered;
        out->relaxed = s.relaxed;
        out->pushes = s.pushes;
        out->unpulled = s.unpulled;
    }
    API_END
}

int blest_rows_phase_times(blest_rows r, uint64_t* out, uint32_t cap, uint32_t* rows) {
    API_BEGIN
    NEED(r && out && rows, "null argument");
    const auto t = r->e->phase_times(cap);
    std::memcpy(out, t.data(), t.size() * 8);
    *rows = (uint32_t)(t.size() / 4);
    API_END
}

int blest_rows_free(blest_rows r) {
    API_BEGIN
    if (r) {
        CK(cudaStreamSynchronize(stream()));
        r->e.reset();
        delete r;
    }
    API_END
}

int blest_bvss_upload(uint32_t n, uint64_t m, uint32_t num_vss, const uint32_t* rp, const uint32_t* v2r,
                      const uint32_t* rows, const uint32_t* masks, int host, blest_bvss* out) {
    API_BEGIN
    NEED(out && rp, "null argument");
    NEED(num_vss == 0 || (v2r && rows && masks), "null BVSS arrays");
    require_device();
    auto h = std::make_unique<blest_bvss_s>();
    h->b = bvss_upload(n, m, num_vss, rp, v2r, rows, masks, host != 0);
    *out = h.release();
    API_END
}

int blest_bvss_get_info(blest_bvss b, blest_bvss_info* out) {
    API_BEGIN
    NEED(b && out, "null argument");
    out->n = b->b.n;
    out->m = b->b.m;
    out->num_slice_sets = b->b.num_sets;
    out->num_vss = b->b.num_vss;
    out->num_unpadded_slices = b->b.num_unpadded;
    out->sigma = kSigma;
    out->tau = kTau;
    API_END
}

int blest_bvss_download(blest_bvss b, uint32_t* rp, uint32_t* v2r, uint32_t* rows, uint32_t* masks) {
    API_BEGIN
    NEED(b, "null argument");
    const DeviceBvss& x = b->b;
    cudaStream_t st = stream();
    if (rp) CK(cudaMemcpyAsync(rp, x.real_ptrs.p, ((size_t)x.num_sets + 1) * 4, cudaMemcpyDeviceToHost, st));
    if (x.num_vss) {
        if (v2r) CK(cudaMemcpyAsync(v2r, x.v2r.p, (size_t)x.num_vss * 4, cudaMemcpyDeviceToHost, st));
        if (rows) CK(cudaMemcpyAsync(rows, x.row_ids.p, (uint64_t)x.num_vss * kTau * 4, cudaMemcpyDeviceToHost, st));
        if (masks) CK(cudaMemcpyAsync(masks, x.masks.p, (uint64_t)x.num_vss * 32 * 4, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    API_END
}

int blest_bvss_stats(blest_bvss b, blest_bvss_stats_t* out) {
    API_BEGIN
    NEED(b && out, "null argument");
    const DeviceBvss& x = b->b;
    std::memset(out, 0, sizeof(*out));
    out->compression_ratio = bvss_compression_ratio(x);
    out->update_divergence = bvss_update_divergence(x);
    out->num_slice_sets = x.num_sets;
    out->num_vss = x.num_vss;
    out->num_slices_padded = (uint64_t)x.num_vss * kTau;
    out->num_unpadded_slices = x.num_unpadded;
    out->connectivity_bits = x.num_unpadded * kSigma;
    out->bytes_real_ptrs = ((uint64_t)x.num_sets + 1) * 4;
    out->bytes_virtual_to_real = (uint64_t)x.num_vss * 4;
    out->bytes_row_ids = (uint64_t)x.num_vss * kTau * 4;
    out->bytes_masks = (uint64_t)x.num_vss * 32 * 4;
    const uint64_t words = ((uint64_t)x.n + 31) / 32;
    out->bytes_dynamic = 4 * words * 4 + 2 * (uint64_t)x.num_vss * 4;  // R:src/bvss.cpp:629-632
    out->bytes_levels = (uint64_t)x.n * 4;
    bvss_slice_histogram(x, out->per_vss_slice_histogram);
    API_END
}

int blest_bvss_update_divergence(blest_bvss b, double* out) {
    API_BEGIN
    NEED(b && out, "null argument");
    *out = bvss_update_divergence(b->b);
    API_END
}

int blest_tile_pull(const uint32_t* masks, const uint8_t* alpha, uint32_t count, uint32_t* counts) {
    API_BEGIN
    NEED((masks && alpha && counts) || !count, "null argument");
    require_device();
    tile_pull_device(masks, alpha, count, counts);
    API_END
}

int blest_bvss_free(blest_bvss b) {
    API_BEGIN
    delete b;
    API_END
}

// ---- BFS --------------------------------------------------------------------------------
namespace {
EngineOptions to_opts(const blest_engine_config* cfg) {
    EngineOptions o;
    if (!cfg) return o;
    if (cfg->mode != BLEST_MODE_EAGER && cfg->mode != BLEST_MODE_LAZY)
        throw InvalidArgument("engine mode must be eager or lazy (resolve auto first)");
    if (cfg->pull != BLEST_PULL_POPC && cfg->pull != BLEST_PULL_MMA) throw InvalidArgument("unknown pull variant");
    o.mode = cfg->mode == BLEST_MODE_LAZY ? Mode::Lazy : Mode::Eager;
    o.pull = cfg->pull == BLEST_PULL_MMA ? Pull::Mma : Pull::Popc;
    o.max_levels = cfg->max_levels;
    o.num_warps = cfg->num_warps;
    o.grid_ctas = cfg->grid_ctas;
    o.threads = cfg->threads_per_cta;
    return o;
}

void fill_counters(const BfsOutcome& r, blest_counters* c, blest_level_trace* trace, uint32_t trace_cap) {
    const uint64_t d = r.sum_queue, pushes = r.sum_pushes, full = r.sum_full, relaxed = r.sum_relaxed;
    if (c) {
        c->vss_dequeues = d;
        c->mma_calls = 2 * d;  // two m8n8k128 tiles per dequeued VSS (SPEC.md MMA exactness)
        c->brs_baseline_mma_calls = 16 * d;
        c->queue_pushes = pushes;
        c->full_atomics = full;
        c->relaxed_atomics = relaxed;
        c->levels_processed = r.max_level;
        c->num_levels = r.max_level + 1;
        c->visited_count = r.visited;
        c->trace_len = r.iterations;
        c->trace_truncated = r.trace_truncated ? 1 : 0;
    }
    if (trace)
        for (uint32_t i = 0; i < trace_cap && i < r.trace.size(); ++i)
            std::memcpy(&trace[i], &r.trace[i], sizeof(blest_level_trace));
}
}  // namespace

int blest_bfs_launch(blest_bvss b, uint32_t src, const blest_engine_config* cfg) {
    API_BEGIN
    NEED(b, "null bvss");
    b->eng().launch(src, to_opts(cfg));
    API_END
}

int blest_bfs_finish(blest_bvss b, uint32_t* levels_out, blest_counters* counters, blest_level_trace* trace,
                     uint32_t trace_cap) {
    API_BEGIN
    NEED(b, "null bvss");
    const BfsOutcome r = b->eng().finish(levels_out);
    b->last_phase_ns = r.phase_ns;
    fill_counters(r, counters, trace, trace_cap);
    API_END
}

int blest_bfs_phase_times(blest_bvss b, uint64_t* out, uint32_t cap, uint32_t* rows) {
    API_BEGIN
    NEED(b, "null bvss");
    const uint32_t n = (uint32_t)(b->last_phase_ns.size() / 3);
    if (rows) *rows = n;
    if (out)
        for (uint32_t i = 0; i < n && i < cap; ++i)
            for (int k = 0; k < 3; ++k) out[3 * i + k] = b->last_phase_ns[3 * i + k];
    API_END
}

int blest_bfs(blest_bvss b, uint32_t src, const blest_engine_config* cfg, uint32_t* levels_out,
              blest_counters* counters, blest_level_trace* trace, uint32_t trace_cap) {
    API_BEGIN
    NEED(b, "null bvss");
    b->eng().launch(src, to_opts(cfg));
    const BfsOutcome r = b->eng().finish(levels_out);
    b->last_phase_ns = r.phase_ns;
    fill_counters(r, counters, trace, trace_cap);
    API_END
}

int blest_bfs_batch(blest_bvss b, const uint32_t* srcs, uint32_t count, const blest_engine_config* cfg,
                    uint32_t* levels_out, blest_counters* counters) {
    API_BEGIN
    NEED(b && (srcs || !count), "null argument");
    const std::vector<BfsOutcome> r = b->eng().run_batch(srcs, count, to_opts(cfg), levels_out);
    if (counters)
        for (uint32_t k = 0; k < count; ++k) fill_counters(r[k], counters + k, nullptr, 0);
    API_END
}

int blest_bfs_prepare(blest_bvss b, const blest_engine_config* cfg, uint64_t* engine_bytes) {
    API_BEGIN
    NEED(b, "null bvss");
    const uint64_t bytes = b->eng().prepare(to_opts(cfg));
    if (engine_bytes) *engine_bytes = bytes;
    API_END
}

int blest_bfs_levels_device(blest_bvss b, const uint32_t** levels) {
    API_BEGIN
    NEED(b && levels, "null argument");
    *levels = b->eng().levels_device();
    API_END
}

int blest_bfs_last_unpulled(blest_bvss b, uint64_t* vss) {
    API_BEGIN
    NEED(b && vss, "null argument");
    *vss = b->eng().last_unpulled();
    API_END
}

int blest_bfs_last_geometry(blest_bvss b, uint32_t* ctas, uint32_t* threads) {
    API_BEGIN
    NEED(b, "null bvss");
    if (ctas) *ctas = b->eng().last_grid_ctas();
    if (threads) *threads = b->eng().last_threads();
    API_END
}

}  // extern "C"
