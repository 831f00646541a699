// Host-side file formats of the reference, for the drop-in boundary:
//   * the BVSS binary cache, 'BVSS' v1 (save_bvss / load_bvss, R:src/bvss.cpp:218-295,
//     R:include/blest/bvss.hpp:106-111): little-endian u32 words — magic, version, sigma,
//     tau, n, m (low, high), numVSS, then realPtrs, virtualToReal, rowIds, masks. The
//     device arrays already have this layout, so save/load stream them through one pinned
//     staging buffer (a 28 GB Kron-27 structure never needs a second host copy);
//   * permutation files (save_permutation / load_permutation, R:src/graph.cpp:396-417):
//     one inverse id per line, blank lines skipped;
//   * graph files (load_graph, R:src/graph.cpp:233-394): Matrix Market coordinate
//     (pattern / real / integer; general / symmetric) and SNAP-style edge lists, parsed
//     on the host with the reference's acceptance rules, then built on the GPU;
//   * Graph::digest (R:src/graph.cpp:62-75): FNV-1a over (n, m, arc list), the cache key.
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <vector>

#include "bvss.cuh"
#include "io.cuh"

namespace blestgpu {

namespace {

constexpr uint32_t kMagic = 0x53535642u;  // "BVSS" little-endian
constexpr uint32_t kVersion = 1;
constexpr size_t kStage = 64u << 20;      // pinned staging bytes

struct Pinned {
    void* p = nullptr;
    explicit Pinned(size_t bytes) { CK(cudaMallocHost(&p, bytes)); }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

struct File {
    FILE* f = nullptr;
    File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

// device array -> file, in staging-buffer chunks
void write_dev(FILE* f, const uint32_t* dev, uint64_t count, Pinned& st, const std::string& path) {
    const uint64_t per = kStage / 4;
    for (uint64_t i = 0; i < count; i += per) {
        const uint64_t k = std::min(per, count - i);
        CK(cudaMemcpyAsync(st.p, dev + i, k * 4, cudaMemcpyDeviceToHost, stream()));
        CK(cudaStreamSynchronize(stream()));
        if (std::fwrite(st.p, 4, k, f) != k) throw RuntimeError("write failed: " + path);
    }
}

// file -> device array
void read_dev(FILE* f, uint32_t* dev, uint64_t count, Pinned& st, const std::string& path) {
    const uint64_t per = kStage / 4;
    for (uint64_t i = 0; i < count; i += per) {
        const uint64_t k = std::min(per, count - i);
        CK(cudaStreamSynchronize(stream()));  // staging buffer free again
        if (std::fread(st.p, 4, k, f) != k) throw RuntimeError("truncated binary structure file");
        CK(cudaMemcpyAsync(dev + i, st.p, k * 4, cudaMemcpyHostToDevice, stream()));
    }
    CK(cudaStreamSynchronize(stream()));
}

uint32_t get_u32(FILE* f) {
    unsigned char b[4];
    if (std::fread(b, 1, 4, f) != 4) throw RuntimeError("truncated binary structure file");
    return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}

void put_u32(FILE* f, uint32_t v) {
    const unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16),
                                (unsigned char)(v >> 24)};
    if (std::fwrite(b, 1, 4, f) != 4) throw RuntimeError("write failed");
}

__global__ void k_count_unpadded(const uint32_t* __restrict__ rows, uint64_t slots, uint32_t n,
                                 unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < slots; i += (uint64_t)gridDim.x * blockDim.x)
        c += rows[i] != n;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// ---- tokenising helpers (the reference's acceptance rules: whitespace-separated
// tokens, integers must parse completely) ----
bool blank(const std::string& s) {
    for (unsigned char c : s)
        if (!std::isspace(c)) return false;
    return true;
}

std::vector<std::string> tokens(const std::string& line) {
    std::vector<std::string> t;
    std::istringstream in(line);
    std::string x;
    while (in >> x) t.push_back(x);
    return t;
}

int64_t to_int(const std::string& tok, size_t line) {
    int64_t v = 0;
    const char* b = tok.data();
    const char* e = b + tok.size();
    auto [p, ec] = std::from_chars(b, e, v);
    if (ec != std::errc{} || p != e) throw ParseError("expected an integer, got '" + tok + "'", line);
    return v;
}

std::string lower(std::string s) {
    for (char& c : s) c = (char)std::tolower((unsigned char)c);
    return s;
}

}  // namespace

void bvss_save(const DeviceBvss& b, const std::string& path) {
    File f(path, "wb");
    if (!f.f) throw RuntimeError("cannot open file for writing: " + path);
    const uint32_t hdr[8] = {kMagic, kVersion, kSigma, kTau, b.n, (uint32_t)(b.m & 0xFFFFFFFFull),
                             (uint32_t)(b.m >> 32), b.num_vss};
    for (uint32_t w : hdr) put_u32(f.f, w);
    Pinned st(kStage);
    write_dev(f.f, b.real_ptrs.p, (uint64_t)b.num_sets + 1, st, path);
    write_dev(f.f, b.v2r.p, b.num_vss, st, path);
    write_dev(f.f, b.row_ids.p, (uint64_t)b.num_vss * kTau, st, path);
    write_dev(f.f, b.masks.p, (uint64_t)b.num_vss * (kTau / 4), st, path);
    if (std::fflush(f.f) != 0) throw RuntimeError("write failed: " + path);
}

DeviceBvss bvss_load(const std::string& path) {
    File f(path, "rb");
    if (!f.f) throw RuntimeError("cannot open file: " + path);
    if (get_u32(f.f) != kMagic) throw RuntimeError("bad magic in " + path);
    if (get_u32(f.f) != kVersion) throw RuntimeError("unsupported version in " + path);
    const uint32_t sigma = get_u32(f.f), tau = get_u32(f.f);
    if (sigma != kSigma) throw InvalidArgument("unsupported tile geometry: sigma must be 8, warp size 32");
    if (tau != kTau) throw RuntimeError("inconsistent tau in " + path);
    DeviceBvss b;
    b.n = get_u32(f.f);
    const uint64_t lo = get_u32(f.f), hi = get_u32(f.f);
    b.m = lo | (hi << 32);
    b.num_vss = get_u32(f.f);
    b.num_sets = (uint32_t)(((uint64_t)b.n + kSigma - 1) / kSigma);
    b.real_ptrs.alloc((size_t)b.num_sets + 1);
    b.v2r.alloc(b.num_vss ? b.num_vss : 1);
    b.row_ids.alloc(b.num_vss ? (size_t)b.num_vss * kTau : 1);
    b.masks.alloc(b.num_vss ? (size_t)b.num_vss * (kTau / 4) : 1);
    Pinned st(kStage);
    read_dev(f.f, b.real_ptrs.p, (uint64_t)b.num_sets + 1, st, path);
    uint32_t last = 0;
    CK(cudaMemcpy(&last, b.real_ptrs.p + b.num_sets, 4, cudaMemcpyDeviceToHost));
    if (last != b.num_vss) throw RuntimeError("corrupt realPtrs in " + path);
    read_dev(f.f, b.v2r.p, b.num_vss, st, path);
    read_dev(f.f, b.row_ids.p, (uint64_t)b.num_vss * kTau, st, path);
    read_dev(f.f, b.masks.p, (uint64_t)b.num_vss * (kTau / 4), st, path);
    DevBuf<unsigned long long> cnt(1);
    CK(cudaMemsetAsync(cnt.p, 0, 8, stream()));
    if (b.num_vss) {
        k_count_unpadded<<<grid_for((uint64_t)b.num_vss * kTau, 256), 256, 0, stream()>>>(
            b.row_ids.p, (uint64_t)b.num_vss * kTau, b.n, cnt.p);
        CK(cudaGetLastError());
    }
    unsigned long long unp = 0;
    CK(cudaMemcpy(&unp, cnt.p, 8, cudaMemcpyDeviceToHost));
    b.num_unpadded = unp;
    return b;
}

void permutation_save(const uint32_t* forward, uint32_t n, const std::string& path) {
    std::vector<uint32_t> inverse(n, n);
    for (uint32_t i = 0; i < n; ++i) {
        if (forward[i] >= n || inverse[forward[i]] != n) throw InvalidArgument("not a permutation");
        inverse[forward[i]] = i;
    }
    std::ofstream out(path);
    if (!out) throw RuntimeError("cannot open file for writing: " + path);
    for (uint32_t p = 0; p < n; ++p) out << inverse[p] << '\n';
    if (!out) throw RuntimeError("write failed: " + path);
}

std::vector<uint32_t> permutation_load(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw RuntimeError("cannot open file: " + path);
    std::vector<uint32_t> inverse;
    std::string line;
    size_t no = 0;
    while (std::getline(in, line)) {
        ++no;
        if (blank(line)) continue;
        std::string t = line;
        while (!t.empty() && std::isspace((unsigned char)t.back())) t.pop_back();
        size_t s = 0;
        while (s < t.size() && std::isspace((unsigned char)t[s])) ++s;
        const int64_t v = to_int(t.substr(s), no);
        if (v < 0) throw ParseError("negative id in permutation", no);
        inverse.push_back((uint32_t)v);
    }
    // Permutation::from_inverse: a bijection on [0, n)
    const uint32_t n = (uint32_t)inverse.size();
    std::vector<uint32_t> forward(n, n);
    for (uint32_t p = 0; p < n; ++p) {
        if (inverse[p] >= n || forward[inverse[p]] != n) throw InvalidArgument("not a permutation");
        forward[inverse[p]] = p;
    }
    return forward;
}

LoadedEdges load_matrix_market(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw RuntimeError("cannot open file: " + path);
    std::string line;
    size_t no = 0;
    if (!std::getline(in, line)) throw ParseError("empty file: " + path, 1);
    ++no;
    auto h = tokens(line);
    for (auto& t : h) t = lower(t);
    if (h.size() < 4 || h[0] != "%%matrixmarket" || h[1] != "matrix")
        throw ParseError("not a Matrix Market file: bad banner", no);
    if (h[2] != "coordinate")
        throw ParseError("unsupported Matrix Market format '" + h[2] + "' (only coordinate is supported)", no);
    const std::string field = h[3];
    if (field != "pattern" && field != "real" && field != "integer")
        throw ParseError("unsupported Matrix Market field '" + field + "'", no);
    const std::string sym = h.size() > 4 ? h[4] : "general";
    if (sym != "general" && sym != "symmetric") throw ParseError("unsupported Matrix Market symmetry '" + sym + "'", no);
    int64_t rows = -1, cols = -1, nnz = -1;
    while (std::getline(in, line)) {
        ++no;
        if ((!line.empty() && line[0] == '%') || blank(line)) continue;
        const auto t = tokens(line);
        if (t.size() != 3) throw ParseError("expected 'rows cols nnz' size line", no);
        rows = to_int(t[0], no);
        cols = to_int(t[1], no);
        nnz = to_int(t[2], no);
        break;
    }
    if (nnz < 0) throw ParseError("missing size line", no);
    if (rows != cols)
        throw ParseError("matrix must be square to be a graph (" + std::to_string(rows) + "x" + std::to_string(cols) +
                             ")", no);
    if (rows < 0) throw ParseError("negative dimension", no);
    LoadedEdges e;
    e.n = (uint32_t)rows;
    e.directed = sym == "general";
    const size_t want_tok = field == "pattern" ? 2 : 3;
    int64_t seen = 0;
    while (std::getline(in, line)) {
        ++no;
        if ((!line.empty() && line[0] == '%') || blank(line)) continue;
        if (seen == nnz)
            throw ParseError("unexpected entry after the " + std::to_string(nnz) + " promised by the header", no);
        const auto t = tokens(line);
        if (t.size() != want_tok)
            throw ParseError("expected " + std::to_string(want_tok) + " tokens per entry, got " +
                                 std::to_string(t.size()), no);
        const int64_t i = to_int(t[0], no), j = to_int(t[1], no);
        if (field == "real") {  // numeric, value discarded (pattern semantics)
            char* endp = nullptr;
            errno = 0;
            std::strtod(t[2].c_str(), &endp);
            if (endp != t[2].c_str() + t[2].size() || t[2].empty())
                throw ParseError("expected a numeric value, got '" + t[2] + "'", no);
        } else if (field == "integer") {
            (void)to_int(t[2], no);
        }
        if (i < 1 || j < 1 || i > rows || j > cols)
            throw ParseError("entry (" + std::to_string(i) + ", " + std::to_string(j) + ") out of bounds", no);
        ++seen;
        const uint32_t u = (uint32_t)(i - 1), v = (uint32_t)(j - 1);
        e.src.push_back(u);
        e.dst.push_back(v);
        if (!e.directed && u != v) {  // symmetric: the mirrored entry too (from_edges mirrors again, dedups)
            e.src.push_back(v);
            e.dst.push_back(u);
        }
    }
    if (seen != nnz)
        throw ParseError("truncated file: header promised " + std::to_string(nnz) + " entries, found " +
                             std::to_string(seen), no);
    return e;
}

LoadedEdges load_edge_list(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw RuntimeError("cannot open file: " + path);
    std::string line;
    size_t no = 0;
    LoadedEdges e;
    e.directed = true;
    int64_t max_id = -1, declared = -1;
    while (std::getline(in, line)) {
        ++no;
        if (!line.empty() && line[0] == '#') {  // "# Nodes: N" pins the vertex count
            const std::string low = lower(line);
            const size_t pos = low.find("nodes");
            if (pos != std::string::npos) {
                size_t i = pos + 5;
                while (i < low.size() && (low[i] == ':' || std::isspace((unsigned char)low[i]))) ++i;
                size_t j = i;
                while (j < low.size() && std::isdigit((unsigned char)low[j])) ++j;
                if (j > i) declared = to_int(low.substr(i, j - i), no);
            }
            continue;
        }
        if (blank(line)) continue;
        const auto t = tokens(line);
        if (t.size() != 2) throw ParseError("expected 'src dst', got " + std::to_string(t.size()) + " tokens", no);
        const int64_t u = to_int(t[0], no), v = to_int(t[1], no);
        if (u < 0 || v < 0) throw InvalidArgument("negative vertex id (line " + std::to_string(no) + ")");
        max_id = std::max(max_id, std::max(u, v));
        e.src.push_back((uint32_t)u);
        e.dst.push_back((uint32_t)v);
    }
    if (declared >= 0 && max_id >= declared)
        throw ParseError("vertex id " + std::to_string(max_id) + " exceeds declared node count " +
                         std::to_string(declared));
    e.n = (uint32_t)(declared >= 0 ? declared : max_id + 1);
    return e;
}

uint64_t graph_digest(const DeviceGraph& g) {
    uint64_t h = 0xcbf29ce484222325ull;
    auto mix = [&h](uint64_t x) {
        for (int i = 0; i < 8; ++i) {
            h ^= (x >> (8 * i)) & 0xFF;
            h *= 0x100000001b3ull;
        }
    };
    mix(g.n);
    mix(g.m);
    std::vector<uint64_t> off((size_t)g.n + 1);
    CK(cudaMemcpyAsync(off.data(), g.off.p, off.size() * 8, cudaMemcpyDeviceToHost, stream()));
    Pinned st(kStage);
    CK(cudaStreamSynchronize(stream()));
    const uint64_t per = kStage / 4;
    const uint32_t* t = static_cast<const uint32_t*>(st.p);
    uint32_t u = 0;
    for (uint64_t i = 0; i < g.m; i += per) {  // arcs stream through the staging buffer
        const uint64_t k = std::min(per, g.m - i);
        CK(cudaMemcpyAsync(st.p, g.tgt.p + i, k * 4, cudaMemcpyDeviceToHost, stream()));
        CK(cudaStreamSynchronize(stream()));
        for (uint64_t a = 0; a < k; ++a) {
            while (off[u + 1] <= i + a) ++u;
            mix(((uint64_t)u << 32) | t[a]);
        }
    }
    return h;
}

}  // namespace blestgpu
