// Orderings: classifier, RCM, random order and source sampling on the host side of the
// library; Jaccard windows on the GPU (jaccard.cu).
#include <algorithm>
#include <cmath>
#include <map>
#include <random>

#include "ordering.cuh"

namespace blestgpu {

namespace {

// Rng (R:include/blest/rng.hpp:11-36): std::mt19937_64's raw stream is fixed by the
// standard; next_below is the reference's explicit rejection sampler.
struct Rng {
    std::mt19937_64 eng;
    explicit Rng(uint64_t seed) : eng(seed) {}
    uint64_t next_below(uint64_t bound) {
        const uint64_t limit = bound * ((~uint64_t{0}) / bound);
        uint64_t x;
        do {
            x = eng();
        } while (x >= limit);
        return x % bound;
    }
};

struct HostCsr {
    uint32_t n = 0;
    std::vector<uint64_t> off;
    std::vector<uint32_t> tgt;
};

HostCsr download(const DeviceGraph& g) {
    HostCsr h;
    h.n = g.n;
    h.off.resize((size_t)g.n + 1);
    h.tgt.resize(g.m);
    CK(cudaMemcpyAsync(h.off.data(), g.off.p, ((size_t)g.n + 1) * 8, cudaMemcpyDeviceToHost, stream()));
    if (g.m) CK(cudaMemcpyAsync(h.tgt.data(), g.tgt.p, g.m * 4, cudaMemcpyDeviceToHost, stream()));
    CK(cudaStreamSynchronize(stream()));
    return h;
}

// Sorted-unique union of out- and in-neighbours (symmetrised_adjacency, R:src/ordering.cpp:171-182).
// An undirected graph's stored arc set is already symmetric, so its out-view is the answer.
HostCsr symmetrised(const DeviceGraph& g) {
    HostCsr out = download(g);
    if (!g.directed) return out;
    const uint32_t n = g.n;
    std::vector<uint64_t> ioff((size_t)n + 1, 0);
    for (uint32_t v : out.tgt) ++ioff[(size_t)v + 1];
    for (uint32_t v = 0; v < n; ++v) ioff[v + 1] += ioff[v];
    std::vector<uint32_t> isrc(out.tgt.size());
    {
        std::vector<uint64_t> cur(ioff.begin(), ioff.end() - 1);
        for (uint32_t u = 0; u < n; ++u)
            for (uint64_t i = out.off[u]; i < out.off[u + 1]; ++i) isrc[cur[out.tgt[i]]++] = u;
    }
    HostCsr s;
    s.n = n;
    s.off.assign((size_t)n + 1, 0);
    s.tgt.reserve(out.tgt.size() * 2);
    for (uint32_t u = 0; u < n; ++u) {
        const size_t before = s.tgt.size();
        std::merge(out.tgt.begin() + out.off[u], out.tgt.begin() + out.off[u + 1], isrc.begin() + ioff[u],
                   isrc.begin() + ioff[u + 1], std::back_inserter(s.tgt));
        s.tgt.erase(std::unique(s.tgt.begin() + before, s.tgt.end()), s.tgt.end());
        s.off[u + 1] = s.tgt.size();
    }
    return s;
}

}  // namespace

SocialReport classify_social_like(const DeviceGraph& g) {
    SocialReport rep;
    const uint32_t n = g.n;
    if (n == 0) return rep;
    std::vector<uint64_t> off((size_t)n + 1);
    CK(cudaMemcpyAsync(off.data(), g.off.p, ((size_t)n + 1) * 8, cudaMemcpyDeviceToHost, stream()));
    CK(cudaStreamSynchronize(stream()));
    std::map<uint64_t, uint32_t> histogram;  // degree -> #vertices (R:src/ordering.cpp:357-362)
    uint64_t total = 0;
    for (uint32_t u = 0; u < n; ++u) {
        const uint64_t d = off[u + 1] - off[u];
        ++histogram[d];
        total += d;
    }
    if (total == 0) return rep;
    // share(percent) (:367-373): top floor(n*p/100 + 1e-9) degrees (clamped to [1, n]),
    // summed from the histogram's descending end — the same integers as the sorted scan.
    auto share = [&](double percent) {
        uint64_t count = (uint64_t)std::floor(n * percent / 100.0 + 1e-9);
        count = std::clamp<uint64_t>(count, 1, n);
        uint64_t acc = 0;
        for (auto it = histogram.rbegin(); it != histogram.rend() && count; ++it) {
            const uint64_t take = std::min<uint64_t>(count, it->second);
            acc += take * it->first;
            count -= take;
        }
        return (double)acc / (double)total;
    };
    rep.top1_share = share(1.0);
    rep.top10_share = share(10.0);
    rep.heavy_tail = rep.top1_share > 0.05 && rep.top10_share > 0.40;
    // fit_log_log (:315-342)
    std::vector<std::pair<double, double>> pts;
    for (const auto& [degree, freq] : histogram)
        if (degree >= 2 && freq >= 1)
            pts.emplace_back(std::log2((double)degree), std::log2((double)freq));
    double slope = 0, r2 = 0;
    if (pts.size() >= 3) {
        double sx = 0, sy = 0;
        for (const auto& [x, y] : pts) {
            sx += x;
            sy += y;
        }
        const double mx = sx / pts.size(), my = sy / pts.size();
        double sxx = 0, sxy = 0, syy = 0;
        for (const auto& [x, y] : pts) {
            sxx += (x - mx) * (x - mx);
            sxy += (x - mx) * (y - my);
            syy += (y - my) * (y - my);
        }
        if (sxx != 0) {
            slope = sxy / sxx;
            const double ss_res = syy - slope * sxy;
            r2 = syy == 0 ? (std::abs(ss_res) < 1e-12 ? 1.0 : 0.0) : std::clamp(1.0 - ss_res / syy, 0.0, 1.0);
        }
    }
    rep.power_law_slope = slope;
    rep.power_law_fit_r2 = r2;
    rep.power_law = pts.size() >= 3 && slope >= -3.5 && slope <= -1.5 && r2 >= 0.8;
    rep.is_social_like = rep.heavy_tail || rep.power_law;
    return rep;
}

std::vector<uint32_t> rcm_forward(const DeviceGraph& g) {
    const HostCsr a = symmetrised(g);
    const uint32_t n = a.n;
    std::vector<uint32_t> degree(n);
    for (uint32_t u = 0; u < n; ++u) degree[u] = (uint32_t)(a.off[u + 1] - a.off[u]);
    std::vector<uint32_t> level(n, kInf);
    std::vector<uint32_t> order_buf;
    order_buf.reserve(n);
    std::vector<uint32_t> children;

    // sym_bfs (R:src/ordering.cpp:190-218) writing the visit order into `out`; levels
    // live in `level` and are reset by the caller from `out` (component-local cost).
    auto sym_bfs = [&](uint32_t start, bool sort_children, std::vector<uint32_t>& out) -> uint32_t {
        out.clear();
        level[start] = 0;
        out.push_back(start);
        uint32_t ecc = 0;
        for (size_t head = 0; head < out.size(); ++head) {
            const uint32_t u = out[head];
            children.clear();
            for (uint64_t i = a.off[u]; i < a.off[u + 1]; ++i) {
                const uint32_t v = a.tgt[i];
                if (level[v] == kInf) {
                    level[v] = level[u] + 1;
                    ecc = std::max(ecc, level[v]);
                    children.push_back(v);
                }
            }
            if (sort_children)
                std::sort(children.begin(), children.end(), [&](uint32_t x, uint32_t y) {
                    return std::pair(degree[x], x) < std::pair(degree[y], y);
                });
            out.insert(out.end(), children.begin(), children.end());
        }
        return ecc;
    };
    auto reset = [&](const std::vector<uint32_t>& touched) {
        for (uint32_t v : touched) level[v] = kInf;
    };

    std::vector<char> placed(n, 0);
    std::vector<uint32_t> order;  // Cuthill-McKee order, reversed at the end
    order.reserve(n);
    std::vector<uint32_t> visit;
    for (uint32_t v = 0; v < n; ++v) {
        if (placed[v]) continue;
        // pseudo_peripheral (R:src/ordering.cpp:220-242)
        uint32_t current = v, best_ecc = 0;
        for (;;) {
            const uint32_t ecc = sym_bfs(current, false, visit);
            if (ecc <= best_ecc && current != v) { reset(visit); break; }
            if (ecc == 0) { reset(visit); break; }
            uint32_t next = current;
            std::pair<uint32_t, uint32_t> best_key{kInf, kInf};
            for (uint32_t x : visit)  // the last level's vertices are all in `visit`
                if (level[x] == ecc && std::pair(degree[x], x) < best_key) {
                    best_key = {degree[x], x};
                    next = x;
                }
            reset(visit);
            if (ecc <= best_ecc) break;
            best_ecc = ecc;
            current = next;
        }
        sym_bfs(current, true, visit);
        reset(visit);
        for (uint32_t u : visit) {
            placed[u] = 1;
            order.push_back(u);
        }
    }
    std::reverse(order.begin(), order.end());
    std::vector<uint32_t> forward(n);  // Permutation::from_inverse(order)
    for (uint32_t i = 0; i < n; ++i) forward[order[i]] = i;
    return forward;
}

std::vector<uint32_t> random_order_forward(uint32_t n, uint64_t seed) {
    std::vector<uint32_t> forward(n);
    for (uint32_t i = 0; i < n; ++i) forward[i] = i;
    Rng rng(seed);
    for (uint32_t i = n; i > 1; --i) std::swap(forward[i - 1], forward[rng.next_below(i)]);
    return forward;
}

std::vector<uint32_t> pick_sources(const DeviceGraph& g, uint32_t count, uint64_t seed, bool skip_isolated) {
    if (g.n == 0) throw RuntimeError("graph has no vertices");
    std::vector<uint64_t> off;
    if (skip_isolated) {
        off.resize((size_t)g.n + 1);
        CK(cudaMemcpyAsync(off.data(), g.off.p, ((size_t)g.n + 1) * 8, cudaMemcpyDeviceToHost, stream()));
        CK(cudaStreamSynchronize(stream()));
        if (off[g.n] == 0) throw RuntimeError("graph has no edges to pick non-isolated sources from");
    }
    Rng rng(seed);
    std::vector<uint32_t> out;
    while (out.size() < count) {
        const uint32_t s = (uint32_t)rng.next_below(g.n);
        if (skip_isolated && off[s + 1] == off[s]) continue;
        out.push_back(s);
    }
    return out;
}

}  // namespace blestgpu
