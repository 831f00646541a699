// Orderings: the classifier (degree histogram on the GPU, the log-log fit on the host in the
// reference's operation order), random order and source sampling (the reference's Rng
// stream). RCM (rcm.cu) and Jaccard windows (jaccard.cu) run on the GPU.
#include <algorithm>
#include <cmath>
#include <map>
#include <random>

#include <cub/cub.cuh>

#include "ordering.cuh"

namespace blestgpu {

namespace {

__global__ void k_out_degrees(const uint64_t* __restrict__ off, uint32_t n, uint64_t* __restrict__ deg) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x)
        deg[u] = off[u + 1] - off[u];
}

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

}  // namespace

SocialReport classify_social_like(const DeviceGraph& g) {
    SocialReport rep;
    const uint32_t n = g.n;
    if (n == 0) return rep;
    // degree histogram (R:src/ordering.cpp:357-362) on the device: out-degrees, radix sort,
    // run-length encode; only the (degree, #vertices) pairs come to the host for the fit
    std::map<uint64_t, uint32_t> histogram;  // degree -> #vertices
    const uint64_t total = g.m;               // Σ out-degrees
    {
        cudaStream_t st = stream();
        DevBuf<uint64_t> deg(n), sorted(n), uniq(n);
        DevBuf<uint32_t> cnt(n);
        DevBuf<uint32_t> nrun(1);
        k_out_degrees<<<grid_for(n, 256), 256, 0, st>>>(g.off.p, n, deg.p);
        CK(cudaGetLastError());
        size_t t1 = 0, t2 = 0;
        CK(cub::DeviceRadixSort::SortKeys(nullptr, t1, deg.p, sorted.p, (int64_t)n, 0, 64, st));
        CK(cub::DeviceRunLengthEncode::Encode(nullptr, t2, sorted.p, uniq.p, cnt.p, nrun.p, (int64_t)n, st));
        DevBuf<unsigned char> tmp(std::max<size_t>({t1, t2, 1}));
        CK(cub::DeviceRadixSort::SortKeys(tmp.p, t1, deg.p, sorted.p, (int64_t)n, 0, 64, st));
        CK(cub::DeviceRunLengthEncode::Encode(tmp.p, t2, sorted.p, uniq.p, cnt.p, nrun.p, (int64_t)n, st));
        uint32_t runs = 0;
        CK(cudaMemcpyAsync(&runs, nrun.p, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::vector<uint64_t> hd(runs);
        std::vector<uint32_t> hc(runs);
        if (runs) {
            CK(cudaMemcpyAsync(hd.data(), uniq.p, runs * 8ull, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(hc.data(), cnt.p, runs * 4ull, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
        for (uint32_t i = 0; i < runs; ++i) histogram.emplace_hint(histogram.end(), hd[i], hc[i]);
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
