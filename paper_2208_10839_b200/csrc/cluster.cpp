// Tensor-core cluster planning (no effect on results: every direction is
// independent and the delay-and-sum is exact integer arithmetic).
//
// A cluster of <= kTcLeafDirs consecutive slots costs R_c = max over channels
// of the channel's shift span over the cluster (+1) accumulating MMAs per
// digit plane and time tile (beamform_tc.cu), and the stage's time tracks that
// MMA count. The shift vectors (delay - advance, 32 channels; pipeline.cpp:
// 432-446 with the delay table of :289-306) are affine images of the 3-D unit
// direction, so they live on a 2-D sheet: clusters should be round in that
// sheet, where a k-d split makes boxes whose diagonal sets R. Balanced k-means
// (capacity kTcLeafDirs) on the top-2 principal components, three
// deterministic restarts, keeping whichever clustering -- k-d or k-means --
// has the smaller sum of R_c (hemisphere3000: 405 -> 362). Members keep their
// k-d order (locality for the 8-direction leaves of the CUDA-core path).
#include "plan.hpp"

#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <numeric>
#include <vector>

namespace snb {

namespace {

int64_t cluster_R_sum(const std::vector<int32_t>& sh /* dir-major n x 32 */, const std::vector<int32_t>& members,
                      const std::vector<int32_t>& bounds) {
    int64_t total = 0;
    for (size_t c = 0; c + 1 < bounds.size(); ++c) {
        int R = 1;
        for (int i = 0; i < kCh; ++i) {
            int lo = INT_MAX, hi = INT_MIN;
            for (int32_t k = bounds[c]; k < bounds[c + 1]; ++k) {
                const int v = sh[(size_t)members[k] * kCh + i];
                lo = std::min(lo, v);
                hi = std::max(hi, v);
            }
            R = std::max(R, hi - lo + 1);
        }
        total += R;
    }
    return total;
}

} // namespace

void rebalance_tc_clusters(Plan& p, uint64_t n, std::vector<int32_t>& leaves, std::vector<int32_t>& tc_leaves) {
    // (beyond ~40k directions the O(n K) Lloyd iterations would dominate
    // workspace creation: keep the k-d clusters there)
    if (n <= (uint64_t)kTcLeafDirs || n > 40000) return;
    std::vector<int32_t> sh(n * kCh);
    for (uint64_t d = 0; d < n; ++d)
        for (int i = 0; i < kCh; ++i) sh[d * kCh + i] = p.delays[d * kCh + i] - p.advances[d];
    const int64_t base_sum = cluster_R_sum(sh, leaves, tc_leaves);

    // top-2 principal components of the shift vectors (power iteration)
    double mean[kCh] = {};
    for (uint64_t d = 0; d < n; ++d)
        for (int i = 0; i < kCh; ++i) mean[i] += sh[d * kCh + i];
    for (double& m : mean) m /= (double)n;
    std::vector<double> cov(kCh * kCh, 0.0);
    for (uint64_t d = 0; d < n; ++d) {
        double x[kCh];
        for (int i = 0; i < kCh; ++i) x[i] = sh[d * kCh + i] - mean[i];
        for (int i = 0; i < kCh; ++i)
            for (int j = 0; j < kCh; ++j) cov[i * kCh + j] += x[i] * x[j];
    }
    double vec[2][kCh];
    for (int e = 0; e < 2; ++e) {
        for (int i = 0; i < kCh; ++i) vec[e][i] = 1.0 + 0.37 * i * (e + 1) - 0.05 * i * i;
        for (int it = 0; it < 200; ++it) {
            double w[kCh] = {};
            for (int i = 0; i < kCh; ++i)
                for (int j = 0; j < kCh; ++j) w[i] += cov[i * kCh + j] * vec[e][j];
            if (e == 1) { // deflate the first component
                double dot = 0;
                for (int i = 0; i < kCh; ++i) dot += w[i] * vec[0][i];
                for (int i = 0; i < kCh; ++i) w[i] -= dot * vec[0][i];
            }
            double nrm = 0;
            for (double v : w) nrm += v * v;
            nrm = std::sqrt(nrm);
            if (!(nrm > 0)) break;
            for (int i = 0; i < kCh; ++i) vec[e][i] = w[i] / nrm;
        }
    }
    std::vector<double> px(n), py(n);
    for (uint64_t d = 0; d < n; ++d) {
        double a = 0, b = 0;
        for (int i = 0; i < kCh; ++i) {
            const double x = sh[d * kCh + i] - mean[i];
            a += x * vec[0][i];
            b += x * vec[1][i];
        }
        px[d] = a;
        py[d] = b;
    }

    const int K = (int)((n + kTcLeafDirs - 1) / kTcLeafDirs);
    std::vector<int32_t> kd_pos(n);
    for (uint64_t k = 0; k < n; ++k) kd_pos[leaves[k]] = (int32_t)k;
    uint64_t rng = 0x9E3779B97F4A7C15ull;
    auto next = [&]() {
        rng ^= rng << 13;
        rng ^= rng >> 7;
        rng ^= rng << 17;
        return rng;
    };
    auto dist = [&](uint64_t d, double x, double y) { return (px[d] - x) * (px[d] - x) + (py[d] - y) * (py[d] - y); };
    std::vector<int32_t> best_members, best_bounds;
    int64_t best_sum = base_sum;
    constexpr int kNear = 8;
    for (int restart = 0; restart < 3; ++restart) {
        // k-means++ initialisation (deterministic generator)
        std::vector<double> cx, cy;
        const uint64_t first = next() % n;
        cx.push_back(px[first]);
        cy.push_back(py[first]);
        std::vector<double> dmin(n, 1e300);
        while ((int)cx.size() < K) {
            double tot = 0;
            for (uint64_t d = 0; d < n; ++d) {
                dmin[d] = std::min(dmin[d], dist(d, cx.back(), cy.back()));
                tot += dmin[d];
            }
            double r = (double)(next() >> 11) / 9007199254740992.0 * tot;
            uint64_t pick = 0;
            for (; pick + 1 < n && r > dmin[pick]; ++pick) r -= dmin[pick];
            cx.push_back(px[pick]);
            cy.push_back(py[pick]);
        }
        // Lloyd iterations with a capacity-respecting assignment: points in
        // order of their distance to the nearest centre take the nearest
        // centre with room among their kNear nearest (else any with room)
        std::vector<int32_t> lab(n, -1), ord(n);
        std::vector<std::array<int32_t, kNear>> nearest(n);
        std::vector<double> nd(n);
        for (int iter = 0; iter < 15; ++iter) {
            for (uint64_t d = 0; d < n; ++d) {
                std::array<std::pair<double, int32_t>, kNear> top;
                top.fill({1e300, -1});
                for (int c = 0; c < K; ++c) {
                    const double dd = dist(d, cx[c], cy[c]);
                    if (dd < top[kNear - 1].first) {
                        int q = kNear - 1;
                        while (q > 0 && top[q - 1].first > dd) {
                            top[q] = top[q - 1];
                            --q;
                        }
                        top[q] = {dd, (int32_t)c};
                    }
                }
                for (int q = 0; q < kNear; ++q) nearest[d][q] = top[q].second;
                nd[d] = top[0].first;
            }
            std::iota(ord.begin(), ord.end(), 0);
            std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return nd[a] < nd[b]; });
            std::vector<int> cap(K, kTcLeafDirs);
            for (int32_t d : ord) {
                int32_t c = -1;
                for (int q = 0; q < kNear && c < 0; ++q)
                    if (nearest[d][q] >= 0 && cap[nearest[d][q]] > 0) c = nearest[d][q];
                if (c < 0) {
                    double m = 1e300;
                    for (int k = 0; k < K; ++k) {
                        const double dd = dist(d, cx[k], cy[k]);
                        if (cap[k] > 0 && dd < m) {
                            m = dd;
                            c = k;
                        }
                    }
                }
                lab[d] = c;
                --cap[c];
            }
            std::vector<double> sx(K, 0.0), sy(K, 0.0);
            std::vector<int> cnt(K, 0);
            for (uint64_t d = 0; d < n; ++d) {
                sx[lab[d]] += px[d];
                sy[lab[d]] += py[d];
                ++cnt[lab[d]];
            }
            for (int k = 0; k < K; ++k) {
                if (cnt[k]) {
                    cx[k] = sx[k] / cnt[k];
                    cy[k] = sy[k] / cnt[k];
                }
            }
        }
        // clusters in order of their first k-d position, members in k-d order
        std::vector<std::vector<int32_t>> mem(K);
        for (uint64_t k = 0; k < n; ++k) mem[lab[leaves[k]]].push_back(leaves[k]);
        std::vector<int> corder(K);
        std::iota(corder.begin(), corder.end(), 0);
        std::stable_sort(corder.begin(), corder.end(), [&](int a, int b) {
            const int32_t fa = mem[a].empty() ? INT32_MAX : kd_pos[mem[a][0]];
            const int32_t fb = mem[b].empty() ? INT32_MAX : kd_pos[mem[b][0]];
            return fa < fb;
        });
        std::vector<int32_t> members, bounds;
        for (int c : corder) {
            if (mem[c].empty()) continue;
            bounds.push_back((int32_t)members.size());
            members.insert(members.end(), mem[c].begin(), mem[c].end());
        }
        bounds.push_back((int32_t)n);
        const int64_t sum = cluster_R_sum(sh, members, bounds);
        if (sum < best_sum) {
            best_sum = sum;
            best_members = std::move(members);
            best_bounds = std::move(bounds);
        }
    }
    if (!best_members.empty()) {
        leaves = std::move(best_members);
        tc_leaves = std::move(best_bounds);
    }
}

} // namespace snb
