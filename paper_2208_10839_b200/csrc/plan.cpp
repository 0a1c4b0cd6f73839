// Host-side plan construction. Restates the reference's setup arithmetic
// (cited per function) so that every table is the same double the reference
// computes; compiled with -ffp-contract=off (see build.py).
#include "plan.hpp"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>

namespace snb {

namespace {

constexpr double kPi = 3.141592653589793; // std::numbers::pi

// xoshiro256++ seeded by splitmix64, polar Box-Muller with a cached spare
// (reference rng.hpp:11-58). Bit-exact generator state is required: the
// microphone layout and the synthetic noise are both drawn from it.
class Xoshiro {
public:
    explicit Xoshiro(uint64_t seed) {
        uint64_t x = seed;
        for (uint64_t& w : s_) {
            x += 0x9e3779b97f4a7c15ULL;
            uint64_t z = x;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
            w = z ^ (z >> 31);
        }
    }
    uint64_t next() {
        const uint64_t r = rotl(s_[0] + s_[3], 23) + s_[0];
        const uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return r;
    }
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double range(double lo, double hi) { return lo + (hi - lo) * unit(); }
    double normal() {
        if (spare_ok_) {
            spare_ok_ = false;
            return spare_;
        }
        double u, v, s;
        do {
            u = 2.0 * unit() - 1.0;
            v = 2.0 * unit() - 1.0;
            s = u * u + v * v;
        } while (s >= 1.0 || s == 0.0);
        const double m = std::sqrt(-2.0 * std::log(s) / s);
        spare_ = v * m;
        spare_ok_ = true;
        return u * m;
    }

private:
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t s_[4]{};
    double spare_ = 0.0;
    bool spare_ok_ = false;
};

struct V3 {
    double x, y, z;
};
inline double dot(const V3& a, const V3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 mic(const sn_pipeline_config& c, int i) {
    return {c.mic_xyz[3 * i], c.mic_xyz[3 * i + 1], c.mic_xyz[3 * i + 2]};
}
inline double dist(const V3& a, const V3& b) {
    const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
    return std::sqrt(dx * dx + dy * dy + dz * dz);
}
// Direction::unit (geometry.cpp:161-164)
inline V3 unit_vector(double az, double el) {
    const double ce = std::cos(el);
    return {ce * std::cos(az), ce * std::sin(az), std::sin(el)};
}

void check_direction(double az, double el) { // geometry.cpp:146-155
    if (!(az >= -kPi && az <= kPi)) {
        argument_error("azimuth " + std::to_string(az) + " outside [-pi, pi]");
    }
    if (!(el >= -kPi / 2 && el <= kPi / 2)) {
        argument_error("elevation " + std::to_string(el) + " outside [-pi/2, pi/2]");
    }
}

void check_geometry(const sn_pipeline_config& c) { // geometry.cpp:27-57
    constexpr double kMaxDisk = 0.05, kMaxAxial = 0.005, kMinSpacing = 0.004;
    for (int i = 0; i < kCh; ++i) {
        const V3 p = mic(c, i);
        const double radial = std::sqrt(p.y * p.y + p.z * p.z);
        if (radial > kMaxDisk) {
            argument_error("microphone " + std::to_string(i) + " outside the disk");
        }
        if (std::abs(p.x) > kMaxAxial) {
            argument_error("microphone " + std::to_string(i) + " axial offset too large");
        }
    }
    for (int i = 0; i < kCh; ++i) {
        for (int j = i + 1; j < kCh; ++j) {
            if (dist(mic(c, i), mic(c, j)) < kMinSpacing) {
                argument_error("microphones " + std::to_string(i) + " and " +
                               std::to_string(j) + " closer than 0.004 m");
            }
        }
    }
}

uint64_t pow2_at_least(uint64_t n) { // fft.cpp:22-26
    uint64_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

uint64_t chirp_samples(double duration, double rate) { // dsp.cpp:84-86
    return static_cast<uint64_t>(std::llround(duration * rate));
}

void check_chirp(const sn_pipeline_config& c, double rate) { // dsp.cpp:88-97
    if (rate <= 0.0) config_error("chirp: sample_rate must be > 0");
    if (c.chirp_duration <= 0.0) config_error("chirp: duration must be > 0");
    if (c.chirp_f_start <= 0.0 || c.chirp_f_start >= rate / 2) {
        config_error("chirp: f_start must lie in (0, sample_rate/2)");
    }
    if (c.chirp_f_end <= 0.0 || c.chirp_f_end >= rate / 2) {
        config_error("chirp: f_end must lie in (0, sample_rate/2)");
    }
}

std::vector<double> chirp(const sn_pipeline_config& c, double rate) { // dsp.cpp:229-240
    check_chirp(c, rate);
    const uint64_t n = chirp_samples(c.chirp_duration, rate);
    const double slope = (c.chirp_f_end - c.chirp_f_start) / (2.0 * c.chirp_duration);
    std::vector<double> s(n);
    for (uint64_t i = 0; i < n; ++i) {
        const double t = static_cast<double>(i) / rate;
        s[i] = std::sin(2.0 * kPi * (c.chirp_f_start * t + slope * t * t));
    }
    return s;
}

std::vector<double> reversed(std::vector<double> v) {
    std::reverse(v.begin(), v.end());
    return v;
}

} // namespace

std::vector<double> design_lowpass(double cutoff_hz, double sample_rate, int taps) {
    // dsp.cpp:129-166: Hamming-windowed sinc, forced Nyquist null, unit DC.
    if (!(cutoff_hz > 0.0 && cutoff_hz < sample_rate / 2)) {
        config_error("design_lowpass: cutoff " + std::to_string(cutoff_hz) + " Hz outside (0, " +
                     std::to_string(sample_rate / 2) + ")");
    }
    if (taps < 3 || taps % 2 == 0) config_error("design_lowpass: taps must be odd and >= 3");
    const double fc = cutoff_hz / sample_rate;
    const int mid = (taps - 1) / 2;
    std::vector<double> h(static_cast<size_t>(taps));
    for (int n = 0; n < taps; ++n) {
        const int m = n - mid;
        const double sinc = m == 0 ? 2.0 * fc : std::sin(2.0 * kPi * fc * m) / (kPi * m);
        const double window = 0.54 - 0.46 * std::cos(2.0 * kPi * n / (taps - 1));
        h[static_cast<size_t>(n)] = sinc * window;
    }
    double alternating = 0.0;
    for (int n = 0; n < taps; ++n) alternating += (n % 2 == 0 ? h[n] : -h[n]);
    const double corr = alternating / taps;
    double dc = 0.0;
    for (int n = 0; n < taps; ++n) {
        h[n] -= (n % 2 == 0 ? corr : -corr);
        dc += h[n];
    }
    for (double& v : h) v /= dc;
    return h;
}

int decimation_filter_taps(int factor) { // dsp.cpp:285-288
    const int t = std::clamp(32 * factor, 63, 1023);
    return t % 2 == 0 ? t + 1 : t;
}

void default_array(uint64_t seed, double* xyz) { // geometry.cpp:69-96
    constexpr double kDisk = 0.046, kAxial = 0.002, kMinSpacing = 0.004;
    Xoshiro rng(seed);
    int placed = 0;
    while (placed < kCh) {
        const double r = kDisk * std::sqrt(rng.unit());
        const double theta = rng.range(0.0, 2.0 * kPi);
        const double x = rng.range(-kAxial, kAxial); // braced init: left to right
        const V3 cand{x, r * std::cos(theta), r * std::sin(theta)};
        bool ok = true;
        for (int i = 0; i < placed && ok; ++i) {
            const V3 p{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
            ok = dist(cand, p) >= kMinSpacing;
        }
        if (ok) {
            xyz[3 * placed] = cand.x;
            xyz[3 * placed + 1] = cand.y;
            xyz[3 * placed + 2] = cand.z;
            ++placed;
        }
    }
}

// Fibonacci lattice on the forward hemisphere (geometry.cpp:206-229 with the
// point count n free: the reference's hemisphere3000 is n = 3000), sorted by
// (elevation, azimuth) as the reference sorts it (geometry.cpp:222-226).
std::vector<double> fibonacci_hemisphere(uint64_t n) {
    if (n == 0) config_error("fibonacci_hemisphere: n must be >= 1");
    const double golden = kPi * (3.0 - std::sqrt(5.0));
    std::vector<std::pair<double, double>> d; // (el, az)
    d.reserve(n);
    for (uint64_t i = 0; i < n; ++i) {
        const double x = (static_cast<double>(i) + 0.5) / static_cast<double>(n);
        const double r = std::sqrt(1.0 - x * x);
        const double phi = golden * static_cast<double>(i);
        const double y = r * std::cos(phi), z = r * std::sin(phi);
        d.emplace_back(std::asin(std::clamp(z, -1.0, 1.0)), std::atan2(y, x));
    }
    std::sort(d.begin(), d.end());
    std::vector<double> out;
    out.reserve(2 * n);
    for (const auto& [el, az] : d) {
        out.push_back(az);
        out.push_back(el);
    }
    return out;
}

std::vector<double> direction_grid(int kind) { // geometry.cpp:181-235
    std::vector<double> out;
    switch (kind) {
        case SN_GRID_HORIZONTAL90: {
            constexpr int n = 90;
            for (int k = 0; k < n; ++k) {
                out.push_back(-kPi / 2 + kPi * static_cast<double>(k) / (n - 1));
                out.push_back(0.0);
            }
            break;
        }
        case SN_GRID_BOX1850: {
            constexpr int n_az = 50, n_el = 37;
            for (int e = 0; e < n_el; ++e) {
                const double el = -kPi / 4 + (kPi / 2) * static_cast<double>(e) / (n_el - 1);
                for (int a = 0; a < n_az; ++a) {
                    out.push_back(-kPi / 4 + (kPi / 2) * static_cast<double>(a) / (n_az - 1));
                    out.push_back(el);
                }
            }
            break;
        }
        case SN_GRID_HEMISPHERE3000: out = fibonacci_hemisphere(3000); break;
        default: config_error("direction_grid: custom grids are built from explicit lists");
    }
    return out;
}

void default_config(int kind, sn_pipeline_config* c) { // pipeline.hpp:22-37, :94-99
    std::memset(c, 0, sizeof(*c));
    default_array(42, c->mic_xyz);
    c->grid_kind = kind;
    c->processing_threads = 0;
    c->pdm_rate = 4.5e6;
    c->chirp_f_start = 90e3;
    c->chirp_f_end = 25e3;
    c->chirp_duration = 3e-3;
    c->demod_cutoff_hz = 126e3;
    c->demod_taps = 255;
    c->demod_decimation = 10;
    c->pre_mf_decimation = 2;
    c->post_envelope_decimation = 10;
    c->smoothing_cutoff_hz = 10e3;
    c->smoothing_taps = 127;
    c->precision = SN_PRECISION_F64;
    c->speed_of_sound = 343.0;
    c->max_range = 5.0;
}

Sizes derive_sizes(const sn_pipeline_config& c) {
    // PipelineConfig::validate, pipeline.cpp:60-92 (same checks, same order).
    if (c.n_directions == 0 || c.directions == nullptr) config_error("pipeline: empty direction set");
    if (c.pdm_rate <= 0.0) config_error("pipeline: pdm_rate must be > 0");
    if (c.demod_decimation < 1 || c.pre_mf_decimation < 1 || c.post_envelope_decimation < 1) {
        config_error("pipeline: decimation factors must be >= 1");
    }
    if (c.demod_taps < 3 || c.demod_taps % 2 == 0) {
        config_error("pipeline: demod taps must be odd and >= 3");
    }
    if (c.smoothing_taps < 3 || c.smoothing_taps % 2 == 0) {
        config_error("pipeline: envelope smoothing taps must be odd and >= 3");
    }
    if (c.speed_of_sound <= 0.0) config_error("pipeline: speed_of_sound must be > 0");
    if (c.max_range <= 0.0) config_error("pipeline: max_range must be > 0");
    if (c.processing_threads < 0) config_error("pipeline: processing_threads must be >= 0");
    Sizes s;
    s.demod_rate = c.pdm_rate / c.demod_decimation;
    s.mf_rate = s.demod_rate / c.pre_mf_decimation;
    s.final_rate = s.mf_rate / c.post_envelope_decimation;
    check_chirp(c, c.pdm_rate);
    check_chirp(c, s.mf_rate);
    if (!(c.demod_cutoff_hz > 0.0 && c.demod_cutoff_hz < c.pdm_rate / 2)) {
        config_error("pipeline: demod cutoff outside (0, pdm_rate/2)");
    }
    if (!(c.smoothing_cutoff_hz > 0.0 && c.smoothing_cutoff_hz < s.mf_rate / 2)) {
        config_error("pipeline: envelope smoothing cutoff outside (0, mf_rate/2)");
    }
    // frames(): window rounded up to lcm(8, D1*D2*D3) (pipeline.cpp:40-48)
    const double window = 2.0 * c.max_range / c.speed_of_sound + c.chirp_duration;
    const auto raw = static_cast<uint64_t>(std::ceil(window * c.pdm_rate));
    const uint64_t stage = static_cast<uint64_t>(c.demod_decimation) *
                           static_cast<uint64_t>(c.pre_mf_decimation) *
                           static_cast<uint64_t>(c.post_envelope_decimation);
    const uint64_t step = std::lcm<uint64_t>(8, stage);
    s.frames = (raw + step - 1) / step * step;
    s.row_bytes = s.frames / 8;
    s.demod_len = s.frames / static_cast<uint64_t>(c.demod_decimation);
    s.mf_len = s.demod_len / static_cast<uint64_t>(c.pre_mf_decimation);
    s.bins = static_cast<uint64_t>(std::floor(2.0 * c.max_range / c.speed_of_sound * s.final_rate));
    s.range_bin_size = c.speed_of_sound / (2.0 * s.final_rate);
    if (s.bins < 1) config_error("pipeline: derived range-bin count is zero");
    s.ref_len = chirp_samples(c.chirp_duration, s.mf_rate);
    if (s.ref_len > s.mf_len) config_error("pipeline: reference chirp longer than the processed window");
    if (s.ref_len < 2) config_error("pipeline: reference chirp shorter than 2 samples");
    s.n_dirs = c.n_directions;
    s.mf_fft = pow2_at_least(s.mf_len + s.ref_len - 1);
    s.env_fft = pow2_at_least(s.mf_len);
    const uint64_t k = static_cast<uint64_t>(c.demod_taps);
    s.lut_octets = (7 + k + 7) / 8; // pipeline.cpp:323
    s.premf_taps = static_cast<uint64_t>(decimation_filter_taps(c.pre_mf_decimation));
    s.comp_len = static_cast<uint64_t>(c.smoothing_taps) +
                 static_cast<uint64_t>(decimation_filter_taps(c.post_envelope_decimation)) - 1;
    // Demodulation window (pipeline.cpp:390-399)
    const int64_t kk = c.demod_taps, d = c.demod_decimation, center = (kk - 1) / 2;
    s.m_lo = (center + d - 1) / d;
    const int64_t limit = (static_cast<int64_t>(s.frames) - kk + center) / d + 1;
    s.m_hi = std::min<int64_t>(static_cast<int64_t>(s.demod_len), std::max(s.m_lo, limit));
    return s;
}

Plan make_plan(const sn_pipeline_config& cin) {
    Plan p;
    p.cfg = cin;
    p.sz = derive_sizes(cin);
    check_geometry(cin);
    p.directions.assign(cin.directions, cin.directions + 2 * cin.n_directions);
    p.cfg.directions = nullptr;
    for (uint64_t d = 0; d < p.sz.n_dirs; ++d) check_direction(p.directions[2 * d], p.directions[2 * d + 1]);
    const Sizes& s = p.sz;
    const sn_pipeline_config& c = p.cfg;

    // Demodulation low-pass and its byte lookup table (pipeline.cpp:260-263,
    // 321-341): LUT[a][t][v] = sum over the 8 bits of v (MSB first) of
    // +/- rev[8t + bit - a], accumulated from +0.0 in bit order.
    p.demod_rev = reversed(design_lowpass(c.demod_cutoff_hz, c.pdm_rate, c.demod_taps));
    const uint64_t K = p.demod_rev.size(), T = s.lut_octets;
    p.demod_lut.assign(8 * T * 256, 0.0);
    for (uint64_t a = 0; a < 8; ++a) {
        for (uint64_t t = 0; t < T; ++t) {
            double* row = p.demod_lut.data() + (a * T + t) * 256;
            for (uint32_t v = 0; v < 256; ++v) {
                double acc = 0.0;
                for (uint32_t bit = 0; bit < 8; ++bit) {
                    const int64_t idx = static_cast<int64_t>(8 * t + bit) - static_cast<int64_t>(a);
                    if (idx < 0 || idx >= static_cast<int64_t>(K)) continue;
                    acc += ((v >> (7 - bit)) & 1u) ? p.demod_rev[idx] : -p.demod_rev[idx];
                }
                row[v] = acc;
            }
        }
    }
    // Pre-MF anti-alias (pipeline.cpp:268-271).
    p.premf_rev = reversed(design_lowpass(0.45 * s.demod_rate / c.pre_mf_decimation, s.demod_rate,
                                          decimation_filter_taps(c.pre_mf_decimation)));
    // Matched-filter reference (pipeline.cpp:274).
    p.chirp_ref = chirp(c, s.mf_rate);
    // Steering tables at the MF rate (pipeline.cpp:284-293; geometry.cpp:245-280).
    p.delays.resize(s.n_dirs * kCh);
    p.advances.resize(s.n_dirs);
    for (uint64_t d = 0; d < s.n_dirs; ++d) {
        const V3 u = unit_vector(p.directions[2 * d], p.directions[2 * d + 1]);
        double raw[kCh];
        double lo = std::numeric_limits<double>::infinity();
        for (int i = 0; i < kCh; ++i) {
            raw[i] = dot(mic(c, i), u) / c.speed_of_sound;
            lo = std::min(lo, raw[i]);
        }
        for (int i = 0; i < kCh; ++i) {
            p.delays[d * kCh + i] = static_cast<int32_t>(std::llround((raw[i] - lo) * s.mf_rate));
        }
        p.advances[d] = static_cast<int32_t>(std::llround(-lo * s.mf_rate));
    }
    // Direction schedule: recursive median bisection (k-d tree) of the
    // boresight-plane components (u_y, u_z) of the unit vectors into leaves of
    // kClusterDirs directions; leaves are laid out consecutively, so the 8
    // directions a beamformer warp processes together are angular neighbours
    // with per-channel shift spreads of a few samples. Scheduling only: every
    // direction is independent (pipeline.cpp:225-226).
    {
        std::vector<double> uy(s.n_dirs), uz(s.n_dirs);
        for (uint64_t d = 0; d < s.n_dirs; ++d) {
            const V3 u = unit_vector(p.directions[2 * d], p.directions[2 * d + 1]);
            uy[d] = u.y;
            uz[d] = u.z;
        }
        std::vector<int32_t> idx(s.n_dirs);
        std::iota(idx.begin(), idx.end(), 0);
        std::vector<int32_t> leaves;
        leaves.reserve(s.n_dirs);
        // two levels: subtrees of <= kTcLeafDirs directions (filled to
        // kTcLeafDirs where possible: the tensor-core beamformer's clusters,
        // compact in direction space so their per-channel shift spans stay
        // small), each split further into kClusterDirs leaves
        std::vector<int32_t> tc_leaves;
        auto split = [&](auto&& self, int32_t* b, int32_t* e, bool in_tc) -> void {
            const int64_t n = e - b;
            if (!in_tc && n <= kTcLeafDirs) {
                tc_leaves.push_back((int32_t)leaves.size());
                in_tc = true;
            }
            if (n <= kClusterDirs) {
                leaves.insert(leaves.end(), b, e);
                return;
            }
            double ylo = 1e9, yhi = -1e9, zlo = 1e9, zhi = -1e9;
            for (int32_t* q = b; q != e; ++q) {
                ylo = std::min(ylo, uy[*q]);
                yhi = std::max(yhi, uy[*q]);
                zlo = std::min(zlo, uz[*q]);
                zhi = std::max(zhi, uz[*q]);
            }
            const std::vector<double>& key = (yhi - ylo >= zhi - zlo) ? uy : uz;
            std::stable_sort(b, e, [&](int32_t x, int32_t y) { return key[x] < key[y]; });
            const int64_t unit = in_tc ? kClusterDirs : kTcLeafDirs;
            int64_t nl = unit * ((n + 2 * unit - 1) / (2 * unit));
            if (nl >= n) nl = n / 2;
            self(self, b, b + nl, in_tc);
            self(self, b + nl, e, in_tc);
        };
        split(split, idx.data(), idx.data() + idx.size(), false);
        tc_leaves.push_back((int32_t)s.n_dirs);
        // tensor-core clusters: balanced k-means in the shift vectors' 2-D
        // embedding when that lowers the MMA work (cluster.cpp)
        rebalance_tc_clusters(p, s.n_dirs, leaves, tc_leaves);
        p.tc_leaves = std::move(tc_leaves);
        std::vector<std::pair<uint64_t, int32_t>> keyed(s.n_dirs);
        for (uint64_t k = 0; k < s.n_dirs; ++k) keyed[k] = {k, leaves[k]};
        p.order.resize(s.n_dirs);
        p.shifts.resize(s.n_dirs * kCh);
        int32_t halo = 0;
        for (uint64_t slot = 0; slot < s.n_dirs; ++slot) {
            const int32_t d = keyed[slot].second;
            p.order[slot] = d;
            for (int i = 0; i < kCh; ++i) {
                const int32_t sh = p.delays[d * kCh + i] - p.advances[d];
                p.shifts[slot * kCh + i] = sh;
                halo = std::max(halo, std::abs(sh));
            }
        }
        p.halo = halo;
    }
    // Composite smoothing (127 taps) * post-envelope anti-alias (321 taps)
    // (pipeline.cpp:307-318).
    const auto smooth = design_lowpass(c.smoothing_cutoff_hz, s.mf_rate, c.smoothing_taps);
    const auto post = design_lowpass(0.45 * s.mf_rate / c.post_envelope_decimation, s.mf_rate,
                                     decimation_filter_taps(c.post_envelope_decimation));
    std::vector<double> comp(smooth.size() + post.size() - 1, 0.0);
    for (size_t i = 0; i < smooth.size(); ++i) {
        for (size_t j = 0; j < post.size(); ++j) comp[i + j] += smooth[i] * post[j];
    }
    p.comp_rev = reversed(std::move(comp));
    return p;
}

SceneEchoes scene_echoes(const sn_pipeline_config& c, const sn_scene& scene) {
    // synthesize_scene (synth.cpp:11-61): per reflector the amplitude and the
    // per-channel onset of the pulse at the PDM rate
    const Sizes s = derive_sizes(c);
    check_geometry(c);
    if (scene.noise_rms < 0.0) argument_error("synthesize_scene: noise_rms < 0");
    SceneEchoes e;
    e.frames = s.frames;
    e.pulse = chirp(c, c.pdm_rate);
    const auto ref_len = static_cast<int64_t>(e.pulse.size());
    for (uint64_t k = 0; k < scene.n_reflectors; ++k) {
        const sn_reflector& r = scene.reflectors[k];
        if (!(r.range > 0.0)) argument_error("reflector " + std::to_string(k) + ": range must be > 0");
        if (!(r.reflectivity >= 0.0) || !std::isfinite(r.reflectivity)) {
            argument_error("reflector " + std::to_string(k) + ": reflectivity must be finite and >= 0");
        }
        const double amplitude = r.reflectivity / (r.range * r.range);
        check_direction(r.azimuth, r.elevation);
        const V3 u = unit_vector(r.azimuth, r.elevation);
        const double round_trip = 2.0 * r.range / c.speed_of_sound;
        e.amplitude.push_back(amplitude);
        for (int ch = 0; ch < kCh; ++ch) {
            const double arrival = round_trip - dot(mic(c, ch), u) / c.speed_of_sound;
            const long onset = std::lround(arrival * c.pdm_rate);
            if (onset + ref_len > static_cast<int64_t>(s.frames)) {
                argument_error("reflector " + std::to_string(k) + ": echo ends past the capture window");
            }
            e.onset.push_back((int64_t)onset);
        }
    }
    return e;
}

void synthesize_packed(const sn_pipeline_config& c, const sn_scene& scene, uint8_t* out) {
    // synth.cpp:116-134 = synthesize_scene (:11-61) -> sigma_delta (:63-94) -> pack (:96-114)
    const SceneEchoes e = scene_echoes(c, scene);
    const uint64_t n = e.frames;
    const std::vector<double>& pulse = e.pulse;
    const auto ref_len = static_cast<int64_t>(pulse.size());
    std::vector<double> x(static_cast<size_t>(kCh) * n, 0.0);
    for (size_t k = 0; k < e.amplitude.size(); ++k) {
        const double amplitude = e.amplitude[k];
        for (int ch = 0; ch < kCh; ++ch) {
            const long onset = (long)e.onset[k * kCh + ch];
            double* dst = x.data() + static_cast<size_t>(ch) * n;
            for (long i = std::max<long>(0, onset); i < onset + ref_len; ++i) {
                dst[i] += amplitude * pulse[static_cast<size_t>(i - onset)];
            }
        }
    }
    if (scene.noise_rms > 0.0) {
        Xoshiro rng(scene.seed);
        for (double& v : x) v += scene.noise_rms * rng.normal();
    }
    std::memset(out, 0, static_cast<size_t>(kCh) * n / 8);
    for (int ch = 0; ch < kCh; ++ch) {
        const double* xc = x.data() + static_cast<size_t>(ch) * n;
        double integ = 0.0;
        for (uint64_t i = 0; i < n; ++i) {
            const double v = std::clamp(xc[i], -1.0, 1.0);
            const int bit = (integ + v >= 0.0) ? 1 : -1;
            integ += v - bit;
            if (bit > 0) {
                const uint64_t bi = i * kCh + static_cast<uint64_t>(ch);
                out[bi / 8] |= static_cast<uint8_t>(1u << (7 - (bi % 8)));
            }
        }
    }
}

} // namespace snb
