/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 *
 * A checker, never the product: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it. Every function cites the
 * reference file:line it restates (paths relative to
 * /root/reference/proj/core/). Pinning: tests/test_oracle.py checks this
 * port against the unmodified reference (oracle/_ref) and against the
 * committed golden fixtures (tests/golden/); the integer and FP64 front-end
 * stages agree bit-for-bit, the FFT-based stages to ~1e-12 relative.
 *
 * Differences that are NOT algorithmic: the matched filter is evaluated as
 * the direct 675-tap correlation the FFT route computes (pipeline.cpp:555-562
 * with N >= mf_len + ref_len - 1, so no circular wrap), and the Hilbert
 * transform uses a plain radix-2 FFT instead of FFTW.
 */
#include "oracle_api.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NCH 32
static const double PI = 3.141592653589793; /* std::numbers::pi */

/* ---- errors ----------------------------------------------------------- */
static __thread char g_err[256];
const char* port_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
    strncpy(g_err, msg, sizeof(g_err) - 1);
    return code;
}

/* ---- rng.hpp:11-58 xoshiro256++ / splitmix64 / polar Box-Muller ---------- */
typedef struct {
    uint64_t s[4];
    double spare;
    int have_spare;
} rng_t;
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static void rng_init(rng_t* r, uint64_t seed) { /* rng.hpp:15-24 */
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) {
        x += 0x9e3779b97f4a7c15ULL;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        r->s[i] = z ^ (z >> 31);
    }
    r->spare = 0.0;
    r->have_spare = 0;
}
static uint64_t rng_next(rng_t* r) { /* rng.hpp:26-36 */
    uint64_t* s = r->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}
static double rng_uniform(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform2(rng_t* r, double lo, double hi) { return lo + (hi - lo) * rng_uniform(r); }
static double rng_gaussian(rng_t* r) { /* rng.hpp:44-58 */
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u, v, s;
    do {
        u = 2.0 * rng_uniform(r) - 1.0;
        v = 2.0 * rng_uniform(r) - 1.0;
        s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    const double m = sqrt(-2.0 * log(s) / s);
    r->spare = v * m;
    r->have_spare = 1;
    return u * m;
}

/* ---- geometry.cpp ------------------------------------------------------ */
static double dist3(const double* a, const double* b) { /* geometry.cpp:18-23 */
    const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
    return sqrt(dx * dx + dy * dy + dz * dz);
}
static double dot3(const double* a, const double* b) { /* geometry.hpp:19-21 */
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

int port_default_array(uint64_t seed, double* out) { /* geometry.cpp:69-96 */
    const double disk = 0.046, axial = 0.002, min_spacing = 0.004;
    rng_t r;
    rng_init(&r, seed);
    int placed = 0;
    while (placed < NCH) {
        const double rad = disk * sqrt(rng_uniform(&r));
        const double theta = rng_uniform2(&r, 0.0, 2.0 * PI);
        double cand[3];
        cand[0] = rng_uniform2(&r, -axial, axial);
        cand[1] = rad * cos(theta);
        cand[2] = rad * sin(theta);
        int ok = 1;
        for (int i = 0; i < placed; ++i) {
            if (dist3(cand, out + 3 * i) < min_spacing) {
                ok = 0;
                break;
            }
        }
        if (ok) {
            memcpy(out + 3 * placed, cand, sizeof cand);
            ++placed;
        }
    }
    return 0;
}

static int cmp_dir(const void* pa, const void* pb) { /* geometry.cpp:224-228 */
    const double* a = (const double*)pa;
    const double* b = (const double*)pb;
    if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
    return 0;
}

int port_direction_grid(int kind, double* out, uint64_t cap, uint64_t* n_out) {
    /* geometry.cpp:181-235 */
    if (kind == 0) {
        const int n = 90;
        *n_out = n;
        if (!out) return 0;
        if (cap < (uint64_t)n) return fail(2, "capacity");
        for (int k = 0; k < n; ++k) {
            out[2 * k] = -PI / 2 + PI * (double)k / (n - 1);
            out[2 * k + 1] = 0.0;
        }
        return 0;
    }
    if (kind == 1) {
        const int n_az = 50, n_el = 37;
        *n_out = n_az * n_el;
        if (!out) return 0;
        if (cap < (uint64_t)(n_az * n_el)) return fail(2, "capacity");
        int i = 0;
        for (int e = 0; e < n_el; ++e) {
            const double el = -PI / 4 + (PI / 2) * (double)e / (n_el - 1);
            for (int a = 0; a < n_az; ++a) {
                out[2 * i] = -PI / 4 + (PI / 2) * (double)a / (n_az - 1);
                out[2 * i + 1] = el;
                ++i;
            }
        }
        return 0;
    }
    if (kind == 2) {
        const int n = 3000;
        *n_out = n;
        if (!out) return 0;
        if (cap < (uint64_t)n) return fail(2, "capacity");
        const double golden = PI * (3.0 - sqrt(5.0));
        for (int i = 0; i < n; ++i) {
            const double x = ((double)i + 0.5) / n;
            const double r = sqrt(1.0 - x * x);
            const double phi = golden * (double)i;
            const double y = r * cos(phi);
            const double z = r * sin(phi);
            double zc = z < -1.0 ? -1.0 : (z > 1.0 ? 1.0 : z);
            out[2 * i] = atan2(y, x);
            out[2 * i + 1] = asin(zc);
        }
        qsort(out, (size_t)n, 2 * sizeof(double), cmp_dir);
        return 0;
    }
    return fail(1, "direction_grid: custom grids are built from explicit lists");
}

static void unit_vec(double az, double el, double* u) { /* geometry.cpp:161-164 */
    const double ce = cos(el);
    u[0] = ce * cos(az);
    u[1] = ce * sin(az);
    u[2] = sin(el);
}

/* geometry.cpp:245-265 steering_delays, :267-280 steering_reference_advance */
static void steering(const double* mics, double az, double el, double c, double fs,
                     int32_t* delays, int32_t* advance) {
    double u[3], raw[NCH];
    unit_vec(az, el, u);
    double lo = INFINITY;
    for (int i = 0; i < NCH; ++i) {
        raw[i] = dot3(mics + 3 * i, u) / c;
        lo = raw[i] < lo ? raw[i] : lo; /* std::min(lo, raw) */
    }
    for (int i = 0; i < NCH; ++i) delays[i] = (int32_t)llround((raw[i] - lo) * fs);
    *advance = (int32_t)llround(-lo * fs);
}

/* ---- dsp.cpp ------------------------------------------------------------- */
static int design_lowpass(double cutoff, double fs, int taps, double* k) {
    /* dsp.cpp:129-166 */
    if (!(cutoff > 0.0 && cutoff < fs / 2)) return fail(1, "design_lowpass: cutoff");
    if (taps < 3 || taps % 2 == 0) return fail(1, "design_lowpass: taps must be odd and >= 3");
    const double fc = cutoff / fs;
    const int mid = (taps - 1) / 2;
    for (int n = 0; n < taps; ++n) {
        const int m = n - mid;
        const double sinc = m == 0 ? 2.0 * fc : sin(2.0 * PI * fc * m) / (PI * m);
        const double window = 0.54 - 0.46 * cos(2.0 * PI * n / (taps - 1));
        k[n] = sinc * window;
    }
    double nyquist = 0.0;
    for (int n = 0; n < taps; ++n) nyquist += (n % 2 == 0 ? k[n] : -k[n]);
    const double correction = nyquist / taps;
    double sum = 0.0;
    for (int n = 0; n < taps; ++n) {
        k[n] -= (n % 2 == 0 ? correction : -correction);
        sum += k[n];
    }
    for (int n = 0; n < taps; ++n) k[n] /= sum;
    return 0;
}

static int decimation_filter_taps(int factor) { /* dsp.cpp:285-288 */
    int t = 32 * factor;
    t = t < 63 ? 63 : (t > 1023 ? 1023 : t);
    return t % 2 == 0 ? t + 1 : t;
}

static size_t chirp_length(double duration, double fs) { /* dsp.cpp:84-86 */
    return (size_t)llround(duration * fs);
}

static void generate_chirp(double f0, double f1, double duration, double fs, double* s,
                           size_t n) { /* dsp.cpp:229-240 */
    const double slope = (f1 - f0) / (2.0 * duration);
    for (size_t i = 0; i < n; ++i) {
        const double t = (double)i / fs;
        s[i] = sin(2.0 * PI * (f0 * t + slope * t * t));
    }
}

/* filters.hpp:14-39 strided_filter, exact 4-lane summation order. */
static void strided_filter(const double* x, size_t len, const double* rev, long k, long start,
                           long stride, double* out, size_t out_len) {
    const long n_in = (long)len;
    for (size_t m = 0; m < out_len; ++m) {
        const long s = start + (long)m * stride;
        const long lo = s > 0 ? s : 0;
        const long hi = (s + k) < n_in ? (s + k) : n_in;
        const double* xs = x + lo;
        const double* h = rev + (lo - s);
        const long n = hi - lo;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        long j = 0;
        for (; j + 4 <= n; j += 4) {
            a0 += h[j] * xs[j];
            a1 += h[j + 1] * xs[j + 1];
            a2 += h[j + 2] * xs[j + 2];
            a3 += h[j + 3] * xs[j + 3];
        }
        double acc = (a0 + a1) + (a2 + a3);
        for (; j < n; ++j) acc += h[j] * xs[j];
        out[m] = acc;
    }
}

/* ---- radix-2 complex FFT (stands in for FFTW, fft.cpp) ---------------- */
static void fft_c(double* re, double* im, size_t n, int sign) {
    size_t j = 0;
    for (size_t i = 1; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            double t = re[i]; re[i] = re[j]; re[j] = t;
            t = im[i]; im[i] = im[j]; im[j] = t;
        }
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len >> 1;
        for (size_t k = 0; k < half; ++k) {
            const double a = (double)sign * 2.0 * PI * (double)k / (double)len;
            const double wr = cos(a), wi = sin(a);
            for (size_t s0 = 0; s0 < n; s0 += len) {
                const size_t p = s0 + k, q = p + half;
                const double tr = re[q] * wr - im[q] * wi;
                const double ti = re[q] * wi + im[q] * wr;
                re[q] = re[p] - tr;
                im[q] = im[p] - ti;
                re[p] += tr;
                im[p] += ti;
            }
        }
    }
}

static size_t next_pow2(size_t n) { /* fft.cpp:22-26 */
    size_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

/* ---- pipeline.cpp -------------------------------------------------------- */
typedef struct {
    size_t frames, demod_len, mf_len, bins, ref_len, n_dirs, mf_fft, env_fft, lut_octets;
    double demod_rate, mf_rate, final_rate, range_bin_size;
} dims_t;

static size_t lcm_sz(size_t a, size_t b) {
    size_t x = a, y = b;
    while (y) {
        size_t t = x % y;
        x = y;
        y = t;
    }
    return a / x * b;
}

static int derive(const orc_config* c, dims_t* d) {
    /* pipeline.cpp:60-92 validate (the numeric subset) */
    if (c->n_directions == 0) return fail(1, "pipeline: empty direction set");
    if (c->pdm_rate <= 0.0) return fail(1, "pipeline: pdm_rate must be > 0");
    if (c->demod_decimation < 1 || c->pre_mf_decimation < 1 || c->post_envelope_decimation < 1)
        return fail(1, "pipeline: decimation factors must be >= 1");
    if (c->demod_taps < 3 || c->demod_taps % 2 == 0) return fail(1, "pipeline: demod taps");
    if (c->smoothing_taps < 3 || c->smoothing_taps % 2 == 0) return fail(1, "pipeline: smoothing taps");
    if (c->speed_of_sound <= 0.0) return fail(1, "pipeline: speed_of_sound must be > 0");
    if (c->max_range <= 0.0) return fail(1, "pipeline: max_range must be > 0");
    d->demod_rate = c->pdm_rate / c->demod_decimation;          /* pipeline.hpp:38 */
    d->mf_rate = d->demod_rate / c->pre_mf_decimation;            /* pipeline.hpp:39 */
    d->final_rate = d->mf_rate / c->post_envelope_decimation;     /* pipeline.hpp:40 */
    /* pipeline.cpp:40-48 frames() */
    const double window = 2.0 * c->max_range / c->speed_of_sound + c->chirp_duration;
    const size_t raw = (size_t)ceil(window * c->pdm_rate);
    const size_t stage = (size_t)c->demod_decimation * (size_t)c->pre_mf_decimation *
                         (size_t)c->post_envelope_decimation;
    const size_t step = lcm_sz(8, stage);
    d->frames = (raw + step - 1) / step * step;
    d->demod_len = d->frames / (size_t)c->demod_decimation;
    d->mf_len = d->demod_len / (size_t)c->pre_mf_decimation;
    /* pipeline.cpp:50-52 range_bins() */
    d->bins = (size_t)floor(2.0 * c->max_range / c->speed_of_sound * d->final_rate);
    d->range_bin_size = c->speed_of_sound / (2.0 * d->final_rate);
    if (d->bins < 1) return fail(1, "pipeline: derived range-bin count is zero");
    d->ref_len = chirp_length(c->chirp_duration, d->mf_rate);
    if (d->ref_len > d->mf_len) return fail(1, "pipeline: reference chirp longer than the processed window");
    if (d->ref_len < 2) return fail(1, "pipeline: reference chirp shorter than 2 samples");
    d->n_dirs = c->n_directions;
    d->mf_fft = next_pow2(d->mf_len + d->ref_len - 1);
    d->env_fft = next_pow2(d->mf_len);
    d->lut_octets = (7 + (size_t)c->demod_taps + 7) / 8;            /* pipeline.cpp:323 */
    return 0;
}

int port_dims(const orc_config* c, uint64_t* dims, double* rbs) {
    dims_t d;
    int rc = derive(c, &d);
    if (rc) return rc;
    dims[0] = d.frames;
    dims[1] = d.demod_len;
    dims[2] = d.mf_len;
    dims[3] = d.bins;
    dims[4] = d.n_dirs;
    dims[5] = d.ref_len;
    dims[6] = d.mf_fft;
    dims[7] = d.env_fft;
    dims[8] = (size_t)c->smoothing_taps + (size_t)decimation_filter_taps(c->post_envelope_decimation) - 1;
    dims[9] = d.lut_octets;
    *rbs = d.range_bin_size;
    return 0;
}

/* pipeline.cpp:321-341 build_demod_lut */
static void build_lut(const double* rev, size_t k, size_t octets, double* lut) {
    for (size_t a = 0; a < 8; ++a)
        for (size_t t = 0; t < octets; ++t) {
            double* entry = lut + (a * octets + t) * 256;
            for (size_t v = 0; v < 256; ++v) {
                double acc = 0.0;
                for (size_t bit = 0; bit < 8; ++bit) {
                    const long idx = (long)(8 * t + bit) - (long)a;
                    if (idx < 0 || idx >= (long)k) continue;
                    const int one = ((v >> (7 - bit)) & 1) != 0;
                    acc += one ? rev[idx] : -rev[idx];
                }
                entry[v] = acc;
            }
        }
}

/* Setup tables (pipeline.cpp:260-318). which: 0 demod_rev, 1 lut, 2 premf_rev,
 * 3 chirp ref @ mf rate, 4 smooth_decimate_rev */
int port_table(const orc_config* c, int which, double* out, uint64_t cap, uint64_t* n_out) {
    dims_t d;
    int rc = derive(c, &d);
    if (rc) return rc;
    size_t n = 0;
    double* tmp = NULL;
    switch (which) {
        case 0:
        case 1: {
            const size_t k = (size_t)c->demod_taps;
            tmp = (double*)malloc(sizeof(double) * k);
            rc = design_lowpass(c->demod_cutoff_hz, c->pdm_rate, c->demod_taps, tmp);
            if (rc) break;
            double* rev = (double*)malloc(sizeof(double) * k);
            for (size_t i = 0; i < k; ++i) rev[i] = tmp[k - 1 - i];
            free(tmp);
            if (which == 0) {
                tmp = rev;
                n = k;
            } else {
                n = 8 * d.lut_octets * 256;
                tmp = (double*)malloc(sizeof(double) * n);
                build_lut(rev, k, d.lut_octets, tmp);
                free(rev);
            }
            break;
        }
        case 2: {
            const int taps = decimation_filter_taps(c->pre_mf_decimation);
            double* k = (double*)malloc(sizeof(double) * taps);
            rc = design_lowpass(0.45 * d.demod_rate / c->pre_mf_decimation, d.demod_rate, taps, k);
            n = (size_t)taps;
            tmp = (double*)malloc(sizeof(double) * n);
            for (size_t i = 0; i < n; ++i) tmp[i] = k[n - 1 - i];
            free(k);
            break;
        }
        case 3:
            n = d.ref_len;
            tmp = (double*)malloc(sizeof(double) * n);
            generate_chirp(c->chirp_f_start, c->chirp_f_end, c->chirp_duration, d.mf_rate, tmp, n);
            break;
        case 4: {
            const int ts = c->smoothing_taps;
            const int tp = decimation_filter_taps(c->post_envelope_decimation);
            double* s = (double*)malloc(sizeof(double) * ts);
            double* p = (double*)malloc(sizeof(double) * tp);
            rc = design_lowpass(c->smoothing_cutoff_hz, d.mf_rate, ts, s);
            if (!rc) rc = design_lowpass(0.45 * d.mf_rate / c->post_envelope_decimation, d.mf_rate, tp, p);
            n = (size_t)(ts + tp - 1);
            double* comp = (double*)calloc(n, sizeof(double));
            for (int i = 0; i < ts; ++i)
                for (int j = 0; j < tp; ++j) comp[i + j] += s[i] * p[j];  /* pipeline.cpp:312-317 */
            tmp = (double*)malloc(sizeof(double) * n);
            for (size_t i = 0; i < n; ++i) tmp[i] = comp[n - 1 - i];
            free(s);
            free(p);
            free(comp);
            break;
        }
        default: return fail(2, "bad table");
    }
    if (rc) {
        free(tmp);
        return rc;
    }
    *n_out = n;
    if (out) {
        if (cap < n) {
            free(tmp);
            return fail(2, "capacity");
        }
        memcpy(out, tmp, n * sizeof(double));
    }
    free(tmp);
    return 0;
}

int port_steering(const orc_config* c, int32_t* delays, int32_t* advances) {
    dims_t d;
    int rc = derive(c, &d);
    if (rc) return rc;
    for (size_t i = 0; i < d.n_dirs; ++i)
        steering(c->mic_xyz, c->directions[2 * i], c->directions[2 * i + 1], c->speed_of_sound,
                 d.mf_rate, delays + NCH * i, advances + i);
    return 0;
}

/* pipeline.cpp:27-36 transpose32 restated bit by bit + :352-385 layout:
 * row c byte b holds frames 8b..8b+7, MSB first. */
static void transpose_rows(const uint8_t* packed, size_t frames, uint8_t* rows, size_t stride) {
    memset(rows, 0, NCH * stride);
    for (size_t f = 0; f < frames; ++f)
        for (int c = 0; c < NCH; ++c) {
            const size_t bit_index = f * NCH + (size_t)c;
            const int bit = (packed[bit_index / 8] >> (7 - (bit_index % 8))) & 1;
            if (bit) rows[(size_t)c * stride + f / 8] |= (uint8_t)(1u << (7 - (f % 8)));
        }
}

/* pipeline.cpp:387-430 demodulate_channel */
static void demodulate(const orc_config* c, const dims_t* d, const uint8_t* row, const double* lut,
                       double* out) {
    const long k = c->demod_taps, dd = c->demod_decimation, center = (k - 1) / 2;
    const long total = (long)d->frames;
    const long m_lo = (center + dd - 1) / dd;
    long m_hi = (long)d->demod_len;
    const long limit = (total - k + center) / dd + 1;
    const long mx = m_lo > limit ? m_lo : limit;
    m_hi = m_hi < mx ? m_hi : mx;
    for (long m = 0; m < (m_lo < (long)d->demod_len ? m_lo : (long)d->demod_len); ++m) out[m] = 0.0;
    for (long m = m_hi; m < (long)d->demod_len; ++m) out[m] = 0.0;
    const size_t octets = d->lut_octets;
    for (long m = m_lo; m < m_hi; ++m) {
        const long s = m * dd - center;
        const size_t base = (size_t)s >> 3, align = (size_t)s & 7;
        const double* table = lut + align * octets * 256;
        const uint8_t* bytes = row + base;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        size_t t = 0;
        for (; t + 4 <= octets; t += 4) {
            a0 += table[(t + 0) * 256 + bytes[t + 0]];
            a1 += table[(t + 1) * 256 + bytes[t + 1]];
            a2 += table[(t + 2) * 256 + bytes[t + 2]];
            a3 += table[(t + 3) * 256 + bytes[t + 3]];
        }
        double acc = (a0 + a1) + (a2 + a3);
        for (; t < octets; ++t) acc += table[t * 256 + bytes[t]];
        out[m] = acc;
    }
}

/* Full process (pipeline.cpp:522-574). Stage outputs optional. */
int port_process(const orc_config* c, const uint8_t* packed, uint64_t packed_len, float* energies,
                 double* demod_out, double* mf_out, double* filt_out) {
    dims_t d;
    int rc = derive(c, &d);
    if (rc) return rc;
    if (packed_len != (uint64_t)NCH * d.frames / 8) return fail(3, "process: payload size");
    const size_t K = (size_t)c->demod_taps;
    uint64_t nt;
    double* lut = (double*)malloc(sizeof(double) * 8 * d.lut_octets * 256);
    port_table(c, 1, lut, 8 * d.lut_octets * 256, &nt);
    const int premf_taps = decimation_filter_taps(c->pre_mf_decimation);
    double* premf_rev = (double*)malloc(sizeof(double) * premf_taps);
    port_table(c, 2, premf_rev, premf_taps, &nt);
    double* ref = (double*)malloc(sizeof(double) * d.ref_len);
    port_table(c, 3, ref, d.ref_len, &nt);
    const size_t comp_len = (size_t)c->smoothing_taps + (size_t)decimation_filter_taps(c->post_envelope_decimation) - 1;
    double* comp_rev = (double*)malloc(sizeof(double) * comp_len);
    port_table(c, 4, comp_rev, comp_len, &nt);
    (void)K;

    const size_t stride = d.frames / 8 + d.lut_octets;
    uint8_t* rows = (uint8_t*)malloc(NCH * stride);
    transpose_rows(packed, d.frames, rows, stride);
    double* demod = (double*)malloc(sizeof(double) * NCH * d.demod_len);
    double* mf = (double*)malloc(sizeof(double) * NCH * d.mf_len);
    double* filt = (double*)malloc(sizeof(double) * NCH * d.mf_len);
    for (int ch = 0; ch < NCH; ++ch) {
        demodulate(c, &d, rows + (size_t)ch * stride, lut, demod + (size_t)ch * d.demod_len);
        strided_filter(demod + (size_t)ch * d.demod_len, d.demod_len, premf_rev, premf_taps,
                       -(long)((premf_taps - 1) / 2), c->pre_mf_decimation,
                       mf + (size_t)ch * d.mf_len, d.mf_len);
        /* matched filter: filt[n] = sum_j mf[n+j] ref[j] (pipeline.cpp:555-562) */
        const double* x = mf + (size_t)ch * d.mf_len;
        for (size_t n = 0; n < d.mf_len; ++n) {
            double acc = 0.0;
            for (size_t j = 0; j < d.ref_len && n + j < d.mf_len; ++j) acc += x[n + j] * ref[j];
            filt[(size_t)ch * d.mf_len + n] = acc;
        }
    }
    if (demod_out) memcpy(demod_out, demod, sizeof(double) * NCH * d.demod_len);
    if (mf_out) memcpy(mf_out, mf, sizeof(double) * NCH * d.mf_len);
    if (filt_out) memcpy(filt_out, filt, sizeof(double) * NCH * d.mf_len);

    int32_t* delays = (int32_t*)malloc(sizeof(int32_t) * NCH * d.n_dirs);
    int32_t* adv = (int32_t*)malloc(sizeof(int32_t) * d.n_dirs);
    port_steering(c, delays, adv);
    const size_t N = d.env_fft, L = d.mf_len;
    double* beam = (double*)malloc(sizeof(double) * L);
    double* re = (double*)malloc(sizeof(double) * N);
    double* im = (double*)malloc(sizeof(double) * N);
    double* env = (double*)malloc(sizeof(double) * L);
    double* fin = (double*)malloc(sizeof(double) * d.bins);
    for (size_t dir = 0; dir < d.n_dirs; ++dir) {
        /* pipeline.cpp:432-446 beamform_into */
        for (size_t n = 0; n < L; ++n) beam[n] = 0.0;
        for (int i = 0; i < NCH; ++i) {
            const long shift = delays[dir * NCH + i] - adv[dir];
            const double* x = filt + (size_t)i * L;
            long n_lo = shift > 0 ? shift : 0;
            long n_hi = (long)L < (long)L + shift ? (long)L : (long)L + shift;
            for (long n = n_lo; n < n_hi; ++n) beam[n] += x[n - shift];
        }
        for (size_t n = 0; n < L; ++n) beam[n] *= 1.0 / NCH;
        /* pipeline.cpp:448-472 envelope_direction: Hilbert with DC/Nyquist zeroed */
        for (size_t n = 0; n < N; ++n) {
            re[n] = n < L ? beam[n] : 0.0;
            im[n] = 0.0;
        }
        fft_c(re, im, N, -1);
        re[0] = im[0] = 0.0;
        re[N / 2] = im[N / 2] = 0.0;
        for (size_t k = 1; k < N / 2; ++k) { /* X -> -i X on positive bins */
            const double a = re[k], b = im[k];
            re[k] = b;
            im[k] = -a;
        }
        for (size_t k = N / 2 + 1; k < N; ++k) { /* Hermitian: conj of the mirror */
            re[k] = re[N - k];
            im[k] = -im[N - k];
        }
        fft_c(re, im, N, +1);
        for (size_t n = 0; n < L; ++n) {
            const double h = re[n] / (double)N;
            env[n] = sqrt(beam[n] * beam[n] + h * h);
        }
        strided_filter(env, L, comp_rev, (long)comp_len, -(long)((comp_len - 1) / 2),
                       c->post_envelope_decimation, fin, d.bins);
        for (size_t k = 0; k < d.bins; ++k) {
            const float v = (float)fin[k];
            energies[dir * d.bins + k] = v > 0.0f ? v : 0.0f; /* std::max(0.0f, v) */
        }
    }
    free(lut); free(premf_rev); free(ref); free(comp_rev); free(rows); free(demod); free(mf);
    free(filt); free(delays); free(adv); free(beam); free(re); free(im); free(env); free(fin);
    return 0;
}

/* ---- synth.cpp:11-134 ----------------------------------------------------- */
int port_synthesize(const orc_config* c, const orc_scene* s, uint8_t* out, uint64_t cap) {
    dims_t d;
    int rc = derive(c, &d);
    if (rc) return rc;
    const size_t n = d.frames;
    if (cap < NCH * n / 8) return fail(2, "capacity");
    const size_t ref_len = chirp_length(c->chirp_duration, c->pdm_rate);
    double* ref = (double*)malloc(sizeof(double) * ref_len);
    generate_chirp(c->chirp_f_start, c->chirp_f_end, c->chirp_duration, c->pdm_rate, ref, ref_len);
    double* x = (double*)calloc(NCH * n, sizeof(double));
    for (uint64_t k = 0; k < s->n_reflectors; ++k) { /* synth.cpp:26-55 */
        const orc_reflector* r = &s->reflectors[k];
        const double amplitude = r->reflectivity / (r->range * r->range);
        double u[3];
        unit_vec(r->azimuth, r->elevation, u);
        const double round_trip = 2.0 * r->range / c->speed_of_sound;
        for (int ch = 0; ch < NCH; ++ch) {
            const double arrival = round_trip - dot3(c->mic_xyz + 3 * ch, u) / c->speed_of_sound;
            const long onset = lround(arrival * c->pdm_rate);
            if (onset + (long)ref_len > (long)n) {
                free(ref);
                free(x);
                return fail(2, "echo ends past the capture window");
            }
            double* dst = x + (size_t)ch * n;
            for (long i = onset > 0 ? onset : 0; i < onset + (long)ref_len; ++i)
                dst[i] += amplitude * ref[i - onset];
        }
    }
    if (s->noise_rms > 0.0) { /* synth.cpp:57-60 */
        rng_t g;
        rng_init(&g, s->seed);
        for (size_t i = 0; i < NCH * n; ++i) x[i] += s->noise_rms * rng_gaussian(&g);
    }
    memset(out, 0, NCH * n / 8);
    for (int ch = 0; ch < NCH; ++ch) { /* synth.cpp:63-94 sigma_delta_modulate */
        double integrator = 0.0;
        const double* xc = x + (size_t)ch * n;
        for (size_t i = 0; i < n; ++i) {
            double v = xc[i];
            if (v > 1.0) v = 1.0;
            else if (v < -1.0) v = -1.0;
            const int bit = (integrator + v >= 0.0) ? 1 : -1;
            integrator += v - bit;
            if (bit > 0) { /* synth.cpp:96-114 pack_pdm */
                const size_t bi = i * NCH + (size_t)ch;
                out[bi / 8] |= (uint8_t)(1u << (7 - (bi % 8)));
            }
        }
    }
    free(ref);
    free(x);
    return 0;
}
