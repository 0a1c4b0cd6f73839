/* TEST INFRASTRUCTURE ONLY — FFTW3 API subset for building the reference
 * oracle (oracle/_ref). See fftw3.h for the contract. Never linked into the
 * product library.
 *
 * Power-of-two complex sizes use an iterative radix-2 DIT transform with a
 * per-plan twiddle table (exact cos/sin per entry, no recurrences); real
 * transforms of even size n run through an n/2-point complex transform plus
 * the standard split/merge step. Everything else falls back to a direct DFT.
 */
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { KIND_R2C = 0, KIND_C2R = 1, KIND_DFT = 2 };

struct fftw_plan_s {
    int kind;
    int n;
    int sign;
    void* in;
    void* out;
    int m;              /* complex transform size used internally */
    double* tw;         /* m/2 twiddles e^{-2 pi i k/m} (re, im) */
    double* rtw;        /* n/2+1 twiddles e^{-2 pi i k/n} for real split/merge */
    int* rev;           /* bit reversal for m */
    double* work;       /* 2*m scratch */
};

static const double kTwoPi = 6.283185307179586476925286766559;

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

double* fftw_alloc_real(size_t n) { return (double*)malloc((n ? n : 1) * sizeof(double)); }
fftw_complex* fftw_alloc_complex(size_t n) {
    return (fftw_complex*)malloc((n ? n : 1) * sizeof(fftw_complex));
}
void fftw_free(void* p) { free(p); }

static void setup_complex(struct fftw_plan_s* p, int m) {
    p->m = m;
    p->work = (double*)calloc((size_t)(2 * (m > 0 ? m : 1)), sizeof(double));
    if (!is_pow2(m) || m < 2) return;
    p->tw = (double*)malloc(sizeof(double) * (size_t)m);
    for (int k = 0; k < m / 2; ++k) {
        const double a = -kTwoPi * (double)k / (double)m;
        p->tw[2 * k] = cos(a);
        p->tw[2 * k + 1] = sin(a);
    }
    p->rev = (int*)malloc(sizeof(int) * (size_t)m);
    int bits = 0;
    while ((1 << bits) < m) ++bits;
    for (int i = 0; i < m; ++i) {
        int r = 0;
        for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
        p->rev[i] = r;
    }
}

/* In-place complex transform of p->m points in buf (interleaved re/im).
 * sign = -1 forward, +1 backward; unnormalised. */
static void complex_transform(const struct fftw_plan_s* p, double* buf, int sign) {
    const int m = p->m;
    if (m <= 1) return;
    if (!is_pow2(m)) {
        double* tmp = p->work;
        for (int k = 0; k < m; ++k) {
            double re = 0.0, im = 0.0;
            for (int j = 0; j < m; ++j) {
                const double a = (double)sign * kTwoPi * (double)(((long long)j * k) % m) / m;
                const double c = cos(a), s = sin(a);
                re += buf[2 * j] * c - buf[2 * j + 1] * s;
                im += buf[2 * j] * s + buf[2 * j + 1] * c;
            }
            tmp[2 * k] = re;
            tmp[2 * k + 1] = im;
        }
        memcpy(buf, tmp, sizeof(double) * 2 * (size_t)m);
        return;
    }
    for (int i = 0; i < m; ++i) {
        const int r = p->rev[i];
        if (r > i) {
            double t0 = buf[2 * i], t1 = buf[2 * i + 1];
            buf[2 * i] = buf[2 * r];
            buf[2 * i + 1] = buf[2 * r + 1];
            buf[2 * r] = t0;
            buf[2 * r + 1] = t1;
        }
    }
    for (int len = 2; len <= m; len <<= 1) {
        const int half = len >> 1;
        const int step = m / len;
        for (int start = 0; start < m; start += len) {
            for (int k = 0; k < half; ++k) {
                const double wr = p->tw[2 * k * step];
                /* forward: w = tw; backward: conj(tw) */
                const double wi = sign < 0 ? p->tw[2 * k * step + 1] : -p->tw[2 * k * step + 1];
                const int a = start + k, b = a + half;
                const double xr = buf[2 * b], xi = buf[2 * b + 1];
                const double tr = xr * wr - xi * wi;
                const double ti = xr * wi + xi * wr;
                buf[2 * b] = buf[2 * a] - tr;
                buf[2 * b + 1] = buf[2 * a + 1] - ti;
                buf[2 * a] += tr;
                buf[2 * a + 1] += ti;
            }
        }
    }
}

static struct fftw_plan_s* new_plan(int kind, int n, int sign, void* in, void* out) {
    struct fftw_plan_s* p = (struct fftw_plan_s*)calloc(1, sizeof(*p));
    p->kind = kind;
    p->n = n;
    p->sign = sign;
    p->in = in;
    p->out = out;
    return p;
}

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
    (void)flags;
    struct fftw_plan_s* p = new_plan(KIND_DFT, n, sign, in, out);
    setup_complex(p, n);
    return p;
}

static void setup_real(struct fftw_plan_s* p) {
    const int n = p->n;
    if (n >= 2 && n % 2 == 0) {
        setup_complex(p, n / 2);
        p->rtw = (double*)malloc(sizeof(double) * (size_t)(n + 2));
        for (int k = 0; k <= n / 2; ++k) {
            const double a = -kTwoPi * (double)k / (double)n;
            p->rtw[2 * k] = cos(a);
            p->rtw[2 * k + 1] = sin(a);
        }
    } else {
        setup_complex(p, n);
    }
}

fftw_plan fftw_plan_dft_r2c_1d(int n, double* in, fftw_complex* out, unsigned flags) {
    (void)flags;
    struct fftw_plan_s* p = new_plan(KIND_R2C, n, -1, in, out);
    setup_real(p);
    return p;
}

fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex* in, double* out, unsigned flags) {
    (void)flags;
    struct fftw_plan_s* p = new_plan(KIND_C2R, n, +1, in, out);
    setup_real(p);
    return p;
}

static void exec_r2c(const struct fftw_plan_s* p) {
    const int n = p->n;
    const double* x = (const double*)p->in;
    double* X = (double*)p->out;
    double* z = p->work;
    if (n % 2 != 0 || n < 2) {
        for (int j = 0; j < n; ++j) {
            z[2 * j] = x[j];
            z[2 * j + 1] = 0.0;
        }
        complex_transform(p, z, -1);
        for (int k = 0; k <= n / 2; ++k) {
            X[2 * k] = z[2 * k];
            X[2 * k + 1] = z[2 * k + 1];
        }
        return;
    }
    const int m = n / 2;
    memcpy(z, x, sizeof(double) * (size_t)n); /* z[j] = x[2j] + i x[2j+1] */
    complex_transform(p, z, -1);
    for (int k = 0; k <= m; ++k) {
        const int k1 = k % m, k2 = (m - k) % m;
        const double zr = z[2 * k1], zi = z[2 * k1 + 1];
        const double cr = z[2 * k2], ci = -z[2 * k2 + 1]; /* conj(Z[m-k]) */
        const double er = 0.5 * (zr + cr), ei = 0.5 * (zi + ci);
        /* O = (Z - conj(Z[m-k])) / (2i) */
        const double dr = zr - cr, di = zi - ci;
        const double or_ = 0.5 * di, oi = -0.5 * dr;
        const double wr = p->rtw[2 * k], wi = p->rtw[2 * k + 1];
        X[2 * k] = er + (or_ * wr - oi * wi);
        X[2 * k + 1] = ei + (or_ * wi + oi * wr);
    }
}

static void exec_c2r(const struct fftw_plan_s* p) {
    const int n = p->n;
    const double* X = (const double*)p->in;
    double* x = (double*)p->out;
    double* z = p->work;
    if (n % 2 != 0 || n < 2) {
        for (int k = 0; k < n; ++k) {
            const int kk = k <= n / 2 ? k : n - k;
            z[2 * k] = X[2 * kk];
            z[2 * k + 1] = k <= n / 2 ? X[2 * kk + 1] : -X[2 * kk + 1];
        }
        z[1] = 0.0;
        complex_transform(p, z, +1);
        for (int j = 0; j < n; ++j) x[j] = z[2 * j];
        return;
    }
    const int m = n / 2;
    for (int k = 0; k < m; ++k) {
        double ar = X[2 * k], ai = X[2 * k + 1];
        double br = X[2 * (m - k)], bi = -X[2 * (m - k) + 1]; /* conj(X[m-k]) */
        if (k == 0) {
            ai = 0.0; /* imag(X[0]) and imag(X[n/2]) are ignored */
            bi = 0.0;
        }
        const double er = 0.5 * (ar + br), ei = 0.5 * (ai + bi);
        const double dr = 0.5 * (ar - br), di = 0.5 * (ai - bi);
        /* O = D * conj(W^k) */
        const double wr = p->rtw[2 * k], wi = -p->rtw[2 * k + 1];
        const double or_ = dr * wr - di * wi, oi = dr * wi + di * wr;
        /* Z = E + i O */
        z[2 * k] = er - oi;
        z[2 * k + 1] = ei + or_;
    }
    complex_transform(p, z, +1);
    for (int j = 0; j < m; ++j) {
        x[2 * j] = 2.0 * z[2 * j];
        x[2 * j + 1] = 2.0 * z[2 * j + 1];
    }
}

void fftw_execute(const fftw_plan p) {
    if (p == NULL) return;
    switch (p->kind) {
        case KIND_R2C: exec_r2c(p); break;
        case KIND_C2R: exec_c2r(p); break;
        default: {
            double* buf = p->work;
            memcpy(buf, p->in, sizeof(double) * 2 * (size_t)p->n);
            complex_transform(p, buf, p->sign);
            memcpy(p->out, buf, sizeof(double) * 2 * (size_t)p->n);
        }
    }
}

void fftw_destroy_plan(fftw_plan p) {
    if (p == NULL) return;
    free(p->tw);
    free(p->rtw);
    free(p->rev);
    free(p->work);
    free(p);
}
