// Hot-path kernels; see kernels.cuh for the stage map and layouts.
#include "fft.cuh"
#include "kernels.cuh"
#include "plan.hpp"

#include <cstdio>
#include <mutex>
#include <string>
#include <map>
#include <utility>

#ifndef SNB_ENV_MINB
#define SNB_ENV_MINB 2 // envelope CTAs per SM the register budget is sized for
#endif
#ifndef SNB_ENV_MINB_F32
#define SNB_ENV_MINB_F32 2
#endif
#include <type_traits>

namespace snb {

// ---------------------------------------------------------------------------
// k_demod: bit transpose + FP64 LUT demodulation, bit-exact with
// pipeline.cpp:352-430.
//
// The output index m of channel c reads the 255-frame window starting at
// s = D*m - center; with P = 8/gcd(D,8), every m of one residue class
// r = m mod P shares the bit alignment a = s & 7, so a CTA serves one class
// and keeps that alignment's 33 x 256 FP64 table (67.6 KB) in shared memory
// for its whole life (persistent grid over (measurement, block of m)).
// Frames are transposed into per-channel MSB-first rows by a 32 x 32 bit
// transpose across the warp (lane l holds frame word l; 5 shuffle stages). The sum per output follows the reference exactly: four lanes
// over octets t = 0 .. 4*floor(T/4)-1 (lane t mod 4), (a0+a1)+(a2+a3), then
// the remaining octets in order; adds only, every add rounded (DADD).
// ---------------------------------------------------------------------------
constexpr int kDemodOctets = 33; // the default 255-tap demodulator: 33 octets per output
__global__ void __launch_bounds__(kThreads) k_demod(DemodArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* lut = reinterpret_cast<double*>(smem);
    uint32_t* rows = reinterpret_cast<uint32_t*>(lut + (size_t)a.octets * 256);
    const int r = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    if (r >= a.demod_len) return;
    const int64_t s_r = (int64_t)a.decim * r - a.center;
    const int align = (int)(((s_r % 8) + 8) % 8);
    {
        const double* src = a.lut + (size_t)align * a.octets * 256;
        for (int i = threadIdx.x; i < a.octets * 256; i += blockDim.x) lut[i] = src[i];
    }
    const int64_t P = a.period;
    const int64_t Jr = (a.demod_len - r + P - 1) / P; // outputs of class r
    const int64_t nblk = (Jr + a.jblock - 1) / a.jblock;
    const int64_t items = nblk * a.batch;
    const int T = a.octets;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t b = it / nblk, jb = it % nblk;
        const int64_t j0 = jb * a.jblock, j1 = min(Jr, j0 + a.jblock);
        // j range whose m lies in [m_lo, m_hi)
        int64_t jv0 = a.m_lo > r ? (a.m_lo - r + P - 1) / P : 0;
        int64_t jv1 = a.m_hi > r ? (a.m_hi - r + P - 1) / P : 0;
        jv0 = max(jv0, j0);
        jv1 = min(jv1, j1);
        int64_t F0 = 0;
        __syncthreads(); // rows of the previous item fully consumed
        if (jv0 < jv1) {
            const int64_t s_first = (int64_t)a.decim * (r + P * jv0) - a.center;
            const int64_t s_last = (int64_t)a.decim * (r + P * (jv1 - 1)) - a.center;
            F0 = s_first & ~int64_t(31);
            const int64_t F1 = s_last + a.taps;
            const int nwords = (int)((F1 - F0 + 31) / 32) + 2; // +2: octet over-read
            const uint8_t* pk = a.packed + b * a.packed_bytes;
            for (int g = warp; g < nwords && g < a.words; g += nwarps) {
                const int64_t f = F0 + 32 * (int64_t)g + lane;
                const uint32_t w = f < a.frames ? *reinterpret_cast<const uint32_t*>(pk + 4 * f) : 0u;
                // 32 x 32 bit transpose across the warp (5 shuffle stages):
                // lane c ends with channel c's bits of the 32 frames. Channel c
                // is bit 7 - c%8 of byte c/8 of a frame word (MSB first); with
                // the byte-swapped word as input, the transpose leaves frame f
                // at bit 31 - f of lane c, and the byte-swapped result is the
                // MSB-first row word (frames 8b..8b+7 in byte b, first frame in
                // the top bit).
                uint32_t x = __byte_perm(w, 0, 0x0123);
                auto stage = [&](int j, uint32_t m) {
                    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
                    if (lane & j) x ^= ((y ^ (x >> j)) & m) << j;
                    else x ^= (x ^ (y >> j)) & m;
                };
                stage(16, 0x0000FFFFu);
                stage(8, 0x00FF00FFu);
                stage(4, 0x0F0F0F0Fu);
                stage(2, 0x33333333u);
                stage(1, 0x55555555u);
                rows[lane * a.words + g] = __byte_perm(x, 0, 0x0123);
            }
        }
        __syncthreads();
        const int64_t nj = j1 - j0;
        double* out_b = a.demod + (size_t)b * 32 * a.demod_len;
        for (int64_t q = threadIdx.x; q < 32 * nj; q += blockDim.x) {
            const int c = (int)(q / nj);
            const int64_t m = r + P * (j0 + q % nj);
            double v = 0.0;
            if (m >= a.m_lo && m < a.m_hi) {
                const int64_t s = (int64_t)a.decim * m - a.center;
                const int off = (int)((s - F0) >> 3); // first octet (byte) of the window in the row
                if (T == kDemodOctets) {
                    // the window's 33 bytes from 10 aligned words, re-aligned by
                    // funnel shifts (10 shared loads instead of 33 byte loads)
                    const uint32_t* rw = rows + c * a.words + (off >> 2);
                    const int sh = 8 * (off & 3);
                    uint32_t w[10];
#pragma unroll
                    for (int i = 0; i < 10; ++i) w[i] = rw[i];
                    uint32_t aw[9];
#pragma unroll
                    for (int i = 0; i < 9; ++i) aw[i] = __funnelshift_r(w[i], w[i + 1], sh);
                    auto lv = [&](int t) { return lut[t * 256 + ((aw[t >> 2] >> (8 * (t & 3))) & 255u)]; };
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                    for (int t = 0; t + 4 <= kDemodOctets; t += 4) {
                        a0 = __dadd_rn(a0, lv(t + 0));
                        a1 = __dadd_rn(a1, lv(t + 1));
                        a2 = __dadd_rn(a2, lv(t + 2));
                        a3 = __dadd_rn(a3, lv(t + 3));
                    }
                    double acc = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
#pragma unroll
                    for (int t = kDemodOctets & ~3; t < kDemodOctets; ++t) acc = __dadd_rn(acc, lv(t));
                    out_b[(size_t)c * a.demod_len + m] = acc;
                    continue;
                }
                const uint8_t* rb = reinterpret_cast<const uint8_t*>(rows + c * a.words) + off;
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                int t = 0;
                for (; t + 4 <= T; t += 4) {
                    a0 = __dadd_rn(a0, lut[(t + 0) * 256 + rb[t + 0]]);
                    a1 = __dadd_rn(a1, lut[(t + 1) * 256 + rb[t + 1]]);
                    a2 = __dadd_rn(a2, lut[(t + 2) * 256 + rb[t + 2]]);
                    a3 = __dadd_rn(a3, lut[(t + 3) * 256 + rb[t + 3]]);
                }
                double acc = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
                for (; t < T; ++t) acc = __dadd_rn(acc, lut[t * 256 + rb[t]]);
                v = acc;
            }
            out_b[(size_t)c * a.demod_len + m] = v;
        }
    }
}

// ---------------------------------------------------------------------------
// k_premf: pre-MF anti-alias FIR + decimation (strided_filter, filters.hpp:
// 14-39, called at pipeline.cpp:551-553), bit-exact: the same clipped window,
// the same four-lane order, products rounded before the add (no FMA).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_premf(PremfArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* taps = reinterpret_cast<double*>(smem);
    double* xs = taps + a.taps;
    const int ch = blockIdx.y, b = blockIdx.z;
    const int64_t n0 = (int64_t)blockIdx.x * blockDim.x;
    const int64_t start = -(int64_t)((a.taps - 1) / 2);
    const double* x = a.demod + ((size_t)b * 32 + ch) * a.demod_len;
    for (int i = threadIdx.x; i < a.taps; i += blockDim.x) taps[i] = a.rev[i];
    const int64_t s0 = start + n0 * a.decim;
    const int span = (int)(blockDim.x - 1) * a.decim + a.taps;
    for (int i = threadIdx.x; i < span; i += blockDim.x) {
        const int64_t g = s0 + i;
        xs[i] = (g >= 0 && g < a.demod_len) ? x[g] : 0.0;
    }
    __syncthreads();
    const int64_t n = n0 + threadIdx.x;
    if (n >= a.mf_len) return;
    const int64_t s = start + n * a.decim;
    const int64_t lo = (s > 0 ? s : (int64_t)0), hi = ((s + a.taps) < a.demod_len ? (s + a.taps) : a.demod_len);
    const double* h = taps + (lo - s);
    const double* xv = xs + (lo - s0);
    const int cnt = (int)(hi - lo);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int j = 0;
    for (; j + 4 <= cnt; j += 4) {
        a0 = __dadd_rn(a0, __dmul_rn(h[j], xv[j]));
        a1 = __dadd_rn(a1, __dmul_rn(h[j + 1], xv[j + 1]));
        a2 = __dadd_rn(a2, __dmul_rn(h[j + 2], xv[j + 2]));
        a3 = __dadd_rn(a3, __dmul_rn(h[j + 3], xv[j + 3]));
    }
    double acc = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
    for (; j < cnt; ++j) acc = __dadd_rn(acc, __dmul_rn(h[j], xv[j]));
    a.mf[((size_t)b * 32 + ch) * a.mf_stride + n] = acc;
}

// ---------------------------------------------------------------------------
// k_matched_filter: per (channel, measurement) row, FP64 real FFT of the
// zero-padded row, product with the spectrum of the reversed chirp, inverse,
// 1/N, and the window [ref_len-1, ref_len-1+mf_len) (pipeline.cpp:555-562).
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(kThreads) k_matched_filter(MfArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int N = 2 * M;
    double2* bufB = reinterpret_cast<double2*>(smem);
    const size_t row = (size_t)blockIdx.y * 32 + blockIdx.x;
    // pre-MF rows are stored zero-padded to N (stride mf_stride >= N): the
    // first FFT pass reads them straight from global memory
    const double* x = a.mf + row * a.mf_stride;
    cfft<M, false, false>(reinterpret_cast<const double2*>(x), bufB, TwGlobal<double2>{a.tw, 2});
    const double scale = 2.0 / (double)N;
    const double2* R = a.ref_spec;
    real_spectral_op(bufB, M, TwGlobal<double2>{a.tw, 2}, [&](double2 X, int k) {
        return cmul(X, double2{R[k].x * scale, R[k].y * scale});
    });
    cfft<M, true, true>(bufB, bufB, TwGlobal<double2>{a.tw, 2});
    // padded rows: sample n at [row * Lp + H + n]; the halo stays zero
    double* out = a.filt + row * a.Lp + a.H;
    float* out32 = a.filt32 ? a.filt32 + row * a.Lp + a.H : nullptr;
    double amax = 0.0;
    for (int64_t n = threadIdx.x; n < a.mf_len; n += blockDim.x) {
        const int64_t q = n + a.ref_len - 1;
        const double2 z = bufB[pad16((int)(q >> 1))];
        const double v = (q & 1) ? z.y : z.x;
        out[n] = v;
        amax = fmax(amax, fabs(v));
        if (out32) out32[n] = (float)v;
    }
    if (a.amax_bits) {
        // per-capture max |filt| (block-floating-point scale of the tensor-core
        // beamformer); non-negative doubles order like their bit patterns
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if ((threadIdx.x & 31) == 0)
            atomicMax(a.amax_bits + blockIdx.y, (unsigned long long)__double_as_longlong(amax));
    }
}

// Forward real FFT of one length-n row (setup: spectrum of the reversed chirp).
template <int M>
__global__ void __launch_bounds__(kThreads) k_rfft_forward(const double* x, double2* X,
                                                           const double2* tw) {
    extern __shared__ __align__(16) unsigned char smem[];
    double2* bufB = reinterpret_cast<double2*>(smem);
    cfft<M, false, false>(reinterpret_cast<const double2*>(x), bufB, TwGlobal<double2>{tw, 2});
    for (int k = threadIdx.x; k <= M; k += blockDim.x) {
        const int k1 = k % M, k2 = (M - k) % M;
        const double2 zk = bufB[pad16(k1)], zkk = bufB[pad16(k2)];
        const double2 e = {0.5 * (zk.x + zkk.x), 0.5 * (zk.y - zkk.y)};
        const double2 d = {0.5 * (zk.x - zkk.x), 0.5 * (zk.y + zkk.y)};
        const double2 o = {d.y, -d.x};
        X[k] = cadd(e, cmul(tw[k], o));
    }
}

// ---------------------------------------------------------------------------
// Per-direction stage, split in two kernels joined by an HBM/L2 beam buffer.
//
// k_beamform_tiles<R>: delay-and-sum (pipeline.cpp:432-446) for 256
// directions x T samples per CTA. The zero-haloed filt rows of one time tile
// (32 channels x (T + 2H), H = max |shift|) are staged in shared memory once
// and reused by all 256 directions; lane = direction. Directions are visited
// in Morton order of their unit vectors (Plan::order), so the 32 lanes of a
// warp need samples a few positions apart and each shared-memory load is
// served by one or two wavefronts. Channels are accumulated in the
// reference order 0..31 and scaled by 1/32 (exact), so the FP64 beam is
// bit-identical to the reference's; the zero halo reproduces its zero-fill
// (adding +0.0 to a partial sum that is never -0.0 is the identity).
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(kThreads) k_beamform_tiles(BeamArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    R* tile = reinterpret_cast<R*>(smem);
    const int W = a.T + 2 * a.H;
    const int64_t t0 = (int64_t)blockIdx.x * a.T;
    const int b = blockIdx.z;
    const R* fb = reinterpret_cast<const R*>(a.filt) + (size_t)b * 32 * a.Lp;
    for (int idx = threadIdx.x; idx < 32 * W; idx += blockDim.x) {
        const int i = idx / W, e = idx - i * W;
        const int64_t g = t0 + e; // padded index: sample t0 - H + e
        tile[idx] = g < a.Lp ? fb[(size_t)i * a.Lp + g] : (R)0;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t slot = ((int64_t)blockIdx.y * (kThreads / 32) + warp) * 32 + lane;
    if (slot >= a.n_dirs) return;
    int off[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) off[i] = i * W + a.H - a.shifts[slot * 32 + i];
    const int nmax = (int)((a.L - t0) < a.T ? (a.L - t0) : (int64_t)a.T);
    R* out = reinterpret_cast<R*>(a.beams) + ((size_t)b * a.n_dirs + slot) * a.N + t0;
    const R scale = (R)(1.0 / 32.0);
    for (int n = 0; n < nmax; n += 4) {
        R c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const R* p = tile + off[i] + n;
            c0 += p[0];
            c1 += p[1];
            c2 += p[2];
            c3 += p[3];
        }
        if (n + 4 <= nmax) {
            if constexpr (sizeof(R) == 8) {
                reinterpret_cast<double2*>(out + n)[0] = double2{c0 * scale, c1 * scale};
                reinterpret_cast<double2*>(out + n)[1] = double2{c2 * scale, c3 * scale};
            } else {
                *reinterpret_cast<float4*>(out + n) = float4{c0 * scale, c1 * scale, c2 * scale, c3 * scale};
            }
        } else {
            if (n < nmax) out[n] = c0 * scale;
            if (n + 1 < nmax) out[n + 1] = c1 * scale;
            if (n + 2 < nmax) out[n + 2] = c2 * scale;
        }
    }
}

// ---------------------------------------------------------------------------
// k_envelope<R, G>: per (measurement, direction): Hilbert transform of the
// beam via a real FFT pair with DC and Nyquist zeroed and X -> -iX
// (pipeline.cpp:448-461), |b + iH(b)| (:462-464), the composite
// smoothing/anti-alias FIR at stride D3 with the reference's clipped window
// and four-lane order (:466-468, filters.hpp:14-39), clamp and f32 write
// (:469-471). G independent 256-thread groups per CTA, each with its own
// shared-memory FFT buffer and named barrier, so one group's barrier waits
// overlap another group's work. The beam is read from global memory twice
// (first FFT pass, magnitude) instead of being held in shared memory; the
// envelope is written over the Hilbert output in place.
// ---------------------------------------------------------------------------
// per group: max(FFT buffer (M + M/16 complex), D * phase_len reals + the FIR
// half-sum scratch), even
__host__ __device__ int envelope_group_reals(int n, int phase_reals) {
    const int M = n / 2;
    const int fft = 2 * (M + M / 16);
    const int ph = phase_reals + kFirScratch;
    const int r = fft > ph ? fft : ph;
    return (r + 1) & ~1;
}

// |b + iH(b)|. FP64: rsqrt seed from the SFU and one third-order step
// instead of the correctly rounded library sequence; FP32: sqrtf.
__device__ __forceinline__ double fast_mag(double b, double h) {
#ifdef SNB_SQRT_TWO_STEP
    // (round-2 form: one Newton step on the reciprocal root, one on the root)
    const double x = b * b + h * h;
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(fmax(x, 1e-300)));
    r = r * fma(-0.5 * x, r * r, 1.5);
    const double s = x * r;
    return fma(0.5 * r, fma(-s, s, x), s);
#else
    // x = b^2 + h^2 + 2^-996: the tiny term keeps the seed finite at b = h = 0
    // (result 2^-498, which every f32 output rounds away) and changes x for
    // no x >= 2^-940. Seed r0 = rsqrt(x)(1 + d) from the SFU (MUFU.RSQ64H),
    // s = x r0, e = s r0 - 1 = (1 + d)^2 - 1 (exact by FMA, so it also
    // corrects the rounding of s), then s (1 + e)^(-1/2) to third order:
    // s (1 - e/2 + 3 e^2 / 8), error ~2.5 d^3. Seven FP64 operations (the
    // round-2 form: ten and a clamp); scripts/micro/rsqrt_acc.cu measures d
    // and the result's error (max 2^-52 relative).
    const double x = fma(b, b, fma(h, h, 0x1p-996));
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double s = x * r;
    const double e = fma(s, r, -1.0);
    return fma(s, e * fma(e, 0.375, -0.5), s);
#endif
}
__device__ __forceinline__ float fast_mag(float b, float h) { return sqrtf(b * b + h * h); }

// Composite smoothing/anti-alias FIR evaluated at stride D (the work of
// detail::strided_filter, filters.hpp:14-39, at pipeline.cpp:466-468), in
// polyphase form: out[k] = sum_p sum_q rev[q*D + p] * e_p[k + q], e_p read
// from the decimation-phase rows `ph` (row p at ph + p * phase_len).
//
// Fast path (D = 10, Q = 45): warps 0-3 of the group sum phases 0-4, warps 4-7
// phases 5-9, for the same kFirR consecutive outputs per thread; a register
// window slides over the row, refilled two samples per 16-byte load, and the
// taps (warp-uniform: broadcast) come two per load; the phase loop is rolled
// (the fully unrolled form overflowed the instruction cache). The upper half
// hands its partial sums to the lower half through `red`.
template <int P0, int NP, typename R>
__device__ __forceinline__ void fir_phases(const R* ph, int phase_len, int k0, R (&acc)[kFirR], const R* staps) {
    using V = typename Cx<R>::T;
#pragma unroll 1
    for (int pp = 0; pp < NP; ++pp) {
        const V* row = reinterpret_cast<const V*>(ph + (P0 + pp) * phase_len + k0);
        const V* tp = reinterpret_cast<const V*>(staps + (P0 + pp) * kFirQP);
        R w[kFirR + kFirQ + 1];
#pragma unroll
        for (int r = 0; r < kFirR / 2; ++r) {
            const V v = row[r];
            w[2 * r] = v.x;
            w[2 * r + 1] = v.y;
        }
        V c2;
#pragma unroll
        for (int q = 0; q < kFirQ; ++q) {
            if ((q & 1) == 0) {
                if (q + 2 < kFirQ) { // w[kFirR + q], w[kFirR + q + 1]: used from step q + 1 on
                    const V v = row[(kFirR + q) / 2];
                    w[kFirR + q] = v.x;
                    w[kFirR + q + 1] = v.y;
                }
                c2 = tp[q / 2];
            }
            const R c = (q & 1) ? c2.y : c2.x;
#pragma unroll
            for (int r = 0; r < kFirR; ++r) acc[r] = fma(c, w[q + r], acc[r]);
        }
    }
}

template <typename R>
__device__ __forceinline__ void fir_polyphase(const R* ph, const R* comp, const EnvArgs& a, float* eo) {
    const int tid = gtid();
    if (a.fir_fast) {
        // rounds of 128 output groups (more than one beyond 768 bins: the
        // 10 m window's 1,311), the exchange scratch reused per round
        const int h = tid >> 7;
        const int groups = (int)((a.bins + kFirR - 1) / kFirR);
        R* red = const_cast<R*>(ph) + kFirD * a.phase_len;
#pragma unroll 1
        for (int g0 = 0; g0 < groups; g0 += 128) {
            const int g = g0 + (tid & 127);
            const int k0 = g * kFirR, kr = (tid & 127) * kFirR;
            R acc[kFirR];
#pragma unroll
            for (int r = 0; r < kFirR; ++r) acc[r] = 0;
            if (g < groups) {
                if (h == 0) fir_phases<0, kFirD / 2>(ph, a.phase_len, k0, acc, comp);
                else fir_phases<kFirD / 2, kFirD / 2>(ph, a.phase_len, k0, acc, comp);
                if (h == 1) {
#pragma unroll
                    for (int r = 0; r < kFirR; ++r) red[kr + r] = acc[r];
                }
            }
            gsync();
            if (h == 0 && g < groups) {
#pragma unroll
                for (int r = 0; r < kFirR; ++r) {
                    if (k0 + r < a.bins) {
                        const float v = (float)(acc[r] + red[kr + r]);
                        eo[k0 + r] = v > 0.0f ? v : 0.0f;
                    }
                }
            }
            if (g0 + 128 < groups) gsync();
        }
    } else {
        // generic decimation / tap count: plain polyphase loops, taps in smem
        for (int64_t k = tid; k < a.bins; k += kGroupThreads) {
            R acc = 0;
            for (int p = 0; p < a.decim; ++p) {
                const R* row = ph + p * a.phase_len + k;
                for (int q = 0; q < a.fir_q; ++q) acc = fma(comp[q * a.decim + p], row[q], acc);
            }
            const float v = (float)acc;
            eo[k] = v > 0.0f ? v : 0.0f;
        }
    }
}

// FF: the smoothing FIR by 768-point FFTs (fir_fft768; M == 4096 only)
template <typename R, int G, int M, bool FF = false>
// (M <= 2048 generic fallbacks -- the 1.5 m window runs k_envelope_pair2048 --
// get the full register file: at 128 registers their Stockham passes spilled)
__global__ void __launch_bounds__(kThreads * G, (M >= 8192 || M <= 2048) ? 1 : ((sizeof(R) == 8 ? SNB_ENV_MINB : SNB_ENV_MINB_F32) / G > 0 ? (sizeof(R) == 8 ? SNB_ENV_MINB : SNB_ENV_MINB_F32) / G : 1))
    k_envelope(EnvArgs a, FirTaps<R> taps) {
    static_assert(!FF || M == 4096, "FFT FIR: N = 8192 only");
    using V = typename Cx<R>::T;
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int N = 2 * M;
    const int grp = gidx(), tid = gtid();
    constexpr bool kSmemTw = M == kTwSharedM;
#ifdef SNB_FF_NOFUSE
    constexpr bool kFfFused = false;
#else
    constexpr bool kFfFused = FF; // the FIR's first pass in the sink
#endif
    V* tws = reinterpret_cast<V*>(smem);                   // compact twiddles (M == 4096)
    // FF: the FFT FIR's spectrum factors and twiddles, shared by the groups
    V* ffu = tws + (kSmemTw ? kTwSharedCount : 0);
    V* ffw = ffu + (FF ? kFfU : 0);
    R* comp = reinterpret_cast<R*>(ffw + (FF ? kFfW : 0));
    // taps in shared memory: phase-major kFirTaps (fast path) or the reversed
    // composite kernel (generic path); none with the FFT FIR
    const int comp_pad = FF ? 0 : a.fir_fast ? kFirTaps : (a.fir_q * a.decim + 1) & ~1;
    const int group_reals = envelope_group_reals(N, FF ? 0 : a.decim * a.phase_len);
    V* bufB = reinterpret_cast<V*>(comp + comp_pad + (size_t)grp * group_reals);
    const R* cr = reinterpret_cast<const R*>(a.comp);
    const V* tw = reinterpret_cast<const V*>(a.tw);
    if constexpr (FF) {
        const V* su = reinterpret_cast<const V*>(a.ff_u);
        const V* sw = reinterpret_cast<const V*>(a.ff_w);
        for (int i = threadIdx.x; i < kFfU; i += blockDim.x) ffu[i] = su[i];
        for (int i = threadIdx.x; i < kFfW; i += blockDim.x) ffw[i] = sw[i];
    } else if (a.fir_fast) {
        for (int i = threadIdx.x; i < comp_pad; i += blockDim.x) comp[i] = taps.c[i]; // phase-major
    } else {
        for (int i = threadIdx.x; i < comp_pad; i += blockDim.x) comp[i] = i < a.comp_len ? cr[i] : (R)0;
    }
    if constexpr (kSmemTw) {
        const V* src = reinterpret_cast<const V*>(a.tw_small);
        for (int i = threadIdx.x; i < kTwSharedCount; i += blockDim.x) tws[i] = src[i];
    }
    __syncthreads();
    using TWT = typename std::conditional<kSmemTw, TwShared<V>, TwGlobal<V>>::type;
    TWT twsrc;
    if constexpr (kSmemTw) twsrc = TwShared<V>{tws};
    else twsrc = TwGlobal<V>{tw, 2};
    const int64_t L = a.mf_len;
    const int64_t items = a.n_dirs * a.batch;
    const R scale = (R)2 / (R)N;
    const int c0 = (a.comp_len - 1) / 2;
    R* env = reinterpret_cast<R*>(bufB); // env[n] at n + 2*(n >> 5) (pad16 of the complex view)
    // M = 4096: the first pass's inputs of the next item are loaded into
    // registers before the current item's FIR, so their L2 latency hides
    // behind it
#ifndef SNB_PRE
#define SNB_PRE 2
#endif
    // of the 16 inputs per thread; direct-FIR path, envelope ms by depth 0-4:
    // 3.56, 3.48, 3.48, 3.60, 3.59 (8+: spills); the FFT-FIR path loads them
    // after its FIR, where depth 0 / 2 / 4 measured 2.95 / 3.04 / 3.05 ms
    // (stack 8 / 56 / 88 B): none
    constexpr int kPre = FF ? 0 : SNB_PRE;
    V pre[16];
    auto load_pre = [&](int64_t item) {
        const V* s = reinterpret_cast<const V*>(a.beams) + (size_t)item * M;
#pragma unroll
        for (int r = 0; r < kPre; ++r) pre[r] = __ldg(s + tid + r * kGroupThreads);
    };
    if constexpr (M == 4096) {
        if ((int64_t)blockIdx.x * G + grp < items) load_pre((int64_t)blockIdx.x * G + grp);
    }
    for (int64_t it = (int64_t)blockIdx.x * G + grp; it < items; it += (int64_t)gridDim.x * G) {
        const int64_t b = it / a.n_dirs, slot = it % a.n_dirs;
        const R* src = reinterpret_cast<const R*>(a.beams) + (size_t)it * N;
#ifndef SNB_NO_BEAM_PREFETCH
        {
            // pull the next item's beam (N reals) into L2 while this one runs
#ifndef SNB_PF_AHEAD
#define SNB_PF_AHEAD 1
#endif
            const int64_t nx = it + (int64_t)gridDim.x * G * SNB_PF_AHEAD;
            if (nx < items && tid == 0) {
                const R* nsrc = reinterpret_cast<const R*>(a.beams) + (size_t)nx * N;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nsrc), "r"((unsigned)(N * sizeof(R)))
                             : "memory");
            }
        }
#endif
        if constexpr (M == 4096) {
#pragma unroll
            for (int r = kPre; r < 16; ++r) pre[r] = __ldg(reinterpret_cast<const V*>(src) + tid + r * kGroupThreads);
            dif_pass1_4096(pre, bufB, twsrc);
            dif_pass2_4096(bufB, twsrc);
            hilbert_mid_dif_4096(bufB, twsrc, scale);
        } else {
            cfft<M, false, false>(reinterpret_cast<const V*>(src), bufB, twsrc);
            hilbert_spectral(bufB, M, twsrc, scale);
        }
        R* ph = env; // phases: D rows of phase_len entries
        {
            // Inverse transform whose last pass feeds |b + iH(b)| straight into
            // the decimation-phase layout e_p[u] = env[u*D - c0 + p] (zero outside
            // [0, L)) that the polyphase FIR reads with unit stride: output n of
            // the last pass is the pair h[2n], h[2n+1]; b[2n], b[2n+1] come from
            // the beam buffer (one 16-byte load). Slot of sample t = n + c0:
            // (t mod D) * phase_len + t / D, t / D by a multiply-high.
            const int D = a.decim, PL = a.phase_len;
            const unsigned dmagic = 0xffffffffu / (unsigned)D + 1u; // exact for t < 2^32 / D
            const V* bsrc = reinterpret_cast<const V*>(src);
            const int Li = (int)L;
            constexpr bool ffir = FF;
            auto sink = [&](int n, V h) {
                const V bv = __ldg(bsrc + n);
                const R m0 = fast_mag(bv.x, h.x);
                const R m1 = fast_mag(bv.y, h.y);
                const unsigned t = 2u * (unsigned)n + (unsigned)c0;
                const int u = (int)__umulhi(t, dmagic);
                const int pp = (int)t - u * D;
                if constexpr (ffir) {
                    // fir_fft768's layout (D == 10, c0 odd: pp odd): both
                    // samples in the complex slot u of sequence (pp - 1) / 2
                    if (2 * n < Li) bufB[ff_slot((pp - 1) >> 1, u)] = V{m0, 2 * n + 1 < Li ? m1 : (R)0};
                } else {
                    if (2 * n < Li) ph[pp * PL + u] = m0;
                    if (2 * n + 1 < Li) ph[pp + 1 == D ? u + 1 : (pp + 1) * PL + u] = m1;
                }
            };
            // FFT FIR, fused: the sink also runs the FIR's first forward pass
            // (radix 3 over u, u + 256, u + 512 of one sequence: samples
            // t, t + 2560, t + 5120 = outputs k, k + 5, k + 10 of this
            // thread's row, t_k = 2 m + c0 + 512 k) and writes every slot of
            // the layout, zeros included. The thread's five butterflies start
            // at the t_k in [0, 2560): k = 0..4 when t_0 < 512, else
            // k = -1..3 (t_-1 < c0: that sample is a zero). k = 15 (t >= 7680)
            // is never needed: by the host check (hi_a < 768) every sample
            // with t >= 7680 lies past L. Needs c0 < 512 (implied by
            // lo_a <= 32).
            auto sink_row = [&](int m, V(&v)[16]) {
                // opaque per item: the slots and twiddles below are
                // loop-invariant, and hoisting them out of the item loop spills
                asm volatile("" : "+r"(m));
                const unsigned t0 = 2u * (unsigned)m + (unsigned)c0;
                const bool hi = t0 >= 512u;
                // (unconditional loads -- n < M, inside the item's beam -- so
                // the compiler can issue them ahead; out-of-range samples
                // selected to zero)
                auto mag = [&](int k) -> V {
                    const int n = m + 256 * k;
                    const V h = v[out_slot<16>(k)];
                    const V bv = __ldg(bsrc + n);
                    const R m0 = fast_mag(bv.x, h.x);
                    const R m1 = fast_mag(bv.y, h.y);
                    return V{2 * n < Li ? m0 : (R)0, 2 * n + 1 < Li ? m1 : (R)0};
                };
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    V x0, x1, x2;
                    unsigned t;
                    if (j < 4) {
                        x0 = mag(j);
                        x1 = mag(j + 5);
                        x2 = mag(j + 10);
                        t = t0 + 512u * j;
                    } else {
                        const V a4 = mag(4), a9 = mag(9), a14 = mag(14);
                        x0 = hi ? V{(R)0, (R)0} : a4;
                        x1 = hi ? a4 : a9;
                        x2 = hi ? a9 : a14;
                        t = hi ? t0 - 512u : t0 + 2048u;
                    }
                    const unsigned u = __umulhi(t, dmagic); // t / 10 (< 256)
                    const int sa = ((int)(t - 10u * u) - 1) >> 1;
                    dft3<false>(x0, x1, x2);
                    const V w1 = ffw[u], w2 = cmul(w1, w1);
                    V* sl = bufB + ff_slot(sa, (int)u);
                    sl[0] = x0;
                    sl[272] = cmul(x1, w1); // pad16(u + 256) = pad16(u) + 272
                    sl[544] = cmul(x2, w2);
                    // (A/B: one butterfly at a time)
#ifdef SNB_FF_FENCE
                    asm volatile("" ::: "memory");
#endif
                }
            };
            if constexpr (M == 4096) {
                dit_pass2_4096(bufB, twsrc);
                if constexpr (kFfFused) dit_pass3_4096_row(bufB, twsrc, sink_row);
                else dit_pass3_4096(bufB, twsrc, sink);
            } else {
                cfft<M, true, true>(bufB, bufB, twsrc, sink);
            }
            // zero the slots whose sample lies outside [0, L): per phase row p,
            // u < ceil((c0 - p) / D) and u >= ceil((L + c0 - p) / D)
            if constexpr (kFfFused) {
            } else if constexpr (ffir) {
                // slot (a, u) holds samples n = 10 u + 2 a + 1 - c0 and n + 1:
                // zero for u < lo_a and u >= hi_a (at most 32 on either side,
                // checked on the host)
                for (int idx = tid; idx < 64 * kFfSeq; idx += kGroupThreads) {
                    const int sa = idx >> 6, k = idx & 63;
                    const int e = c0 - 1 - 2 * sa;
                    const int lo = e > 0 ? (e + kFirD - 1) / kFirD : 0; // D == kFirD (host check)
                    const int hi = (int)((L + e + kFirD - 1) / kFirD);
                    const int u = k < 32 ? k : hi + (k - 32);
                    if (k < 32 ? u < lo : u < kFfL) bufB[ff_slot(sa, u)] = V{(R)0, (R)0};
                }
            } else if (tid < D) {
                const int p = tid;
                const int lo = c0 >= p ? (c0 - p + D - 1) / D : 0;
                const int hi = (int)((L + c0 - p + D - 1) / D);
                R* row = ph + p * a.phase_len;
                for (int k = 0; k < lo; ++k) row[k] = 0;
                for (int k = hi; k < a.phase_len; ++k) row[k] = 0;
            }
        }
        const int64_t nx = it + (int64_t)gridDim.x * G;
        if constexpr (M == 4096) {
            if (!FF && nx < items) load_pre(nx);
        }
        gsync();
        float* eo = a.energy + ((size_t)b * a.n_dirs + a.order[slot]) * a.bins;
        if constexpr (M == 4096) {
            if constexpr (FF) {
                // (the next item's early first-pass loads come after the FFT FIR:
                // its radix-16 passes need the whole register budget)
                fir_fft768<!kFfFused>(bufB, ffu, ffw, eo, (int)a.bins);
                if (nx < items) load_pre(nx);
            } else {
                fir_polyphase<R>(ph, comp, a, eo);
            }
        } else {
            fir_polyphase<R>(ph, comp, a, eo);
        }
        gsync();
    }
}

// ---------------------------------------------------------------------------
// k_envelope_pair2048: the envelope for N = 4096 (M = 2048; the 1.5 m window)
// with TWO beams per 256-thread group, 128 threads per beam, so every pass
// keeps all threads busy with one 16- or two 8-point butterflies and the
// register budget of the M = 4096 path (the generic Stockham path left half
// the threads idle in two passes and spilled 620 B at 128 registers).
// In-place DIF/DIT pair, indices n = 128 n1 + 8 n2 + n3, k = k1 + 16 k2 + 256 k3:
//   forward pass 1 (thread m = n mod 128): DFT16 over n1, * W2048^{m k1}, to 128 k1 + m
//   forward pass 2 (thread (k1, n3)):      DFT16 over n2, * W128^{n3 k2}, to 128 k1 + 8 k2 + n3
//   middle (thread u: rows a = k1 + 16 k2 and 256 - a, or rows 0 and 128 for u = 0):
//     DFT8 over n3 -> X[a + 256 k3]; the Hilbert operator pairs bin a + 256 k3
//     with (256 - a) + 256 (7 - k3), both rows in this thread's registers (no
//     exchange); inverse DFT8 over k3, in place
//   inverse B (thread (k1, n3)): * conj W128^{n3 k2}, DFT16 over k2
//   inverse C (thread m): * conj W2048^{m k1}, DFT16 over k1 -> z[m + 128 n1] -> sink
// then the polyphase FIR of each beam (fir_polyphase, all 256 threads).
// ---------------------------------------------------------------------------
constexpr int kP2M = 2048, kP2Buf = kP2M + kP2M / 8; // complex slots per beam (pad8)
// one pad slot per 8 complex: the middle pass's 8-element rows 128 k1 + 8 k2
// land at 144 k1 + 9 k2, distinct 16-byte bank groups for the 8 consecutive
// k2 of a quarter-warp; the passes' runs of 8 consecutive positions stay
// conflict-free
__device__ __forceinline__ int pad8(int i) { return i + (i >> 3); }

template <typename V, typename TW>
__device__ __forceinline__ void tw_powers_m(const TW& tw, int M, int ns, int k, V (&w)[16]) {
    w[1] = tw.w(M, ns, 16, k, 1);
    w[2] = tw.w(M, ns, 16, k, 2);
    w[4] = tw.w(M, ns, 16, k, 4);
    w[8] = tw.w(M, ns, 16, k, 8);
    w[3] = cmul(w[1], w[2]);
    w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]);
    w[7] = cmul(w[3], w[4]);
#pragma unroll
    for (int r = 9; r < 16; ++r) w[r] = cmul(w[r - 8], w[8]);
}

template <typename R>
__global__ void __launch_bounds__(kThreads, SNB_ENV_MINB) k_envelope_pair2048(EnvArgs a, FirTaps<R> taps) {
    using V = typename Cx<R>::T;
    constexpr int M = kP2M, N = 2 * M;
    extern __shared__ __align__(16) unsigned char smem[];
    R* comp = reinterpret_cast<R*>(smem);
    V* buf0 = reinterpret_cast<V*>(comp + kFirTaps);
    const int t = threadIdx.x, h = t >> 7, u = t & 127;
    V* buf = buf0 + h * kP2Buf;
    for (int i = t; i < kFirTaps; i += blockDim.x) comp[i] = taps.c[i];
    __syncthreads();
    const TwGlobal<V> tw{reinterpret_cast<const V*>(a.tw), 2};
    const int64_t items = a.n_dirs * a.batch, pairs = (items + 1) / 2;
    const R s = (R)2 / (R)N;
    const int c0 = (a.comp_len - 1) / 2, D = a.decim, PL = a.phase_len;
    const int Li = (int)a.mf_len;
    auto cosS = [](int S) { return (R)(S <= 8 ? cos_pi16(S) : -cos_pi16(16 - S)); };
    auto sinS = [](int S) { return (R)cos_pi16(S <= 8 ? 8 - S : S - 8); };
    for (int64_t p = blockIdx.x; p < pairs; p += gridDim.x) {
        const int64_t it = 2 * p + h;
        const bool live = it < items;
        const int64_t src_it = live ? it : items - 1; // the idle half recomputes a beam (barriers)
        const V* src = reinterpret_cast<const V*>(a.beams) + (size_t)src_it * M;
        {
            const int64_t nx = 2 * (p + gridDim.x) + h;
            if (nx < items && u == 0) {
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const V*>(a.beams) + (size_t)nx * M),
                             "r"((unsigned)(M * sizeof(V))) : "memory");
            }
        }
        {   // forward pass 1
            V v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = __ldg(src + u + 128 * r);
            dft16<false>(v);
            V w[16];
            tw_powers_m(tw, M, 128, u, w);
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int k1 = out_slot<16>(r);
                buf[pad8(u + 128 * k1)] = k1 ? cmul(v[r], w[k1 ? k1 : 1]) : v[r];
            }
        }
        __syncthreads();
        {   // forward pass 2
            const int k1 = u >> 3, n3 = u & 7;
            V v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = buf[pad8(128 * k1 + 8 * r + n3)];
            dft16<false>(v);
            V w[16];
            tw_powers_m(tw, M, 8, n3, w);
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int k2 = out_slot<16>(r);
                buf[pad8(128 * k1 + 8 * k2 + n3)] = k2 ? cmul(v[r], w[k2 ? k2 : 1]) : v[r];
            }
        }
        __syncthreads();
        {   // middle: DFT8, Hilbert operator, inverse DFT8 (thread-local rows)
            // rows: u = 8 c + d -> ra = c + 16 d (k1 = c fixed, k2 = d spread
            // over a quarter-warp), rb = 256 - ra (u = 0: rows 0 and 128)
            const int ra = (u >> 3) + 16 * (u & 7), rb = u == 0 ? 128 : 256 - ra;
            const int ba = 128 * (ra & 15) + 8 * (ra >> 4), bb = 128 * (rb & 15) + 8 * (rb >> 4);
            V xa[8], xb[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                xa[r] = buf[pad8(ba + r)];
                xb[r] = buf[pad8(bb + r)];
            }
            dft8<false>(xa);
            dft8<false>(xb);
            // op(zk, zc, c, sn) = s (cos t conj(zc) + i sin t zk), c = s cos t, sn = s sin t
            auto op = [](V zk, V zc, R c, R sn) { return V{c * zc.x - sn * zk.y, sn * zk.x - c * zc.y}; };
            V na[8], nb[8];
            const V ha = tw.h(ra), hb = tw.h(rb);
            const R cja = s * ha.x, sja = -s * ha.y, cjb = s * hb.x, sjb = -s * hb.y;
            if (u != 0) {
                // bin ra + 256 k3 <-> rb + 256 (7 - k3), angle of the partner = pi - t
#pragma unroll
                for (int k3 = 0; k3 < 8; ++k3) {
                    const R c = cja * cosS(2 * k3) - sja * sinS(2 * k3);
                    const R sn = sja * cosS(2 * k3) + cja * sinS(2 * k3);
                    na[k3] = op(xa[k3], xb[7 - k3], c, sn);
                    nb[7 - k3] = op(xb[7 - k3], xa[k3], -c, sn);
                }
            } else {
                // row 0: bins 256 k3 <-> 256 (8 - k3) (k3 = 4 with itself), DC
                // and Nyquist (Z[0]) zeroed; row 128: k3 <-> 7 - k3
                na[0] = V{(R)0, (R)0};
#pragma unroll
                for (int k3 = 1; k3 < 8; ++k3) na[k3] = op(xa[k3], xa[8 - k3], s * cosS(2 * k3), s * sinS(2 * k3));
#pragma unroll
                for (int k3 = 0; k3 < 8; ++k3) {
                    const R c = cjb * cosS(2 * k3) - sjb * sinS(2 * k3);
                    const R sn = sjb * cosS(2 * k3) + cjb * sinS(2 * k3);
                    nb[k3] = op(xb[k3], xb[7 - k3], c, sn);
                }
            }
            dft8<true>(na);
            dft8<true>(nb);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                buf[pad8(ba + r)] = na[r];
                buf[pad8(bb + r)] = nb[r];
            }
        }
        __syncthreads();
        {   // inverse B
            const int k1 = u >> 3, n3 = u & 7;
            V v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = buf[pad8(128 * k1 + 8 * r + n3)];
            V w[16];
            tw_powers_m(tw, M, 8, n3, w);
#pragma unroll
            for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], cconj(w[r]));
            dft16<true>(v);
#pragma unroll
            for (int r = 0; r < 16; ++r) buf[pad8(128 * k1 + 8 * out_slot<16>(r) + n3)] = v[r];
        }
        __syncthreads();
        {   // inverse C + sink: |b + iH(b)| into the decimation-phase rows of this beam
            V v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = buf[pad8(128 * r + u)];
            V w[16];
            tw_powers_m(tw, M, 128, u, w);
#pragma unroll
            for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], cconj(w[r]));
            dft16<true>(v);
            __syncthreads();
            R* ph = reinterpret_cast<R*>(buf);
            const unsigned dmagic = 0xffffffffu / (unsigned)D + 1u;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int n = u + 128 * out_slot<16>(r);
                const V hv = v[r];
                const V bv = __ldg(src + n);
                const R m0 = fast_mag(bv.x, hv.x);
                const R m1 = fast_mag(bv.y, hv.y);
                const unsigned tt = 2u * (unsigned)n + (unsigned)c0;
                const int uu = (int)__umulhi(tt, dmagic);
                const int pp = (int)tt - uu * D;
                if (2 * n < Li) ph[pp * PL + uu] = m0;
                if (2 * n + 1 < Li) ph[pp + 1 == D ? uu + 1 : (pp + 1) * PL + uu] = m1;
            }
            if (u < D) {
                const int pr = u;
                const int lo = c0 >= pr ? (c0 - pr + D - 1) / D : 0;
                const int hi = (int)((a.mf_len + c0 - pr + D - 1) / D);
                R* row = ph + pr * PL;
                for (int k = 0; k < lo; ++k) row[k] = 0;
                for (int k = hi; k < PL; ++k) row[k] = 0;
            }
        }
        __syncthreads();
        {
            // polyphase FIR of this half's beam over its 4 warps: units (output
            // group, phase half) with the half warp-uniform (warps 0, 2: phases
            // 0-4; 1, 3: 5-9), 64 groups per round; the upper half's partial
            // sums through shared memory after the phase rows
            const R* ph = reinterpret_cast<const R*>(buf);
            R* red = reinterpret_cast<R*>(buf) + D * PL;
            const int groups = (int)((a.bins + kFirR - 1) / kFirR);
            const int wl = u >> 5, q = wl & 1, gl = (wl >> 1) * 32 + (u & 31);
            const int64_t b = src_it / a.n_dirs, slot = src_it % a.n_dirs;
            float* eo = a.energy + ((size_t)b * a.n_dirs + a.order[slot]) * a.bins;
#pragma unroll 1
            for (int g0 = 0; g0 < groups; g0 += 64) {
                const int g = g0 + gl, k0 = g * kFirR;
                R acc[kFirR];
#pragma unroll
                for (int r = 0; r < kFirR; ++r) acc[r] = 0;
                if (g < groups) {
                    if (q == 0) fir_phases<0, kFirD / 2>(ph, PL, k0, acc, comp);
                    else fir_phases<kFirD / 2, kFirD / 2>(ph, PL, k0, acc, comp);
                    if (q) {
#pragma unroll
                        for (int r = 0; r < kFirR; ++r) red[gl * kFirR + r] = acc[r];
                    }
                }
                __syncthreads();
                if (live && g < groups && q == 0) {
#pragma unroll
                    for (int r = 0; r < kFirR; ++r) {
                        if (k0 + r < a.bins) {
                            const float v = (float)(acc[r] + red[gl * kFirR + r]);
                            eo[k0 + r] = v > 0.0f ? v : 0.0f;
                        }
                    }
                }
                __syncthreads();
            }
        }
    }
}

// ---------------------------------------------------------------------------
// k_envelope_split8192: the envelope for N = 16384 (M = 8192; the 8-11.7 m
// windows). One radix-2 DIF stage splits the 8192-point transform into its
// even- and odd-bin 4096-point halves, each run by one 256-thread half of the
// CTA with the in-place M = 4096 passes (dif_pass1/2, the Hilbert middle pass
// -- the even half's pairing and angles are exactly the M = 4096 ones, the
// odd half pairs k' with 4095 - k' -- and dit_pass2/3); the inverse radix-2
// stage recombines z'[n] = e'[n] +- W8192^{-n} o'[n] and feeds the sink. The
// polyphase FIR then runs over all 512 threads (units of output group x
// phase part). Replaces the generic Stockham path (two butterflies per thread
// per pass, 241 registers, 8 warps per SM).
// ---------------------------------------------------------------------------
constexpr int kS8Buf = 4096 + 256; // complex slots per half (pad16)

template <typename R>
__global__ void __launch_bounds__(2 * kThreads, 1) k_envelope_split8192(EnvArgs a, FirTaps<R> taps) {
    using V = typename Cx<R>::T;
    constexpr int M = 8192, N = 2 * M;
    extern __shared__ __align__(16) unsigned char smem[];
    V* tws = reinterpret_cast<V*>(smem);
    R* comp = reinterpret_cast<R*>(tws + kTwSharedCount);
    V* buf0 = reinterpret_cast<V*>(comp + kFirTaps);
    for (int i = threadIdx.x; i < kTwSharedCount; i += blockDim.x) tws[i] = reinterpret_cast<const V*>(a.tw_small)[i];
    for (int i = threadIdx.x; i < kFirTaps; i += blockDim.x) comp[i] = taps.c[i];
    __syncthreads();
    const TwShared<V> tw4{tws};
    const V* tw = reinterpret_cast<const V*>(a.tw); // e^{-2 pi i k / 16384}
    const int64_t items = a.n_dirs * a.batch;
    const R s = (R)2 / (R)N;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        // per-item thread indices, opaque to the compiler: loop-invariant
        // addresses hoisted out of the item loop would not fit the registers
        int t = threadIdx.x;
        asm volatile("" : "+r"(t));
        const int h = t >> 8, j = t & 255;
        V* buf = buf0 + h * kS8Buf;
        const int c0 = (a.comp_len - 1) / 2, D = a.decim, PL = a.phase_len;
        const int Li = (int)a.mf_len;
        const V* src = reinterpret_cast<const V*>(a.beams) + (size_t)it * M;
        {
            const int64_t nx = it + gridDim.x;
            if (nx < items && t == 0) {
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const V*>(a.beams) + (size_t)nx * M),
                             "r"((unsigned)(M * sizeof(V))) : "memory");
            }
        }
        {   // radix-2 DIF stage: e[n] = z[n] + z[n + 4096], o[n] = (z[n] - z[n + 4096]) W8192^n
            V v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int n = j + 256 * r;
                const V z0 = __ldg(src + n), z1 = __ldg(src + n + 4096);
                v[r] = h == 0 ? cadd(z0, z1) : cmul(csub(z0, z1), __ldg(tw + 2 * n));
            }
            dif_pass1_4096(v, buf, tw4);
        }
        dif_pass2_4096(buf, tw4);
        if (h == 0) hilbert_mid_dif_4096(buf, tw4, s);
        else hilbert_mid_dif_4096_odd(buf, tw4, tw, s);
        dit_pass2_4096(buf, tw4);
        dit_pass3_4096(buf, tw4, [&](int n, V v) { buf[pad16(n)] = v; });
        __syncthreads();
        // inverse radix-2 stage + sink: z'[n + 4096 h] = e'[n] +- conj(W8192^n) o'[n]
        V zz[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int n = j + 256 * r;
            const V e = buf0[pad16(n)];
            const V o = cmul(buf0[kS8Buf + pad16(n)], cconj(__ldg(tw + 2 * n)));
            zz[r] = h == 0 ? cadd(e, o) : csub(e, o);
        }
        __syncthreads();
        {
            R* ph = reinterpret_cast<R*>(buf0);
            const unsigned dmagic = 0xffffffffu / (unsigned)D + 1u;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int n = j + 256 * r + 4096 * h;
                const V hv = zz[r];
                const V bv = __ldg(src + n);
                const R m0 = fast_mag(bv.x, hv.x);
                const R m1 = fast_mag(bv.y, hv.y);
                const unsigned tt = 2u * (unsigned)n + (unsigned)c0;
                const int uu = (int)__umulhi(tt, dmagic);
                const int pp = (int)tt - uu * D;
                if (2 * n < Li) ph[pp * PL + uu] = m0;
                if (2 * n + 1 < Li) ph[pp + 1 == D ? uu + 1 : (pp + 1) * PL + uu] = m1;
            }
            if (t < D) {
                const int pr = t;
                const int lo = c0 >= pr ? (c0 - pr + D - 1) / D : 0;
                const int hi = (int)((a.mf_len + c0 - pr + D - 1) / D);
                R* row = ph + pr * PL;
                for (int k = 0; k < lo; ++k) row[k] = 0;
                for (int k = hi; k < PL; ++k) row[k] = 0;
            }
        }
        __syncthreads();
        {
            // polyphase FIR: units (output group, phase part), the part
            // warp-uniform (warp w: part w mod 4 of 3 + 3 + 2 + 2 phases), 128
            // groups per round; partial sums of parts 1-3 through shared
            // memory after the phase rows
            const R* ph = reinterpret_cast<const R*>(buf0);
            R* red = reinterpret_cast<R*>(buf0) + D * PL;
            const int groups = (int)((a.bins + kFirR - 1) / kFirR);
            const int q = (t >> 5) & 3, gl = (t >> 7) * 32 + (t & 31);
            const int64_t b = it / a.n_dirs, slot = it % a.n_dirs;
            float* eo = a.energy + ((size_t)b * a.n_dirs + a.order[slot]) * a.bins;
#pragma unroll 1
            for (int g0 = 0; g0 < groups; g0 += 128) {
                const int g = g0 + gl, k0 = g * kFirR;
                R acc[kFirR];
#pragma unroll
                for (int r = 0; r < kFirR; ++r) acc[r] = 0;
                if (g < groups) {
                    if (q == 0) fir_phases<0, 3>(ph, PL, k0, acc, comp);
                    else if (q == 1) fir_phases<3, 3>(ph, PL, k0, acc, comp);
                    else if (q == 2) fir_phases<6, 2>(ph, PL, k0, acc, comp);
                    else fir_phases<8, 2>(ph, PL, k0, acc, comp);
                    if (q) {
#pragma unroll
                        for (int r = 0; r < kFirR; ++r) red[((q - 1) * 128 + gl) * kFirR + r] = acc[r];
                    }
                }
                __syncthreads();
                if (g < groups && q == 0) {
#pragma unroll
                    for (int r = 0; r < kFirR; ++r) {
                        if (k0 + r < a.bins) {
                            const R sum = acc[r] + red[gl * kFirR + r] + red[(128 + gl) * kFirR + r] +
                                          red[(256 + gl) * kFirR + r];
                            const float v = (float)sum;
                            eo[k0 + r] = v > 0.0f ? v : 0.0f;
                        }
                    }
                }
                __syncthreads();
            }
        }
    }
}

size_t envelope_split8192_smem_bytes(bool f32) {
    const size_t rb = f32 ? 4 : 8;
    return (size_t)kTwSharedCount * 2 * rb + (size_t)kFirTaps * rb + (size_t)2 * kS8Buf * 2 * rb;
}

int envelope_split8192_blocks_per_sm(bool f32) {
    int n = 0;
    const size_t smem = envelope_split8192_smem_bytes(f32);
    if (f32) {
        set_smem((const void*)k_envelope_split8192<float>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_envelope_split8192<float>, 2 * kThreads, smem);
    } else {
        set_smem((const void*)k_envelope_split8192<double>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_envelope_split8192<double>, 2 * kThreads, smem);
    }
    return n;
}

size_t envelope_pair2048_smem_bytes(bool f32) {
    const size_t rb = f32 ? 4 : 8;
    return (size_t)kFirTaps * rb + (size_t)2 * kP2Buf * 2 * rb;
}

// Workspace::beamform accessor (pipeline.cpp:576-591): materialised beams
// [n_dirs][L] f64, channels accumulated in order then * (1/32).
__global__ void __launch_bounds__(kThreads) k_beamform(const double* filt, double* beams,
                                                      const int32_t* shifts, int64_t L) {
    const int64_t d = blockIdx.y;
    __shared__ int sh[32];
    if (threadIdx.x < 32) sh[threadIdx.x] = shifts[d * 32 + threadIdx.x];
    __syncthreads();
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= L) return;
    double acc = 0.0;
    for (int i = 0; i < 32; ++i) {
        const int64_t src = n - sh[i];
        if (src >= 0 && src < L) acc += filt[(size_t)i * L + src];
    }
    beams[d * L + n] = acc * (1.0 / 32.0);
}

void launch_beamform(const double* filt, double* beams, const int32_t* shifts, int64_t L,
                     int64_t n_dirs, cudaStream_t s) {
    k_beamform<<<dim3((unsigned)((L + kThreads - 1) / kThreads), (unsigned)n_dirs), kThreads, 0, s>>>(
        filt, beams, shifts, L);
}

// FMA-throughput microbenchmark (roofline denominator for the CUDA-core
// stages: MEASURED_PEAKS.json carries only HBM and bf16 tensor figures).
// 8 independent FMA chains per thread, 4 x 148 CTAs x 256 threads.
template <typename R>
__global__ void __launch_bounds__(kThreads) k_fma_peak(R* out, int iters, R seed) {
    R a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed + (R)(threadIdx.x + i);
    const R m = (R)0.999999, c = (R)1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fma(a[i], m, c);
        }
    }
    R s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == (R)12345.678) out[threadIdx.x] = s; // keep the chains live
}

double measure_fma_peak(int sms, bool f32) {
    void* out = nullptr;
    cudaMalloc(&out, kThreads * 8);
    const int blocks = sms * 4, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        if (f32) k_fma_peak<float><<<blocks, kThreads>>>((float*)out, iters, 1.0f);
        else k_fma_peak<double><<<blocks, kThreads>>>((double*)out, iters, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0) best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 2.0 * 8 * 16 * (double)iters * kThreads * blocks;
    return flops / (best * 1e-3) / 1e12;
}

// ---------------------------------------------------------------------------
size_t demod_smem_bytes(int octets, int words) {
    return (size_t)octets * 256 * sizeof(double) + (size_t)32 * words * sizeof(uint32_t);
}

size_t fft_smem_bytes(int n, int real_bytes) {
    const int M = n / 2;
    return (size_t)(M + M / 16) * 2 * real_bytes;
}

// Dynamic shared-memory opt-in of a kernel, raised once per (kernel, size)
// (workspaces on several host threads share the table); a failure is thrown
// as SN_ERR_CUDA through the C ABI instead of surfacing as a launch error.
void set_smem(const void* fn, size_t smem) {
    static std::mutex m;
    static std::map<std::pair<int, const void*>, size_t> done; // per device: the attribute is per context
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(dev, fn);
    std::lock_guard<std::mutex> lk(m);
    auto it = done.find(key);
    if (it != done.end() && it->second >= smem) return;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(SN_ERR_CUDA, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize = " + std::to_string(smem) +
                                     "): " + cudaGetErrorString(e));
    }
    done[key] = smem;
}

void launch_demod(const DemodArgs& a, int grid_x, size_t smem, cudaStream_t s) {
    set_smem((const void*)k_demod, smem);
    k_demod<<<dim3(grid_x, a.period), kThreads, smem, s>>>(a);
}

// ---------------------------------------------------------------------------
// k_premf_rw: the same filter for the reference's default (65 taps, /2), with
// a register window: a thread computes kPremfR consecutive outputs, whose
// 65-sample windows overlap in all but 2 samples, so 2 R + 63 loads serve
// 65 R products; taps are kernel-parameter (constant-bank) operands. Each
// output keeps the reference's exact order (lane j mod 4 over j < 64, then
// (a0 + a1) + (a2 + a3), then j = 64; rounded products, no FMA). Blocks
// whose windows are clipped by the row ends take the generic loop.
// ---------------------------------------------------------------------------
constexpr int kPremfTaps = 65, kPremfR = 8, kPremfThreads = 128;
struct PremfTaps { double h[kPremfTaps]; };

// the CTA's input span staged in shared memory with one pad double per 16
// (thread t reads from 16 t + j: stride 17, bank-conflict free)
__device__ __forceinline__ int premf_pad(int i) { return i + (i >> 4); }

__global__ void __launch_bounds__(kPremfThreads) k_premf_rw(PremfArgs a, const __grid_constant__ PremfTaps t) {
    constexpr int kSpan = 2 * kPremfThreads * kPremfR + kPremfTaps; // inputs of the CTA's outputs
    __shared__ double xs[kSpan + kSpan / 16 + 1];
    const int ch = blockIdx.y, b = blockIdx.z;
    const int64_t nb = (int64_t)blockIdx.x * kPremfThreads * kPremfR;
    const int64_t n0 = nb + (int64_t)threadIdx.x * kPremfR;
    const double* x = a.demod + ((size_t)b * 32 + ch) * a.demod_len;
    double* out = a.mf + ((size_t)b * 32 + ch) * a.mf_stride;
    constexpr int start = -(kPremfTaps - 1) / 2;
    const int64_t sb = start + 2 * nb;
    for (int i = threadIdx.x; i < kSpan; i += kPremfThreads) {
        const int64_t g = sb + i;
        xs[premf_pad(i)] = (g >= 0 && g < a.demod_len) ? x[g] : 0.0;
    }
    __syncthreads();
    if (n0 >= a.mf_len) return;
    const int64_t s0 = start + 2 * n0;
    if (s0 >= 0 && s0 + 2 * (kPremfR - 1) + kPremfTaps <= a.demod_len && n0 + kPremfR <= a.mf_len) {
        const int l0 = (int)(s0 - sb); // = 2 kPremfR threadIdx.x
        double acc[kPremfR][4];
#pragma unroll
        for (int r = 0; r < kPremfR; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.0;
        double w[2 * kPremfR + kPremfTaps];
#pragma unroll
        for (int i = 0; i < 2 * kPremfR - 2; ++i) w[i] = xs[premf_pad(l0 + i)];
#pragma unroll
        for (int j = 0; j < kPremfTaps - 1; ++j) {
            w[2 * kPremfR - 2 + j] = xs[premf_pad(l0 + 2 * kPremfR - 2 + j)];
#pragma unroll
            for (int r = 0; r < kPremfR; ++r) acc[r][j & 3] = __dadd_rn(acc[r][j & 3], __dmul_rn(t.h[j], w[2 * r + j]));
        }
        w[2 * kPremfR - 2 + kPremfTaps - 1] = xs[premf_pad(l0 + 2 * kPremfR - 2 + kPremfTaps - 1)];
#pragma unroll
        for (int r = 0; r < kPremfR; ++r) {
            double v = __dadd_rn(__dadd_rn(acc[r][0], acc[r][1]), __dadd_rn(acc[r][2], acc[r][3]));
            v = __dadd_rn(v, __dmul_rn(t.h[kPremfTaps - 1], w[2 * r + kPremfTaps - 1]));
            out[n0 + r] = v;
        }
        return;
    }
    // clipped windows (row ends): generic per-output loop, same order
    for (int r = 0; r < kPremfR; ++r) {
        const int64_t n = n0 + r;
        if (n >= a.mf_len) break;
        const int64_t s = start + 2 * n;
        const int64_t lo = s > 0 ? s : 0, hi = (s + kPremfTaps) < a.demod_len ? (s + kPremfTaps) : a.demod_len;
        const int cnt = (int)(hi - lo);
        const int h0 = (int)(lo - s);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int j = 0;
        for (; j + 4 <= cnt; j += 4) {
            a0 = __dadd_rn(a0, __dmul_rn(t.h[h0 + j], x[lo + j]));
            a1 = __dadd_rn(a1, __dmul_rn(t.h[h0 + j + 1], x[lo + j + 1]));
            a2 = __dadd_rn(a2, __dmul_rn(t.h[h0 + j + 2], x[lo + j + 2]));
            a3 = __dadd_rn(a3, __dmul_rn(t.h[h0 + j + 3], x[lo + j + 3]));
        }
        double acc = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
        for (; j < cnt; ++j) acc = __dadd_rn(acc, __dmul_rn(t.h[h0 + j], x[lo + j]));
        out[n] = acc;
    }
}

void launch_premf(const PremfArgs& a, int batch, cudaStream_t s) {
    if (a.taps == kPremfTaps && a.decim == 2 && a.rev_host) {
        PremfTaps t;
        for (int i = 0; i < kPremfTaps; ++i) t.h[i] = a.rev_host[i];
        const int64_t per = (int64_t)kPremfThreads * kPremfR;
        k_premf_rw<<<dim3((unsigned)((a.mf_len + per - 1) / per), 32, batch), kPremfThreads, 0, s>>>(a, t);
        return;
    }
    const size_t smem = (size_t)(a.taps + (kThreads - 1) * a.decim + a.taps) * sizeof(double);
    set_smem((const void*)k_premf, smem);
    const int gx = (int)((a.mf_len + kThreads - 1) / kThreads);
    k_premf<<<dim3(gx, 32, batch), kThreads, smem, s>>>(a);
}

template <int M>
static void mf_launch(const MfArgs& a, int batch, size_t smem, cudaStream_t s) {
    set_smem((const void*)k_matched_filter<M>, smem);
    k_matched_filter<M><<<dim3(32, batch), kThreads, smem, s>>>(a);
}

template <typename R>
static void launch_bf(const BeamArgs& a, cudaStream_t s) {
    const size_t smem = (size_t)32 * (a.T + 2 * a.H) * sizeof(R);
    set_smem((const void*)k_beamform_tiles<R>, smem);
    dim3 grid((unsigned)((a.L + a.T - 1) / a.T), (unsigned)((a.n_dirs + kThreads - 1) / kThreads),
              (unsigned)a.batch);
    k_beamform_tiles<R><<<grid, kThreads, smem, s>>>(a);
}

void launch_beamform_tiles(const BeamArgs& a, bool f32, cudaStream_t s) {
    if (f32) launch_bf<float>(a, s);
    else launch_bf<double>(a, s);
}

size_t envelope_smem_bytes(int n, int comp_taps_padded, int phase_reals, bool f32, int groups) {
    const size_t rb = f32 ? 4 : 8;
    return (n / 2 == kTwSharedM ? (size_t)kTwSharedCount * 2 * rb : 0) +
           (size_t)((comp_taps_padded + 1) & ~1) * rb +
           (size_t)groups * envelope_group_reals(n, phase_reals) * rb;
}

// Compile-time FFT sizes: N = 2M real points, 32 <= N <= 8192.
#define SNB_DISPATCH_M(M_RUNTIME, CALL)                                  \
    switch (M_RUNTIME) {                                                 \
        case 16: { constexpr int MM = 16; CALL; break; }                 \
        case 32: { constexpr int MM = 32; CALL; break; }                 \
        case 64: { constexpr int MM = 64; CALL; break; }                 \
        case 128: { constexpr int MM = 128; CALL; break; }               \
        case 256: { constexpr int MM = 256; CALL; break; }               \
        case 512: { constexpr int MM = 512; CALL; break; }               \
        case 1024: { constexpr int MM = 1024; CALL; break; }             \
        case 2048: { constexpr int MM = 2048; CALL; break; }             \
        case 4096: { constexpr int MM = 4096; CALL; break; }             \
        case 8192: { constexpr int MM = 8192; CALL; break; }             \
        default: break;                                                  \
    }

template <typename R, int G, int M>
static int env_occ(size_t smem) {
    int n = 1;
    set_smem((const void*)k_envelope<R, G, M>, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_envelope<R, G, M>, kThreads * G, smem);
    return n;
}

int envelope_blocks_per_sm(bool f32, int n_fft, size_t smem) {
    int n = 1;
    if (f32) { SNB_DISPATCH_M(n_fft / 2, (n = env_occ<float, kEnvGroupsF32, MM>(smem))) }
    else { SNB_DISPATCH_M(n_fft / 2, (n = env_occ<double, kEnvGroupsF64, MM>(smem))) }
    return n > 0 ? n : 1;
}

template <typename R, int G, int M>
static void env_launch(const EnvArgs& a, const FirTaps<R>& taps, int grid, size_t smem, cudaStream_t s) {
    set_smem((const void*)k_envelope<R, G, M>, smem);
    k_envelope<R, G, M><<<grid, kThreads * G, smem, s>>>(a, taps);
}

// FFT FIR variant (N = 8192): kFfGroups groups per CTA share the spectrum
// factors and twiddles in shared memory
size_t envelope_ff_smem_bytes(bool f32) {
    const size_t rb = f32 ? 4 : 8;
    return ((size_t)kTwSharedCount + kFfU + kFfW) * 2 * rb +
           (size_t)(f32 ? kFfGroupsF32 : kFfGroups) * envelope_group_reals(8192, 0) * rb;
}

int envelope_ff_blocks_per_sm(bool f32) {
    int n = 1;
    const size_t smem = envelope_ff_smem_bytes(f32);
    if (f32) {
        set_smem((const void*)k_envelope<float, kFfGroupsF32, 4096, true>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_envelope<float, kFfGroupsF32, 4096, true>, kThreads * kFfGroupsF32,
                                                      smem);
    } else {
        set_smem((const void*)k_envelope<double, kFfGroups, 4096, true>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_envelope<double, kFfGroups, 4096, true>, kThreads * kFfGroups, smem);
    }
    return n > 0 ? n : 0;
}

template <typename R>
static void env_ff_launch(const EnvArgs& a, const FirTaps<R>& taps, int grid, cudaStream_t s) {
    const size_t smem = envelope_ff_smem_bytes(sizeof(R) == 4);
    constexpr int G = ff_groups<R>();
    set_smem((const void*)k_envelope<R, G, 4096, true>, smem);
    k_envelope<R, G, 4096, true><<<grid, kThreads * G, smem, s>>>(a, taps);
}

int envelope_pair2048_blocks_per_sm(bool f32) {
    int n = 0;
    const size_t smem = envelope_pair2048_smem_bytes(f32);
    if (f32) {
        set_smem((const void*)k_envelope_pair2048<float>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_envelope_pair2048<float>, kThreads, smem);
    } else {
        set_smem((const void*)k_envelope_pair2048<double>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_envelope_pair2048<double>, kThreads, smem);
    }
    return n;
}

void launch_envelope(const EnvArgs& a, const FirTaps<float>& t32, const FirTaps<double>& t64, bool f32,
                     int grid, cudaStream_t s) {
    if (a.split8192) {
        const size_t smem = envelope_split8192_smem_bytes(f32);
        if (f32) {
            set_smem((const void*)k_envelope_split8192<float>, smem);
            k_envelope_split8192<float><<<grid, 2 * kThreads, smem, s>>>(a, t32);
        } else {
            set_smem((const void*)k_envelope_split8192<double>, smem);
            k_envelope_split8192<double><<<grid, 2 * kThreads, smem, s>>>(a, t64);
        }
        return;
    }
    if (a.pair2048) {
        const size_t smem = envelope_pair2048_smem_bytes(f32);
        if (f32) {
            set_smem((const void*)k_envelope_pair2048<float>, smem);
            k_envelope_pair2048<float><<<grid, kThreads, smem, s>>>(a, t32);
        } else {
            set_smem((const void*)k_envelope_pair2048<double>, smem);
            k_envelope_pair2048<double><<<grid, kThreads, smem, s>>>(a, t64);
        }
        return;
    }
    if (a.fir_fft) {
        if (f32) env_ff_launch<float>(a, t32, grid, s);
        else env_ff_launch<double>(a, t64, grid, s);
        return;
    }
    if (f32) {
        const size_t smem = envelope_smem_bytes(a.n, a.fir_fast ? kFirTaps : a.fir_q * a.decim, a.decim * a.phase_len, true, kEnvGroupsF32);
        SNB_DISPATCH_M(a.n / 2, (env_launch<float, kEnvGroupsF32, MM>(a, t32, grid, smem, s)))
    } else {
        const size_t smem = envelope_smem_bytes(a.n, a.fir_fast ? kFirTaps : a.fir_q * a.decim, a.decim * a.phase_len, false, kEnvGroupsF64);
        SNB_DISPATCH_M(a.n / 2, (env_launch<double, kEnvGroupsF64, MM>(a, t64, grid, smem, s)))
    }
}

template <int M>
static void rfft_launch(const double* x, double2* X, const double2* tw, size_t smem, cudaStream_t s) {
    set_smem((const void*)k_rfft_forward<M>, smem);
    k_rfft_forward<M><<<1, kThreads, smem, s>>>(x, X, tw);
}

void launch_rfft_forward(const double* x, double2* X, const double2* tw, int n, size_t smem,
                         cudaStream_t s) {
    SNB_DISPATCH_M(n / 2, (rfft_launch<MM>(x, X, tw, smem, s)))
}

void launch_matched_filter(const MfArgs& a, int batch, size_t smem, cudaStream_t s) {
    SNB_DISPATCH_M(a.n / 2, (mf_launch<MM>(a, batch, smem, s)))
}

} // namespace snb
