// CTA-cooperative FFTs over shared memory (sm_100a).
//
// Replaces the reference's FFTW calls on the hot path (fft.cpp:81-92 RealFft
// forward/inverse, reached from pipeline.cpp:558-560 for the matched filter
// and :454-461 for the Hilbert envelope). FFTW conventions are kept:
// forward e^{-i}, unnormalised; the inverse is scaled by 1/n (fft.cpp:87-92).
//
// Layout: a real signal of N = 2M samples is viewed as M complex points
// z[n] = x[2n] + i x[2n+1] and transformed by an M-point complex Stockham FFT
// (radix-16 passes, one radix-2/4/8 pass to finish); a split/merge step maps
// Z <-> the half spectrum X[0..M]. Complex scratch lives in shared memory with
// one pad element per 16 (index i -> i + i/16) so that the strided Stockham
// stores are bank-conflict free for 16-byte elements.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

namespace snb {

template <typename R> struct Cx;
template <> struct Cx<double> { using T = double2; };
template <> struct Cx<float> { using T = float2; };

__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

// Thread groups: a CTA may run several independent 256-thread groups, each on
// its own work item and shared-memory region; FFT phases synchronise with a
// per-group named barrier (id 1 + group) instead of __syncthreads.
constexpr int kGroupThreads = 256;
__device__ __forceinline__ int gtid() { return threadIdx.x & (kGroupThreads - 1); }
__device__ __forceinline__ int gidx() { return threadIdx.x / kGroupThreads; }
__device__ __forceinline__ void gsync() {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + gidx()), "r"(kGroupThreads) : "memory");
}

template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return {a.x + b.x, a.y + b.y}; }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return {a.x - b.x, a.y - b.y}; }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
    return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename V> __device__ __forceinline__ V cconj(V a) { return {a.x, -a.y}; }
// multiply by -i (forward) or +i (inverse)
template <bool INV, typename V> __device__ __forceinline__ V rot90(V a) {
    return INV ? V{-a.y, a.x} : V{a.y, -a.x};
}

template <bool INV, typename V>
__device__ __forceinline__ void dft2(V& a, V& b) {
    const V t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

template <bool INV, typename V>
__device__ __forceinline__ void dft4(V& x0, V& x1, V& x2, V& x3) {
    const V a = cadd(x0, x2), b = csub(x0, x2);
    const V c = cadd(x1, x3), d = rot90<INV>(csub(x1, x3));
    x0 = cadd(a, c);
    x2 = csub(a, c);
    x1 = cadd(b, d);
    x3 = csub(b, d);
}

// Constant twiddles e^{-+2 pi i k/16}
template <bool INV, typename V, typename R>
__device__ __forceinline__ V tw16(V v, int k) {
    constexpr R c1 = (R)0.92387953251128675613, s1 = (R)0.38268343236508977173;
    constexpr R h = (R)0.70710678118654752440;
    const R sg = INV ? (R)1 : (R)-1; // sign of the sine term
    switch (k & 15) {
        case 0: return v;
        case 1: return cmul(v, V{c1, sg * s1});
        case 2: return cmul(v, V{h, sg * h});
        case 3: return cmul(v, V{s1, sg * c1});
        case 4: return rot90<INV>(v);
        case 6: return cmul(v, V{-h, sg * h});
        case 9: return cmul(v, V{-c1, -sg * s1});
        default: {
            // not used by the 4x4 decomposition (n2*k1 in {0,1,2,3,4,6,9})
            return v;
        }
    }
}

template <bool INV, typename V>
__device__ __forceinline__ void dft8(V* x) {
    using R = decltype(x[0].x);
    // radix-2 x 4: even/odd split
    dft4<INV>(x[0], x[2], x[4], x[6]);
    dft4<INV>(x[1], x[3], x[5], x[7]);
    constexpr R h = (R)0.70710678118654752440;
    const R sg = INV ? (R)1 : (R)-1;
    // twiddle odd outputs by W8^k
    const V o1 = cmul(x[3], V{h, sg * h});
    const V o2 = rot90<INV>(x[5]);
    const V o3 = cmul(x[7], V{-h, sg * h});
    const V e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6], o0 = x[1];
    x[0] = cadd(e0, o0);
    x[4] = csub(e0, o0);
    x[1] = cadd(e1, o1);
    x[5] = csub(e1, o1);
    x[2] = cadd(e2, o2);
    x[6] = csub(e2, o2);
    x[3] = cadd(e3, o3);
    x[7] = csub(e3, o3);
}

// In-register 16-point DFT (4x4 Cooley-Tukey). Input natural order; the
// output is left TRANSPOSED: register 4*k1 + k2 holds X[k1 + 4*k2]
// (see out_slot), which saves a 16-element register shuffle.
template <bool INV, typename V>
__device__ __forceinline__ void dft16(V* x) {
    using R = decltype(x[0].x);
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(x[n2], x[4 + n2], x[8 + n2], x[12 + n2]);
    // x[4*k1 + n2] = T[k1][n2]; twiddle by W16^{n2*k1}
#pragma unroll
    for (int k1 = 1; k1 < 4; ++k1) {
#pragma unroll
        for (int n2 = 1; n2 < 4; ++n2) x[4 * k1 + n2] = tw16<INV, V, R>(x[4 * k1 + n2], n2 * k1);
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(x[4 * k1], x[4 * k1 + 1], x[4 * k1 + 2], x[4 * k1 + 3]);
}

// Output index held by register slot i after dft_r<RADIX>.
template <int RADIX>
__device__ __forceinline__ constexpr int out_slot(int i) {
    return RADIX == 16 ? (i >> 2) + 4 * (i & 3) : i;
}

template <int RADIX, bool INV, typename V>
__device__ __forceinline__ void dft_r(V* x) {
    if constexpr (RADIX == 16) dft16<INV>(x);
    else if constexpr (RADIX == 8) dft8<INV>(x);
    else if constexpr (RADIX == 4) dft4<INV>(x[0], x[1], x[2], x[3]);
    else dft2<INV>(x[0], x[1]);
}

// Twiddle sources. A pass of radix R at sub-transform length ns needs
// w(k, e) = e^{-2 pi i step e / M}, step = (M / (ns R)) k; the real split/merge
// needs h(k) = e^{-2 pi i k / N}, N = 2M, k in [0, M].
//   TwGlobal: one table e^{-2 pi i k / Nt} in global memory, read at stride
//             tws (Nt = tws * N for a table shared with a larger size).
//   TwShared: compact per-pass tables in shared memory for M = 4096
//             (radix-16 passes at ns = 16 and 256 need e in {1,2,4,8} only)
//             and a two-level table for h(k) = A[k >> 6] * B[k & 63].
template <typename V> struct TwGlobal {
    const V* __restrict__ tw;
    int tws;
    __device__ __forceinline__ V w(int M, int ns, int R, int k, int e) const {
        return tw[(size_t)((M / (ns * R)) * k * e) * tws];
    }
    __device__ __forceinline__ V h(int k) const { return tw[k]; }
};

constexpr int kTwSharedM = 4096;
constexpr int kTwSharedCount = 16 * 4 + 256 * 4 + 65 + 64; // complex entries
template <typename V> struct TwShared {
    const V* t; // [t16: 4 x 16][t256: 4 x 256][A: 65][B: 64], exponent-major (lanes = k: conflict-free)
    __device__ __forceinline__ V w(int, int ns, int, int k, int e) const {
        const int le = e == 1 ? 0 : e == 2 ? 1 : e == 4 ? 2 : 3;
        return ns == 16 ? t[le * 16 + k] : t[64 + le * 256 + k];
    }
    __device__ __forceinline__ V h(int k) const {
        const V a = t[64 + 1024 + (k >> 6)], b = t[64 + 1024 + 65 + (k & 63)];
        return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
    }
};

// One Stockham pass: radix RADIX, current sub-transform length ns, M points.
// src element i at src[SRC_PADDED ? pad16(i) : i]; dst always padded.
// In place (src == dst) is allowed: every thread loads all of its inputs
// before a CTA barrier, then stores. M / RADIX butterflies over kGroupThreads
// threads: BPT = ceil(M / RADIX / kGroupThreads) per thread (1 up to M = 4096
// with radix 16, 2 for M = 8192).
// Sink: the last pass of a transform may hand its outputs (index, value) to a
// consumer instead of storing them (the consumer runs after the pre-store
// barrier, so it may overwrite the buffer; no trailing barrier).
struct NoSink {
    template <typename V> __device__ __forceinline__ void operator()(int, V) const {}
};

template <int RADIX, bool INV, bool SRC_PADDED, int M, typename V, typename TW, typename Sink = NoSink>
__device__ __forceinline__ void stockham_pass(const V* src, V* dst, int ns, const TW& tw, Sink sink = {}) {
    constexpr bool kSink = !std::is_same<Sink, NoSink>::value;
    static_assert(!kSink || SRC_PADDED, "a sink pass runs in place");
    // SRC_PADDED: in place in the shared buffer, so every thread's loads must
    // finish before any store (barrier below). Otherwise src is a different
    // (global) array and dst is free (callers end their previous use of the
    // buffer with a barrier): no pre-store barrier.
    constexpr int nj = M / RADIX;
    constexpr int BPT = (nj + kGroupThreads - 1) / kGroupThreads;
    V v[BPT][RADIX];
#pragma unroll
    for (int bt = 0; bt < BPT; ++bt) {
        const int j = gtid() + bt * kGroupThreads;
        if (j < nj) {
#pragma unroll
            for (int r = 0; r < RADIX; ++r) {
                const int i = j + r * nj;
                v[bt][r] = src[SRC_PADDED ? pad16(i) : i];
            }
            const int k = j % ns;
            if (ns > 1) {
                if constexpr (RADIX == 16) {
                    // w^1, w^2, w^4, w^8 from the table, the other powers by at most
                    // three products (<= 3 roundings): 4 loads instead of 15
                    V w[16];
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
#pragma unroll
                    for (int r = 1; r < 16; ++r) v[bt][r] = cmul(v[bt][r], INV ? cconj(w[r]) : w[r]);
                } else {
#pragma unroll
                    for (int r = 1; r < RADIX; ++r) {
                        V w = tw.w(M, ns, RADIX, k, r);
                        if (INV) w.y = -w.y;
                        v[bt][r] = cmul(v[bt][r], w);
                    }
                }
            }
            dft_r<RADIX, INV>(v[bt]);
        }
    }
    if constexpr (SRC_PADDED) gsync();
#pragma unroll
    for (int bt = 0; bt < BPT; ++bt) {
        const int j = gtid() + bt * kGroupThreads;
        if (j < nj) {
            const int k = j % ns;
            const int base = (j / ns) * ns * RADIX + k;
#pragma unroll
            for (int r = 0; r < RADIX; ++r) {
                if constexpr (kSink) sink(base + out_slot<RADIX>(r) * ns, v[bt][r]);
                else dst[pad16(base + out_slot<RADIX>(r) * ns)] = v[bt][r];
            }
        }
    }
    if constexpr (!kSink) gsync();
}

// Full M-point complex FFT, M a compile-time power of two in [16, 8192]:
// radix-16 passes, then one radix-2/4/8 pass for the remaining factor. The
// first pass reads `src` (padded or not); later passes work in place on `buf`.
// With a sink, the last pass hands its outputs to it (see stockham_pass).
template <int M, bool INV, bool SRC_PADDED, int NS = 1, typename V, typename TW, typename Sink = NoSink>
__device__ __forceinline__ void cfft(const V* src, V* buf, const TW& tw, Sink sink = {}) {
    constexpr int REM = M / NS;
    if constexpr (REM == 16) {
        stockham_pass<16, INV, SRC_PADDED, M>(src, buf, NS, tw, sink);
    } else if constexpr (REM > 16) {
        stockham_pass<16, INV, SRC_PADDED, M>(src, buf, NS, tw);
        cfft<M, INV, true, NS * 16>(buf, buf, tw, sink);
    } else if constexpr (REM > 1) {
        stockham_pass<REM, INV, SRC_PADDED, M>(src, buf, NS, tw, sink);
    }
}

// Split/merge between the M-point complex transform of a packed real signal
// and its half spectrum, fused with a per-bin spectral operator, then merged
// back for the inverse real transform (all in place in padded `buf`).
//   forward:  X[k] = E[k] + W_N^k O[k],  E = (Z_k + Z*_{M-k})/2, O = (Z_k - Z*_{M-k})/(2i)
//   op:       Y[k] = op(X[k], k)         (must keep Y Hermitian-consistent)
//   inverse:  Z'[k] = E' + i O',  E' = (Y_k + Y*_{M-k})/2, O' = (Y_k - Y*_{M-k}) conj(W_N^k)/2
// tw.h(k) = e^{-2 pi i k / N} for k in [0, M].
template <typename V, typename TW, typename Op>
__device__ __forceinline__ void real_spectral_op(V* buf, int M, const TW& tw, Op op) {
    using R = decltype(V{}.x);
    for (int k = gtid(); k <= M / 2; k += kGroupThreads) {
        if (k == 0) {
            const V z0 = buf[0];
            const V x0 = {z0.x + z0.y, (R)0};
            const V xm = {z0.x - z0.y, (R)0};
            const V y0 = op(x0, 0);
            const V ym = op(xm, M);
            // imag(Y[0]), imag(Y[M]) ignored (FFTW c2r convention)
            const R e = (R)0.5 * (y0.x + ym.x);
            const R o = (R)0.5 * (y0.x - ym.x);
            buf[0] = V{e, o};
            continue;
        }
        const int kk = M - k;
        const V zk = buf[pad16(k)], zkk = buf[pad16(kk)];
        const V wk = tw.h(k), wkk = tw.h(kk);
        // forward split
        const V ek = {(R)0.5 * (zk.x + zkk.x), (R)0.5 * (zk.y - zkk.y)};
        const V dk = {(R)0.5 * (zk.x - zkk.x), (R)0.5 * (zk.y + zkk.y)}; // (Z_k - Z*_kk)/2
        const V ok = {dk.y, -dk.x};                                    // / i
        const V xk = cadd(ek, cmul(wk, ok));
        const V ekk = {ek.x, -ek.y};       // E_{M-k} = conj(E_k)
        const V okk = {ok.x, -ok.y};       // O_{M-k} = conj(O_k)
        const V xkk = cadd(ekk, cmul(wkk, okk));
        const V yk = op(xk, k), ykk = op(xkk, kk);
        // inverse merge
        const V e2 = {(R)0.5 * (yk.x + ykk.x), (R)0.5 * (yk.y - ykk.y)};
        const V d2 = {(R)0.5 * (yk.x - ykk.x), (R)0.5 * (yk.y + ykk.y)};
        const V o2 = cmul(d2, cconj(wk));
        buf[pad16(k)] = V{e2.x - o2.y, e2.y + o2.x};
        if (kk != k) {
            const V e3 = {(R)0.5 * (ykk.x + yk.x), (R)0.5 * (ykk.y - yk.y)};
            const V d3 = {(R)0.5 * (ykk.x - yk.x), (R)0.5 * (ykk.y + yk.y)};
            const V o3 = cmul(d3, cconj(wkk));
            buf[pad16(kk)] = V{e3.x - o3.y, e3.y + o3.x};
        }
    }
    gsync();
}

// real_spectral_op specialised to the Hilbert operator of pipeline.cpp:456-459
// (Y[k] = -i s X[k], DC and Nyquist zeroed, s = 2/N the inverse scaling).
// Substituting the operator into split -> op -> merge collapses to
//   Z'[k]   = s (cos t_k conj(Z[M-k]) + i sin t_k Z[k]),
//   Z'[M-k] = s (i sin t_k Z[M-k] - cos t_k conj(Z[k])),   t_k = 2 pi k / N,
// one twiddle and 4 multiply-adds per bin pair instead of ~50 operations
// (s is a power of two, so folding it into the twiddle is exact).
template <typename V, typename TW, typename R>
__device__ __forceinline__ void hilbert_spectral(V* buf, int M, const TW& tw, R s) {
    for (int k = gtid(); k < M / 2; k += kGroupThreads) {
        if (k == 0) {
            buf[0] = V{(R)0, (R)0}; // DC and Nyquist (packed in Z[0]) zeroed
            const V z = buf[pad16(M / 2)];
            const V w = tw.h(M / 2);
            const R c = s * w.x, sn = -s * w.y;
            buf[pad16(M / 2)] = V{c * z.x - sn * z.y, sn * z.x - c * z.y};
            continue;
        }
        const int kk = M - k;
        const V zk = buf[pad16(k)], zkk = buf[pad16(kk)];
        const V w = tw.h(k); // (cos t_k, -sin t_k)
        const R c = s * w.x, sn = -s * w.y;
        buf[pad16(k)] = V{c * zkk.x - sn * zk.y, sn * zk.x - c * zkk.y};
        buf[pad16(kk)] = V{-c * zk.x - sn * zkk.y, c * zk.y + sn * zkk.x};
    }
    gsync();
}

// cos(k pi / 16) as exact literals (twiddles of the Hilbert operator)
__device__ __forceinline__ constexpr double cos_pi16(int k) { // cos(k pi / 16), k in [0, 8]
    return k == 0 ? 1.0 : k == 1 ? 0.98078528040323044913 : k == 2 ? 0.92387953251128675613
         : k == 3 ? 0.83146961230254523708 : k == 4 ? 0.70710678118654752440 : k == 5 ? 0.55557023301960222474
         : k == 6 ? 0.38268343236508977173 : k == 7 ? 0.19509032201612826785 : 0.0;
}

// ---------------------------------------------------------------------------
// In-place M = 4096 transform pair for the Hilbert envelope (3 radix-16
// passes each way, one butterfly per thread): every pass after the first
// loads and stores the SAME 16 positions, so no barrier is needed between a
// pass's loads and its stores (the Stockham passes above need one).
// Forward: decimation in frequency, natural input, output digit-reversed:
//   position 256 k1 + 16 k2 + k3 holds X[k1 + 16 k2 + 256 k3].
// Inverse: decimation in time from that digit-reversed order, natural output.
// Index digits: n = 256 n1 + 16 n2 + n3, k = k1 + 16 k2 + 256 k3.
// ---------------------------------------------------------------------------
// the 15 twiddle powers w^e, e = 1..15, from w^1, w^2, w^4, w^8 (4 table loads)
template <typename V, typename TW>
__device__ __forceinline__ void tw_powers(const TW& tw, int ns, int k, V (&w)[16]) {
    w[1] = tw.w(4096, ns, 16, k, 1);
    w[2] = tw.w(4096, ns, 16, k, 2);
    w[4] = tw.w(4096, ns, 16, k, 4);
    w[8] = tw.w(4096, ns, 16, k, 8);
    w[3] = cmul(w[1], w[2]);
    w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]);
    w[7] = cmul(w[3], w[4]);
#pragma unroll
    for (int r = 9; r < 16; ++r) w[r] = cmul(w[r - 8], w[8]);
}

// forward pass 1: v[r] = x[j + 256 r] (j = gtid()); A[k1][j] = DFT16_n1 * W4096^{j k1}
// stored at j + 256 k1
template <typename V, typename TW>
__device__ __forceinline__ void dif_pass1_4096(V (&v)[16], V* buf, const TW& tw) {
    const int j = gtid();
    dft16<false>(v);
    V w[16];
    tw_powers(tw, 256, j, w);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int k1 = out_slot<16>(r);
        const V y = k1 ? cmul(v[r], w[k1 ? k1 : 1]) : v[r];
        buf[pad16(j + 256 * k1)] = y;
    }
    gsync();
}

// forward pass 2 (thread (k1, n3)): DFT16 over n2, * W256^{n3 k2}, in place
template <typename V, typename TW>
__device__ __forceinline__ void dif_pass2_4096(V* buf, const TW& tw) {
    const int t = gtid(), k1 = t >> 4, n3 = t & 15;
    V v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[pad16(256 * k1 + 16 * r + n3)];
    dft16<false>(v);
    V w[16];
    tw_powers(tw, 16, n3, w);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int k2 = out_slot<16>(r);
        const V y = k2 ? cmul(v[r], w[k2 ? k2 : 1]) : v[r];
        buf[pad16(256 * k1 + 16 * k2 + n3)] = y;
    }
    gsync();
}

// Forward pass 3 + the Hilbert operator + inverse stage A, in registers and in
// place. Thread (k1, k2), a = k1 + 16 k2, holds X[a + 256 k3], k3 = 0..15; the
// complementary bins M - a - 256 k3 = (256 - a) + 256 (15 - k3) belong to
// thread 256 - a: lanes l < 16 of warp w < 7 take k1 = w + 1, k2 = l, lanes
// l + 16 the partner (k1 = 15 - w, k2 = 15 - l); warp 7 holds k1 = 0 (lanes
// 0-15) and k1 = 8 (lanes 16-31), partners inside the half-warp (a = 0 and
// a = 128 pair with themselves). Row 16 k1 + k2 of the padded buffer differs
// mod 8 within every quarter-warp: conflict-free 16-byte accesses.
template <typename V, typename TW, typename R>
__device__ __forceinline__ void hilbert_mid_dif_4096(V* buf, const TW& tw, R s) {
    const int t = gtid(), w = t >> 5, l = t & 31;
    int k1, k2, src;
    if (w < 7) {
        k1 = l < 16 ? w + 1 : 15 - w;
        k2 = l < 16 ? l : 31 - l;
        src = l ^ 16;
    } else {
        k1 = l < 16 ? 0 : 8;
        k2 = l & 15;
        src = l < 16 ? ((16 - l) & 15) : 47 - l;
    }
    const int a = k1 + 16 * k2, row = 256 * k1 + 16 * k2;
    const bool self0 = a == 0;
    V z[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) z[r] = buf[pad16(row + r)];
    dft16<false>(z); // z[out_slot(S)] = X[a + 256 S]
    const V ha = tw.h(a);
    const R cj = s * ha.x, sj = -s * ha.y;
    auto cosS = [](int S) { return (R)(S <= 8 ? cos_pi16(S) : -cos_pi16(16 - S)); };
    auto sinS = [](int S) { return (R)cos_pi16(S <= 8 ? 8 - S : S - 8); };
    auto op = [&](V zk, V zc, int S) {
        const R c = cj * cosS(S) - sj * sinS(S), sn = sj * cosS(S) + cj * sinS(S);
        return V{c * zc.x - sn * zk.y, sn * zk.x - c * zc.y};
    };
    auto shfl = [&](V v) {
        return V{__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)};
    };
#pragma unroll
    for (int S = 0; S < 8; ++S) {
        V& x0 = z[out_slot<16>(S)];
        V& x1 = z[out_slot<16>(15 - S)];
        const V pa = shfl(x1), pb = shfl(x0); // partner's X[. + 256 (15 - S)], X[. + 256 S]
        if (!self0) {
            const V n0 = op(x0, pa, S), n1 = op(x1, pb, 15 - S);
            x0 = n0;
            x1 = n1;
        }
    }
    if (self0) {
        // bins 256 S pair with 256 (16 - S); DC and Nyquist (Z[0]) zeroed
        z[0] = V{(R)0, (R)0};
#pragma unroll
        for (int S = 1; S <= 8; ++S) {
            V& x0 = z[out_slot<16>(S)];
            V& x1 = z[out_slot<16>(16 - S)];
            const V n0 = op(x0, x1, S), n1 = op(x1, x0, 16 - S);
            x0 = n0;
            if (S != 8) x1 = n1;
        }
    }
    // inverse stage A: DFT16 over k3 of Z'[a + 256 k3] -> A[k1][k2][n3], stored
    // in place (this thread's own row: no barrier before the stores)
    V x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = z[out_slot<16>(r)];
    dft16<true>(x);
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[pad16(row + out_slot<16>(r))] = x[r];
    gsync();
}

// The ODD-bin half of an M = 8192 transform split by one radix-2 DIF stage
// (k = 2 k' + 1, k' < 4096, held like the M = 4096 forward output): bin k'
// pairs with 4095 - k' (M - k = 2 (4095 - k') + 1), i.e. row a = k1 + 16 k2
// with row 255 - a = (15 - k1) + 16 (15 - k2) at k3 -> 15 - k3 (no bin pairs
// with itself). Lanes l < 16 of warp w take k1 = w, k2 = l, lanes l + 16 the
// partner rows; t_k = 2 pi (2 k' + 1) / 16384: the row part e^{-2 pi i (2a+1)/16384}
// comes from the N = 16384 table `h16384`, the k3 part is pi k3 / 16 as above.
template <typename V, typename TW, typename R>
__device__ __forceinline__ void hilbert_mid_dif_4096_odd(V* buf, const TW& tw, const V* h16384, R s) {
    const int t = gtid(), w = t >> 5, l = t & 31;
    const int k1 = l < 16 ? w : 15 - w;
    const int k2 = l < 16 ? l : 31 - l;
    const int src = l ^ 16;
    const int a = k1 + 16 * k2, row = 256 * k1 + 16 * k2;
    V z[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) z[r] = buf[pad16(row + r)];
    dft16<false>(z); // z[out_slot(S)] = O[a + 256 S]
    const V ha = h16384[2 * a + 1];
    const R cj = s * ha.x, sj = -s * ha.y;
    auto cosS = [](int S) { return (R)(S <= 8 ? cos_pi16(S) : -cos_pi16(16 - S)); };
    auto sinS = [](int S) { return (R)cos_pi16(S <= 8 ? 8 - S : S - 8); };
    auto shfl = [&](V v) {
        return V{__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)};
    };
    V nz[16];
#pragma unroll
    for (int S = 0; S < 16; ++S) {
        // partner's O[(255 - a) + 256 (15 - S)]
        const V pc = shfl(z[out_slot<16>(15 - S)]);
        const R c = cj * cosS(S) - sj * sinS(S), sn = sj * cosS(S) + cj * sinS(S);
        const V zk = z[out_slot<16>(S)];
        nz[S] = V{c * pc.x - sn * zk.y, sn * zk.x - c * pc.y};
    }
    V x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = nz[r];
    dft16<true>(x);
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[pad16(row + out_slot<16>(r))] = x[r];
    gsync();
}

// inverse stage B (thread (k1, n3)): * conj W256^{k2 n3}, DFT16 over k2, in place
template <typename V, typename TW>
__device__ __forceinline__ void dit_pass2_4096(V* buf, const TW& tw) {
    const int t = gtid(), k1 = t >> 4, n3 = t & 15;
    V v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[pad16(256 * k1 + 16 * r + n3)];
    V w[16];
    tw_powers(tw, 16, n3, w);
#pragma unroll
    for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], cconj(w[r]));
    dft16<true>(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[pad16(256 * k1 + 16 * out_slot<16>(r) + n3)] = v[r];
    gsync();
}

// inverse stage C (thread m = n3 + 16 n2): * conj W4096^{k1 m}, DFT16 over k1;
// output z[m + 256 n1] (natural order) handed to sink(n, value) after a
// barrier (the sink may overwrite the buffer)
template <typename V, typename TW, typename Sink>
__device__ __forceinline__ void dit_pass3_4096(V* buf, const TW& tw, Sink sink) {
    const int m = gtid();
    V v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[pad16(256 * r + m)];
    V w[16];
    tw_powers(tw, 256, m, w);
#pragma unroll
    for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], cconj(w[r]));
    dft16<true>(v);
    gsync();
#pragma unroll
    for (int r = 0; r < 16; ++r) sink(m + 256 * out_slot<16>(r), v[r]);
}

// inverse stage C as above, the thread's whole output row handed to
// sink(m, v) after the barrier: v[r] = z[m + 256 out_slot(r)]
template <typename V, typename TW, typename Sink>
__device__ __forceinline__ void dit_pass3_4096_row(V* buf, const TW& tw, Sink sink) {
    const int m = gtid();
    V v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[pad16(256 * r + m)];
    V w[16];
    tw_powers(tw, 256, m, w);
#pragma unroll
    for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], cconj(w[r]));
    dft16<true>(v);
    gsync();
    sink(m, v);
}

// ---------------------------------------------------------------------------
// Smoothing FIR by FFT (the composite 447-tap filter at stride 10 of
// pipeline.cpp:466-468, default shapes). In polyphase form the decimated
// output is a sum of ten 45-tap correlations,
//     out[o] = sum_p sum_q G_p[q] E_p[o + q],  E_p[u] = env[10 u - c0 + p],
// G_p[q] = rev[10 q + p]; with o < bins and q < 45 every index stays below
// 768 >= bins + 44, so a cyclic length-768 correlation is exact (entries
// [bins + 44, 768) of a phase only reach discarded outputs; they hold
// envelope samples or zeros, never garbage).
// The two samples of one magnitude pair (t = n + c0 odd, t + 1) land in one
// complex slot: sequence a = (t mod 10 - 1) / 2 carries
//     c_a[u] = E_{2a+1}[u] + i E_{2a+2}[u]       (a < 4)
//     c_4[u] = E_9[u]      + i E_0[u + 1]         (phase 0 advanced by one:
//                                                  its taps delayed by one, cyclically)
// and for real filters the ten correlations collapse to
//     out = Re( IDFT768( sum_a C_a U_a ) ),
//     U_a = (conj Ghat_re - i conj Ghat_im) / 768            (host table)
// i.e. five forward FFTs, one multiply-accumulate and one inverse FFT:
// ~180k FP64 operations per beam instead of 655 x 450 = 295k FMAs.
// 768 = 3 x 16 x 16, in place over the group buffer:
//   forward (decimation in frequency, natural input): radix 3 over n1
//   (stride 256), radix 16 over n2 (stride 16), radix 16 over n3; position
//   256 k1 + 16 k2 + k3 ends up holding C[k1 + 3 k2 + 48 k3];
//   inverse (decimation in time from that order back to natural order).
// Slot of (sequence a, position x): a * kFfStride + pad16(x); kFfStride = 5
// mod 8 so the sink's lanes (a = 0..4 cycling, u advancing every 5 lanes)
// hit distinct bank groups. Every pass loads and stores the same slots per
// thread (no barrier between a pass's loads and its stores).
// ---------------------------------------------------------------------------
constexpr int kFfL = 768, kFfSeq = 5, kFfThreads = 240; // radix-16 butterflies of the 5 forward FFTs
constexpr int kFfStride = 821;                           // >= pad16(767) + 1, = 5 mod 8
constexpr int kFfSlots = 4 * kFfStride + 816;            // complex slots of the FIR layout
constexpr int kFfU = 16 * kFfThreads;                    // spectrum factors (complex)
constexpr int kFfW = 512;                                // twiddles: w768^j (j < 256), w256^{n3 k2} (16 x 16)
__device__ __forceinline__ int ff_slot(int a, int x) { return a * kFfStride + pad16(x); }

// w16^k = w256^{16 k} from the 16 x 16 table w256^{n3 k2} (at 16 k2 + n3),
// k = q m in {0, 1, 2, 3, 4, 6, 9} (lane-dependent: a table load, not a branch)
template <typename V>
__device__ __forceinline__ V w16_pow(const V* w256, int k) { return w256[k == 9 ? 16 * 12 + 12 : 16 * 8 + 2 * k]; }

template <bool INV, typename V>
__device__ __forceinline__ void dft3(V& x0, V& x1, V& x2) {
    using R = decltype(V{}.x);
    constexpr R h = (R)0.86602540378443864676; // sin(2 pi / 3)
    const V s = cadd(x1, x2);
    const V t = {x0.x - (R)0.5 * s.x, x0.y - (R)0.5 * s.y};
    const V d = csub(x1, x2);
    // forward: (x1 - x2) * (-i h); inverse: (x1 - x2) * (+i h)
    const V u = INV ? V{-h * d.y, h * d.x} : V{h * d.y, -h * d.x};
    x0 = cadd(x0, s);
    x1 = cadd(t, u);
    x2 = csub(t, u);
}

// out[o] = max(0, float(r[o])) for o < bins. U: [16][kFfThreads] in the
// register order of the third forward pass; W: [w768^j, j < 256][w256^{n3 k2}
// at 16 k2 + n3] (e^{-2 pi i . / n}); both in shared memory.
// PASS1 == false: the first forward pass was done by the producer of the
// layout (the envelope's fused sink, which holds the three samples of each
// radix-3 butterfly in one thread).
template <bool PASS1 = true, typename V>
__device__ __forceinline__ void fir_fft768(V* buf, const V* U, const V* W, float* __restrict__ eo, int bins) {
    using R = decltype(V{}.x);
    int t = gtid();
    // opaque per call: keeps the compiler from hoisting every pass's
    // (loop-invariant) shared-memory addresses out of the item loop and
    // spilling them
    asm volatile("" : "+r"(t));
    const V* w256 = W + 256;
    if constexpr (PASS1) {
        // forward pass 1: radix 3 over n1, * w768^{j k1}, the five sequences
        const int j = t;
        const V w1 = W[j], w2 = cmul(w1, w1);
#pragma unroll
        for (int a = 0; a < kFfSeq; ++a) {
            V x0 = buf[ff_slot(a, j)], x1 = buf[ff_slot(a, j + 256)], x2 = buf[ff_slot(a, j + 512)];
            dft3<false>(x0, x1, x2);
            buf[ff_slot(a, j)] = x0;
            buf[ff_slot(a, j + 256)] = cmul(x1, w1);
            buf[ff_slot(a, j + 512)] = cmul(x2, w2);
        }
        gsync();
    }
    if (t < kFfThreads) {
        // forward pass 2 (thread (a, k1, n3)): DFT16 over n2, * w256^{n3 k2}
        const int a = t / 48, rem = t - 48 * a, k1 = rem >> 4, n3 = rem & 15;
        V* s = buf + a * kFfStride;
        const int b = 256 * k1 + n3;
        V v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = s[pad16(b + 16 * r)];
        dft16<false>(v);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int k2 = out_slot<16>(r);
            s[pad16(b + 16 * k2)] = k2 ? cmul(v[r], w256[16 * k2 + n3]) : v[r];
        }
    }
    gsync();
    if (t < kFfThreads) {
        // forward pass 3 (thread (a, k1, k2)): DFT16 over n3, times U_a
        const int a = t / 48, rem = t - 48 * a;
        V* s = buf + a * kFfStride;
        const int b = 16 * rem; // 256 k1 + 16 k2
        V v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = s[pad16(b + r)];
        dft16<false>(v);
#pragma unroll
        for (int r = 0; r < 16; ++r) s[pad16(b + out_slot<16>(r))] = cmul(v[r], U[r * kFfThreads + t]);
    }
    gsync();
    if (t < 192) {
        // inverse pass A: DFT16 over k3 of the sum over the five sequences, for
        // group g = (k1, k2) (positions 16 g + k3), four lanes per group:
        // lane q takes k3 = q + 4 i, DFT4 over i, * w16^{q m}, exchange
        // through shared memory (slot 4 q + m), DFT4 over q; output n3 = m + 4 p
        // at slot m + 4 p. Lanes of a quarter-warp serve 8 different groups
        // (rows 17 apart): conflict-free.
        const int l = t & 31, g = 8 * (t >> 5) + (l & 7), q = l >> 3;
        V* s = buf + pad16(16 * g);
        V x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            V acc = s[q + 4 * i];
#pragma unroll
            for (int a = 1; a < kFfSeq; ++a) acc = cadd(acc, s[a * kFfStride + q + 4 * i]);
            x[i] = acc;
        }
        dft4<true>(x[0], x[1], x[2], x[3]);
#pragma unroll
        for (int m = 1; m < 4; ++m) x[m] = cmul(x[m], cconj(w16_pow(w256, q * m)));
        __syncwarp();
#pragma unroll
        for (int m = 0; m < 4; ++m) s[4 * q + m] = x[m];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = s[4 * i + q]; // T_i[m = q]
        dft4<true>(x[0], x[1], x[2], x[3]);
#pragma unroll
        for (int p = 0; p < 4; ++p) s[q + 4 * p] = x[p];
    }
    gsync();
    if (t < 192) {
        // inverse pass B: * conj w256^{n3 k2}, DFT16 over k2 for group
        // g = (k1, n3) (positions 256 k1 + n3 + 16 k2), four lanes per group as
        // in pass A
        const int l = t & 31, g = 8 * (t >> 5) + (l & 7), q = l >> 3;
        const int n3 = g & 15;
        V* s = buf + 272 * (g >> 4) + n3; // pad16(256 k1 + 16 k2 + n3) = 272 k1 + 17 k2 + n3
        auto at = [&](int k2) -> V& { return s[17 * k2]; };
        V x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k2 = q + 4 * i;
            x[i] = k2 ? cmul(at(k2), cconj(w256[16 * k2 + n3])) : at(k2);
        }
        dft4<true>(x[0], x[1], x[2], x[3]);
#pragma unroll
        for (int m = 1; m < 4; ++m) x[m] = cmul(x[m], cconj(w16_pow(w256, q * m)));
        __syncwarp();
#pragma unroll
        for (int m = 0; m < 4; ++m) at(4 * q + m) = x[m];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = at(4 * i + q);
        dft4<true>(x[0], x[1], x[2], x[3]);
#pragma unroll
        for (int p = 0; p < 4; ++p) at(q + 4 * p) = x[p];
    }
    gsync();
    {
        // inverse pass C (thread j = 16 n2 + n3): * conj w768^{j k1}, radix 3
        // over k1, real parts only; out[256 n1 + j]
        const int j = t;
        constexpr R h = (R)0.86602540378443864676;
        const V w1 = W[j], w2 = cmul(w1, w1);
        const V y0 = buf[pad16(j)];
        const V y1 = cmul(buf[pad16(j + 256)], cconj(w1));
        const V y2 = cmul(buf[pad16(j + 512)], cconj(w2));
        const R c = y0.x - (R)0.5 * (y1.x + y2.x), sn = h * (y1.y - y2.y);
        const R r0 = y0.x + y1.x + y2.x, r1 = c - sn, r2 = c + sn;
        auto put = [&](int o, R r) {
            if (o < bins) {
                const float f = (float)r;
                eo[o] = f > 0.0f ? f : 0.0f;
            }
        };
        put(j, r0);
        put(j + 256, r1);
        put(j + 512, r2);
    }
}
} // namespace snb
