// Delay-and-sum beamforming on the int8 tensor cores (tcgen05.mma kind::i8),
// exact in integer arithmetic.
//
// The reference (beamform_into, pipeline.cpp:432-446) forms, per direction d,
//     y_d[n] = (1/32) sum_i x_i[n - s_{d,i}]          (zero outside [0, L))
// with integer shifts s_{d,i} = delay - advance. For a cluster of 128
// directions (consecutive k-d slots, Plan::order) the shifts of channel i lie
// in [b_i, b_i + R) with R ~ 23 on the hemisphere3000 grid, so with the
// re-centred channels x'_i[t] = x_i[t - b_i]
//     y_d[n] = sum_{r < R} sum_{i < 32} A_r[d][i] * x'_i[n - r],
//     A_r[d][i] = (s_{d,i} - b_i == r)  in {0, 1}
// i.e. R accumulating GEMMs D(128 x N) += A_r(128 x 32) * X_r^T(32 x N): a
// dense steering-matrix contraction (the "0/1 steering matrix" of the
// north star) whose B operand for shift r is the same time window displaced
// by r rows. The samples are quantised to 46-bit block floating point per
// capture (X = round(x * 2^46 / max|x|)), split into six balanced base-256
// digits (int8), and each digit plane is contracted separately with int32
// accumulation in tensor memory (|sum| <= 32 * 128: exact). The epilogue
// recombines Y = sum_j 256^j Y_j exactly in int64 and scales once:
//     beam = fl(Y * max|x| * 2^-46 / 32)
// — the exactly rounded sum of the quantised samples, whose error
// (<= 2^-47 max|x|) is the same size as the reference's own FP64 summation
// error (32 roundings of 2^-53 |partial|).
//
// Shared-memory operand layouts (SWIZZLE_NONE, K-major, 16-byte core rows):
//   B window, per digit j and channel half h: rows q = 0 .. N + R - 2 of 16
//     bytes (16 channels), i.e. a uniform 16-byte row stride (SBO = 128 B per
//     8 rows), the halves LBO apart. The operand for shift r starts at row
//     R - 1 - r: any r is a 16-byte aligned descriptor offset, so the shifted
//     operands are free (no copies).
//   A_r: [half][128 rows][16 B], LBO = 2048 B, SBO = 128 B; built by the
//     threads from their direction's residual bytes with one SIMD compare per
//     4 channels, double-buffered in chunks of kTcRChunk shifts whose reuse is
//     gated by tcgen05.commit -> mbarrier.
// TMEM: 6 accumulators of N = 80 int32 columns (480 of 512), lane = direction.
#include "kernels.cuh"

#include <cstdint>

namespace snb {

namespace {

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor (SWIZZLE_NONE, version 1 = sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}

// Instruction descriptor: kind::i8, signed A and B, S32 accumulate, K-major
// A and B, M x N.
constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SNB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SNB_WAIT_%=;\n}\n" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(smem_dst)), "l"(gsrc) : "memory");
}

constexpr int kTcThreads = 128;
constexpr int kTmemCols = 512;
constexpr int kABytes = 2 * kTcM * 16; // one shift: two channel halves x 128 rows x 16 B

} // namespace

// ---------------------------------------------------------------------------
// k_digits: filt (FP64) -> per-cluster re-centred digit planes.
// planes[((b * C + c) * 12 + 2 j + h) * rows + row][l] = digit j of
// X_i[row - pad - base[c][i]], i = 16 h + l, X = round(x * 2^46 / max|x|).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_digits(DigitArgs a) {
    const int c = blockIdx.y, b = blockIdx.z;
    const int nblk = (a.rows + 127) / 128;
    const int h = blockIdx.x / nblk;
    const int row = (blockIdx.x % nblk) * 128 + threadIdx.x;
    if (row >= a.rows) return;
    double amax = __longlong_as_double((long long)a.amax_bits[b]);
    const double inv = amax > 0.0 ? 70368744177664.0 / amax : 0.0; // 2^46 / max|x|
    const int64_t t = (int64_t)row - a.pad;
    const double* fb = a.filt + ((size_t)b * 32 + 16 * h) * a.Lp + a.H;
    const int32_t* base = a.base + (size_t)c * 32 + 16 * h;
    uint32_t w[kTcSlices][4];
#pragma unroll
    for (int j = 0; j < kTcSlices; ++j) w[j][0] = w[j][1] = w[j][2] = w[j][3] = 0;
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        const int64_t tp = t - base[l];
        const double x = (tp >= 0 && tp < a.L) ? fb[(size_t)l * a.Lp + tp] : 0.0;
        long long X = __double2ll_rn(x * inv);
#pragma unroll
        for (int j = 0; j < kTcSlices; ++j) {
            const int d = (int)((X + 128) & 255) - 128; // balanced digit in [-128, 127]
            X = (X - d) >> 8;
            w[j][l >> 2] |= (uint32_t)(d & 255) << (8 * (l & 3));
        }
    }
    const size_t plane = ((size_t)b * a.clusters + c) * 12;
#pragma unroll
    for (int j = 0; j < kTcSlices; ++j) {
        uint4* dst = reinterpret_cast<uint4*>(a.planes + ((plane + 2 * j + h) * a.rows + row) * 16);
        *dst = make_uint4(w[j][0], w[j][1], w[j][2], w[j][3]);
    }
}

// ---------------------------------------------------------------------------
// k_beamform_tc: persistent, one CTA (4 warps) per SM; the work list of
// (cluster, capture, time tile) is cut into contiguous per-CTA ranges of
// equal estimated work (TcSched).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTcThreads, 1) k_beamform_tc(TcArgs a, const __grid_constant__ TcSched sched) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int wrows = kTcN + a.pad;                 // window rows per (digit, half)
    uint8_t* Bw = smem;                             // [12][wrows][16]
    uint8_t* Ab = Bw + (size_t)12 * wrows * 16;     // [2][kTcRChunk][kABytes]
    Ab = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(Ab) + 127) & ~uintptr_t(127));
    uint64_t* bars = reinterpret_cast<uint64_t*>(Ab + 2 * kTcRChunk * kABytes); // chunk 0, chunk 1, acc
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = idesc_i8(kTcM, kTcN);
    const uint32_t bw_addr = su32(Bw), ab_addr = su32(Ab);
    uint32_t ph0 = 0, ph1 = 0, ph_acc = 0;
    bool pend0 = false, pend1 = false;
    const int per_cb = a.batch * a.ntiles;
    for (int t = sched.start[blockIdx.x]; t < sched.start[blockIdx.x + 1]; ++t) {
        const int c = t / per_cb, rem = t - c * per_cb;
        const int b = rem / a.ntiles, tt = rem - b * a.ntiles;
        const int64_t t0 = (int64_t)tt * kTcN;
        const int R = a.R[c];
        // ---- B window: 12 planes x (N + R - 1) rows, async copies
        {
            const int nq = kTcN + R - 1;
            const int8_t* pb = a.planes + (((size_t)b * a.clusters + c) * 12 * a.rows + (a.pad + t0 - (R - 1))) * 16;
            for (int idx = tid; idx < 12 * nq; idx += kTcThreads) {
                const int jh = idx / nq, q = idx - jh * nq;
                cp_async16(Bw + ((size_t)jh * wrows + q) * 16, pb + ((size_t)jh * a.rows + q) * 16);
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        }
        // my direction's residual bytes (0xFF on padding rows: never equal to r)
        uint32_t res[8];
        {
            const uint4* rp = reinterpret_cast<const uint4*>(a.resid + ((size_t)c * kTcM + tid) * 32);
            const uint4 r0 = rp[0], r1 = rp[1];
            res[0] = r0.x; res[1] = r0.y; res[2] = r0.z; res[3] = r0.w;
            res[4] = r1.x; res[5] = r1.y; res[6] = r1.z; res[7] = r1.w;
        }
        const int nchunks = (R + kTcRChunk - 1) / kTcRChunk;
        for (int q = 0; q < nchunks; ++q) {
            const int buf = q & 1;
            if (buf == 0 && pend0) { mbar_wait(&bars[0], ph0); ph0 ^= 1; pend0 = false; }
            if (buf == 1 && pend1) { mbar_wait(&bars[1], ph1); ph1 ^= 1; pend1 = false; }
            uint8_t* abuf = Ab + (size_t)buf * kTcRChunk * kABytes;
#pragma unroll
            for (int rr = 0; rr < kTcRChunk; ++rr) {
                const int r = q * kTcRChunk + rr;
                if (r < R) {
                    const uint32_t pat = 0x01010101u * (uint32_t)r;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint4 v;
                        v.x = __vcmpeq4(res[4 * h + 0], pat) & 0x01010101u;
                        v.y = __vcmpeq4(res[4 * h + 1], pat) & 0x01010101u;
                        v.z = __vcmpeq4(res[4 * h + 2], pat) & 0x01010101u;
                        v.w = __vcmpeq4(res[4 * h + 3], pat) & 0x01010101u;
                        *reinterpret_cast<uint4*>(abuf + (size_t)rr * kABytes + h * (kTcM * 16) + tid * 16) = v;
                    }
                }
            }
            if (q == 0) asm volatile("cp.async.wait_all;\n" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                for (int rr = 0; rr < kTcRChunk; ++rr) {
                    const int r = q * kTcRChunk + rr;
                    if (r >= R) break;
                    const uint64_t ad = sdesc(ab_addr + (uint32_t)((buf * kTcRChunk + rr) * kABytes), kTcM * 16, 128);
#pragma unroll
                    for (int j = 0; j < kTcSlices; ++j) {
                        const uint32_t boff = (uint32_t)(((2 * j) * wrows + (R - 1 - r)) * 16);
                        const uint64_t bd = sdesc(bw_addr + boff, (uint32_t)(wrows * 16), 128);
                        mma_i8(tmem + (uint32_t)(j * kTcN), ad, bd, idesc, r > 0 ? 1u : 0u);
                    }
                }
                mma_commit(&bars[buf]);
                if (q == nchunks - 1) mma_commit(&bars[2]);
            }
            if (buf == 0) pend0 = true;
            else pend1 = true;
        }
        // ---- epilogue: exact recombination of the six digit products
        mbar_wait(&bars[2], ph_acc);
        ph_acc ^= 1;
        if (pend0) { mbar_wait(&bars[0], ph0); ph0 ^= 1; pend0 = false; }
        if (pend1) { mbar_wait(&bars[1], ph1); ph1 ^= 1; pend1 = false; }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const int64_t slot = (int64_t)c * kTcM + tid;
        const double amax = __longlong_as_double((long long)a.amax_bits[b]);
        const double scale = amax * (1.0 / 70368744177664.0) * (1.0 / 32.0);
        const bool live = slot < a.n_dirs;
        const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
        for (int cc = 0; cc < kTcN / 16; ++cc) {
            uint32_t y[kTcSlices][16];
#pragma unroll
            for (int j = 0; j < kTcSlices; ++j) tmem_ld16(trow + (uint32_t)(j * kTcN + cc * 16), y[j]);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (live) {
                const int64_t n0 = t0 + cc * 16;
                double v[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    long long Y = 0;
#pragma unroll
                    for (int j = kTcSlices - 1; j >= 0; --j) Y = Y * 256 + (long long)(int32_t)y[j][i];
                    v[i] = (double)Y * scale;
                }
                if (a.f32) {
                    float* out = reinterpret_cast<float*>(a.beams) + ((size_t)b * a.n_dirs + slot) * a.N + n0;
                    if (n0 + 16 <= a.L) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            *reinterpret_cast<float4*>(out + i) = make_float4((float)v[i], (float)v[i + 1], (float)v[i + 2], (float)v[i + 3]);
                    } else {
                        for (int i = 0; i < 16; ++i) if (n0 + i < a.L) out[i] = (float)v[i];
                    }
                } else {
                    double* out = reinterpret_cast<double*>(a.beams) + ((size_t)b * a.n_dirs + slot) * a.N + n0;
                    if (n0 + 16 <= a.L) {
#pragma unroll
                        for (int i = 0; i < 16; i += 2) *reinterpret_cast<double2*>(out + i) = make_double2(v[i], v[i + 1]);
                    } else {
                        for (int i = 0; i < 16; ++i) if (n0 + i < a.L) out[i] = v[i];
                    }
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads(); // TMEM drained and smem windows free before the next tile
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols) : "memory");
    }
}

size_t beamform_tc_smem_bytes(int pad) {
    const size_t b = (size_t)12 * (kTcN + pad) * 16;
    const size_t need = ((b + 127) & ~size_t(127)) + 2 * kTcRChunk * kABytes + 64 + 1024;
    // >= 115 KB so at most one CTA (and one 512-column TMEM allocation) per SM
    return need > 118 * 1024 ? need : 118 * 1024;
}

void launch_digits(const DigitArgs& a, int batch, cudaStream_t s) {
    const int nblk = (a.rows + 127) / 128;
    k_digits<<<dim3(2 * nblk, a.clusters, batch), 128, 0, s>>>(a);
}

void launch_beamform_tc(const TcArgs& a, const TcSched& sched, int grid, cudaStream_t s) {
    const size_t smem = beamform_tc_smem_bytes(a.pad);
    cudaFuncSetAttribute((const void*)k_beamform_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_beamform_tc<<<grid, kTcThreads, smem, s>>>(a, sched);
}

} // namespace snb
