// Hot-path kernels of the eRTIS image-formation pipeline (sm_100a).
//
// One measurement = 32 channels of packed 1-bit PDM (frame-major); output =
// n_dirs x bins f32 energyscape. Reference: sonarnet::Workspace::process
// (pipeline.cpp:522-574). Stage -> kernel:
//   transpose_bits + demodulate_channel (pipeline.cpp:352-430) -> k_demod
//   strided_filter pre-MF /2         (filters.hpp:14-39)      -> k_premf
//   matched filter via RealFft       (pipeline.cpp:555-562)    -> k_matched_filter
//   run_directions: beamform_into + envelope_direction
//                                    (pipeline.cpp:432-505)    -> k_beamform_tiles + k_envelope
// Device layouts (batch index b outermost):
//   packed  [b][frames*4 bytes]           u8   (as received)
//   demod   [b][32][demod_len]            f64
//   mf      [b][32][mf_len]               f64
//   filt    [b][32][Lp]  zero halo H      f64  (+ f32 copy in F32 mode)
//   beams   [b][n_dirs][N] slot order     f64/f32 (tail [L, N) zero)
//   energy  [b][n_dirs][bins]             f32
#pragma once

#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace snb {

constexpr int kThreads = 256;

struct DemodArgs {
    const uint8_t* packed;    // [B][packed_bytes]
    double* demod;            // [B][32][demod_len]
    const double* lut;        // [8][octets][256]
    int64_t frames, packed_bytes, demod_len, m_lo, m_hi;
    int taps, decim, center, octets, period; // period P = 8/gcd(D,8)
    int jblock;               // outputs (of one class) per work item
    int words;                // row words per channel staged in smem
    int batch;
};

struct PremfArgs {
    const double* demod; // [B][32][demod_len]
    double* mf;          // [B][32][mf_stride], samples [0, mf_len), zero tail
    const double* rev;   // premf reversed taps
    int64_t demod_len, mf_len, mf_stride;
    int taps, decim;
    const double* rev_host; // the same taps on the host (register-window kernel params) or null
};

struct MfArgs {
    const double* mf;       // [B][32][mf_stride] zero-padded rows (mf_stride >= n)
    double* filt;           // [B][32][mf_len]
    float* filt32;          // optional f32 copy (F32 mode) or null
    const double2* ref_spec;// M+1 bins of rfft(reversed chirp, N)
    const double2* tw;      // e^{-2 pi i k/N}, k < N
    int64_t mf_len, Lp, mf_stride;
    int n, ref_len, H;
    unsigned long long* amax_bits; // optional [B] max |filt| (as double bits), zeroed by the caller
};

struct BeamArgs {
    const void* filt;        // [B][32][Lp] f64/f32, sample n at H + n, zero halo
    void* beams;             // [B][n_dirs][N] slot order, tail [L, N) zero
    const int32_t* shifts;   // [n_dirs][32] slot order: delay - advance
    int64_t L, Lp, N, n_dirs;
    int H, T, batch;
};

struct EnvArgs {
    const void* beams;       // [B][n_dirs][N] slot order
    float* energy;           // [B][n_dirs][bins] direction order
    const int32_t* order;    // slot -> direction
    const void* comp;        // composite reversed kernel (f64 or f32)
    const void* tw;          // twiddles for N (double2 or float2)
    const void* tw_small;    // TwShared tables (fft.cuh), used when N == 8192
    int64_t mf_len, bins, n_dirs;
    int n, comp_len, decim, batch;
    int fir_q;               // ceil(comp_len / decim): taps per phase
    int phase_len;           // entries per phase row (>= bins + fir_q + FIR_R)
    int fir_fast;            // decim == kFirD, fir_q == kFirQ, bins <= 128 * kFirR
    int fir_fft;             // FIR by 768-point FFTs (fir_fft768, fft.cuh): N == 8192 and the shapes fit
    const void* ff_u;        // [16][240] spectrum factors U_a in register order (double2 or float2)
    const void* ff_w;        // e^{-2 pi i e / 768}, e < 768
    int pair2048;            // N = 4096 with the fast FIR: k_envelope_pair2048 (two beams per group)
    int split8192;           // N = 16384 with the fast FIR: k_envelope_split8192 (radix-2 + two 4096 halves)
};

// Polyphase smoothing FIR fast path (the reference's default composite
// filter: 447 taps at stride 10 -> 10 phases x 45 taps): every thread owns
// kFirR consecutive outputs over one half of the phases; kFirR = 2 mod 4 so
// that the row window and the taps are read as 16-byte pairs without bank
// conflicts (lane stride kFirR / 2 = odd 16-byte chunks). The phase-major
// taps (kFirQP per phase, zero-padded to even) travel in the kernel
// parameters and are copied to shared memory once per CTA.
constexpr int kFirR = 6;
constexpr int kFirD = 10, kFirQ = 45;              // decimation, taps per phase
constexpr int kFirQP = kFirQ + 1;                  // taps per phase, padded to even
constexpr int kFirTaps = kFirD * kFirQP;           // 460 (zero-padded)
constexpr int kFirScratch = 128 * kFirR;           // half-sum exchange (reals)
static_assert(kFirR % 4 == 2, "paired conflict-free loads");
template <typename R> struct FirTaps { R c[kFirTaps]; }; // c[p * kFirQP + q] = comp[q * kFirD + p]
constexpr int kEnvGroupsF64 = 1;
constexpr int kEnvGroupsF32 = 1;

void launch_demod(const DemodArgs& a, int grid_x, size_t smem, cudaStream_t s);
void launch_premf(const PremfArgs& a, int batch, cudaStream_t s);
void launch_matched_filter(const MfArgs& a, int batch, size_t smem, cudaStream_t s);
void launch_beamform_tiles(const BeamArgs& a, bool f32, cudaStream_t s);
void launch_envelope(const EnvArgs& a, const FirTaps<float>& t32, const FirTaps<double>& t64, bool f32,
                     int grid, cudaStream_t s);
size_t envelope_smem_bytes(int n, int comp_taps_padded, int phase_reals, bool f32, int groups);
constexpr int kFfGroups = 2;        // FFT FIR envelope: groups per CTA (shared factor tables)
#ifndef SNB_FF_G32
#define SNB_FF_G32 3 // FP32 envelope ms by groups per CTA: 2: 2.14, 3: 1.86, 4: 1.89 (64 registers: spills)
#endif
constexpr int kFfGroupsF32 = SNB_FF_G32; // FP32 mode: half the registers per value, more groups fit
template <typename R> constexpr int ff_groups() { return sizeof(R) == 4 ? kFfGroupsF32 : kFfGroups; }
size_t envelope_ff_smem_bytes(bool f32);
int envelope_ff_blocks_per_sm(bool f32); // 0: does not fit
__host__ __device__ int envelope_group_reals(int n, int phase_reals);
int envelope_blocks_per_sm(bool f32, int n_fft, size_t smem);
size_t envelope_pair2048_smem_bytes(bool f32);
int envelope_pair2048_blocks_per_sm(bool f32); // 0: does not fit
size_t envelope_split8192_smem_bytes(bool f32);
int envelope_split8192_blocks_per_sm(bool f32); // 0: does not fit
void launch_rfft_forward(const double* x, double2* X, const double2* tw, int n, size_t smem,
                         cudaStream_t s);

void launch_beamform(const double* filt, double* beams, const int32_t* shifts, int64_t L,
                     int64_t n_dirs, cudaStream_t s);

double measure_fma_peak(int sms, bool f32);

// ---- wire-format frames on the GPU (frames.cu) ------------------------------
constexpr int kCrcShiftMats = 48;   // A_{2^k}, k < 48: messages up to 2^48 bytes
struct CrcTables {
    const uint32_t* slice;          // [4][256] slicing-by-4 tables
    const uint32_t* shift;          // [kCrcShiftMats][32] columns of A_{2^k}
    const uint32_t* lane;           // [32][32] columns of A_{128 (31 - l)} (warp-segment encoder)
    const uint32_t* seg;            // [full segments][32] columns of A_{n - 4096 (s + 1)} for the
                                    // launch's string length n (crc_segment_shifts_host), or null
};
struct FrameIds {                   // per-capture header fields
    uint32_t serial;
    uint64_t ts, seq;
};
struct ImageFrameArgs {
    const float* energies;          // [count][cells] direction order
    const uint8_t* tpl;             // header + direction table template (tpl_len bytes)
    const FrameIds* ids;            // [count]
    uint8_t* frames;                // [count][frame_stride]
    uint32_t* acc;                  // [count] CRC accumulators (zeroed)
    uint64_t cells, tpl_len, frame_len, frame_stride;
};
void launch_crc_partial(const uint8_t* base, uint64_t stride, uint64_t n, uint64_t count, const CrcTables& ct,
                        uint32_t* acc, cudaStream_t s);
void launch_encode_image_frames(const ImageFrameArgs& a, uint64_t count, const CrcTables& ct, cudaStream_t s);
void launch_unpack_frames(const uint8_t* src, uint64_t sstride, uint8_t* dst, uint64_t nbytes, uint64_t count,
                          cudaStream_t s);
void launch_crc_finalize(uint32_t* acc, uint32_t k_n, uint64_t count, uint8_t* out, uint64_t stride, uint64_t n,
                         bool store, int32_t* ok, cudaStream_t s);
uint32_t crc32_host(const uint8_t* p, uint64_t n);
void launch_energyscape_transform(const float* in, float* out, uint64_t count, uint64_t cells, int mode,
                                  float floor_db, cudaStream_t s);

// ---- synthetic captures on the GPU (synth.cu) -------------------------------
constexpr int kSynthMaxReflectors = 8;
struct SynthScene {
    uint64_t seed;
    double noise_rms;
    int n_refl;
    double amp[kSynthMaxReflectors];
    int64_t onset[kSynthMaxReflectors][32];
};
struct SynthArgs {
    const double* pulse;        // PDM-rate pulse (ref_len)
    const SynthScene* scenes;   // [count]
    uint32_t* words;            // [count][32][nwords] scratch
    unsigned long long* states; // [count][32][4] noise-stream state at each channel start (scratch)
    uint8_t* packed;            // [count][packed_bytes]
    int64_t frames, ref_len, nwords, packed_bytes;
    int count;
};
void launch_synth(const SynthArgs& a, cudaStream_t s);
void crc_tables_host(uint32_t* slice, uint32_t* shift);
uint32_t crc_init_term(const uint32_t* shift, uint64_t n);
// A_n(v) on the host (shift: crc_tables_host's A_{2^k} columns)
uint32_t crc_advance_host(const uint32_t* shift, uint32_t v, uint64_t n);
// CrcTables::seg for strings of n bytes: per full 4 KB segment s the map that
// moves its CRC to the string end (one warp-parallel step on the device
// instead of a chain of up to log2(n) matrix products)
std::vector<uint32_t> crc_segment_shifts_host(const uint32_t* shift, uint64_t n);

// ---- tensor-core delay-and-sum (beamform_tc.cu) ---------------------------
constexpr int kTcM = 128;      // directions per cluster (MMA M)
constexpr int kTcN = 64;       // narrow tile (MMA N, TMEM ring of 8 x 64); 128 where shared memory allows
constexpr int kTcSlices = 6;   // balanced base-256 digits of the 46-bit fixed-point samples
constexpr int kTcRMax = 40;    // max shift values per cluster (A resident in smem: 4 KB each)
struct DigitArgs {
    const double* filt;                // [B][32][Lp], sample n at H + n
    const unsigned long long* amax_bits; // [B]
    const int32_t* base;               // [C][32] per-cluster channel base shift
    int8_t* planes;                    // [B][C][6][2][rows][16]
    uint2* words;                      // [B][32][L] the 6 digits of each sample, byte j = digit j
    int64_t L, Lp;
    int H, rows, pad, clusters;
};
struct TcArgs {
    const int8_t* planes;              // as DigitArgs
    const uint8_t* resid;              // [C * 128][32] shift - base (0xFF: unused row)
    const int32_t* R;                  // [C] shift values per cluster (<= kTcRMax)
    const int32_t* cl_start;           // [C] first slot of the cluster
    const int32_t* cl_size;            // [C] slots in the cluster (<= 128)
    const unsigned long long* amax_bits;
    void* beams;                       // [B][n_dirs][N] slot order, f64 or f32
    int64_t L, N, n_dirs;
    int rows, pad, clusters, ntiles, batch, f32, rmax;
    int n;                             // tile width (MMA N): 64 or 128
};
constexpr int kTcMaxGrid = 512;
struct TcSched { int start[kTcMaxGrid + 1]; }; // CTA k processes tiles [start[k], start[k+1])
void launch_digits(const DigitArgs& a, int batch, cudaStream_t s);
cudaError_t launch_beamform_tc(const TcArgs& a, const TcSched& sched, int grid, cudaStream_t s);
size_t beamform_tc_smem_bytes(int rmax, int pad, int tn);

size_t demod_smem_bytes(int octets, int words);
// raise a kernel's dynamic shared-memory limit (cached; throws Error(SN_ERR_CUDA))
void set_smem(const void* fn, size_t smem);
size_t fft_smem_bytes(int n, int real_bytes);

} // namespace snb
