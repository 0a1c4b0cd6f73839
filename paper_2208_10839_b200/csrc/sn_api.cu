// C ABI (include/sonarnet_b200.h) over the device pipeline.
//
// sn_workspace is the B200 counterpart of sonarnet::Workspace::Impl
// (pipeline.cpp:191-319): everything is derived and allocated at creation
// (device tables, per-stage buffers for max_batch measurements, pinned
// staging, one CUDA stream); process calls only enqueue kernels and copies.
#include "fft.cuh"
#include "kernels.cuh"
#include "plan.hpp"
#include "sonarnet_b200.h"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

using namespace snb;

namespace {

thread_local std::string g_last_error;

struct CudaError : Error {
    explicit CudaError(const std::string& w) : Error(SN_ERR_CUDA, w) {}
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

template <typename F>
sn_status guarded(F&& f) {
    try {
        f();
        return SN_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SN_ERR_INTERNAL;
    }
}

// NVTX ranges around the host-side entry points (header-only nvtx3: no
// link dependency; zero cost unless a profiler injects itself)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (dev >= 0) {
            cudaGetDevice(&prev);
            if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
        }
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

template <typename T>
T* dmalloc(size_t n, uint64_t& count) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)), "cudaMalloc");
    ++count;
    return static_cast<T*>(p);
}

template <typename T>
void upload(T* d, const std::vector<T>& h, cudaStream_t s) {
    ck(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s), "upload");
}

std::vector<double2> twiddles(uint64_t n) {
    std::vector<double2> tw(n);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (uint64_t k = 0; k < n; ++k) {
        const long double a = two_pi * (long double)k / (long double)n;
        tw[k] = double2{(double)cosl(a), (double)-sinl(a)};
    }
    return tw;
}

// Compact twiddle set of TwShared (fft.cuh) for M = 4096 (N = 8192): per-pass
// tables e^{-2 pi i step e / M} for the radix-16 passes at ns = 16 and 256
// (e = 1, 2, 4, 8) and the two-level split/merge table A[a] = e^{-2 pi i 64a/N},
// B[b] = e^{-2 pi i b/N}.
std::vector<double2> twiddles_small() {
    const long double two_pi = 6.283185307179586476925286766559005768L;
    auto e = [&](long double num, long double den) {
        const long double a = two_pi * num / den;
        return double2{(double)cosl(a), (double)-sinl(a)};
    };
    std::vector<double2> t;
    const int M = kTwSharedM, N = 2 * kTwSharedM;
    for (int ns : {16, 256}) {
        for (int ex : {1, 2, 4, 8}) {
            for (int k = 0; k < ns; ++k) t.push_back(e((long double)(M / (ns * 16)) * k * ex, M));
        }
    }
    for (int a = 0; a <= 64; ++a) t.push_back(e(64.0L * a, N));
    for (int b = 0; b < 64; ++b) t.push_back(e(b, N));
    return t;
}

} // namespace

void snb::set_last_error(const std::string& m) { g_last_error = m; }

struct sn_workspace {
    Plan plan;
    int device = -1;
    uint64_t max_batch = 1;
    cudaStream_t stream = nullptr;
    // host path: copies run on their own streams so that chunk j+1's H2D and
    // chunk j-1's D2H overlap chunk j's kernels
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    // second compute stream: envelope chunks alternate between `stream` and
    // s_env2 so that a chunk's CTAs fill the SMs its predecessor's tail frees
    cudaStream_t s_env2 = nullptr;
    cudaEvent_t ev_beams = nullptr;
    // completion of the most recent call's device work, whatever stream it
    // ran on: every entry point orders its first device operation after it
    // (a device call on a caller stream followed by a host call, or two
    // device calls on different streams, share the scratch buffers)
    cudaEvent_t ev_last = nullptr;
    // host path, blocks of one call: front end done (d_packed free), the
    // block's downloads done (d_energy free)
    cudaEvent_t ev_front = nullptr, ev_d2h[2] = {};
    float* d_energy_cur = nullptr; // the half the current block's envelope writes
    void after_last(cudaStream_t s) const { ck(cudaStreamWaitEvent(s, ev_last, 0), "wait last"); }
    void mark_last(cudaStream_t s) const { ck(cudaEventRecord(ev_last, s), "record last"); }
    static constexpr int kMaxChunks = 16;
    // envelope chunk sizes of a block of c captures: ~2 per chunk, the last
    // chunk a single capture (its download is the exposed one)
#ifndef SNB_ENV_SUB
#define SNB_ENV_SUB 2 // captures per envelope sub-chunk (the last one: 1)
#endif
#ifndef SNB_ENV_SUB_FRAMES
// the frame path: 3 per chunk (an encoder launch per chunk between the
// envelope chunks; e2e_wire A/B 2 / 3 / 4: 3,502 / 3,557-3,564 / 3,513-3,518 /s)
#define SNB_ENV_SUB_FRAMES 3
#endif
    static std::vector<uint64_t> env_chunks(uint64_t c, uint64_t sub = SNB_ENV_SUB) {
        std::vector<uint64_t> v;
        if (c <= 2) {
            v.assign(c, 1);
            return v;
        }
        uint64_t rest = c - 1;
        const uint64_t n = std::min<uint64_t>((rest + sub - 1) / sub, kMaxChunks - 1);
        for (uint64_t j = 0; j < n; ++j) v.push_back(rest / n + (j < rest % n ? 1 : 0));
        v.push_back(1);
        return v;
    }
    cudaEvent_t ev_in[kMaxChunks] = {}, ev_done[kMaxChunks] = {};
    bool f32 = false;
    // device buffers
    uint8_t* d_packed = nullptr;
    double* d_demod = nullptr;
    double* d_mf = nullptr;
    double* d_filt = nullptr;
    float* d_filt32 = nullptr;
    // beam ring: the per-direction stage (digit planes, delay-and-sum,
    // envelope) runs over chunks of at most `chunk_cap` captures of a batch,
    // so its buffers are bounded by the beam budget instead of growing as
    // max_batch x n_dirs x N (30k directions at 10 m: 3.9 GB per capture)
    void* d_beams = nullptr;
    uint64_t chunk_cap = 1, beam_budget = 0;
    int32_t* d_order = nullptr;
    int32_t* d_shifts_slot = nullptr;

    float* d_energy = nullptr;
    double* d_lut = nullptr;
    double* d_premf = nullptr;
    double* d_comp = nullptr;
    float* d_comp32 = nullptr;
    int32_t* d_shifts = nullptr;
    double2* d_ref_spec = nullptr;
    double2* d_tw_mf = nullptr;
    double2* d_tw_env = nullptr;
    float2* d_tw_env32 = nullptr;
    double2* d_tw_small = nullptr;
    float2* d_tw_small32 = nullptr;
    // FIR by FFT (fir_fft768): spectrum factors and 768-point twiddles
    int fir_fft = 0;
    double2* d_ff_u = nullptr;
    float2* d_ff_u32 = nullptr;
    double2* d_ff_w = nullptr;
    float2* d_ff_w32 = nullptr;
    uint8_t* h_in = nullptr;
    float* h_out = nullptr;
    // launch shapes
    DemodArgs demod{};
    int demod_grid = 0;
    size_t demod_smem = 0, mf_smem = 0, dir_smem = 0;
    int dir_grid = 0, halo = 0, tile = 0, fir_q = 0, phase_len = 0, fir_fast = 0, pair2048 = 0, split8192 = 0;
    // wire-format frames (frames.cu)
    uint32_t* d_crc_slice = nullptr;
    uint32_t* d_crc_shift = nullptr;
    uint32_t* d_crc_lane = nullptr;
    uint32_t* d_crc_seg_in = nullptr;  // CrcTables::seg for the input frames' CRC length
    uint32_t* d_crc_seg_out = nullptr; // ... and the image frames'
    std::vector<uint32_t> h_crc_shift;
    uint8_t* d_img_tpl = nullptr;
    uint64_t img_tpl_len = 0, img_frame_len = 0, img_frame_stride = 0;
    uint64_t in_frame_len = 0, in_frame_stride = 0;
    uint8_t* d_frames_out = nullptr;
    uint8_t* h_frames_out = nullptr;
    uint8_t* d_frames_in = nullptr;
    uint8_t* h_frames_in = nullptr;
    FrameIds* d_ids = nullptr;
    FrameIds* h_ids = nullptr;
    uint32_t* d_crc_acc = nullptr;   // [2][max_batch]: inputs, outputs
    int32_t* d_crc_ok = nullptr;
    int32_t* h_crc_ok = nullptr;
    // tensor-core beamformer (beamform_tc.cu)
    bool tc = false;
    int tc_clusters = 0, tc_pad = 0, tc_rows = 0, tc_ntiles = 0, tc_grid = 0, tc_n = kTcN;
    std::vector<int32_t> tc_R;
    int8_t* d_planes = nullptr;
    uint2* d_dwords = nullptr;
    uint8_t* d_resid = nullptr;
    int32_t* d_tc_R = nullptr;
    int32_t* d_tc_start = nullptr;
    int32_t* d_tc_size = nullptr;
    int tc_rmax = 0;
    int32_t* d_tc_base = nullptr;
    unsigned long long* d_amax = nullptr;
    FirTaps<double> taps64{};
    FirTaps<float> taps32{};
    uint64_t packed_bytes = 0, energy_per = 0, lp = 0;
    // device_allocs: buffers allocated while the workspace is built;
    // alloc_events (Workspace::allocation_events, pipeline.cpp:343-348): every
    // allocation after construction, all of which go through runtime_alloc
    uint64_t alloc_events = 0, device_allocs = 0, last_launches = 0;
    template <typename T>
    T* runtime_alloc(size_t n) {
        ++alloc_events;
        return dmalloc<T>(n, device_allocs);
    }
    // scratch of the beamform() accessor, allocated on its first call
    double* d_bf_in = nullptr;
    double* d_bf_out = nullptr;
    // optional per-stage timing (events on the launching stream)
    bool profiling = false;
    // ev[0..3]: front end boundaries; per beam-ring chunk c: ev_ch[2c]
    // (delay-and-sum done), ev_ch[2c + 1] (envelope done); stage times sum
    // over the chunks of the last call
    cudaEvent_t ev[4] = {};
    std::vector<cudaEvent_t> ev_ch;
    uint64_t prof_chunks = 0;
    // graph cache
    cudaGraphExec_t graph = nullptr;
    const uint8_t* g_in = nullptr;
    float* g_out = nullptr;
    uint64_t g_count = 0;

    ~sn_workspace() {
        if (device < 0) return;
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        if (graph) cudaGraphExecDestroy(graph);
        for (cudaEvent_t e : ev) {
            if (e) cudaEventDestroy(e);
        }
        for (cudaEvent_t e : ev_ch) {
            if (e) cudaEventDestroy(e);
        }
        for (int j = 0; j < kMaxChunks; ++j) {
            if (ev_in[j]) cudaEventDestroy(ev_in[j]);
            if (ev_done[j]) cudaEventDestroy(ev_done[j]);
        }
        if (s_h2d) cudaStreamDestroy(s_h2d);
        if (s_d2h) cudaStreamDestroy(s_d2h);
        if (s_env2) cudaStreamDestroy(s_env2);
        if (ev_beams) cudaEventDestroy(ev_beams);
        if (ev_last) cudaEventDestroy(ev_last);
        if (ev_front) cudaEventDestroy(ev_front);
        for (cudaEvent_t e : ev_d2h)
            if (e) cudaEventDestroy(e);
        for (void* p : {(void*)d_packed, (void*)d_demod, (void*)d_mf, (void*)d_filt,
                        (void*)d_filt32, (void*)d_beams, (void*)d_order, (void*)d_shifts_slot,  (void*)d_energy, (void*)d_lut, (void*)d_premf,
                        (void*)d_comp, (void*)d_comp32, (void*)d_shifts, (void*)d_ref_spec,
                        (void*)d_tw_mf, (void*)d_tw_env, (void*)d_tw_env32, (void*)d_tw_small, (void*)d_tw_small32, (void*)d_ff_u, (void*)d_ff_u32, (void*)d_ff_w, (void*)d_ff_w32, (void*)d_planes, (void*)d_dwords, (void*)d_resid,
                        (void*)d_tc_R, (void*)d_tc_base, (void*)d_amax, (void*)d_tc_start, (void*)d_tc_size,
                        (void*)d_crc_slice, (void*)d_crc_shift, (void*)d_crc_lane, (void*)d_crc_seg_in, (void*)d_crc_seg_out, (void*)d_img_tpl, (void*)d_frames_out,
                        (void*)d_frames_in, (void*)d_ids, (void*)d_crc_acc, (void*)d_crc_ok, (void*)d_bf_in, (void*)d_bf_out}) {
            if (p) cudaFree(p);
        }
        if (h_in) cudaFreeHost(h_in);
        for (void* p : {(void*)h_frames_out, (void*)h_frames_in, (void*)h_ids, (void*)h_crc_ok}) {
            if (p) cudaFreeHost(p);
        }
        if (h_out) cudaFreeHost(h_out);
        if (stream) cudaStreamDestroy(stream);
        if (prev >= 0) cudaSetDevice(prev);
    }

    void require_device() const {
        if (device < 0) throw CudaError("workspace was created without a device (device < 0)");
    }

    void init_device() {
        NvtxRange nv("sn_workspace_create");
        const Sizes& s = plan.sz;
        if (s.mf_fft > 16384 || s.env_fft > 16384) {
            config_error("pipeline: FFT size " + std::to_string(std::max(s.mf_fft, s.env_fft)) +
                         " exceeds the shared-memory FFT limit (16384; max_range <= ~11.7 m at 4.5 MHz)");
        }
        if (s.mf_fft < 32 || s.env_fft < 32) config_error("pipeline: processed window too short for the device FFT");
        DeviceGuard g(device);
        ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&s_h2d, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&s_env2, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaEventCreateWithFlags(&ev_beams, cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&ev_last, cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&ev_front, cudaEventDisableTiming), "cudaEventCreate");
        for (cudaEvent_t& e : ev_d2h) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        for (int j = 0; j < kMaxChunks; ++j) {
            ck(cudaEventCreateWithFlags(&ev_in[j], cudaEventDisableTiming), "cudaEventCreate");
            ck(cudaEventCreateWithFlags(&ev_done[j], cudaEventDisableTiming), "cudaEventCreate");
        }
        packed_bytes = static_cast<uint64_t>(kCh) * s.frames / 8;
        energy_per = s.n_dirs * s.bins;
        const uint64_t B = max_batch;
        uint64_t& n = device_allocs;
        d_packed = dmalloc<uint8_t>(B * packed_bytes, n);
        d_demod = dmalloc<double>(B * kCh * s.demod_len, n);
        d_mf = dmalloc<double>(B * kCh * s.mf_fft, n); // rows zero-padded to the MF FFT size
        ck(cudaMemsetAsync(d_mf, 0, B * kCh * s.mf_fft * sizeof(double), stream), "memset");
        halo = plan.halo;
        lp = s.mf_len + 2 * static_cast<uint64_t>(halo);
        d_filt = dmalloc<double>(B * kCh * lp, n);
        ck(cudaMemsetAsync(d_filt, 0, B * kCh * lp * sizeof(double), stream), "memset");
        if (f32) {
            d_filt32 = dmalloc<float>(B * kCh * lp, n);
            ck(cudaMemsetAsync(d_filt32, 0, B * kCh * lp * sizeof(float), stream), "memset");
        }
        {
            // captures per chunk: as many as the budget holds (beams + digit
            // planes per capture), at least one
            const uint64_t per = s.n_dirs * s.env_fft * (f32 ? sizeof(float) : sizeof(double)) +
                                 (tc ? (uint64_t)tc_clusters * 12 * tc_rows * 16 + (uint64_t)kCh * s.mf_len * 8 : 0);
            chunk_cap = std::max<uint64_t>(1, std::min<uint64_t>(B, beam_budget / per));
        }
        const size_t beam_bytes = chunk_cap * s.n_dirs * s.env_fft * (f32 ? sizeof(float) : sizeof(double));
        d_beams = dmalloc<uint8_t>(beam_bytes, n);
        ck(cudaMemsetAsync(d_beams, 0, beam_bytes, stream), "memset");
        d_order = dmalloc<int32_t>(s.n_dirs, n);
        d_shifts_slot = dmalloc<int32_t>(s.n_dirs * kCh, n);
        upload(d_order, plan.order, stream);
        upload(d_shifts_slot, plan.shifts, stream);

        // two halves: consecutive blocks of one host-path call alternate, so
        // block j's downloads overlap block j + 1's kernels
        d_energy = dmalloc<float>(2 * B * energy_per, n);
        d_lut = dmalloc<double>(plan.demod_lut.size(), n);
        d_premf = dmalloc<double>(plan.premf_rev.size(), n);
        d_comp = dmalloc<double>(plan.comp_rev.size(), n);
        d_comp32 = dmalloc<float>(plan.comp_rev.size(), n);
        d_shifts = dmalloc<int32_t>(s.n_dirs * kCh, n);
        d_ref_spec = dmalloc<double2>(s.mf_fft / 2 + 1, n);
        d_tw_mf = dmalloc<double2>(s.mf_fft, n);
        d_tw_env = dmalloc<double2>(s.env_fft, n);
        d_tw_env32 = dmalloc<float2>(s.env_fft, n);
        ck(cudaMallocHost(&h_in, B * packed_bytes), "cudaMallocHost");
        for (cudaEvent_t& e : ev) ck(cudaEventCreate(&e), "cudaEventCreate");
        ev_ch.assign(2 * ((B + chunk_cap - 1) / chunk_cap), nullptr);
        for (cudaEvent_t& e : ev_ch) ck(cudaEventCreate(&e), "cudaEventCreate");
        ck(cudaMallocHost(&h_out, B * energy_per * sizeof(float)), "cudaMallocHost");

        upload(d_lut, plan.demod_lut, stream);
        upload(d_premf, plan.premf_rev, stream);
        upload(d_comp, plan.comp_rev, stream);
        std::vector<float> comp32(plan.comp_rev.begin(), plan.comp_rev.end());
        upload(d_comp32, comp32, stream);
        std::vector<int32_t> shifts(s.n_dirs * kCh);
        for (uint64_t d = 0; d < s.n_dirs; ++d) {
            for (int i = 0; i < kCh; ++i) shifts[d * kCh + i] = plan.delays[d * kCh + i] - plan.advances[d];
        }
        upload(d_shifts, shifts, stream);
        const auto tw_mf = twiddles(s.mf_fft), tw_env = twiddles(s.env_fft);
        upload(d_tw_mf, tw_mf, stream);
        upload(d_tw_env, tw_env, stream);
        std::vector<float2> tw32(s.env_fft);
        for (uint64_t k = 0; k < s.env_fft; ++k) tw32[k] = float2{(float)tw_env[k].x, (float)tw_env[k].y};
        upload(d_tw_env32, tw32, stream);
        {
            const auto ts = twiddles_small();
            d_tw_small = dmalloc<double2>(ts.size(), n);
            d_tw_small32 = dmalloc<float2>(ts.size(), n);
            upload(d_tw_small, ts, stream);
            std::vector<float2> ts32(ts.size());
            for (size_t k = 0; k < ts.size(); ++k) ts32[k] = float2{(float)ts[k].x, (float)ts[k].y};
            upload(d_tw_small32, ts32, stream);
        }
        // reference spectrum: rfft of the reversed chirp zero-padded to mf_fft
        // (pipeline.cpp:274-278)
        {
            std::vector<double> padded(s.mf_fft, 0.0);
            std::reverse_copy(plan.chirp_ref.begin(), plan.chirp_ref.end(), padded.begin());
            double* d_tmp = nullptr;
            ck(cudaMalloc(&d_tmp, padded.size() * sizeof(double)), "cudaMalloc");
            upload(d_tmp, padded, stream);
            mf_smem = fft_smem_bytes((int)s.mf_fft, sizeof(double));
            launch_rfft_forward(d_tmp, d_ref_spec, d_tw_mf, (int)s.mf_fft, mf_smem, stream);
            ck(cudaGetLastError(), "rfft launch");
            ck(cudaStreamSynchronize(stream), "setup sync");
            cudaFree(d_tmp);
        }
        // demod launch shape
        const int D = plan.cfg.demod_decimation;
        const int P = 8 / std::gcd(D, 8);
        demod = DemodArgs{};
        demod.lut = d_lut;
        demod.frames = (int64_t)s.frames;
        demod.packed_bytes = (int64_t)packed_bytes;
        demod.demod_len = (int64_t)s.demod_len;
        demod.m_lo = s.m_lo;
        demod.m_hi = s.m_hi;
        demod.taps = plan.cfg.demod_taps;
        demod.decim = D;
        demod.center = (plan.cfg.demod_taps - 1) / 2;
        demod.octets = (int)s.lut_octets;
        demod.period = P;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        // outputs of one residue class per work item: among the candidates
        // that keep the most CTAs per SM (LUT + staged rows in shared
        // memory), the one with the fewest estimated item-waves x (block +
        // staging margin) for a full batch (hemisphere3000: 48 -> 0.160 ms;
        // 64 -> 0.221 ms at 2 CTAs/SM; 32 -> 0.170 ms)
        auto words_for = [&](int jb) {
            int w = (int)((int64_t)D * P * (jb - 1) + demod.taps + 62) / 32 + 3;
            return w % 2 == 0 ? w + 1 : w;
        };
        auto per_sm_for = [&](int jb) {
            return std::max(1, (int)((228 * 1024) / (demod_smem_bytes(demod.octets, words_for(jb)) + 1024)));
        };
        const int64_t Jr = ((int64_t)s.demod_len + P - 1) / P;
        const int cands[] = {64, 56, 48, 40, 32, 24};
        int max_per = 1;
        for (int jb : cands) max_per = std::max(max_per, per_sm_for(jb));
        double best = 1e300;
        demod.jblock = 32;
        for (int jb : cands) {
            if (per_sm_for(jb) != max_per) continue;
            const int64_t grid = std::max(1, sms * max_per / P);
            const int64_t items = (Jr + jb - 1) / jb * (int64_t)max_batch;
            const double cost = (double)((items + grid - 1) / grid) * (jb + (double)demod.taps / (D * P));
            if (cost < best - 1e-9) {
                best = cost;
                demod.jblock = jb;
            }
        }
        const int words = words_for(demod.jblock);
        demod.words = words;
        demod_smem = demod_smem_bytes(demod.octets, words);
        if (demod_smem > 227 * 1024) {
            config_error("pipeline: demod taps " + std::to_string(demod.taps) + " exceed the shared-memory LUT limit");
        }
        const int per_sm = std::max(1, (int)((228 * 1024) / (demod_smem + 1024)));
        demod_grid = std::max(1, sms * per_sm / P);
        // beamformer time tile: 32 x (T + 2H) samples staged per CTA
        tile = 128;
        init_tensor_core_beamformer(sms);
        {
            // polyphase FIR rows (fir_polyphase in kernels.cu): every envelope
            // sample needs a slot and every FIR read stays inside its row
            const int D = plan.cfg.post_envelope_decimation;
            const int c0 = (int)(plan.comp_rev.size() - 1) / 2;
            fir_q = (int)((plan.comp_rev.size() + D - 1) / D);
            const int groups = (int)((s.bins + kFirR - 1) / kFirR);
            phase_len = std::max(groups * kFirR + fir_q + 1, (int)((s.mf_len + c0) / D) + 1);
            phase_len = std::max(phase_len, (int)s.bins + fir_q + 1);
            phase_len = (phase_len + 1) & ~1; // even: rows stay 16-byte aligned (paired loads)
            fir_fast = D == kFirD && fir_q == kFirQ && groups <= 4 * 128;
            init_fir_fft(D, c0);
            if (fir_fast) {
                for (int p = 0; p < kFirD; ++p) {
                    for (int q = 0; q < kFirQ; ++q) {
                        const size_t j = (size_t)q * kFirD + p;
                        const double v = j < plan.comp_rev.size() ? plan.comp_rev[j] : 0.0;
                        taps64.c[p * kFirQP + q] = v;
                        taps32.c[p * kFirQP + q] = (float)v;
                    }
                }
            }
        }
        dir_smem = envelope_smem_bytes((int)s.env_fft,
                                       fir_fast ? kFirTaps : fir_q * plan.cfg.post_envelope_decimation,
                                       plan.cfg.post_envelope_decimation * phase_len, f32,
                                       f32 ? kEnvGroupsF32 : kEnvGroupsF64);
        {
            dir_grid = sms * envelope_blocks_per_sm(f32, (int)s.env_fft, dir_smem);
            // N = 4096 (the 1.5 m window): two beams per group, when the phase
            // rows + FIR scratch of a beam fit its FFT buffer
            pair2048 = s.env_fft == 4096 && fir_fast &&
                       plan.cfg.post_envelope_decimation * phase_len + 64 * kFirR <= 2 * (2048 + 256);
            if (pair2048) {
                const int per = envelope_pair2048_blocks_per_sm(f32);
                if (per > 0) dir_grid = sms * per;
                else pair2048 = 0;
            }
            // N = 16384 (8-11.7 m): radix-2 split into two M = 4096 halves
            split8192 = s.env_fft == 16384 && fir_fast &&
                        plan.cfg.post_envelope_decimation * phase_len + 3 * 128 * kFirR <= 2 * 2 * (4096 + 256);
            if (split8192) {
                const int per = envelope_split8192_blocks_per_sm(f32);
                if (per > 0) dir_grid = sms * per;
                else split8192 = 0;
            }
            if (fir_fft) {
                const int per = envelope_ff_blocks_per_sm(f32);
                if (per > 0) dir_grid = sms * per;
                else fir_fft = 0; // does not fit: direct polyphase FIR
            }
        }
        mf_smem = fft_smem_bytes((int)s.mf_fft, sizeof(double));
        init_frames();
        ck(cudaStreamSynchronize(stream), "setup sync");
    }

    // ---- wire-format frames (protocol.md): CRC tables, the processed-image
    // frame template (packet header + AIMG header + direction table,
    // pipeline.cpp:109-125, wire.cpp:66-81,268-276) and frame buffers
    static void put(std::vector<uint8_t>& v, const void* p, size_t n) {
        const uint8_t* b = static_cast<const uint8_t*>(p);
        v.insert(v.end(), b, b + n);
    }
    std::vector<uint8_t> image_template() const {
        const Sizes& z = plan.sz;
        std::vector<uint8_t> t;
        const uint32_t magic = 0x45525449u, aimg = 0x41494D47u, zero32 = 0;
        const uint16_t version = 1, msg = 2;
        const uint64_t zero64 = 0;
        const uint64_t payload = 34 + 8 * z.n_dirs + 4 * z.n_dirs * z.bins;
        put(t, &magic, 4); put(t, &version, 2); put(t, &msg, 2); put(t, &zero32, 4);
        put(t, &zero64, 8); put(t, &zero64, 8); put(t, &payload, 8);
        const uint32_t nd = (uint32_t)z.n_dirs, nb = (uint32_t)z.bins;
        const uint16_t iv = 1;
        put(t, &aimg, 4); put(t, &iv, 2); put(t, &zero32, 4); put(t, &zero64, 8);
        put(t, &nd, 4); put(t, &nb, 4); put(t, &z.range_bin_size, 8);
        for (uint64_t d = 0; d < z.n_dirs; ++d) {
            const float az = (float)plan.directions[2 * d], el = (float)plan.directions[2 * d + 1];
            put(t, &az, 4); put(t, &el, 4);
        }
        return t;
    }
    void init_frames() {
        const Sizes& z = plan.sz;
        uint64_t& n = device_allocs;
        std::vector<uint32_t> slice(1024);
        h_crc_shift.assign((size_t)kCrcShiftMats * 32, 0);
        crc_tables_host(slice.data(), h_crc_shift.data());
        d_crc_slice = dmalloc<uint32_t>(slice.size(), n);
        d_crc_shift = dmalloc<uint32_t>(h_crc_shift.size(), n);
        upload(d_crc_slice, slice, stream);
        upload(d_crc_shift, h_crc_shift, stream);
        std::vector<uint32_t> lane(1024);
        for (int l = 0; l < 32; ++l)
            for (int b = 0; b < 32; ++b) lane[32 * l + b] = crc_advance_host(h_crc_shift.data(), 1u << b, 128u * (31 - l));
        d_crc_lane = dmalloc<uint32_t>(lane.size(), n);
        upload(d_crc_lane, lane, stream);
        const auto tpl = image_template();
        img_tpl_len = tpl.size();
        img_frame_len = img_tpl_len + 4 * z.n_dirs * z.bins + 4;
        img_frame_stride = (img_frame_len + 15) & ~uint64_t(15);
        d_img_tpl = dmalloc<uint8_t>(tpl.size(), n);
        upload(d_img_tpl, tpl, stream);
        in_frame_len = 36 + 38 + packed_bytes + 4;
        in_frame_stride = (in_frame_len + 15) & ~uint64_t(15);
        {
            const auto si = crc_segment_shifts_host(h_crc_shift.data(), in_frame_len - 4);
            const auto so = crc_segment_shifts_host(h_crc_shift.data(), img_frame_len - 4);
            d_crc_seg_in = dmalloc<uint32_t>(std::max<size_t>(si.size(), 1), n);
            d_crc_seg_out = dmalloc<uint32_t>(std::max<size_t>(so.size(), 1), n);
            if (!si.empty()) upload(d_crc_seg_in, si, stream);
            if (!so.empty()) upload(d_crc_seg_out, so, stream);
        }
        const uint64_t B = max_batch;
        // output frames, host-side ids and CRC verdicts in two halves: the
        // blocks of one process_frames call alternate (block j + 1 is
        // enqueued while block j's frames download)
        d_frames_out = dmalloc<uint8_t>(2 * B * img_frame_stride, n);
        d_frames_in = dmalloc<uint8_t>(B * in_frame_stride, n);
        d_ids = dmalloc<FrameIds>(2 * B, n);
        d_crc_acc = dmalloc<uint32_t>(2 * B, n);
        d_crc_ok = dmalloc<int32_t>(2 * B, n);
        ck(cudaMallocHost(&h_frames_out, B * img_frame_len), "cudaMallocHost");
        ck(cudaMallocHost(&h_frames_in, B * in_frame_len), "cudaMallocHost");
        ck(cudaMallocHost(&h_ids, 2 * B * sizeof(FrameIds)), "cudaMallocHost");
        ck(cudaMallocHost(&h_crc_ok, 2 * B * sizeof(int32_t)), "cudaMallocHost");
    }
    // seg: the per-length segment maps of the input (false) or image (true) frames
    CrcTables crc_tables(bool image) const {
        return CrcTables{d_crc_slice, d_crc_shift, d_crc_lane, image ? d_crc_seg_out : d_crc_seg_in};
    }

    // Tensor-core delay-and-sum setup (beamform_tc.cu): clusters of <= kTcM
    // consecutive slots cut greedily so that R_c (the largest per-channel
    // shift span) stays <= kTcRMax; per cluster the channel base shifts b_i
    // (min over the cluster) and per slot the residual bytes s - b_i.
    // SNB_BEAMFORMER=tiles selects the CUDA-core tiled kernel instead.
    std::vector<int32_t> tc_base, tc_start, tc_size;
    std::vector<uint8_t> tc_resid;
    void plan_tensor_core_beamformer(const sn_workspace_options& opt) {
        tc = opt.beamformer != SN_BEAMFORMER_CUDA_CORE;
        if (!tc) return;
        const Sizes& s = plan.sz;
        tc_R.clear();
        tc_base.clear();
        tc_start.clear();
        tc_size.clear();
        tc_resid.clear();
        // clusters: the planner's <= 128-direction k-d subtrees, each cut
        // greedily further only if its shift span exceeds kTcRMax
        for (size_t leaf = 0; leaf + 1 < plan.tc_leaves.size(); ++leaf) {
            uint64_t s0 = (uint64_t)plan.tc_leaves[leaf];
            const uint64_t s_end = (uint64_t)plan.tc_leaves[leaf + 1];
            while (s0 < s_end) {
                int lo[kCh], hi[kCh];
                for (int i = 0; i < kCh; ++i) { lo[i] = 1 << 30; hi[i] = -(1 << 30); }
                uint64_t s1 = s0;
                int R = 1;
                while (s1 < s_end && s1 - s0 < (uint64_t)kTcM) {
                    int Rn = 1;
                    for (int i = 0; i < kCh; ++i) {
                        const int v = plan.shifts[s1 * kCh + i];
                        Rn = std::max(Rn, std::max(hi[i], v) - std::min(lo[i], v) + 1);
                    }
                    if (Rn > kTcRMax) break;
                    for (int i = 0; i < kCh; ++i) {
                        const int v = plan.shifts[s1 * kCh + i];
                        lo[i] = std::min(lo[i], v);
                        hi[i] = std::max(hi[i], v);
                    }
                    R = Rn;
                    ++s1;
                }
                const size_t c = tc_R.size();
                tc_R.push_back(R);
                tc_start.push_back((int32_t)s0);
                tc_size.push_back((int32_t)(s1 - s0));
                tc_base.resize((c + 1) * kCh);
                tc_resid.resize((c + 1) * kTcM * kCh, 0xFF);
                for (int i = 0; i < kCh; ++i) tc_base[c * kCh + i] = lo[i];
                for (uint64_t sl = s0; sl < s1; ++sl) {
                    for (int i = 0; i < kCh; ++i)
                        tc_resid[(c * kTcM + (sl - s0)) * kCh + i] = (uint8_t)(plan.shifts[sl * kCh + i] - lo[i]);
                }
                s0 = s1;
            }
        }
        tc_clusters = (int)tc_R.size();
        tc_rmax = *std::max_element(tc_R.begin(), tc_R.end());
        tc_pad = (tc_rmax + 6) & ~7; // >= rmax - 1, multiple of 8
        // wide tiles (N = 128: 3 TMEM slots, ~1.4x the int8 MMA rate per
        // instruction) when the resident A_r and three B windows fit in
        // shared memory; SNB_TC_N=64 forces the narrow tiles
        const int want = opt.tc_tile_n ? opt.tc_tile_n : 96;
        tc_n = kTcN;
        for (int n : {128, 96})
            if (want >= n && tc_n == kTcN && beamform_tc_smem_bytes(tc_rmax, tc_pad, n) <= 220 * 1024) tc_n = n;
        tc_ntiles = (int)((s.mf_len + tc_n - 1) / tc_n);
        tc_rows = tc_pad + tc_ntiles * tc_n;
    }

    void init_tensor_core_beamformer(int sms) {
        if (!tc) return;
        uint64_t& n = device_allocs;
        d_planes = dmalloc<int8_t>(chunk_cap * (uint64_t)tc_clusters * 12 * tc_rows * 16, n);
        d_dwords = dmalloc<uint2>(chunk_cap * (uint64_t)kCh * plan.sz.mf_len, n);
        d_resid = dmalloc<uint8_t>(tc_resid.size(), n);
        d_tc_R = dmalloc<int32_t>(tc_R.size(), n);
        d_tc_base = dmalloc<int32_t>(tc_base.size(), n);
        d_tc_start = dmalloc<int32_t>(tc_start.size(), n);
        d_tc_size = dmalloc<int32_t>(tc_size.size(), n);
        d_amax = dmalloc<unsigned long long>(max_batch, n);
        upload(d_resid, tc_resid, stream);
        upload(d_tc_R, tc_R, stream);
        upload(d_tc_base, tc_base, stream);
        upload(d_tc_start, tc_start, stream);
        upload(d_tc_size, tc_size, stream);
        tc_grid = std::min(sms, kTcMaxGrid);
    }

    // contiguous per-CTA tile ranges of equal estimated work. A tile costs
    // the larger of its MMA time (R_c units of six MMAs) and an epilogue
    // floor (SNB_TC_EPI_UNITS), plus a fixed part. Per-CTA busy times
    // (scripts/tc_times.py, globaltimer per CTA) showed the fixed part
    // dominating: ~3.8 us + 0.06 us x R_c per tile, i.e. R_c + ~60 units, and
    // the round-1 model max(R_c, 20) + 2 leaving a max/mean CTA time of 1.08.
    // A/B (beamform stage vs max(R, 20) + 2, sweep grids, min of 2 runs):
    // R + 20: hemi3000 0.97, box1850 0.93, fib10k 0.98-1.00, fib30k 1.04;
    // R + 30: 0.96-0.98, 0.95-0.96, 0.95-0.98, 1.02-1.03;
    // R + 40: 0.96, 0.97-0.99, 0.93-0.97, 1.015 (1- and 2-cluster grids
    // within run-to-run noise)
#ifndef SNB_TC_EPI_UNITS
#define SNB_TC_EPI_UNITS 0
#endif
#ifndef SNB_TC_FIXED_UNITS
#define SNB_TC_FIXED_UNITS 30
#endif
    static double tc_tile_cost(int R) {
        return std::max<double>(R, SNB_TC_EPI_UNITS) + SNB_TC_FIXED_UNITS;
    }
    TcSched tc_schedule(int count) const {
        TcSched sc{};
        const int per_c = count * tc_ntiles;
        double total = 0;
        for (int c = 0; c < tc_clusters; ++c) total += tc_tile_cost(tc_R[c]) * per_c;
        int k = 1;
        double acc = 0;
        sc.start[0] = 0;
        for (int c = 0; c < tc_clusters && k < tc_grid; ++c) {
            const double w = tc_tile_cost(tc_R[c]);
            while (k < tc_grid && acc + w * per_c >= total * k / tc_grid) {
                const double need = total * k / tc_grid - acc;
                int m = (int)std::ceil(need / w);
                m = std::max(0, std::min(per_c, m));
                sc.start[k++] = c * per_c + m;
            }
            acc += w * per_c;
        }
        for (; k <= tc_grid; ++k) sc.start[k] = tc_clusters * per_c;
        return sc;
    }

    // Enqueue the whole pipeline for `count` measurements (count <= max_batch).
    // Front end (demod, pre-MF FIR, matched filter) of captures
    // [off, off + count), whose packed bits are at d_in.
    void enqueue_front(const uint8_t* d_in, uint64_t off, uint64_t count, cudaStream_t s) {
        const Sizes& z = plan.sz;
        double* dm = d_demod + off * kCh * z.demod_len;
        double* mf = d_mf + off * kCh * z.mf_fft;
        DemodArgs da = demod;
        da.packed = d_in;
        da.demod = dm;
        da.batch = (int)count;
        if (profiling) cudaEventRecord(ev[0], s);
        launch_demod(da, demod_grid, demod_smem, s);
        if (profiling) cudaEventRecord(ev[1], s);
        PremfArgs pa{dm, mf, d_premf, (int64_t)z.demod_len, (int64_t)z.mf_len, (int64_t)z.mf_fft,
                     (int)plan.premf_rev.size(), plan.cfg.pre_mf_decimation, plan.premf_rev.data()};
        launch_premf(pa, (int)count, s);
        if (profiling) cudaEventRecord(ev[2], s);
        MfArgs ma{mf, d_filt + off * kCh * lp, f32 && !tc ? d_filt32 + off * kCh * lp : nullptr, d_ref_spec, d_tw_mf,
                  (int64_t)z.mf_len, (int64_t)lp, (int64_t)z.mf_fft, (int)z.mf_fft, (int)z.ref_len, halo,
                  tc ? d_amax + off : nullptr};
        if (tc) ck(cudaMemsetAsync(d_amax + off, 0, count * sizeof(unsigned long long), s), "memset");
        launch_matched_filter(ma, (int)count, mf_smem, s);
        if (profiling) cudaEventRecord(ev[3], s);
    }

    // Delay-and-sum of captures [off, off + count) of the batch (count <=
    // chunk_cap) into the beam ring (ring position 0 = capture off).
    void enqueue_beams(uint64_t off, uint64_t count, cudaStream_t s) {
        const Sizes& z = plan.sz;
        if (tc) {
            DigitArgs dg{d_filt + off * kCh * lp, d_amax + off, d_tc_base, d_planes, d_dwords, (int64_t)z.mf_len,
                         (int64_t)lp, halo, tc_rows, tc_pad, tc_clusters};
            launch_digits(dg, (int)count, s);
            TcArgs ta{};
            ta.planes = d_planes;
            ta.resid = d_resid;
            ta.R = d_tc_R;
            ta.cl_start = d_tc_start;
            ta.cl_size = d_tc_size;
            ta.rmax = tc_rmax;
            ta.amax_bits = d_amax + off;
            ta.beams = d_beams;
            ta.L = (int64_t)z.mf_len;
            ta.N = (int64_t)z.env_fft;
            ta.n_dirs = (int64_t)z.n_dirs;
            ta.rows = tc_rows;
            ta.pad = tc_pad;
            ta.clusters = tc_clusters;
            ta.ntiles = tc_ntiles;
            ta.batch = (int)count;
            ta.f32 = f32 ? 1 : 0;
            ta.n = tc_n;
            ck(launch_beamform_tc(ta, tc_schedule((int)count), tc_grid, s), "tensor-core beamformer");
        } else {
            BeamArgs ba{};
            ba.filt = f32 ? (const void*)(d_filt32 + off * kCh * lp) : (const void*)(d_filt + off * kCh * lp);
            ba.beams = d_beams;
            ba.shifts = d_shifts_slot;
            ba.L = (int64_t)z.mf_len;
            ba.Lp = (int64_t)lp;
            ba.N = (int64_t)z.env_fft;
            ba.n_dirs = (int64_t)z.n_dirs;
            ba.H = halo;
            ba.T = tile;
            ba.batch = (int)count;
            launch_beamform_tiles(ba, f32, s);
        }
    }
    uint64_t beam_launches() const { return tc ? 3 : 1; } // k_digit_words + k_digits + k_beamform_tc

    // The device pipeline for `count` captures (<= max_batch): front end for
    // the batch, then per chunk of the beam ring delay-and-sum + envelope.
    void enqueue(const uint8_t* d_in, uint64_t count, float* d_out, cudaStream_t s) {
        enqueue_front(d_in, 0, count, s);
        uint64_t launches = 3, c = 0;
        for (uint64_t off = 0; off < count; off += chunk_cap, ++c) {
            const uint64_t k = std::min(chunk_cap, count - off);
            enqueue_beams(off, k, s);
            if (profiling) cudaEventRecord(ev_ch[2 * c], s);
            enqueue_envelope(0, k, d_out + off * energy_per, s);
            if (profiling) cudaEventRecord(ev_ch[2 * c + 1], s);
            launches += beam_launches() + 1;
        }
        prof_chunks = c;
        ck(cudaGetLastError(), "kernel launch");
        last_launches = launches;
    }

    // Envelope stage for ring positions [b0, b0 + count) of the beam ring;
    // energies to d_out (ring position b0 first).
    void enqueue_envelope(uint64_t b0, uint64_t count, float* d_out, cudaStream_t s) {
        const Sizes& z = plan.sz;
        const size_t rb = f32 ? sizeof(float) : sizeof(double);
        EnvArgs ea{};
        ea.beams = static_cast<const uint8_t*>(d_beams) + b0 * z.n_dirs * z.env_fft * rb;
        ea.energy = d_out;
        ea.order = d_order;
        ea.comp = f32 ? (const void*)d_comp32 : (const void*)d_comp;
        ea.tw = f32 ? (const void*)d_tw_env32 : (const void*)d_tw_env;
        ea.tw_small = f32 ? (const void*)d_tw_small32 : (const void*)d_tw_small;
        ea.mf_len = (int64_t)z.mf_len;
        ea.bins = (int64_t)z.bins;
        ea.n_dirs = (int64_t)z.n_dirs;
        ea.n = (int)z.env_fft;
        ea.comp_len = (int)plan.comp_rev.size();
        ea.decim = plan.cfg.post_envelope_decimation;
        ea.batch = (int)count;
        ea.fir_q = fir_q;
        ea.phase_len = phase_len;
        ea.fir_fast = fir_fast;
        ea.fir_fft = fir_fft;
        ea.pair2048 = pair2048;
        ea.split8192 = split8192;
        ea.ff_u = f32 ? (const void*)d_ff_u32 : (const void*)d_ff_u;
        ea.ff_w = f32 ? (const void*)d_ff_w32 : (const void*)d_ff_w;
        launch_envelope(ea, taps32, taps64, f32, dir_grid, s);
    }

    // FIR by 768-point FFTs (fir_fft768 in fft.cuh) for the default shapes:
    // N = 8192, decimation 10, 45 taps per phase, bins + 44 <= 768 and at most
    // 32 zero slots per phase on either side of the envelope. Host tables: the
    // spectrum factors U_a[k] = (conj Ghat_re[k] - i conj Ghat_im[k]) / 768 (re/im
    // phases of sequence a as laid out by the sink, fft.cuh),
    // Ghat_p = DFT768 of the phase taps G_p[q] = rev[10 q + p] (long double),
    // stored in the register order of the third forward pass, and the
    // twiddles w768^j (j < 256) and w256^{n3 k2} (16 x 16). SNB_FIR_DIRECT (build macro, A/B) keeps
    // the direct polyphase FIR.
    void init_fir_fft(int D, int c0) {
        const Sizes& s = plan.sz;
        fir_fft = 0;
#ifndef SNB_FIR_DIRECT
        if (s.env_fft != 8192 || D != kFirD || fir_q != kFirQ || c0 % 2 != 1 || s.bins + kFirQ - 1 > (uint64_t)kFfL)
            return;
        for (int sa = 0; sa < kFfSeq; ++sa) {
            // slot (sa, u) holds samples 10 u + 2 sa + 1 - c0 and the next one
            const int64_t e = c0 - 1 - 2 * sa;
            const int64_t lo = e > 0 ? (e + D - 1) / D : 0;
            const int64_t hi = ((int64_t)s.mf_len + e + D - 1) / D;
            // hi < 768: the last slot of sequence 4 (E_0 advanced by one, read
            // cyclically at index -1) must be a zero
            if (lo > 32 || hi >= kFfL || kFfL - hi > 32) return;
        }
        const long double pi2 = 6.283185307179586476925286766559L;
        std::vector<long double> gr(D * kFfL), gi(D * kFfL); // conj Ghat_p[k]
        for (int p = 0; p < D; ++p) {
            for (int k = 0; k < kFfL; ++k) {
                long double re = 0, im = 0;
                for (int q = 0; q < kFirQ; ++q) {
                    const size_t j = (size_t)q * D + p;
                    if (j >= plan.comp_rev.size()) continue;
                    const long double g = plan.comp_rev[j];
                    const long double ang = pi2 * (long double)((k * q) % kFfL) / kFfL;
                    re += g * cosl(ang);
                    im += g * sinl(ang); // conj: e^{+2 pi i k q / 768}
                }
                gr[p * kFfL + k] = re;
                gi[p * kFfL + k] = im;
            }
        }
        // sequence a: real part phase 2a + 1, imaginary part phase 2a + 2
        // (a < 4) or phase 0 advanced by one sample (a = 4: conj Ghat_0 times
        // e^{-2 pi i k / 768}, its taps delayed by one cyclically)
        std::vector<double2> u(kFfU);
        for (int t = 0; t < kFfThreads; ++t) {
            const int a = t / 48, k1 = (t % 48) / 16, k2 = t % 16;
            for (int r = 0; r < 16; ++r) {
                const int k3 = (r >> 2) + 4 * (r & 3); // out_slot<16>(r)
                const int k = k1 + 3 * k2 + 48 * k3;
                const size_t pr = (size_t)(2 * a + 1) * kFfL + k, pi = (size_t)((2 * a + 2) % D) * kFfL + k;
                long double ir = gr[pi], ii = gi[pi];
                if (a == kFfSeq - 1) {
                    const long double ang = pi2 * k / kFfL, c = cosl(ang), sn = -sinl(ang);
                    const long double xr = ir * c - ii * sn, xi = ir * sn + ii * c;
                    ir = xr;
                    ii = xi;
                }
                // (conj Ghat_re - i conj Ghat_im) / 768
                u[(size_t)r * kFfThreads + t] = double2{(double)((gr[pr] + ii) / kFfL), (double)((gi[pr] - ir) / kFfL)};
            }
        }
        std::vector<double2> w(kFfW); // w768^j (j < 256); w256^{n3 k2} at 256 + 16 k2 + n3
        for (int e = 0; e < 256; ++e) {
            const long double a1 = pi2 * e / kFfL, a2 = pi2 * ((e >> 4) * (e & 15)) / 256;
            w[e] = double2{(double)cosl(a1), (double)-sinl(a1)};
            w[256 + e] = double2{(double)cosl(a2), (double)-sinl(a2)};
        }
        uint64_t& n = device_allocs;
        d_ff_u = dmalloc<double2>(u.size(), n);
        d_ff_w = dmalloc<double2>(w.size(), n);
        d_ff_u32 = dmalloc<float2>(u.size(), n);
        d_ff_w32 = dmalloc<float2>(w.size(), n);
        upload(d_ff_u, u, stream);
        upload(d_ff_w, w, stream);
        std::vector<float2> u32(u.size()), w32(w.size());
        for (size_t i = 0; i < u.size(); ++i) u32[i] = float2{(float)u[i].x, (float)u[i].y};
        for (size_t i = 0; i < w.size(); ++i) w32[i] = float2{(float)w[i].x, (float)w[i].y};
        upload(d_ff_u32, u32, stream);
        upload(d_ff_w32, w32, stream);
        fir_fft = 1;
#else
        (void)s;
        (void)D;
        (void)c0;
#endif
    }

    void validate(const sn_raw_measurement& m) const { // pipeline.cpp:524-540
        const Sizes& z = plan.sz;
        if (m.channels != kCh) {
            decode_error("process: measurement has " + std::to_string(m.channels) +
                         " channels, expected " + std::to_string(kCh));
        }
        if (m.frames != z.frames) {
            decode_error("process: measurement has " + std::to_string(m.frames) +
                         " frames, config expects " + std::to_string(z.frames));
        }
        if (std::abs(m.pdm_rate - plan.cfg.pdm_rate) > 1e-6 * plan.cfg.pdm_rate) {
            decode_error("process: measurement pdm_rate " + std::to_string(m.pdm_rate) +
                         " does not match config " + std::to_string(plan.cfg.pdm_rate));
        }
        const uint64_t expected = static_cast<uint64_t>(kCh) * z.frames / 8;
        if (m.packed_len != expected || m.packed == nullptr) {
            decode_error("process: payload is " + std::to_string(m.packed_len) +
                         " bytes, expected " + std::to_string(expected));
        }
    }

    static bool is_pinned(const void* p) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    }

    // Per-direction stage of a block of c captures whose front end is
    // enqueued on `stream`: per beam-ring chunk the delay-and-sum (on
    // `stream`), then the envelope in sub-chunks alternating between the two
    // compute streams so a sub-chunk's CTAs fill the SMs its predecessor's
    // tail frees; `after(o, k, stream, event)` enqueues the consumer of the
    // energies of captures [o, o + k) (downloads, frame encoding) on that
    // sub-chunk's stream and returns its launch count. A later chunk's
    // delay-and-sum waits until the ring's previous contents are read.
    template <typename After>
    uint64_t enqueue_per_direction(uint64_t c, After&& after, cudaEvent_t energies_free = nullptr,
                                   uint64_t sub = SNB_ENV_SUB) {
        uint64_t nlaunch = 0, ev_j = 0;
        for (uint64_t o = 0; o < c; o += chunk_cap) {
            const uint64_t kc = std::min(chunk_cap, c - o);
            enqueue_beams(o, kc, stream);
            nlaunch += beam_launches();
            // the energies buffer may still be read by the previous block's
            // downloads: the envelope (not the delay-and-sum) waits for them
            if (energies_free && o == 0) ck(cudaStreamWaitEvent(stream, energies_free, 0), "wait");
            ck(cudaEventRecord(ev_beams, stream), "event");
            ck(cudaStreamWaitEvent(s_env2, ev_beams, 0), "wait");
            // sub-chunks on two streams (measured: also for the inner blocks of
            // a pipelined call, where one launch per block was 2% slower: the
            // next block's front end starts under the other stream's tail)
            const std::vector<uint64_t> chunks = env_chunks(kc, sub);
            uint64_t off = 0;
            for (uint64_t j = 0; j < chunks.size(); ++j, ++ev_j) {
                const uint64_t k = chunks[j];
                cudaStream_t cs = (j & 1) ? s_env2 : stream;
                enqueue_envelope(off, k, (d_energy_cur ? d_energy_cur : d_energy) + (o + off) * energy_per, cs);
                nlaunch += 1 + after(o + off, k, cs, ev_done[ev_j % kMaxChunks]);
                off += k;
            }
            if (chunks.size() > 1) {
                ck(cudaEventRecord(ev_beams, s_env2), "event");
                ck(cudaStreamWaitEvent(stream, ev_beams, 0), "wait");
            }
        }
        return nlaunch;
    }

    // Host path: H2D of every capture, the device pipeline, D2H of the
    // energyscapes, one synchronisation per max_batch block. A block is cut
    // into up to kMaxChunks chunks pipelined over three streams (H2D, kernels,
    // D2H) so only the first chunk's upload and the last chunk's download are
    // exposed. Caller buffers that are page-locked are DMA'd directly;
    // pageable ones go through the workspace's pinned staging buffers.
    void process_host(const sn_raw_measurement* ms, uint64_t count, float* out) {
        NvtxRange nv("sn_workspace_process_batch");
        for (uint64_t i = 0; i < count; ++i) validate(ms[i]); // all-or-error
        require_device();
        DeviceGuard g(device);
        const bool out_pinned = is_pinned(out);
        bool in_pinned = true;
        for (uint64_t i = 0; i < count && in_pinned; ++i) in_pinned = is_pinned(ms[i].packed);
        // with page-locked caller buffers the blocks of a call pipeline into
        // each other (block j + 1's upload and front end run under block j's
        // envelope and downloads; ordered by events on the buffers they
        // share); otherwise each block ends with a host synchronisation
        // (the staging buffers are reused)
        const bool pipelined = out_pinned && in_pinned;
        after_last(s_h2d);
        after_last(stream);
        uint64_t done = 0, blk = 0;
        while (done < count) {
            const uint64_t c = std::min(max_batch, count - done);
            const int half = (int)(blk & 1);
            float* d_en = d_energy + (uint64_t)half * max_batch * energy_per;
            // the first block's captures uploaded in up to 4 parts (copy
            // stream), the front end of part p running while part p + 1 is on
            // the bus; the beamformer for the whole block; then the envelope
            // in chunks whose energyscapes are downloaded (D2H stream) while
            // the next chunk computes: only the first part's upload and the
            // last chunk's download are exposed. Later blocks upload in one
            // part: their upload runs under the previous block's envelope,
            // and a front end split in 4 costs more than it hides (e2e A/B,
            // 128 captures per call: 4 parts every block 3,685 /s, 2 parts
            // 3,759, 1 part 3,786)
#ifndef SNB_E2E_PARTS
#define SNB_E2E_PARTS 4
#endif
#ifndef SNB_E2E_PARTS_LATER
#define SNB_E2E_PARTS_LATER 1
#endif
            const uint64_t parts = std::min<uint64_t>(c, blk == 0 ? SNB_E2E_PARTS : SNB_E2E_PARTS_LATER);
            if (blk > 0) ck(cudaStreamWaitEvent(s_h2d, ev_front, 0), "wait"); // d_packed consumed
            uint64_t p0 = 0;
            for (uint64_t p = 0; p < parts; ++p) {
                const uint64_t p1 = c * (p + 1) / parts;
                for (uint64_t i = p0; i < p1; ++i) {
                    const uint8_t* src = ms[done + i].packed;
                    if (!in_pinned) {
                        std::memcpy(h_in + i * packed_bytes, src, packed_bytes);
                        src = h_in + i * packed_bytes;
                    }
                    ck(cudaMemcpyAsync(d_packed + i * packed_bytes, src, packed_bytes, cudaMemcpyHostToDevice, s_h2d),
                       "H2D");
                }
                ck(cudaEventRecord(ev_in[p], s_h2d), "event");
                ck(cudaStreamWaitEvent(stream, ev_in[p], 0), "wait");
                enqueue_front(d_packed + p0 * packed_bytes, p0, p1 - p0, stream);
                p0 = p1;
            }
            ck(cudaEventRecord(ev_front, stream), "event");
            d_energy_cur = d_en;
            const uint64_t nlaunch = enqueue_per_direction(c, [&](uint64_t o, uint64_t k, cudaStream_t cs, cudaEvent_t ed) {
                float* d_e = d_en + o * energy_per;
                ck(cudaEventRecord(ed, cs), "event");
                ck(cudaStreamWaitEvent(s_d2h, ed, 0), "wait");
                float* dst = (out_pinned ? out + done * energy_per : h_out) + o * energy_per;
                ck(cudaMemcpyAsync(dst, d_e, k * energy_per * sizeof(float), cudaMemcpyDeviceToHost, s_d2h), "D2H");
                return uint64_t{0};
            }, blk >= 2 ? ev_d2h[half] : nullptr);
            d_energy_cur = nullptr;
            ck(cudaEventRecord(ev_d2h[half], s_d2h), "event"); // this half's downloads
            ck(cudaGetLastError(), "kernel launch");
            last_launches = 3 * parts + nlaunch;
            if (!pipelined) {
                ck(cudaStreamSynchronize(s_d2h), "process sync");
                if (!out_pinned) std::memcpy(out + done * energy_per, h_out, c * energy_per * sizeof(float));
            }
            done += c;
            ++blk;
        }
        if (pipelined) ck(cudaStreamSynchronize(s_d2h), "process sync");
        mark_last(s_d2h);
    }

    // wire::error_frame(serial, ts, seq, message) (wire.cpp:278-287)
    static std::vector<uint8_t> error_frame(uint32_t serial, uint64_t ts, uint64_t seq, const std::string& msg) {
        std::vector<uint8_t> f;
        const uint32_t magic = 0x45525449u;
        const uint16_t version = 1, type = 5;
        const uint64_t plen = msg.size();
        put(f, &magic, 4); put(f, &version, 2); put(f, &type, 2); put(f, &serial, 4);
        put(f, &ts, 8); put(f, &seq, 8); put(f, &plen, 8);
        put(f, msg.data(), msg.size());
        const uint32_t crc = crc32_host(f.data(), f.size());
        put(f, &crc, 4);
        return f;
    }

    // Central-node processing of received frames (central_node.cpp:130-160,
    // 238-270, 316-323): packet checks (wire.cpp:95-168) and payload decode
    // (wire.cpp:196-223) on the host from the 74 header bytes; the CRC of
    // every well-formed measurement frame on the GPU; the pipeline; the
    // processed-image frames (AIMG + CRC) encoded on the GPU. Per frame:
    //   SN_OK          image frame (image_frame(img, m.seq))
    //   SN_ERR_DECODE  process() rejected the measurement: error frame
    //   SN_ERR_IO      malformed / integrity error / not a measurement: discarded
    void process_frames(const uint8_t* const* frames, const uint64_t* lens, uint64_t count, uint8_t* out,
                        uint64_t slot, uint64_t* out_lens, int32_t* status) {
        NvtxRange nv("sn_workspace_process_frames");
        require_device();
        DeviceGuard g(device);
        const Sizes& z = plan.sz;
        const bool out_pinned = is_pinned(out);
        after_last(stream);
        after_last(s_h2d);
        after_last(s_d2h);
        // Blocks of up to max_batch accepted frames. A block whose frames are
        // all page-locked and whose output slots are consecutive in a
        // page-locked `out` (frames DMA'd both ways, no staging) is left in
        // flight: the next block is enqueued behind it (its upload on the copy
        // stream under this block's envelope, its front end after this
        // block's beams), and its verdicts are read once its downloads are
        // done; the two halves of the output frames / ids / verdicts
        // alternate. Any other block is finished before the next one starts.
        std::vector<uint64_t> batch;
        batch.reserve(max_batch);
        std::vector<uint64_t> pend[2];
        uint64_t blk = 0;
        auto finish = [&](int half, bool staged) {
            if (pend[half].empty()) return;
            ck(cudaEventSynchronize(ev_d2h[half]), "frames sync");
            const int32_t* ok = h_crc_ok + (uint64_t)half * max_batch;
            for (uint64_t i = 0; i < pend[half].size(); ++i) {
                const uint64_t k = pend[half][i];
                if (ok[i]) {
                    if (staged) std::memcpy(out + k * slot, h_frames_out + i * img_frame_len, img_frame_len);
                    out_lens[k] = img_frame_len;
                    status[k] = SN_OK;
                } else {
                    out_lens[k] = 0; // integrity error: frame discarded (wire.cpp:141-145)
                    status[k] = SN_ERR_IO;
                }
            }
            pend[half].clear();
        };
        auto flush = [&]() {
            if (batch.empty()) return;
            const uint64_t c = batch.size();
            const int half = (int)(blk & 1);
            finish(half, false); // block blk - 2 (pipelined: no staging)
            bool in_pinned = true;
            for (uint64_t i = 0; i < c && in_pinned; ++i) in_pinned = is_pinned(frames[batch[i]]);
            const bool direct = out_pinned && batch.back() - batch.front() == c - 1;
            const bool pipelined = direct && in_pinned;
            if (!pipelined) finish(half ^ 1, false); // staging buffers are shared: drain first
            FrameIds* hid = h_ids + (uint64_t)half * max_batch;
            uint8_t* dfo = d_frames_out + (uint64_t)half * max_batch * img_frame_stride;
            // the input frames (and d_packed) are free once the previous
            // block's front end has run
            if (blk > 0) ck(cudaStreamWaitEvent(s_h2d, ev_front, 0), "wait");
            for (uint64_t i = 0; i < c; ++i) {
                const uint8_t* f = frames[batch[i]];
                if (in_pinned) {
                    ck(cudaMemcpyAsync(d_frames_in + i * in_frame_stride, f, in_frame_len, cudaMemcpyHostToDevice,
                                       s_h2d), "H2D frame");
                } else {
                    std::memcpy(h_frames_in + i * in_frame_len, f, in_frame_len);
                    ck(cudaMemcpyAsync(d_frames_in + i * in_frame_stride, h_frames_in + i * in_frame_len,
                                       in_frame_len, cudaMemcpyHostToDevice, s_h2d), "H2D frame");
                }
                FrameIds id{};
                std::memcpy(&id.serial, f + 36, 4);
                std::memcpy(&id.ts, f + 40, 8);
                std::memcpy(&id.seq, f + 48, 8);
                hid[i] = id;
            }
            // ids on the copy stream too (an upload on the compute stream can
            // queue behind the next upload); d_ids alternates halves
            FrameIds* did = d_ids + (uint64_t)half * max_batch;
            ck(cudaMemcpyAsync(did, hid, c * sizeof(FrameIds), cudaMemcpyHostToDevice, s_h2d), "H2D ids");
            ck(cudaEventRecord(ev_in[0], s_h2d), "event");
            ck(cudaStreamWaitEvent(stream, ev_in[0], 0), "wait");
            ck(cudaMemsetAsync(d_crc_acc, 0, 2 * max_batch * sizeof(uint32_t), stream), "memset");
            const CrcTables ct = crc_tables(true), ct_in = crc_tables(false);
            const uint64_t nin = in_frame_len - 4;
            launch_crc_partial(d_frames_in, in_frame_stride, nin, c, ct_in, d_crc_acc, stream);
            int32_t* dok = d_crc_ok + (uint64_t)half * max_batch;
            launch_crc_finalize(d_crc_acc, crc_init_term(h_crc_shift.data(), nin), c, d_frames_in, in_frame_stride,
                                nin, false, dok, stream);
            launch_unpack_frames(d_frames_in + 74, in_frame_stride, d_packed, packed_bytes, c, stream);
            enqueue_front(d_packed, 0, c, stream);
            ck(cudaEventRecord(ev_front, stream), "event");
            // the verdicts download on the D2H stream (a copy on the compute
            // stream would queue behind the previous block's frame downloads
            // on the copy engine and hold up this block's kernels); they
            // precede ev_d2h[half], and dok is next written by block blk + 2
            ck(cudaStreamWaitEvent(s_d2h, ev_front, 0), "wait");
            ck(cudaMemcpyAsync(h_crc_ok + (uint64_t)half * max_batch, dok, c * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, s_d2h), "D2H ok");
            // envelope + frame encode in chunks; each chunk's frames download
            // (D2H stream) while the next chunk computes. D2H straight into the
            // caller's slots when they are page-locked and consecutive. The
            // envelope of this half waits for block blk - 2's downloads.
            const uint64_t nout = img_frame_len - 4;
            const uint32_t kout = crc_init_term(h_crc_shift.data(), nout);
            enqueue_per_direction(c, [&](uint64_t off, uint64_t k, cudaStream_t cs, cudaEvent_t ed) {
                ImageFrameArgs ia{d_energy + off * energy_per, d_img_tpl, did + off,
                                  dfo + off * img_frame_stride, d_crc_acc + max_batch + off, energy_per,
                                  img_tpl_len, img_frame_len, img_frame_stride};
                launch_encode_image_frames(ia, k, ct, cs);
                launch_crc_finalize(d_crc_acc + max_batch + off, kout, k, dfo + off * img_frame_stride,
                                    img_frame_stride, nout, true, nullptr, cs);
                ck(cudaEventRecord(ed, cs), "event");
                ck(cudaStreamWaitEvent(s_d2h, ed, 0), "wait");
                uint8_t* dst = direct ? out + (batch.front() + off) * slot : h_frames_out + off * img_frame_len;
                const uint64_t dpitch = direct ? slot : img_frame_len;
                for (uint64_t i = 0; i < k; ++i) {
                    ck(cudaMemcpyAsync(dst + i * dpitch, dfo + (off + i) * img_frame_stride, img_frame_len,
                                       cudaMemcpyDeviceToHost, s_d2h), "D2H frame");
                }
                return uint64_t{2};
            }, blk >= 2 ? ev_d2h[half] : nullptr, SNB_ENV_SUB_FRAMES);
            ck(cudaEventRecord(ev_d2h[half], s_d2h), "event");
            ck(cudaGetLastError(), "frame kernels");
            pend[half] = batch;
            if (!pipelined) finish(half, !direct);
            ++blk;
            batch.clear();
        };
        for (uint64_t k = 0; k < count; ++k) {
            out_lens[k] = 0;
            status[k] = SN_ERR_IO;
            const uint8_t* f = frames[k];
            const uint64_t len = lens[k];
            if (!f || len < 40) continue;
            uint32_t magic;
            uint16_t version, type;
            uint64_t plen;
            std::memcpy(&magic, f, 4);
            std::memcpy(&version, f + 4, 2);
            std::memcpy(&type, f + 6, 2);
            std::memcpy(&plen, f + 28, 8);
            if (magic != 0x45525449u || plen > (uint64_t{1} << 32) || len != 40 + plen) continue;
            if (len != in_frame_len) {
                // not this configuration's measurement size: host CRC, then the
                // reference's decisions (discard, or an error frame from process())
                uint32_t stored;
                std::memcpy(&stored, f + 36 + plen, 4);
                if (stored != crc32_host(f, 36 + plen)) continue;
            }
            if (version != 1 || type != 1) continue; // framing error / not a measurement
            if (plen < 38) continue;                 // decode_raw_measurement: truncated
            sn_raw_measurement m{};
            std::memcpy(&m.sensor_serial, f + 36, 4);
            std::memcpy(&m.timestamp_us, f + 40, 8);
            std::memcpy(&m.seq, f + 48, 8);
            std::memcpy(&m.channels, f + 56, 2);
            std::memcpy(&m.frames, f + 58, 8);
            std::memcpy(&m.pdm_rate, f + 66, 8);
            m.packed = f + 74;
            m.packed_len = plen - 38;
            if (m.channels == 0 || m.frames == 0 || m.frames % 8 != 0 ||
                m.packed_len != (uint64_t)m.channels * m.frames / 8) {
                continue; // decode_raw_measurement rejects: malformed, discarded
            }
            try {
                validate(m);
            } catch (const Error& e) {
                // the nominal-size frames skipped the host CRC above (it runs on
                // the GPU with the batch); a rejected one is checked here first,
                // so a corrupted header is discarded as an integrity error
                // (wire.cpp:136-145) instead of answered with an error frame
                // carrying corrupted ids
                if (len == in_frame_len) {
                    uint32_t stored;
                    std::memcpy(&stored, f + 36 + plen, 4);
                    if (stored != crc32_host(f, 36 + plen)) continue;
                }
                const auto ef = error_frame(m.sensor_serial, m.timestamp_us, m.seq, e.what());
                if (ef.size() <= slot) {
                    std::memcpy(out + k * slot, ef.data(), ef.size());
                    out_lens[k] = ef.size();
                }
                status[k] = SN_ERR_DECODE;
                continue;
            }
            batch.push_back(k);
            if (batch.size() == max_batch) flush();
        }
        flush();
        if (blk >= 2) finish((int)(blk & 1), false); // block blk - 2
        if (blk >= 1) finish((int)((blk - 1) & 1), false);
        mark_last(stream); // every block was waited for above
        (void)z;
    }

    // SN_STAGE_BEAMS: the delay-and-sum of capture `item` of the last batch,
    // recomputed into ring position 0 from the retained matched-filter output
    // (and its block-floating-point scale), slot order -> direction order.
    void dump_beams(uint64_t item, double* out) {
        const Sizes& z = plan.sz;
        DeviceGuard g(device);
        after_last(stream);
        enqueue_beams(item, 1, stream);
        ck(cudaGetLastError(), "beams launch");
        const size_t rb = f32 ? sizeof(float) : sizeof(double);
        std::vector<uint8_t> h(z.n_dirs * z.env_fft * rb);
        ck(cudaMemcpyAsync(h.data(), d_beams, h.size(), cudaMemcpyDeviceToHost, stream), "D2H beams");
        mark_last(stream);
        ck(cudaStreamSynchronize(stream), "beams sync");
        for (uint64_t sl = 0; sl < z.n_dirs; ++sl) {
            double* dst = out + (uint64_t)plan.order[sl] * z.mf_len;
            const uint8_t* src = h.data() + sl * z.env_fft * rb;
            for (uint64_t t = 0; t < z.mf_len; ++t) {
                if (f32) dst[t] = reinterpret_cast<const float*>(src)[t];
                else dst[t] = reinterpret_cast<const double*>(src)[t];
            }
        }
    }

    void process_device(const uint8_t* d_in, uint64_t count, float* d_out, cudaStream_t s) {
        NvtxRange nv("sn_workspace_process_device");
        require_device();
        DeviceGuard g(device);
        if (!s) s = stream;
        after_last(s);
        uint64_t done = 0;
        while (done < count) {
            const uint64_t c = std::min(max_batch, count - done);
            enqueue(d_in + done * packed_bytes, c, d_out + done * energy_per, s);
            done += c;
        }
        mark_last(s);
    }
};

extern "C" {

int sn_abi_version(void) { return SN_ABI_VERSION; }
const char* sn_last_error(void) { return g_last_error.c_str(); }

const char* sn_status_name(sn_status s) {
    switch (s) {
        case SN_OK: return "ok";
        case SN_ERR_CONFIG: return "config";
        case SN_ERR_ARGUMENT: return "argument";
        case SN_ERR_DECODE: return "decode";
        case SN_ERR_IO: return "io";
        case SN_ERR_CUDA: return "cuda";
        case SN_ERR_NOT_READY: return "not ready";
        default: return "internal";
    }
}

sn_status sn_default_array(uint64_t seed, double* out) {
    return guarded([&] {
        if (!out) argument_error("null output");
        default_array(seed, out);
    });
}

sn_status sn_direction_grid(int32_t kind, double* out, uint64_t capacity, uint64_t* n_out) {
    return guarded([&] {
        const auto g = direction_grid(kind);
        const uint64_t n = g.size() / 2;
        if (n_out) *n_out = n;
        if (!out) return;
        if (capacity < n) argument_error("direction buffer too small");
        std::copy(g.begin(), g.end(), out);
    });
}

sn_status sn_fibonacci_hemisphere(uint64_t n, double* out, uint64_t capacity) {
    return guarded([&] {
        if (!out) argument_error("null argument");
        if (capacity < n) argument_error("buffer too small");
        const std::vector<double> d = fibonacci_hemisphere(n);
        std::copy(d.begin(), d.end(), out);
    });
}

sn_status sn_default_config(int32_t kind, sn_pipeline_config* cfg, double* dir_buf,
                            uint64_t dir_capacity) {
    return guarded([&] {
        if (!cfg) argument_error("null config");
        default_config(kind, cfg);
        if (kind != SN_GRID_CUSTOM) {
            const auto g = direction_grid(kind);
            const uint64_t n = g.size() / 2;
            if (!dir_buf || dir_capacity < n) argument_error("direction buffer too small");
            std::copy(g.begin(), g.end(), dir_buf);
            cfg->directions = dir_buf;
            cfg->n_directions = n;
        }
    });
}

sn_status sn_config_dims(const sn_pipeline_config* cfg, sn_dims* dims) {
    return guarded([&] {
        if (!cfg || !dims) argument_error("null argument");
        const Sizes s = derive_sizes(*cfg);
        *dims = sn_dims{s.frames, s.demod_len, s.mf_len, s.bins, s.n_dirs, s.ref_len, s.mf_fft,
                        s.env_fft, s.comp_len, s.range_bin_size, s.demod_rate, s.mf_rate,
                        s.final_rate, 0};
    });
}

sn_status sn_synthesize_packed(const sn_pipeline_config* cfg, const sn_scene* scene,
                               uint8_t* packed_out, uint64_t capacity) {
    return guarded([&] {
        if (!cfg || !scene || !packed_out) argument_error("null argument");
        const Sizes s = derive_sizes(*cfg);
        if (capacity < static_cast<uint64_t>(kCh) * s.frames / 8) argument_error("packed buffer too small");
        synthesize_packed(*cfg, *scene, packed_out);
    });
}

sn_status sn_workspace_create(const sn_pipeline_config* cfg, int device, uint64_t max_batch,
                              sn_workspace** out) {
    return sn_workspace_create_ex(cfg, device, max_batch, nullptr, out);
}

sn_status sn_workspace_create_ex(const sn_pipeline_config* cfg, int device, uint64_t max_batch,
                                 const sn_workspace_options* options, sn_workspace** out) {
    return guarded([&] {
        if (!cfg || !out) argument_error("null argument");
        *out = nullptr;
        const sn_workspace_options opt = options ? *options : sn_workspace_options{};
        if (opt.beamformer != SN_BEAMFORMER_TENSOR_CORE && opt.beamformer != SN_BEAMFORMER_CUDA_CORE)
            argument_error("options: unknown beamformer kind");
        if (opt.tc_tile_n != 0 && opt.tc_tile_n != 64 && opt.tc_tile_n != 96 && opt.tc_tile_n != 128)
            argument_error("options: tensor-core tile width must be 64, 96 or 128");
        auto ws = std::make_unique<sn_workspace>();
        ws->plan = make_plan(*cfg);
        ws->device = device;
        ws->max_batch = std::max<uint64_t>(1, max_batch);
        ws->f32 = cfg->precision == SN_PRECISION_F32;
        ws->beam_budget = opt.beam_budget_bytes ? opt.beam_budget_bytes : (uint64_t{4} << 30);
        ws->plan_tensor_core_beamformer(opt);
        if (cfg->precision != SN_PRECISION_F64 && cfg->precision != SN_PRECISION_F32) {
            config_error("pipeline: unknown precision mode");
        }
        if (ws->max_batch * ws->plan.sz.n_dirs >= (uint64_t{1} << 31)) {
            argument_error("max_batch x directions must stay below 2^31 (per-launch work items)");
        }
        if (device >= 0) ws->init_device();
        *out = ws.release();
    });
}

void sn_workspace_destroy(sn_workspace* ws) { delete ws; }

sn_status sn_workspace_dims(const sn_workspace* ws, sn_dims* dims) {
    return guarded([&] {
        if (!ws || !dims) argument_error("null argument");
        const Sizes& s = ws->plan.sz;
        *dims = sn_dims{s.frames, s.demod_len, s.mf_len, s.bins, s.n_dirs, s.ref_len, s.mf_fft,
                        s.env_fft, s.comp_len, s.range_bin_size, s.demod_rate, s.mf_rate,
                        s.final_rate, ws->max_batch};
    });
}

sn_status sn_workspace_process(sn_workspace* ws, const sn_raw_measurement* m, float* out) {
    return guarded([&] {
        if (!ws || !m || !out) argument_error("null argument");
        ws->process_host(m, 1, out);
    });
}

sn_status sn_workspace_process_batch(sn_workspace* ws, const sn_raw_measurement* ms,
                                     uint64_t count, float* out) {
    return guarded([&] {
        if (!ws || (!ms && count) || (!out && count)) argument_error("null argument");
        if (count) ws->process_host(ms, count, out);
    });
}

sn_status sn_workspace_process_device(sn_workspace* ws, const uint8_t* d_packed, uint64_t count,
                                      float* d_energies, void* stream) {
    return guarded([&] {
        if (!ws || (!d_packed && count) || (!d_energies && count)) argument_error("null argument");
        ws->process_device(d_packed, count, d_energies, static_cast<cudaStream_t>(stream));
    });
}

sn_status sn_workspace_process_device_graph(sn_workspace* ws, const uint8_t* d_packed,
                                            uint64_t count, float* d_energies, void* stream) {
    return guarded([&] {
        if (!ws || !d_packed || !d_energies || count == 0) argument_error("null argument");
        ws->require_device();
        if (count > ws->max_batch) argument_error("graph replay: count exceeds max_batch");
        DeviceGuard g(ws->device);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ws->stream;
        if (!ws->graph || ws->g_in != d_packed || ws->g_out != d_energies || ws->g_count != count) {
            if (ws->graph) {
                cudaGraphExecDestroy(ws->graph);
                ws->graph = nullptr;
            }
            ws->after_last(ws->stream);
            ck(cudaStreamSynchronize(ws->stream), "sync before capture");
            cudaGraph_t graph;
            ck(cudaStreamBeginCapture(ws->stream, cudaStreamCaptureModeThreadLocal), "capture");
            ws->enqueue(d_packed, count, d_energies, ws->stream);
            ck(cudaStreamEndCapture(ws->stream, &graph), "capture end");
            ck(cudaGraphInstantiate(&ws->graph, graph, 0), "graph instantiate");
            cudaGraphDestroy(graph);
            ws->g_in = d_packed;
            ws->g_out = d_energies;
            ws->g_count = count;
        }
        ws->after_last(s);
        ck(cudaGraphLaunch(ws->graph, s), "graph launch");
        ws->mark_last(s);
        ws->last_launches = ws->tc ? 7 : 5;
    });
}

sn_status sn_workspace_delay_table(const sn_workspace* ws, int32_t* out, uint64_t capacity) {
    return guarded([&] {
        if (!ws || !out) argument_error("null argument");
        if (capacity < ws->plan.delays.size()) argument_error("buffer too small");
        std::copy(ws->plan.delays.begin(), ws->plan.delays.end(), out);
    });
}

sn_status sn_workspace_reference_advances(const sn_workspace* ws, int32_t* out, uint64_t capacity) {
    return guarded([&] {
        if (!ws || !out) argument_error("null argument");
        if (capacity < ws->plan.advances.size()) argument_error("buffer too small");
        std::copy(ws->plan.advances.begin(), ws->plan.advances.end(), out);
    });
}

uint64_t sn_workspace_allocation_events(const sn_workspace* ws) { return ws ? ws->alloc_events : 0; }
uint64_t sn_workspace_last_launches(const sn_workspace* ws) { return ws ? ws->last_launches : 0; }

sn_status sn_workspace_table(const sn_workspace* ws, int32_t table, double* out, uint64_t capacity,
                             uint64_t* n_out) {
    return guarded([&] {
        if (!ws) argument_error("null argument");
        const std::vector<double>* v = nullptr;
        switch (table) {
            case SN_TABLE_DEMOD_TAPS_REV: v = &ws->plan.demod_rev; break;
            case SN_TABLE_DEMOD_LUT: v = &ws->plan.demod_lut; break;
            case SN_TABLE_PREMF_TAPS_REV: v = &ws->plan.premf_rev; break;
            case SN_TABLE_CHIRP_REF: v = &ws->plan.chirp_ref; break;
            case SN_TABLE_SMOOTH_REV: v = &ws->plan.comp_rev; break;
            default: argument_error("unknown table");
        }
        if (n_out) *n_out = v->size();
        if (!out) return;
        if (capacity < v->size()) argument_error("buffer too small");
        std::copy(v->begin(), v->end(), out);
    });
}

sn_status sn_workspace_stage(sn_workspace* ws, int32_t stage, uint64_t item, double* out,
                             uint64_t capacity) {
    return guarded([&] {
        if (!ws || !out) argument_error("null argument");
        ws->require_device();
        if (item >= ws->max_batch) argument_error("item out of range");
        const Sizes& z = ws->plan.sz;
        const double* src = nullptr;
        uint64_t n = 0;
        if (stage == SN_STAGE_BEAMS) {
            if (capacity < z.n_dirs * z.mf_len) argument_error("buffer too small");
            ws->dump_beams(item, out);
            return;
        }
        switch (stage) {
            case SN_STAGE_DEMOD: src = ws->d_demod + item * kCh * z.demod_len; n = kCh * z.demod_len; break;
            case SN_STAGE_PREMF: src = ws->d_mf + item * kCh * z.mf_fft; n = kCh * z.mf_len; break;
            case SN_STAGE_FILT: src = ws->d_filt + item * kCh * ws->lp + ws->halo; n = kCh * z.mf_len; break;
            default: argument_error("unknown stage");
        }
        if (capacity < n) argument_error("buffer too small");
        DeviceGuard g(ws->device);
        ck(cudaEventSynchronize(ws->ev_last), "sync");
        if (stage == SN_STAGE_FILT || stage == SN_STAGE_PREMF) {
            const uint64_t pitch = stage == SN_STAGE_FILT ? ws->lp : z.mf_fft;
            ck(cudaMemcpy2D(out, z.mf_len * sizeof(double), src, pitch * sizeof(double),
                            z.mf_len * sizeof(double), kCh, cudaMemcpyDeviceToHost), "stage copy");
        } else {
            ck(cudaMemcpy(out, src, n * sizeof(double), cudaMemcpyDeviceToHost), "stage copy");
        }
    });
}

sn_status sn_workspace_beamform(sn_workspace* ws, const double* filtered, uint64_t channels,
                                uint64_t samples, double* out) {
    return guarded([&] {
        if (!ws || !filtered || !out) argument_error("null argument");
        const Sizes& z = ws->plan.sz;
        // pipeline.cpp:576-591 argument checks
        if (channels != static_cast<uint64_t>(kCh)) {
            argument_error("beamform: expected 32 channels, got " + std::to_string(channels));
        }
        if (samples != z.mf_len) {
            argument_error("beamform: expected " + std::to_string(z.mf_len) +
                           " samples per channel, got " + std::to_string(samples));
        }
        ws->require_device();
        DeviceGuard g(ws->device);
        const uint64_t L = z.mf_len;
        // the accessor is off the hot path: its two scratch buffers are
        // allocated on the first call (counted in allocation_events) and reused
        if (!ws->d_bf_in) ws->d_bf_in = ws->runtime_alloc<double>(kCh * L);
        if (!ws->d_bf_out) ws->d_bf_out = ws->runtime_alloc<double>(z.n_dirs * L);
        ws->after_last(ws->stream);
        ck(cudaMemcpyAsync(ws->d_bf_in, filtered, kCh * L * sizeof(double), cudaMemcpyHostToDevice, ws->stream), "H2D");
        launch_beamform(ws->d_bf_in, ws->d_bf_out, ws->d_shifts, (int64_t)L, (int64_t)z.n_dirs, ws->stream);
        ck(cudaGetLastError(), "beamform launch");
        ck(cudaMemcpyAsync(out, ws->d_bf_out, z.n_dirs * L * sizeof(double), cudaMemcpyDeviceToHost, ws->stream), "D2H");
        ws->mark_last(ws->stream);
        ck(cudaStreamSynchronize(ws->stream), "beamform");
    });
}

sn_status sn_workspace_set_profiling(sn_workspace* ws, int enable) {
    return guarded([&] {
        if (!ws) argument_error("null argument");
        ws->profiling = enable != 0;
    });
}

sn_status sn_workspace_stage_times(sn_workspace* ws, float* ms5) {
    return guarded([&] {
        if (!ws || !ms5) argument_error("null argument");
        ws->require_device();
        if (!ws->profiling) argument_error("profiling is not enabled");
        DeviceGuard g(ws->device);
        if (ws->prof_chunks == 0) argument_error("no profiled device-path call yet");
        ck(cudaEventSynchronize(ws->ev_ch[2 * ws->prof_chunks - 1]), "event sync");
        for (int i = 0; i < 3; ++i) ck(cudaEventElapsedTime(&ms5[i], ws->ev[i], ws->ev[i + 1]), "elapsed");
        ms5[3] = ms5[4] = 0;
        cudaEvent_t prev = ws->ev[3];
        for (uint64_t c = 0; c < ws->prof_chunks; ++c) {
            float a = 0, b = 0;
            ck(cudaEventElapsedTime(&a, prev, ws->ev_ch[2 * c]), "elapsed");
            ck(cudaEventElapsedTime(&b, ws->ev_ch[2 * c], ws->ev_ch[2 * c + 1]), "elapsed");
            ms5[3] += a;
            ms5[4] += b;
            prev = ws->ev_ch[2 * c + 1];
        }
    });
}

sn_status sn_workspace_beamformer_info(const sn_workspace* ws, sn_beamformer_info* info) {
    return guarded([&] {
        if (!ws || !info) argument_error("null argument");
        *info = sn_beamformer_info{};
        info->kind = ws->tc ? 1 : 0;
        if (!ws->tc) return;
        info->clusters = ws->tc_clusters;
        for (int32_t r : ws->tc_R) info->sum_R += r;
        info->max_R = ws->tc_rmax;
        info->ntiles = ws->tc_ntiles;
        info->slices = kTcSlices;
        info->m = kTcM;
        info->n = ws->tc_n;
        info->k = 32;
    });
}

uint32_t sn_crc32(const uint8_t* bytes, uint64_t n) { return bytes || !n ? crc32_host(bytes, n) : 0; }

uint64_t sn_workspace_image_frame_bytes(const sn_workspace* ws) { return ws ? ws->img_frame_len : 0; }

sn_status sn_measurement_frame(const sn_raw_measurement* m, uint8_t* out, uint64_t capacity, uint64_t* n_out) {
    return guarded([&] {
        if (!m || (!m->packed && m->packed_len)) argument_error("null argument");
        std::vector<uint8_t> f;
        const uint32_t magic = 0x45525449u;
        const uint16_t version = 1, type = 1;
        const uint64_t plen = 38 + m->packed_len;
        sn_workspace::put(f, &magic, 4); sn_workspace::put(f, &version, 2); sn_workspace::put(f, &type, 2);
        sn_workspace::put(f, &m->sensor_serial, 4); sn_workspace::put(f, &m->timestamp_us, 8);
        sn_workspace::put(f, &m->seq, 8); sn_workspace::put(f, &plen, 8);
        sn_workspace::put(f, &m->sensor_serial, 4); sn_workspace::put(f, &m->timestamp_us, 8);
        sn_workspace::put(f, &m->seq, 8); sn_workspace::put(f, &m->channels, 2);
        sn_workspace::put(f, &m->frames, 8); sn_workspace::put(f, &m->pdm_rate, 8);
        sn_workspace::put(f, m->packed, m->packed_len);
        const uint32_t crc = crc32_host(f.data(), f.size());
        sn_workspace::put(f, &crc, 4);
        if (n_out) *n_out = f.size();
        if (!out) return;
        if (capacity < f.size()) argument_error("buffer too small");
        std::memcpy(out, f.data(), f.size());
    });
}

sn_status sn_workspace_process_frames(sn_workspace* ws, const uint8_t* const* frames, const uint64_t* lens,
                                      uint64_t count, uint8_t* out, uint64_t slot_bytes, uint64_t* out_lens,
                                      int32_t* status) {
    return guarded([&] {
        if (!ws || (count && (!frames || !lens || !out || !out_lens || !status))) argument_error("null argument");
        ws->require_device();
        if (slot_bytes < ws->img_frame_len) argument_error("output slot smaller than an image frame");
        ws->process_frames(frames, lens, count, out, slot_bytes, out_lens, status);
    });
}

sn_status sn_synthesize_device(const sn_pipeline_config* cfg, const sn_scene* scenes, uint64_t count, int device,
                               uint8_t* d_packed, void* stream) {
    return guarded([&] {
        if (!cfg || (!scenes && count) || (!d_packed && count)) argument_error("null argument");
        if (device < 0) argument_error("device must be >= 0");
        if (count == 0) return;
        std::vector<SynthScene> sc(count);
        std::vector<double> pulse;
        uint64_t frames = 0;
        for (uint64_t i = 0; i < count; ++i) {
            const SceneEchoes e = scene_echoes(*cfg, scenes[i]);
            if (e.amplitude.size() > (size_t)kSynthMaxReflectors)
                argument_error("synthesize_device: more than 8 reflectors in a scene");
            if (i == 0) {
                pulse = e.pulse;
                frames = e.frames;
            }
            SynthScene& s = sc[i];
            s = SynthScene{};
            s.seed = scenes[i].seed;
            s.noise_rms = scenes[i].noise_rms;
            s.n_refl = (int)e.amplitude.size();
            for (int k = 0; k < s.n_refl; ++k) {
                s.amp[k] = e.amplitude[k];
                for (int ch = 0; ch < kCh; ++ch) s.onset[k][ch] = e.onset[(size_t)k * kCh + ch];
            }
        }
        DeviceGuard g(device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int64_t nwords = (int64_t)((frames + 31) / 32);
        double* d_pulse = nullptr;
        SynthScene* d_sc = nullptr;
        uint32_t* d_words = nullptr;
        unsigned long long* d_states = nullptr;
        ck(cudaMallocAsync(&d_states, count * kCh * 4 * sizeof(unsigned long long), st), "cudaMallocAsync");
        ck(cudaMallocAsync(&d_pulse, pulse.size() * sizeof(double), st), "cudaMallocAsync");
        ck(cudaMallocAsync(&d_sc, count * sizeof(SynthScene), st), "cudaMallocAsync");
        ck(cudaMallocAsync(&d_words, count * 32 * nwords * sizeof(uint32_t), st), "cudaMallocAsync");
        ck(cudaMemcpyAsync(d_pulse, pulse.data(), pulse.size() * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemcpyAsync(d_sc, sc.data(), count * sizeof(SynthScene), cudaMemcpyHostToDevice, st), "H2D");
        SynthArgs a{d_pulse, d_sc, d_words, d_states, d_packed, (int64_t)frames, (int64_t)pulse.size(), nwords,
                    (int64_t)(kCh * frames / 8), (int)count};
        launch_synth(a, st);
        ck(cudaGetLastError(), "synth launch");
        cudaFreeAsync(d_states, st);
        cudaFreeAsync(d_pulse, st);
        cudaFreeAsync(d_sc, st);
        cudaFreeAsync(d_words, st);
        ck(cudaStreamSynchronize(st), "synth sync");
    });
}

sn_status sn_energyscape_transform(const float* d_energies, float* d_out, uint64_t count, uint64_t cells,
                                   int32_t mode, float floor_db, void* stream) {
    return guarded([&] {
        if ((!d_energies || !d_out) && count) argument_error("null argument");
        if (mode != SN_TRANSFORM_NORMALIZE && mode != SN_TRANSFORM_DB) argument_error("unknown transform mode");
        if (d_energies == d_out && count) argument_error("the transform writes a separate buffer (in == out)");
        launch_energyscape_transform(d_energies, d_out, count, cells, mode, floor_db,
                                     static_cast<cudaStream_t>(stream));
        ck(cudaGetLastError(), "transform launch");
    });
}

sn_status sn_measure_fp_peak(int device, int precision, double* tflops) {
    return guarded([&] {
        if (!tflops) argument_error("null argument");
        DeviceGuard g(device);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        *tflops = measure_fma_peak(sms, precision == SN_PRECISION_F32);
    });
}

} // extern "C"
