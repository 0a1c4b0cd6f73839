// Synthetic captures on the GPU (load generation).
//
// Restates synthesize_measurement (synth.cpp:116-134): echoes of the PDM-rate
// pulse per reflector and channel (synthesize_scene :11-61), white Gaussian
// noise from one xoshiro256++ stream in channel-major sample order with the
// polar Box-Muller method and its cached spare (rng.hpp), the first-order
// sigma-delta modulator per channel (:63-94) and frame-major MSB-first packing
// (:96-114). The noise stream is sequential by definition (the Box-Muller
// rejection makes the stream position of every sample data dependent), but
// its expensive part is not: k_synth_skip walks each capture's stream once
// with only the cheap acceptance test (two draws, q = u^2 + v^2, the same
// rounded operations) and records the generator state at every channel
// start; k_synth_sd then runs one thread per (capture, channel) with the
// logarithm, square root and the sigma-delta modulator. With an even frame
// count every channel consumes whole accepted pairs, so no cached spare
// crosses a channel boundary (odd frame counts run the whole capture in one
// thread). The FP64 operations are issued in the reference's order without
// contraction (__dadd_rn / __dmul_rn). Echo
// geometry (pulse, amplitudes, onsets) comes from the host planner
// (plan.cpp scene_echoes), so it is the reference's to the bit. log() on the
// device may differ from the host's in the last place; a sigma-delta decision
// can only change where |integrator + x| is within ~1e-16 of zero.
#include "kernels.cuh"

#include <cstdint>

namespace snb {

namespace {

struct DevRng {
    uint64_t s[4];
    double spare;
    bool have;
    __device__ explicit DevRng(uint64_t seed) : spare(0.0), have(false) {
        uint64_t x = seed;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            x += 0x9e3779b97f4a7c15ULL;
            uint64_t z = x;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
            s[i] = z ^ (z >> 31);
        }
    }
    __device__ static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    __device__ uint64_t next() {
        const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return r;
    }
    __device__ double uniform() { return __dmul_rn((double)(next() >> 11), 0x1.0p-53); }
    __device__ double gaussian() {
        if (have) {
            have = false;
            return spare;
        }
        double u, v, q;
        do {
            u = __dsub_rn(__dmul_rn(2.0, uniform()), 1.0);
            v = __dsub_rn(__dmul_rn(2.0, uniform()), 1.0);
            q = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
        } while (q >= 1.0 || q == 0.0);
        const double m = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(q)), q));
        spare = __dmul_rn(v, m);
        have = true;
        return __dmul_rn(u, m);
    }
};

} // namespace

// Generator state at the start of every channel: frames / 2 accepted pairs
// per channel (even frame count), rejections included.
__global__ void k_synth_skip(SynthArgs a) {
    const int cap = blockIdx.x * blockDim.x + threadIdx.x;
    if (cap >= a.count) return;
    const SynthScene sc = a.scenes[cap];
    DevRng rng(sc.seed);
    unsigned long long* st = a.states + (size_t)cap * 32 * 4;
    const int64_t pairs = a.frames / 2;
    for (int ch = 0; ch < 32; ++ch) {
#pragma unroll
        for (int k = 0; k < 4; ++k) st[4 * ch + k] = rng.s[k];
        if (sc.noise_rms <= 0.0) continue;
        for (int64_t i = 0; i < pairs; ++i) {
            double q;
            do {
                const double u = __dsub_rn(__dmul_rn(2.0, rng.uniform()), 1.0);
                const double v = __dsub_rn(__dmul_rn(2.0, rng.uniform()), 1.0);
                q = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
            } while (q >= 1.0 || q == 0.0);
        }
    }
}

// Echoes + noise + sigma-delta for channels [ch0, ch1) of a capture, starting
// from the generator state `rng`; bits land channel-major in
// words[capture][32][nwords] (bit i of word w = frame 32 w + i).
__device__ void synth_channels(const SynthArgs& a, const SynthScene& sc, DevRng& rng, int cap, int ch0, int ch1) {
    uint32_t* words = a.words + (size_t)cap * 32 * a.nwords;
    for (int ch = ch0; ch < ch1; ++ch) {
        double integ = 0.0;
        uint32_t w = 0;
        for (int64_t i = 0; i < a.frames; ++i) {
            double x = 0.0;
            for (int k = 0; k < sc.n_refl; ++k) {
                const int64_t o = sc.onset[k][ch];
                if (i >= o && i < o + a.ref_len) x = __dadd_rn(x, __dmul_rn(sc.amp[k], __ldg(a.pulse + (i - o))));
            }
            if (sc.noise_rms > 0.0) x = __dadd_rn(x, __dmul_rn(sc.noise_rms, rng.gaussian()));
            const double v = x > 1.0 ? 1.0 : (x < -1.0 ? -1.0 : x);
            const double bit = __dadd_rn(integ, v) >= 0.0 ? 1.0 : -1.0;
            integ = __dadd_rn(integ, __dsub_rn(v, bit));
            if (bit > 0.0) w |= 1u << (i & 31);
            if ((i & 31) == 31 || i == a.frames - 1) {
                words[(size_t)ch * a.nwords + (i >> 5)] = w;
                w = 0;
            }
        }
    }
}

// one thread per (capture, channel), from the recorded channel-start states
__global__ void k_synth_sd(SynthArgs a) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)a.count * 32) return;
    const int cap = (int)(t / 32), ch = (int)(t % 32);
    const SynthScene sc = a.scenes[cap];
    DevRng rng(0);
    const unsigned long long* st = a.states + ((size_t)cap * 32 + ch) * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) rng.s[k] = st[k];
    synth_channels(a, sc, rng, cap, ch, ch + 1);
}

// odd frame counts: one thread per capture, all channels in stream order
__global__ void k_synth_sd_serial(SynthArgs a) {
    const int cap = blockIdx.x * blockDim.x + threadIdx.x;
    if (cap >= a.count) return;
    const SynthScene sc = a.scenes[cap];
    DevRng rng(sc.seed);
    synth_channels(a, sc, rng, cap, 0, 32);
}

// Channel-major bit words -> frame-major packed bytes (pack_pdm, synth.cpp:
// 96-114): one warp per (capture, 32 frames); lane c holds channel c's word,
// a ballot per frame gathers the 32 channel bits of that frame.
__global__ void k_synth_pack(SynthArgs a) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int64_t per = a.nwords;
    if (warp >= (int64_t)a.count * per) return;
    const int cap = (int)(warp / per);
    const int64_t wi = warp % per;
    const uint32_t mine = a.words[((size_t)cap * 32 + lane) * a.nwords + wi];
    uint32_t out = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const uint32_t m = __ballot_sync(0xffffffffu, (mine >> i) & 1u); // bit c = channel c of frame 32 wi + i
        if (lane == i) out = __byte_perm(__brev(m), 0, 0x0123);          // byte c/8, bit 7 - c%8
    }
    const int64_t f = 32 * wi + lane;
    if (f < a.frames) reinterpret_cast<uint32_t*>(a.packed + (size_t)cap * a.packed_bytes)[f] = out;
}

void launch_synth(const SynthArgs& a, cudaStream_t s) {
    if (a.frames % 2 == 0) {
        k_synth_skip<<<(a.count + 31) / 32, 32, 0, s>>>(a);
        k_synth_sd<<<(unsigned)((a.count * 32 + 31) / 32), 32, 0, s>>>(a);
    } else {
        k_synth_sd_serial<<<(a.count + 31) / 32, 32, 0, s>>>(a);
    }
    const int64_t warps = (int64_t)a.count * a.nwords;
    k_synth_pack<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(a);
}

} // namespace snb
