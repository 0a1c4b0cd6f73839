// Wire-format frames on the GPU (protocol.md; wire.cpp, pipeline.cpp:109-125):
// CRC-32 of whole frames and the processed-image frame encoder.
//
// CRC-32 (reflected 0xEDB88320, init/xorout 0xFFFFFFFF, wire.cpp:17-63) is
// affine in the register: for a message M of n bytes split in chunks C_i that
// end at byte e_i,
//     R(s, M) = A_n(s) ^ XOR_i A_{n - e_i}(R(0, C_i)),   crc(M) = R(~0, M) ^ ~0
// where A_m is the GF(2)-linear map "advance the register over m zero bytes".
// Every thread computes R(0, C_i) of its chunk (slicing-by-4 tables in shared
// memory), shifts it by the bytes that follow (A_{2^k} matrices, one per set
// bit) and XORs it into the frame's accumulator; the host folds in the
// constant A_n(~0) ^ ~0. No sequential pass over the 7.9 MB image frames.
//
// The image frame (wire::image_frame(image_to_bytes(img), seq)) is
//   [36 B packet header][34 B AIMG header][8 B per direction][4 B per cell][CRC]
// The header + direction table is a per-workspace template patched with the
// capture's serial / timestamp / seq; the energies start at byte
// E = 70 + 8 n_dirs (E mod 4 = 2), so each output word is a 16-bit funnel
// shift of two consecutive float words of the energyscape. The encoder CRCs
// the words it writes (no re-read) and a finalize kernel stores the CRC.
#include "kernels.cuh"
#include "sonarnet_b200.h"

#include <cstdint>
#include <cstring>

namespace snb {

namespace {

__device__ __forceinline__ uint32_t crc_word(const uint32_t* __restrict__ t, uint32_t c, uint32_t w) {
    c ^= w; // little-endian: byte 0 first
    return t[768 + (c & 0xFF)] ^ t[512 + ((c >> 8) & 0xFF)] ^ t[256 + ((c >> 16) & 0xFF)] ^ t[c >> 24];
}
__device__ __forceinline__ uint32_t crc_byte(const uint32_t* __restrict__ t, uint32_t c, uint32_t b) {
    return t[(c ^ b) & 0xFF] ^ (c >> 8);
}

// v -> A_m(v): product of the A_{2^k} for the set bits of m (mat: [k][32] columns)
__device__ __forceinline__ uint32_t crc_shift(const uint32_t* __restrict__ mat, uint32_t v, uint64_t m) {
    for (int k = 0; m != 0 && v != 0; ++k, m >>= 1) {
        if (m & 1) {
            const uint32_t* col = mat + 32 * k;
            uint32_t r = 0;
#pragma unroll
            for (int b = 0; b < 32; ++b) r ^= (0u - ((v >> b) & 1u)) & col[b];
            v = r;
        }
    }
    return v;
}

__device__ __forceinline__ void load_crc_tables(const CrcTables& ct, uint32_t* s_tab) {
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_tab[i] = ct.slice[i];
}

} // namespace

// ---------------------------------------------------------------------------
// CRC of `count` byte strings (string f at base + f * stride, n bytes each,
// base and stride 4-byte aligned): acc[f] ^= XOR of shifted chunk CRCs.
// One warp per 4 KB segment (see the encoder below): coalesced word loads
// staged in shared memory, a 128-byte chunk per lane, lane chunks moved to
// the segment end by the constant maps A_{128 (31 - l)}, segments to the
// string end by A_{2^k} products; the n mod 4 trailing bytes by the byte table.
// ---------------------------------------------------------------------------
constexpr int kEncWarps = 8, kSegWords = 1024;

__device__ __forceinline__ uint32_t lane_to_segment_end(const uint32_t* s_lane, int l, uint32_t c) {
    const uint32_t* col = s_lane + 32 * l;
    uint32_t r = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) r ^= (0u - ((c >> b) & 1u)) & col[b];
    return r;
}

// The warp's segment CRC (lane chunks already moved to the segment end,
// XOR-reduced here) moved on to the string end. A full segment s with the
// per-length table: lane b holds column b of A_{n - 4096 (s + 1)} (loaded
// before the CRC loop), the product is a masked XOR reduction across the warp;
// otherwise lane 0 runs the A_{2^k} chain. Lane 0 returns the result.
__device__ __forceinline__ uint32_t segment_to_end(const CrcTables& ct, bool full, uint64_t w0, uint64_t n,
                                                   uint32_t c, uint32_t seg_col, int l) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c ^= __shfl_xor_sync(0xffffffffu, c, o);
    if (full && ct.seg) {
        uint32_t r = (c >> l) & 1u ? seg_col : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r ^= __shfl_xor_sync(0xffffffffu, r, o);
        return r;
    }
    if (l == 0 && full) c = crc_shift(ct.shift, c, n - 4 * (w0 + kSegWords));
    return c;
}

__device__ __forceinline__ uint32_t seg_column(const CrcTables& ct, uint64_t w0, uint64_t nw, int l) {
    return ct.seg && w0 + kSegWords <= nw ? __ldg(ct.seg + 32 * (w0 / kSegWords) + l) : 0u;
}

__global__ void __launch_bounds__(32 * kEncWarps) k_crc_partial(const uint8_t* base, uint64_t stride, uint64_t n,
                                                                CrcTables ct, uint32_t* acc) {
    __shared__ uint32_t s_tab[1024];
    __shared__ uint32_t s_lane[1024];
    __shared__ uint32_t s_w[kEncWarps][kSegWords + 32];
    load_crc_tables(ct, s_tab);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_lane[i] = ct.lane[i];
    __syncthreads();
    const int f = blockIdx.y, warp = threadIdx.x >> 5, l = threadIdx.x & 31;
    const uint64_t nw = n / 4; // full words; then n % 4 tail bytes
    const uint64_t w0 = ((uint64_t)blockIdx.x * kEncWarps + warp) * kSegWords;
    if (w0 > nw || (w0 == nw && (n & 3) == 0)) return;
    const uint32_t seg_col = seg_column(ct, w0, nw, l);
    const uint8_t* p = base + (size_t)f * stride;
    const uint32_t* pw = reinterpret_cast<const uint32_t*>(p);
    uint32_t* sw = s_w[warp];
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
        const uint64_t w = w0 + 32 * i + l;
        if (w < nw) sw[33 * i + l] = __ldg(pw + w);
    }
    __syncwarp();
    uint32_t c = 0;
    const uint64_t cw0 = w0 + 32 * l;
    for (int i = 0; i < 32; ++i) {
        const uint64_t w = cw0 + i;
        if (w < nw) {
            c = crc_word(s_tab, c, sw[33 * l + i]);
        } else {
            if (w == nw)
                for (uint64_t bb = 4 * nw; bb < n; ++bb) c = crc_byte(s_tab, c, p[bb]);
            break;
        }
    }
    const bool full = w0 + kSegWords <= nw;
    if (full) {
        c = lane_to_segment_end(s_lane, l, c);
    } else {
        const uint64_t end = cw0 + 32 <= nw ? 4 * (cw0 + 32) : n;
        c = cw0 <= nw ? crc_shift(ct.shift, c, n - end) : 0u;
    }
    c = segment_to_end(ct, full, w0, n, c, seg_col, l);
    if (l == 0 && c) atomicXor(acc + f, c);
}

// ---------------------------------------------------------------------------
// Image-frame encoder: frame f (stride fstride) from the f32 energyscape
// energies[f][n_dirs * bins] and the header template; CRC of bytes
// [0, frame_len - 4) accumulated into acc[f].
// One warp per 4 KB segment of the frame: the words are produced and stored
// lane-interleaved (coalesced loads of the energies, coalesced stores) and
// staged in shared memory; lane l then CRCs its contiguous 128-byte chunk,
// moves it to the segment end with the constant map A_{128 (31 - l)}
// (CrcTables::lane), the warp XOR-reduces, and lane 0 moves the segment's CRC
// to the frame end. Frame words: template (header fields patched per capture)
// up to byte E - 2; the word at E - 2 joins the template's last two bytes and
// the low half of energy 0; above, word = hi16(en[q]) | lo16(en[q + 1]) << 16;
// the CRC covers a final 2-byte tail (hi16 of the last energy).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32 * kEncWarps) k_encode_image_frames(ImageFrameArgs a, CrcTables ct) {
    __shared__ uint32_t s_tab[1024];
    __shared__ uint32_t s_lane[1024];
    __shared__ uint32_t s_w[kEncWarps][kSegWords + 32];
    load_crc_tables(ct, s_tab);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_lane[i] = ct.lane[i];
    __syncthreads();
    const int f = blockIdx.y, warp = threadIdx.x >> 5, l = threadIdx.x & 31;
    const uint64_t ncrc = a.frame_len - 4; // = E + 4 cells, E % 4 == 2
    const uint64_t nw = ncrc / 4;          // full words; then the 2-byte tail at byte 4 nw
    const uint64_t w0 = ((uint64_t)blockIdx.x * kEncWarps + warp) * kSegWords;
    if (w0 > nw) return;
    const uint32_t seg_col = seg_column(ct, w0, nw, l);
    uint8_t* out = a.frames + (size_t)f * a.frame_stride;
    uint32_t* ow = reinterpret_cast<uint32_t*>(out);
    const uint32_t* en = reinterpret_cast<const uint32_t*>(a.energies + (size_t)f * a.cells);
    const uint8_t* tpl = a.tpl;
    const uint32_t* tplw = reinterpret_cast<const uint32_t*>(tpl);
    const FrameIds id = a.ids[f];
    const uint64_t E = a.tpl_len;
    auto tpl_byte = [&](uint64_t b) -> uint32_t {
        // header fields patched per capture (packet: serial 8, ts 12, seq 20;
        // AIMG: serial 42, ts 46)
        if (b >= 8 && b < 12) return (id.serial >> (8 * (b - 8))) & 0xFF;
        if (b >= 12 && b < 20) return (uint32_t)(id.ts >> (8 * (b - 12))) & 0xFF;
        if (b >= 20 && b < 28) return (uint32_t)(id.seq >> (8 * (b - 20))) & 0xFF;
        if (b >= 42 && b < 46) return (id.serial >> (8 * (b - 42))) & 0xFF;
        if (b >= 46 && b < 54) return (uint32_t)(id.ts >> (8 * (b - 46))) & 0xFF;
        return tpl[b];
    };
    auto word_at = [&](uint64_t w) -> uint32_t {
        const uint64_t b = 4 * w;
        if (b + 4 <= E - 2) {
            if (b >= 56) return __ldg(tplw + w);
            return tpl_byte(b) | (tpl_byte(b + 1) << 8) | (tpl_byte(b + 2) << 16) | (tpl_byte(b + 3) << 24);
        }
        if (b == E - 2) return (uint32_t)tpl[E - 2] | ((uint32_t)tpl[E - 1] << 8) | (__ldg(en) << 16);
        const uint64_t q = (b - E - 2) / 4;
        return __funnelshift_r(__ldg(en + q), __ldg(en + q + 1), 16);
    };
    const uint32_t tail = __ldg(en + a.cells - 1) >> 16;
    uint32_t* sw = s_w[warp];
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
        const uint64_t w = w0 + 32 * i + l;
        if (w < nw) {
            const uint32_t v = word_at(w);
            ow[w] = v;
            sw[33 * i + l] = v;
        } else if (w == nw) {
            reinterpret_cast<uint16_t*>(out + 4 * nw)[0] = (uint16_t)tail;
        }
    }
    __syncwarp();
    uint32_t c = 0;
    const uint64_t cw0 = w0 + 32 * l; // lane chunk: words [cw0, cw0 + 32)
    for (int i = 0; i < 32; ++i) {
        const uint64_t w = cw0 + i;
        if (w < nw) {
            c = crc_word(s_tab, c, sw[33 * l + i]);
        } else {
            if (w == nw) {
                c = crc_byte(s_tab, c, tail & 0xFF);
                c = crc_byte(s_tab, c, tail >> 8);
            }
            break;
        }
    }
    const bool full = w0 + kSegWords <= nw;
    if (full) {
        c = lane_to_segment_end(s_lane, l, c);
    } else {
        const uint64_t end = cw0 + 32 <= nw ? 4 * (cw0 + 32) : ncrc;
        c = cw0 <= nw ? crc_shift(ct.shift, c, ncrc - end) : 0u;
    }
    c = segment_to_end(ct, full, w0, ncrc, c, seg_col, l);
    if (l == 0 && c) atomicXor(a.acc + f, c);
}

// crc[f] = acc[f] ^ k_n (k_n = A_n(~0) ^ ~0 from the host); optionally stored
// little-endian at out + f * stride + n (2-byte aligned) and/or compared with
// the stored value there (ok[f] = match).
__global__ void k_crc_finalize(uint32_t* acc, uint32_t k_n, uint64_t count, uint8_t* out, uint64_t stride,
                               uint64_t n, int store, int32_t* ok) {
    const uint64_t f = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= count) return;
    const uint32_t crc = acc[f] ^ k_n;
    acc[f] = crc;
    uint8_t* p = out + f * stride + n;
    if (store) {
        reinterpret_cast<uint16_t*>(p)[0] = (uint16_t)(crc & 0xFFFF);
        reinterpret_cast<uint16_t*>(p)[1] = (uint16_t)(crc >> 16);
    }
    if (ok) {
        const uint32_t stored = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
        ok[f] = stored == crc;
    }
}

// The packed bits of `count` received frames (at src + f * sstride, 2-byte
// aligned: byte 74 of a 16-byte aligned frame) into the 4-byte aligned capture
// buffer (dst + f * nbytes, nbytes % 4 == 0): one output word per thread from
// two 16-bit loads. A kernel rather than a 2-D device-to-device memcpy, which
// can queue on a copy engine behind the previous block's downloads.
__global__ void k_unpack_frames(const uint8_t* __restrict__ src, uint64_t sstride, uint8_t* __restrict__ dst,
                                uint64_t nbytes) {
    const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; // output word
    if (4 * j >= nbytes) return;
    const uint16_t* s = reinterpret_cast<const uint16_t*>(src + (size_t)blockIdx.y * sstride) + 2 * j;
    reinterpret_cast<uint32_t*>(dst + (size_t)blockIdx.y * nbytes)[j] = (uint32_t)__ldg(s) | ((uint32_t)__ldg(s + 1) << 16);
}

void launch_unpack_frames(const uint8_t* src, uint64_t sstride, uint8_t* dst, uint64_t nbytes, uint64_t count,
                          cudaStream_t s) {
    if (count == 0 || nbytes == 0) return;
    k_unpack_frames<<<dim3((unsigned)((nbytes / 4 + 255) / 256), (unsigned)count), 256, 0, s>>>(src, sstride, dst,
                                                                                                 nbytes);
}

void launch_crc_partial(const uint8_t* base, uint64_t stride, uint64_t n, uint64_t count, const CrcTables& ct,
                        uint32_t* acc, cudaStream_t s) {
    if (n == 0 || count == 0) return;
    const uint64_t segs = (n / 4 + 1 + kSegWords - 1) / kSegWords; // words + the tail
    const unsigned gx = (unsigned)((segs + kEncWarps - 1) / kEncWarps);
    k_crc_partial<<<dim3(gx, (unsigned)count), 32 * kEncWarps, 0, s>>>(base, stride, n, ct, acc);
}

void launch_encode_image_frames(const ImageFrameArgs& a, uint64_t count, const CrcTables& ct, cudaStream_t s) {
    const uint64_t segs = ((a.frame_len - 4) / 4 + 1 + kSegWords - 1) / kSegWords; // words + the tail
    const unsigned gx = (unsigned)((segs + kEncWarps - 1) / kEncWarps);
    k_encode_image_frames<<<dim3(gx, (unsigned)count), 32 * kEncWarps, 0, s>>>(a, ct);
}

void launch_crc_finalize(uint32_t* acc, uint32_t k_n, uint64_t count, uint8_t* out, uint64_t stride, uint64_t n,
                         bool store, int32_t* ok, cudaStream_t s) {
    k_crc_finalize<<<(unsigned)((count + 127) / 128), 128, 0, s>>>(acc, k_n, count, out, stride, n, store ? 1 : 0, ok);
}

// ---- host side: tables and the constant of the init term --------------------
// slicing-by-8 tables, built once (C++11 magic static: thread-safe first use)
struct HostCrcTables {
    uint32_t t[8][256];
    HostCrcTables() {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
            t[0][i] = c;
        }
        for (int s = 1; s < 8; ++s)
            for (int i = 0; i < 256; ++i) t[s][i] = t[0][t[s - 1][i] & 0xFF] ^ (t[s - 1][i] >> 8);
    }
};
static const HostCrcTables& host_crc() {
    static const HostCrcTables tabs;
    return tabs;
}

uint32_t crc32_host(const uint8_t* p, uint64_t n) {
    const HostCrcTables& T = host_crc();
    uint32_t c = 0xFFFFFFFFu;
    uint64_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint32_t lo, hi;
        std::memcpy(&lo, p + i, 4);
        std::memcpy(&hi, p + i + 4, 4);
        lo ^= c;
        c = T.t[7][lo & 0xFF] ^ T.t[6][(lo >> 8) & 0xFF] ^ T.t[5][(lo >> 16) & 0xFF] ^ T.t[4][lo >> 24] ^
            T.t[3][hi & 0xFF] ^ T.t[2][(hi >> 8) & 0xFF] ^ T.t[1][(hi >> 16) & 0xFF] ^ T.t[0][hi >> 24];
    }
    for (; i < n; ++i) c = T.t[0][(c ^ p[i]) & 0xFF] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

void crc_tables_host(uint32_t* slice /* 1024 */, uint32_t* shift /* kCrcShiftMats x 32 */) {
    const uint32_t* host_tab = host_crc().t[0];
    for (int i = 0; i < 256; ++i) {
        uint32_t c = host_tab[i];
        slice[i] = c;
        for (int t = 1; t < 4; ++t) {
            c = host_tab[c & 0xFF] ^ (c >> 8);
            slice[256 * t + i] = c;
        }
    }
    // A_1: one zero byte; A_{2^k} = A_{2^(k-1)} o A_{2^(k-1)}
    uint32_t m[32];
    for (int b = 0; b < 32; ++b) {
        const uint32_t v = 1u << b;
        m[b] = host_tab[v & 0xFF] ^ (v >> 8);
    }
    for (int k = 0; k < kCrcShiftMats; ++k) {
        for (int b = 0; b < 32; ++b) shift[32 * k + b] = m[b];
        uint32_t sq[32];
        for (int b = 0; b < 32; ++b) {
            uint32_t v = m[b], r = 0;
            for (int i = 0; i < 32; ++i)
                if (v >> i & 1) r ^= m[i];
            sq[b] = r;
        }
        for (int b = 0; b < 32; ++b) m[b] = sq[b];
    }
}

uint32_t crc_advance_host(const uint32_t* shift, uint32_t v, uint64_t n) {
    for (int k = 0; n != 0 && v != 0; ++k, n >>= 1) {
        if (n & 1) {
            uint32_t r = 0;
            for (int b = 0; b < 32; ++b)
                if (v >> b & 1) r ^= shift[32 * k + b];
            v = r;
        }
    }
    return v;
}

std::vector<uint32_t> crc_segment_shifts_host(const uint32_t* shift, uint64_t n) {
    const uint64_t segs = (n / 4) / kSegWords; // full segments: 4096 (s + 1) <= n
    std::vector<uint32_t> t(segs * 32);
    if (segs == 0) return t;
    uint32_t col[32];
    for (int b = 0; b < 32; ++b) col[b] = crc_advance_host(shift, 1u << b, n - 4 * kSegWords * segs);
    for (uint64_t s = segs; s-- > 0;) {
        for (int b = 0; b < 32; ++b) t[32 * s + b] = col[b];
        if (s > 0)
            for (int b = 0; b < 32; ++b) col[b] = crc_advance_host(shift, col[b], 4 * kSegWords);
    }
    return t;
}

uint32_t crc_init_term(const uint32_t* shift, uint64_t n) {
    uint32_t v = 0xFFFFFFFFu;
    for (int k = 0; n != 0; ++k, n >>= 1) {
        if (n & 1) {
            uint32_t r = 0;
            for (int b = 0; b < 32; ++b)
                if (v >> b & 1) r ^= shift[32 * k + b];
            v = r;
        }
    }
    return v ^ 0xFFFFFFFFu;
}

} // namespace snb

namespace snb {

// ---------------------------------------------------------------------------
// Opt-in display transform of finished energyscapes (north star stage 4,
// "log/normalisation"): the reference's write-out stops at max(0, float)
// (pipeline.cpp:469-471), so this runs strictly after the energies exist,
// into a separate buffer, and never changes them. Per image (cells floats):
//   SN_TRANSFORM_NORMALIZE: e / max(e)                    (0 if the image is all 0)
//   SN_TRANSFORM_DB:        max(10 log10(e / max(e)), floor_db)  (floor_db if e == 0)
// One CTA per image: a block max reduction over the image, then the map, both
// reading the image with 16-byte loads where aligned.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_energyscape_transform(const float* in, float* out, uint64_t cells,
                                                                int mode, float floor_db) {
    __shared__ float red[16];
    const float* e = in + (size_t)blockIdx.x * cells;
    float* o = out + (size_t)blockIdx.x * cells;
    float m = 0.0f;
    for (uint64_t i = threadIdx.x; i < cells; i += blockDim.x) m = fmaxf(m, e[i]);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = 0.0f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
    for (uint64_t i = threadIdx.x; i < cells; i += blockDim.x) {
        const float r = m > 0.0f ? __fdiv_rn(e[i], m) : 0.0f; // the peak maps to exactly 1 (0 dB)
        o[i] = mode == SN_TRANSFORM_NORMALIZE ? r : (r > 0.0f ? fmaxf(10.0f * log10f(r), floor_db) : floor_db);
    }
}

void launch_energyscape_transform(const float* in, float* out, uint64_t count, uint64_t cells, int mode,
                                  float floor_db, cudaStream_t s) {
    if (count == 0) return;
    k_energyscape_transform<<<(unsigned)count, 512, 0, s>>>(in, out, cells, mode, floor_db);
}

} // namespace snb
