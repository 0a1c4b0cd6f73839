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

#include <cstdint>

namespace snb {

namespace {

constexpr int kCrcThreads = 256;

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
// Chunks of kCrcChunk bytes per thread.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kCrcThreads) k_crc_partial(const uint8_t* base, uint64_t stride, uint64_t n,
                                                             CrcTables ct, uint32_t* acc) {
    __shared__ uint32_t s_tab[1024];
    load_crc_tables(ct, s_tab);
    __syncthreads();
    const int f = blockIdx.y;
    const uint64_t c0 = ((uint64_t)blockIdx.x * kCrcThreads + threadIdx.x) * kCrcChunk;
    if (c0 >= n) return;
    const uint64_t c1 = c0 + kCrcChunk < n ? c0 + kCrcChunk : n;
    const uint8_t* p = base + (size_t)f * stride;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(p + c0);
    uint32_t c = 0;
    const uint64_t nw = (c1 - c0) / 4;
    for (uint64_t i = 0; i < nw; ++i) c = crc_word(s_tab, c, __ldg(w + i));
    for (uint64_t b = c0 + 4 * nw; b < c1; ++b) c = crc_byte(s_tab, c, p[b]);
    c = crc_shift(ct.shift, c, n - c1);
    if (c) atomicXor(acc + f, c);
}

// ---------------------------------------------------------------------------
// Image-frame encoder: frame f (stride fstride) from the f32 energyscape
// energies[f][n_dirs * bins] and the header template; CRC of bytes
// [0, frame_len - 4) accumulated into acc[f].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kCrcThreads) k_encode_image_frames(ImageFrameArgs a, CrcTables ct) {
    __shared__ uint32_t s_tab[1024];
    load_crc_tables(ct, s_tab);
    __syncthreads();
    const int f = blockIdx.y;
    const uint64_t F = a.frame_len, ncrc = F - 4;
    const uint64_t c0 = ((uint64_t)blockIdx.x * kCrcThreads + threadIdx.x) * kCrcChunk;
    if (c0 >= ncrc) return;
    const uint64_t c1 = c0 + kCrcChunk < ncrc ? c0 + kCrcChunk : ncrc;
    uint8_t* out = a.frames + (size_t)f * a.frame_stride;
    const uint32_t* en = reinterpret_cast<const uint32_t*>(a.energies + (size_t)f * a.cells);
    const uint8_t* tpl = a.tpl;
    const FrameIds id = a.ids[f];
    const uint64_t E = a.tpl_len; // first energy byte (E % 4 == 2)
    auto byte_at = [&](uint64_t b) -> uint32_t {
        if (b < E) {
            // header fields patched per capture (packet: serial 8, ts 12, seq 20;
            // AIMG: serial 42, ts 46)
            if (b >= 8 && b < 12) return (id.serial >> (8 * (b - 8))) & 0xFF;
            if (b >= 12 && b < 20) return (uint32_t)(id.ts >> (8 * (b - 12))) & 0xFF;
            if (b >= 20 && b < 28) return (uint32_t)(id.seq >> (8 * (b - 20))) & 0xFF;
            if (b >= 42 && b < 46) return (id.serial >> (8 * (b - 42))) & 0xFF;
            if (b >= 46 && b < 54) return (uint32_t)(id.ts >> (8 * (b - 46))) & 0xFF;
            return tpl[b];
        }
        const uint64_t e = b - E;
        return (__ldg(en + e / 4) >> (8 * (e & 3))) & 0xFF;
    };
    uint32_t c = 0;
    uint64_t b = c0;
    uint32_t* ow = reinterpret_cast<uint32_t*>(out);
    // bytes below the first full energy word, and the partial last word: byte path
    const uint64_t fast0 = E + 2;            // 4-aligned, first word made of two energy halves
    const uint64_t fast1 = ncrc & ~uint64_t(3); // words below this are complete
    while (b < c1 && (b < fast0 || b >= fast1 || (b & 3))) {
        const uint32_t v = byte_at(b);
        if ((b & 3) == 0 && b + 4 <= c1 && b + 4 <= ncrc && b < fast0) {
            // whole header word
            const uint32_t word = v | (byte_at(b + 1) << 8) | (byte_at(b + 2) << 16) | (byte_at(b + 3) << 24);
            ow[b / 4] = word;
            c = crc_word(s_tab, c, word);
            b += 4;
            continue;
        }
        out[b] = (uint8_t)v;
        c = crc_byte(s_tab, c, v);
        ++b;
    }
    // fast path: word w at byte 4w >= E + 2: hi16(en[q]) | lo16(en[q + 1]) << 16
    for (; b + 4 <= c1 && b + 4 <= fast1; b += 4) {
        const uint64_t q = (b - E - 2) / 4;
        const uint32_t word = __funnelshift_r(__ldg(en + q), __ldg(en + q + 1), 16);
        ow[b / 4] = word;
        c = crc_word(s_tab, c, word);
    }
    for (; b < c1; ++b) {
        const uint32_t v = byte_at(b);
        out[b] = (uint8_t)v;
        c = crc_byte(s_tab, c, v);
    }
    c = crc_shift(ct.shift, c, ncrc - c1);
    if (c) atomicXor(a.acc + f, c);
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

void launch_crc_partial(const uint8_t* base, uint64_t stride, uint64_t n, uint64_t count, const CrcTables& ct,
                        uint32_t* acc, cudaStream_t s) {
    if (n == 0 || count == 0) return;
    const uint64_t chunks = (n + kCrcChunk - 1) / kCrcChunk;
    const unsigned gx = (unsigned)((chunks + kCrcThreads - 1) / kCrcThreads);
    k_crc_partial<<<dim3(gx, (unsigned)count), kCrcThreads, 0, s>>>(base, stride, n, ct, acc);
}

void launch_encode_image_frames(const ImageFrameArgs& a, uint64_t count, const CrcTables& ct, cudaStream_t s) {
    const uint64_t chunks = (a.frame_len - 4 + kCrcChunk - 1) / kCrcChunk;
    const unsigned gx = (unsigned)((chunks + kCrcThreads - 1) / kCrcThreads);
    k_encode_image_frames<<<dim3(gx, (unsigned)count), kCrcThreads, 0, s>>>(a, ct);
}

void launch_crc_finalize(uint32_t* acc, uint32_t k_n, uint64_t count, uint8_t* out, uint64_t stride, uint64_t n,
                         bool store, int32_t* ok, cudaStream_t s) {
    k_crc_finalize<<<(unsigned)((count + 127) / 128), 128, 0, s>>>(acc, k_n, count, out, stride, n, store ? 1 : 0, ok);
}

// ---- host side: tables and the constant of the init term --------------------
static uint32_t host_tab[256];

static void host_tables_init() {
    static bool done = false;
    if (done) return;
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
        host_tab[i] = c;
    }
    done = true;
}

uint32_t crc32_host(const uint8_t* p, uint64_t n) {
    host_tables_init();
    uint32_t c = 0xFFFFFFFFu;
    for (uint64_t i = 0; i < n; ++i) c = host_tab[(c ^ p[i]) & 0xFF] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

void crc_tables_host(uint32_t* slice /* 1024 */, uint32_t* shift /* kCrcShiftMats x 32 */) {
    host_tables_init();
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
