// Microbenchmark: the tensor-core beamformer's MMA issue structure in
// isolation -- tiles of 6 digit-plane chains of R MMAs (M=128, N=96, K=32,
// kind::i8, A_r resident, B window displaced one 16-byte row per r), each
// chain into the next slot of a 5-slot TMEM ring -- with and without the
// per-chain tcgen05.commit and tcgen05.fence::after_thread_sync the kernel
// issues, to find what keeps the tensor pipe idle (developer diagnostic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_planes mma_planes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
constexpr int N = 96, SLOTS = 5, PLANES = 6;
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\nWT%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WT%=;\n}\n" ::"r"(su32(b)), "r"(parity) : "memory");
}

// MODE bit 0: commit per chain; bit 1: fence per chain; bit 2: one chain of
// 6R MMAs per tile (no slot switching); bit 3: 16 more warps poll an
// mbarrier (try_wait loop) meanwhile, as the kernel's epilogue warps do;
// bit 4: they poll with a 1 us suspend-time hint
template <int MODE, int R = 17>
__global__ void k(int tiles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ __align__(8) uint64_t sfull[SLOTS], sempty[SLOTS];
    for (int i = threadIdx.x; i < 20 * 128 * 32 + 12 * (N + 32) * 16; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&bar[0])), "r"(1 << 20)); // never completes
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[1])));
        for (int i = 0; i < SLOTS; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&sfull[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;\n" ::"r"(su32(&sempty[i])));
        }
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = slot;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (threadIdx.x < 32) {
        uint32_t pred;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
        const bool leader = pred;
        const uint32_t wrows = N + 32;
        const uint64_t a0 = sdesc(su32(smem), 128 * 16, 128);
        const uint64_t b0 = sdesc(su32(smem + 20 * 128 * 32 + (R - 1) * 16), wrows * 16, 128);
        for (int g = 0; g < tiles; ++g) {
            for (int p = 0; p < PLANES; ++p) {
                const int q = PLANES * g + p, sl = (MODE & 4) ? 0 : q % SLOTS;
                if ((MODE & 32) && q >= SLOTS) mbar_wait(&sempty[sl], (uint32_t)(((q - SLOTS) / SLOTS) & 1));
                if (MODE & 2) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                if (leader) {
                    uint64_t ad = a0, bd = b0 + (uint64_t)(2 * wrows * (PLANES - 1 - p));
                    for (int r = 0; r < R; ++r) {
                        const uint32_t acc = ((MODE & 4) ? (p > 0 || r > 0) : r > 0) ? 1u : 0u;
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)(sl * N)),
                                     "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                        ad += 256;
                        bd -= 1;
                    }
                    if (MODE & 32)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&sfull[sl])));
                    else if (MODE & 1)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar[0])));
                }
                __syncwarp();
            }
        }
        if (leader) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar[1])));
            asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}\n" ::"r"(su32(&bar[1])));
        }
        __syncwarp();
    } else if (MODE & 32) {
        // consumers, as the kernel's epilogue warps with no work (NOEPI):
        // wait for slot q's chain, fence, arrive on its empty barrier
        const int tiles_ = tiles;
        for (int q = 0; q < PLANES * tiles_; ++q) {
            const int sl = q % SLOTS;
            mbar_wait(&sfull[sl], (uint32_t)((q / SLOTS) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (MODE & 64) {
                uint32_t y[8];
                const uint32_t src = slot + ((uint32_t)((threadIdx.x / 32) & 3) * 32 << 16) + (uint32_t)(sl * N + (((threadIdx.x / 32 - 1) >> 2) * (N / 4)));
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                             : "=r"(y[0]), "=r"(y[1]), "=r"(y[2]), "=r"(y[3]), "=r"(y[4]), "=r"(y[5]), "=r"(y[6]), "=r"(y[7])
                             : "r"(src));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                if (y[0] == 0x12345678u && y[7] == 1u) asm volatile("trap;");
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&sempty[sl])) : "memory");
        }
    } else if (MODE & 8) {
        // pollers: wait for phase 0 of bar[1], completed by the MMA warp's
        // final commit (they poll for the whole run)
        if (MODE & 16) {
            asm volatile("{\n\t.reg .pred p;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, 1000;\n\t@!p bra W2;\n}\n" ::"r"(su32(&bar[1])));
        } else {
            asm volatile("{\n\t.reg .pred p;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n}\n" ::"r"(su32(&bar[1])));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <int MODE, int R = 17> void run(int sms, const char* name) {
    const int tiles = 400;
    const size_t sm = 20 * 128 * 32 + 12 * (N + 32) * 16 + 1024;
    cudaFuncSetAttribute(k<MODE, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int threads = (MODE & (8 | 32)) ? 32 * 17 : 128;
    k<MODE, R><<<sms, threads, sm>>>(4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<MODE, R><<<sms, threads, sm>>>(tiles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double mmas = (double)tiles * PLANES * R;
    printf("%-34s R=%2d %.3f ms  %.1f clk/MMA (floor 48)  %s\n", name, R, ms, ms * 1e-3 * 1.965e9 / mmas,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<4>(sms, "one chain per tile, no commits");
    run<0>(sms, "6 chains x 5 slots, no commit/fence");
    run<1>(sms, "6 chains, commit per chain");
    run<2>(sms, "6 chains, fence per chain");
    run<3>(sms, "6 chains, commit + fence (kernel)");
    run<4>(sms, "one chain per tile, no commits");
    run<3 | 8>(sms, "kernel + 16 polling warps");
    run<3 | 8 | 16>(sms, "kernel + 16 warps, 1 us hint");
    run<2 | 32>(sms, "slot ring with 16 consumer warps");
    run<2 | 32 | 64>(sms, "ring + consumers tcgen05.ld x8");
    run<2, 7>(sms, "6 chains, fence per chain");
    run<2 | 32 | 64, 7>(sms, "ring + consumers tcgen05.ld x8");
    run<2, 13>(sms, "6 chains, fence per chain");
    run<2 | 32 | 64, 13>(sms, "ring + consumers tcgen05.ld x8");
    run<2, 21>(sms, "6 chains, fence per chain");
    run<2 | 32 | 64, 21>(sms, "ring + consumers tcgen05.ld x8");
}
