// Microbenchmark: tcgen05.mma kind::i8 issue rate for M=128, N in {32,64,128,256},
// K=32, A/B from shared memory (SWIZZLE_NONE, K-major) -- developer diagnostic.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
template <int N, int ROT, bool TS = false, bool VAR = false>
__global__ void k(int iters, int* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 20 * 128 * 32 + (N + 32) * 32; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = slot;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (threadIdx.x == 0) {
        const uint64_t ad = sdesc(su32(smem), 128 * 16, 128);
        const uint64_t bd = sdesc(su32(smem + 128 * 32), N * 16, 128);
        if (TS) {
          for (int it = 0; it < iters; ++it) {
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)((it % ROT) * N)),
                         "r"(tmem + 384u), "l"(bd), "r"(idesc), "r"(1));
          }
        } else if (VAR) {
          // as k_beamform_tc: 20 resident A_r (4 KB apart), B window shifted by one 16-byte row per r
          const uint64_t bd0 = sdesc(su32(smem + 20 * 128 * 32 + 19 * 16), (N + 32) * 16, 128);
          for (int it = 0; it < iters; it += 20) {
            uint64_t a_ = sdesc(su32(smem), 128 * 16, 128), b_ = bd0;
            for (int r = 0; r < 20; ++r) {
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)(((it / 20) % 2) * N)),
                           "l"(a_), "l"(b_), "r"(idesc), "r"(r));
              a_ += 256; b_ -= 1;
            }
          }
        } else
        for (int it = 0; it < iters; ++it) {
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)((it % ROT) * N)),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(1));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}\n" ::"r"(su32(&bar)));
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    if (threadIdx.x == 0 && out) out[blockIdx.x] = 1;
}
template <int N, int ROT, bool TS = false, bool VAR = false> void run(int sms) {
    const int iters = 20000;
    cudaFuncSetAttribute(k<N, ROT, TS, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    k<N, ROT, TS, VAR><<<sms, 128, 150 * 1024>>>(100, nullptr);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<N, ROT, TS, VAR><<<sms, 128, 150 * 1024>>>(iters, nullptr);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double macs = (double)sms * iters * 128.0 * N * 32;
    printf("TS=%d ROT=%d VAR=%d ", (int)TS, ROT, (int)VAR); printf("N=%3d: %.3f ms, %.2f TOPS (int8, 2 ops/MAC), %.1f clk/MMA at 1.965 GHz, err=%s\n", N, ms, 2 * macs / ms / 1e9,
           ms * 1e-3 * 1.965e9 / iters, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<32,2>(sms); run<32,2,true>(sms); run<64,2>(sms); run<64,2,true>(sms); run<128,2>(sms); run<128,2,true>(sms);
    run<64,1>(sms); run<128,1>(sms); run<64,6>(sms); run<128,3>(sms);
    run<64,2,false,true>(sms); run<96,2,false,true>(sms); run<128,2,false,true>(sms); run<96,2>(sms);
}
