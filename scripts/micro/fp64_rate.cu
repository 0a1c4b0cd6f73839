// FP64 pipe microbenchmark: DFMA vs DADD vs DMUL throughput (developer diagnostic)
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double seed) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x + i;
    const double m = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (OP == 0) a[i] = fma(a[i], m, c);
                else if (OP == 1) a[i] = __dadd_rn(a[i], c);
                else a[i] = __dmul_rn(a[i], m);
            }
        }
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.678) out[0] = s;
}
template <int OP> void run(const char* name, int sms) {
    double* o; cudaMalloc(&o, 8);
    k<OP><<<sms * 4, 256>>>(o, 100, 1.0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<OP><<<sms * 4, 256>>>(o, 4096, 1.0); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = 8.0 * 16 * 4096 * 256 * sms * 4;
    printf("%s: %.2f Gop/s = %.1f lanes/clk/SM at 1.965 GHz\n", name, ops / ms / 1e6, ops / (ms * 1e-3) / 1.965e9 / sms);
}
int main() { int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); run<0>("DFMA", sms); run<1>("DADD", sms); run<2>("DMUL", sms); }
