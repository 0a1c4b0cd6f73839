// FP64 tensor (DMMA, mma.sync f64) vs FP64 pipe (DFMA) microbenchmark:
// does the FP64 MMA issue on a unit separate from the DFMA pipe, i.e. do the
// two rates add when a kernel mixes them? (developer diagnostic)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_rate dmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                 "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// MODE 0: DFMA only; 1: m8n8k4 only; 2: m16n8k16 only; 3: m8n8k4 + DFMA in
// every warp (same counts as modes 0 and 1 together); 4: m16n8k16 + DFMA
template <int MODE>
__global__ void k(double* out, int iters, double seed) {
    double f[8];
    for (int i = 0; i < 8; ++i) f[i] = seed + threadIdx.x + i;
    double d4[4][2] = {}, d16[2][4] = {};
    double a8[8], b4[4];
    for (int i = 0; i < 8; ++i) a8[i] = seed * (i + 1);
    for (int i = 0; i < 4; ++i) b4[i] = seed / (i + 2);
    const double m = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE == 0 || MODE == 3 || MODE == 4) {
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] = fma(f[i], m, c);
            }
            if (MODE == 1 || MODE == 3) {
#pragma unroll
                for (int j = 0; j < 4; ++j) mma884(d4[j], a8[j], b4[j]);
            }
            if (MODE == 2 || MODE == 4) {
#pragma unroll
                for (int j = 0; j < 2; ++j) mma16816(d16[j], a8, b4);
            }
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += f[i];
    for (int j = 0; j < 4; ++j) s += d4[j][0] + d4[j][1];
    for (int j = 0; j < 2; ++j) s += d16[j][0] + d16[j][1] + d16[j][2] + d16[j][3];
    if (s == 12345.678) out[0] = s;
}

template <int MODE>
void run(const char* name, int sms, int blocks_per_sm) {
    double* o;
    cudaMalloc(&o, 8);
    const int iters = 2048;
    k<MODE><<<sms * blocks_per_sm, 256>>>(o, 10, 1.0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<MODE><<<sms * blocks_per_sm, 256>>>(o, iters, 1.0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warps = (double)sms * blocks_per_sm * 8;
    const double per_warp_iter = 8.0; // u loop
    double dfma = 0, mma_fma = 0;
    if (MODE == 0 || MODE == 3 || MODE == 4) dfma = warps * 32 * iters * per_warp_iter * 8;
    if (MODE == 1 || MODE == 3) mma_fma = warps * iters * per_warp_iter * 4 * (8 * 8 * 4);
    if (MODE == 2 || MODE == 4) mma_fma = warps * iters * per_warp_iter * 2 * (16 * 8 * 16);
    const double s = ms * 1e-3;
    printf("%-22s %7.3f ms  DFMA %6.2f TFLOP/s  MMA %6.2f TFLOP/s  total %6.2f TFLOP/s  (%s)\n", name, ms,
           2 * dfma / s / 1e12, 2 * mma_fma / s / 1e12, 2 * (dfma + mma_fma) / s / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bps : {2, 4}) {
        printf("-- %d blocks x 256 threads per SM\n", bps);
        run<0>("DFMA", sms, bps);
        run<1>("DMMA m8n8k4", sms, bps);
        run<2>("DMMA m16n8k16", sms, bps);
        run<3>("m8n8k4 + DFMA", sms, bps);
        run<4>("m16n8k16 + DFMA", sms, bps);
    }
}
