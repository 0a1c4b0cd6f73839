// Accuracy of the FP64 magnitude sequences in k_envelope's sink against the
// correctly rounded sqrt (developer diagnostic):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rsqrt_acc rsqrt_acc.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ double seed(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ double two_step(double x) {
    double r = seed(fmax(x, 1e-300));
    r = r * fma(-0.5 * x, r * r, 1.5);
    const double s = x * r;
    return fma(0.5 * r, fma(-s, s, x), s);
}
__device__ double coupled(double x) {
    const double r = seed(x + 1e-300), s = x * r;
    return fma(0.5 * r, fma(-s, s, x), s);
}
__device__ double third(double x) {
    const double r = seed(x + 1e-300), s = x * r;
    const double e = fma(s, r, -1.0);
    return fma(s, e * fma(e, 0.375, -0.5), s);
}
__global__ void k(double* err, unsigned long long n) {
    double e[4] = {0, 0, 0, 0};
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n; i += (unsigned long long)gridDim.x * blockDim.x) {
        // log-uniform x over [2^-200, 2^200) plus mantissa sweep
        unsigned long long h = i * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 32;
        const double m = 1.0 + (double)(h >> 12) * 0x1p-52;
        const double x = ldexp(m, (int)(i % 400) - 200);
        const double t = sqrt(x);
        e[0] = fmax(e[0], fabs(seed(x) * t - 1.0));
        e[1] = fmax(e[1], fabs(two_step(x) / t - 1.0));
        e[2] = fmax(e[2], fabs(coupled(x) / t - 1.0));
        e[3] = fmax(e[3], fabs(third(x) / t - 1.0));
    }
    for (int j = 0; j < 4; ++j) {
        unsigned long long* p = reinterpret_cast<unsigned long long*>(err + j);
        atomicMax(p, (unsigned long long)__double_as_longlong(e[j]));
    }
}
int main() {
    double* d;
    cudaMalloc(&d, 32);
    cudaMemset(d, 0, 32);
    k<<<592, 256>>>(d, 1ull << 30);
    double h[4];
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    const char* nm[4] = {"rsqrt.approx.f64 seed", "two Newton steps (r02 sink)", "coupled step", "third-order step"};
    for (int j = 0; j < 4; ++j) printf("%-30s max rel err %.3e (2^%.1f)\n", nm[j], h[j], log2(h[j]));
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
