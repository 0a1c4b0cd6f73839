/* TEST INFRASTRUCTURE ONLY — never linked into the product.
 *
 * Minimal FFTW3 double-precision API subset so the UNMODIFIED reference
 * sources (/root/reference/proj/core/src/fft.cpp) compile and link without
 * FFTW, which is absent from this image.
 *
 * Symbols used by the reference: fft.cpp:33-36 (plans), :83/:89/:150/:156
 * (execute), :41-46 (alloc/free/destroy).
 *
 * Semantics follow the published FFTW3 conventions:
 *   r2c  : out[k] = sum_j in[j] e^{-2 pi i jk/n}, k = 0..n/2, unnormalised
 *   c2r  : out[j] = sum_k X[k] e^{+2 pi i jk/n} over the Hermitian extension,
 *          imag(X[0]) and imag(X[n/2]) ignored, unnormalised
 *   dft  : sign -1 forward / +1 backward, unnormalised
 * Sizes: any n >= 1 (powers of two take the fast path; others a direct DFT).
 */
#ifndef SONARNET_ORACLE_FFTW3_SHIM_H
#define SONARNET_ORACLE_FFTW3_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)

double* fftw_alloc_real(size_t n);
fftw_complex* fftw_alloc_complex(size_t n);
void fftw_free(void* p);

fftw_plan fftw_plan_dft_r2c_1d(int n, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex* in, double* out, unsigned flags);
fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
