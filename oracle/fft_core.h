/* ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product path.
 *
 * fp64 complex 2-D DFT used by (a) the FFTW-API shim that lets the reference's
 * own proj/src/fft.cpp link (FFTW3 is absent from this image),
 * and (b) the C restatement of the NCS path in ncs_oracle.c.  Sharing one
 * transform makes the restatement bitwise comparable with the reference build.
 *
 * Convention follows proj/include/ncstomo/fft.hpp:8-28 / FFTW: sign -1 is the
 * unnormalised forward transform, sign +1 the unnormalised backward transform
 * (the 1/N^2 is applied by the caller, as proj/src/fft.cpp:45-47 does).
 * Radix-2 iterative Cooley-Tukey for power-of-two lengths, direct O(n^2) DFT
 * otherwise; every twiddle is evaluated directly with cos/sin (no recurrence).
 */
#ifndef NCS_ORACLE_FFT_CORE_H
#define NCS_ORACLE_FFT_CORE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* In-place 1-D transform of n complex values (interleaved re,im) with stride. */
void ncs_fft1d(double* data, int n, ptrdiff_t stride, int sign);

/* 2-D n0 x n1 row-major complex transform, in -> out (may alias). */
void ncs_fft2d(const double* in, double* out, int n0, int n1, int sign);

#ifdef __cplusplus
}
#endif

#endif
