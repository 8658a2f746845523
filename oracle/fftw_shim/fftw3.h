/* ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * Minimal FFTW3-API shim so the reference's proj/src/fft.cpp compiles and links
 * unchanged in this image, where FFTW3 is not installed.  It
 * covers exactly the calls fft.cpp makes (fft.cpp:3,23-34,39,45):
 * fftw_complex, fftw_plan, FFTW_FORWARD/BACKWARD/ESTIMATE, fftw_plan_dft_2d,
 * fftw_execute, fftw_destroy_plan.  The transform itself is oracle/fft_core.c.
 * FFTW3 (third-party, unpinned: proj/src/CMakeLists.txt:8-9) computes the same
 * unnormalised DFT; only its rounding differs.
 */
#ifndef NCS_FFTW_SHIM_H
#define NCS_FFTW_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
