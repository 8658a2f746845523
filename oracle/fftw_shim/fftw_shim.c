/* ORACLE / TEST INFRASTRUCTURE ONLY -- FFTW3-API shim, see fftw3.h. */
#include "fftw3.h"

#include <stdlib.h>

#include "../fft_core.h"

struct fftw_plan_s {
  int n0, n1, sign;
  double* in;
  double* out;
};

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
  (void)flags;
  if (n0 < 1 || n1 < 1) return NULL;
  fftw_plan p = (fftw_plan)malloc(sizeof(struct fftw_plan_s));
  p->n0 = n0;
  p->n1 = n1;
  p->sign = sign;
  p->in = (double*)in;
  p->out = (double*)out;
  return p;
}

void fftw_execute(const fftw_plan p) { ncs_fft2d(p->in, p->out, p->n0, p->n1, p->sign); }

void fftw_destroy_plan(fftw_plan p) { free(p); }
