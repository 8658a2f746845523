/* ORACLE / TEST INFRASTRUCTURE ONLY -- see fft_core.h. */
#include "fft_core.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846;

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

/* Radix-2 DIT on a contiguous buffer of n complex values. */
static void fft_pow2(double* a, int n, int sign) {
  for (int i = 1, j = 0; i < n; ++i) {
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double tr = a[2 * i], ti = a[2 * i + 1];
      a[2 * i] = a[2 * j];
      a[2 * i + 1] = a[2 * j + 1];
      a[2 * j] = tr;
      a[2 * j + 1] = ti;
    }
  }
  for (int len = 2; len <= n; len <<= 1) {
    int half = len >> 1;
    for (int k = 0; k < half; ++k) {
      double ang = sign * 2.0 * kPi * (double)k / (double)len;
      double wr = cos(ang), wi = sin(ang);
      for (int i = 0; i < n; i += len) {
        double* u = a + 2 * (i + k);
        double* v = a + 2 * (i + k + half);
        double vr = v[0] * wr - v[1] * wi;
        double vi = v[0] * wi + v[1] * wr;
        v[0] = u[0] - vr;
        v[1] = u[1] - vi;
        u[0] += vr;
        u[1] += vi;
      }
    }
  }
}

static void dft_direct(double* a, int n, int sign, double* tmp) {
  for (int k = 0; k < n; ++k) {
    double sr = 0.0, si = 0.0;
    for (int j = 0; j < n; ++j) {
      /* reduce k*j mod n before forming the angle to keep it small */
      long long kj = ((long long)k * j) % n;
      double ang = sign * 2.0 * kPi * (double)kj / (double)n;
      double wr = cos(ang), wi = sin(ang);
      sr += a[2 * j] * wr - a[2 * j + 1] * wi;
      si += a[2 * j] * wi + a[2 * j + 1] * wr;
    }
    tmp[2 * k] = sr;
    tmp[2 * k + 1] = si;
  }
  memcpy(a, tmp, sizeof(double) * 2 * (size_t)n);
}

static void transform_contig(double* a, int n, int sign, double* tmp) {
  if (is_pow2(n))
    fft_pow2(a, n, sign);
  else
    dft_direct(a, n, sign, tmp);
}

void ncs_fft1d(double* data, int n, ptrdiff_t stride, int sign) {
  double* buf = (double*)malloc(sizeof(double) * 4 * (size_t)n);
  for (int i = 0; i < n; ++i) {
    buf[2 * i] = data[2 * i * stride];
    buf[2 * i + 1] = data[2 * i * stride + 1];
  }
  transform_contig(buf, n, sign, buf + 2 * n);
  for (int i = 0; i < n; ++i) {
    data[2 * i * stride] = buf[2 * i];
    data[2 * i * stride + 1] = buf[2 * i + 1];
  }
  free(buf);
}

void ncs_fft2d(const double* in, double* out, int n0, int n1, int sign) {
  size_t total = (size_t)n0 * n1;
  if (out != in) memcpy(out, in, sizeof(double) * 2 * total);
  /* rows (contiguous) */
#pragma omp parallel
  {
    double* tmp = (double*)malloc(sizeof(double) * 4 * (size_t)(n0 > n1 ? n0 : n1));
#pragma omp for schedule(static)
    for (int r = 0; r < n0; ++r) {
      double* row = out + 2 * (size_t)r * n1;
      memcpy(tmp, row, sizeof(double) * 2 * (size_t)n1);
      transform_contig(tmp, n1, sign, tmp + 2 * n1);
      memcpy(row, tmp, sizeof(double) * 2 * (size_t)n1);
    }
#pragma omp for schedule(static)
    for (int c = 0; c < n1; ++c) {
      for (int r = 0; r < n0; ++r) {
        tmp[2 * r] = out[2 * ((size_t)r * n1 + c)];
        tmp[2 * r + 1] = out[2 * ((size_t)r * n1 + c) + 1];
      }
      transform_contig(tmp, n0, sign, tmp + 2 * n0);
      for (int r = 0; r < n0; ++r) {
        out[2 * ((size_t)r * n1 + c)] = tmp[2 * r];
        out[2 * ((size_t)r * n1 + c) + 1] = tmp[2 * r + 1];
      }
    }
    free(tmp);
  }
}
