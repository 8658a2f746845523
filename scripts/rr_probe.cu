#include <cstdio>
#include "../paper_1810_13100_b200/csrc/ncsg_internal.cuh"
__device__ __forceinline__ void ray_range(const ncsg::AngleGeom& g, float c, float x0, float x1,
                                          float y0, float y1, int s_mid, float eps, int& lo, int& hi) {
  float a = (x0 - c) * g.aXf, b = (x1 - c) * g.aXf;
  float e = (y0 - c) * g.aYf, f = (y1 - c) * g.aYf;
  float mn = fminf(a, b) + fminf(e, f);
  float mx = fmaxf(a, b) + fmaxf(e, f);
  lo = max(-s_mid, static_cast<int>(floorf(mn - eps)));
  hi = min(s_mid, static_cast<int>(ceilf(mx + eps)));
  printf("a %f b %f e %f f %f mn %f mx %f eps %f lo %d hi %d\n", a, b, e, f, mn, mx, eps, lo, hi);
}
__global__ void k(ncsg::AngleGeom g) { int lo, hi; ray_range(g, 7.5f, -1.f, 129.f, -1.f, 33.f, 12, 1.0f, lo, hi); }
int main() { ncsg::AngleGeom g{}; g.aXf = 1.f; g.aYf = 0.f; k<<<1,1>>>(g); cudaDeviceSynchronize(); return 0; }
