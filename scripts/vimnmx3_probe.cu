// Repro: ptxas (CUDA 12.9, sm_100a) folds max(-a, x) followed by max(., y) into
// one VIMNMX3 whose first bound is +a (the negation is lost).
#include <cstdio>
__global__ void k(const float* in, int s_mid, const int* sl, int* out) {
  float mn = in[threadIdx.x];
  int lo = max(-s_mid, (int)floorf(mn - 1.0f));
  lo = max(lo, sl[0]);
  out[threadIdx.x] = lo;
}
int main() {
  float h[32]; for (int i = 0; i < 32; ++i) h[i] = -8.5f;
  int sl[2] = {-12, 12}, o[32];
  float* di; int *ds, *dout;
  cudaMalloc(&di, 128); cudaMalloc(&ds, 8); cudaMalloc(&dout, 128);
  cudaMemcpy(di, h, 128, cudaMemcpyHostToDevice); cudaMemcpy(ds, sl, 8, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(di, 12, ds, dout);
  cudaMemcpy(o, dout, 128, cudaMemcpyDeviceToHost);
  printf("max(max(-12, floor(-9.5)), -12) = %d (expected -10)\n", o[0]);
  return 0;
}
