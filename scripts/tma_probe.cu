// Stand-alone probe of the TMA tile load used by fp_strip_kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile("{\n .reg .pred p;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2, unsigned bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(dst), "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}

template <int BW, int BH, int MODE>
__global__ void probe(float* out, const __grid_constant__ CUtensorMap map, int x0, int y0) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  unsigned pad = ((base + 127u) & ~127u) - base;
  if (threadIdx.x == 0) {
    mbar_init(b, 1);
    if (MODE >= 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(b, BW * BH * 4);
    tma_load_3d(base + pad, &map, x0, y0, 0, b);
  }
  mbar_wait(b, 0);
  for (int i = threadIdx.x; i < BW * BH; i += blockDim.x) out[i] = sm[pad / 4 + i];
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int BW, int BH, int MODE>
int run(int n, int x0, int y0) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<EncodeTiledFn>(p);
  std::vector<float> h(n * n);
  for (int i = 0; i < n * n; ++i) h[i] = i + 1;
  float *d, *o;
  cudaMalloc(&d, n * n * 4);
  cudaMalloc(&o, BW * BH * 4);
  cudaMemcpy(d, h.data(), n * n * 4, cudaMemcpyHostToDevice);
  CUtensorMap m{};
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, 1};
  cuuint64_t str[2] = {(cuuint64_t)n * 4, (cuuint64_t)n * n * 4};
  cuuint32_t box[3] = {BW, BH, 1}, es[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("n=%d box=%dx%d mode=%d at (%d,%d): encode=%d ", n, BW, BH, MODE, x0, y0, (int)r);
  size_t smem = BW * BH * 4 + 128;
  cudaFuncSetAttribute(probe<BW, BH, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<BW, BH, MODE><<<1, 128, smem>>>(o, m, x0, y0);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> ho(BW * BH);
  cudaMemcpy(ho.data(), o, BW * BH * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int yy = 0; yy < BH; ++yy)
    for (int xx = 0; xx < BW; ++xx) {
      int gx = x0 + xx, gy = y0 + yy;
      float want = (gx >= 0 && gx < n && gy >= 0 && gy < n) ? h[gy * n + gx] : 0.f;
      bad += ho[yy * BW + xx] != want;
    }
  printf("err=%s bad=%d\n", cudaGetErrorString(e), bad);
  cudaFree(d);
  cudaFree(o);
  return e != cudaSuccess;
}

int main(int argc, char** argv) {
  int v = argc > 1 ? atoi(argv[1]) : 0;
  switch (v) {
    case 0: return run<132, 36, 0>(512, -2, -2);
    case 1: return run<32, 8, 0>(512, 0, 0);
    case 2: return run<32, 8, 0>(512, -2, -2);
    case 3: return run<128, 32, 0>(512, 0, 0);
    case 4: return run<132, 36, 0>(512, 0, 0);
    case 5: return run<64, 16, 0>(512, 0, 0);
    case 6: return run<16, 4, 0>(512, 0, 0);
    case 7: return run<256, 2, 0>(512, 0, 0);
    case 8: return run<132, 36, 0>(512, 400, 490);
    case 9: return run<132, 36, 0>(200, 126, 30);
    case 10: return run<132, 36, 0>(200, 126, 190);
    case 11: return run<132, 36, 0>(512, 382, 0);
    case 12: return run<132, 36, 0>(512, 0, 478);
    case 13: return run<128, 32, 0>(512, 400, 0);
  }
  return 0;
}
