// Explicit sparse projector (SparseMap, sparse.cpp:55-71) on the device:
// y = A x with the CSR rows, A^T u with the stored transpose -- both gathers,
// one warp per output row, lanes striding the row's entries and a fixed-order
// shuffle reduction (deterministic, no atomics).  HBM-bound: each nonzero
// moves 8 B (fp32 value + int32 index) plus the gathered operand, which the
// 126 MB L2 mostly serves.
#include <cuda_runtime.h>

#include <algorithm>

#include "ncsg_internal.cuh"

namespace ncsg {

namespace {

__global__ void csr_spmv_kernel(const int64_t* __restrict__ row_ptr, const int* __restrict__ col,
                                const float* __restrict__ val, const float* __restrict__ x,
                                size_t x_stride, float* __restrict__ y, size_t y_stride,
                                size_t rows) {
  const int b = blockIdx.y;
  const float* xb = x + b * x_stride;
  float* yb = y + b * y_stride;
  const int lane = threadIdx.x & 31;
  const size_t warps = static_cast<size_t>(gridDim.x) * (blockDim.x >> 5);
  for (size_t r = blockIdx.x * static_cast<size_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
       r < rows; r += warps) {
    const int64_t e0 = row_ptr[r], e1 = row_ptr[r + 1];
    float acc = 0.f;
    for (int64_t i = e0 + lane; i < e1; i += 32) acc = fmaf(__ldg(val + i), __ldg(xb + __ldg(col + i)), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) yb[r] = acc;
  }
}

}  // namespace

void SparseDev::upload(const SparseHost& h) {
  n = h.n;
  views = h.views;
  rays = h.rays;
  rows = static_cast<size_t>(h.views) * h.rays;
  cols = static_cast<size_t>(h.n) * h.n;
  nnz = h.val.size();
  std::vector<float> v(h.val.begin(), h.val.end()), tv(h.t_val.begin(), h.t_val.end());
  row_ptr.alloc(h.row_ptr.size());
  t_row_ptr.alloc(h.t_row_ptr.size());
  col.alloc(std::max<size_t>(1, nnz));
  t_col.alloc(std::max<size_t>(1, nnz));
  val.alloc(std::max<size_t>(1, nnz));
  t_val.alloc(std::max<size_t>(1, nnz));
  NCSG_CUDA_CHECK(cudaMemcpy(row_ptr.p, h.row_ptr.data(), h.row_ptr.size() * 8, cudaMemcpyHostToDevice));
  NCSG_CUDA_CHECK(cudaMemcpy(t_row_ptr.p, h.t_row_ptr.data(), h.t_row_ptr.size() * 8,
                             cudaMemcpyHostToDevice));
  if (nnz) {
    NCSG_CUDA_CHECK(cudaMemcpy(col.p, h.col.data(), nnz * 4, cudaMemcpyHostToDevice));
    NCSG_CUDA_CHECK(cudaMemcpy(t_col.p, h.t_col.data(), nnz * 4, cudaMemcpyHostToDevice));
    NCSG_CUDA_CHECK(cudaMemcpy(val.p, v.data(), nnz * 4, cudaMemcpyHostToDevice));
    NCSG_CUDA_CHECK(cudaMemcpy(t_val.p, tv.data(), nnz * 4, cudaMemcpyHostToDevice));
  }
}

void launch_sparse_forward(const SparseDev& A, const float* x, size_t x_stride, float* y,
                           size_t y_stride, int batch, cudaStream_t s) {
  const int per = 256 / 32;
  const int blocks = static_cast<int>(std::min<size_t>((A.rows + per - 1) / per, 148 * 16));
  csr_spmv_kernel<<<dim3(std::max(1, blocks), batch), 256, 0, s>>>(
      A.row_ptr.p, A.col.p, A.val.p, x, x_stride, y, y_stride, A.rows);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_sparse_adjoint(const SparseDev& A, const float* u, size_t u_stride, float* y,
                           size_t y_stride, int batch, cudaStream_t s) {
  const int per = 256 / 32;
  const int blocks = static_cast<int>(std::min<size_t>((A.cols + per - 1) / per, 148 * 16));
  csr_spmv_kernel<<<dim3(std::max(1, blocks), batch), 256, 0, s>>>(
      A.t_row_ptr.p, A.t_col.p, A.t_val.p, u, u_stride, y, y_stride, A.cols);
  NCSG_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

}  // namespace ncsg
