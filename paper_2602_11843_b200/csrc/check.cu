// check.cu -- NSERIES_CHECK_FINITE for the paths without a fused count (the tiled fp64 engine
// and the warp-group batched kernel count in their final epilogue): one grid-stride pass over
// S that counts NaN / Inf entries into a device counter.  Matrices of a batch at S + b*stride
// (or S_ptrs[b]), rows x d row-major (rows = d, or a row block of the sharded chain).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.h"

namespace nseries {
namespace {

template <typename T>
__global__ void count_nonfinite_kernel(const T* __restrict__ S, int64_t stride, const T* const* __restrict__ S_ptrs,
                                       int batch, int64_t per, int* __restrict__ count) {
  const int64_t n = per * batch;
  int c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / per, e = i % per;
    const T v = S_ptrs ? S_ptrs[b][e] : S[b * stride + e];
    c += isfinite(v) ? 0 : 1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

}  // namespace

int launch_count_nonfinite(nseries_dtype dt, const void* S, int64_t stride, const void* const* S_ptrs, int batch,
                           int rows, int d, int* count, void* stream) {
  const int64_t per = (int64_t)rows * d, n = per * batch;
  if (n == 0) return 0;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dt == NSERIES_F64)
    count_nonfinite_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(S), stride,
                                                          reinterpret_cast<const double* const*>(S_ptrs), batch, per, count);
  else
    count_nonfinite_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(S), stride,
                                                         reinterpret_cast<const float* const*>(S_ptrs), batch, per, count);
  return (int)cudaGetLastError();
}

}  // namespace nseries
