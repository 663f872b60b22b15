// selftest.cu — device self-tests of the exact-arithmetic helpers (test hook,
// not part of the reference interface): exact_div_pos against IEEE `/`.
#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

__global__ void k_selftest_div(const double* __restrict__ n, const double* __restrict__ d,
                               double* __restrict__ fast, double* __restrict__ ieee, size_t count) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    fast[i] = exact_div_pos(n[i], d[i]);
    double ns = n[i];
    asm("mov.b64 %0, %0;" : "+d"(ns));
    ieee[i] = ns / d[i];
  }
}

}  // namespace disb200

extern "C" DIS_API int dis_selftest_div(const double* n, const double* d, double* fast,
                                        double* ieee, size_t count, void* stream) {
  disb200::k_selftest_div<<<148 * 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, d, fast, ieee, count);
  return cudaGetLastError() == cudaSuccess ? DIS_OK : DIS_ERR_CUDA;
}
