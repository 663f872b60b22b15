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

// FP64 roofline denominator: 8 independent chains per thread of DADD (or
// DMUL), no FMA (the exact-parity kernels never contract).  The constants
// keep every value finite and normal.
template <bool MUL>
__global__ void __launch_bounds__(256) k_fp64_peak(double* out, int n, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = a + (double)(threadIdx.x + i);
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = MUL ? x[i] * b : x[i] + b;
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // never true; keeps the chains live
}

}  // namespace disb200

extern "C" DIS_API int dis_selftest_fp64_peak(double* dadd_gops, double* dmul_gops,
                                              void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return DIS_ERR_CUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, th = 256, n = 4096;
  const double ops = (double)blocks * th * n * 8;
  double best[2] = {0.0, 0.0};
  for (int rep = 0; rep < 4; ++rep) {
    for (int m = 0; m < 2; ++m) {
      cudaEventRecord(e0, st);
      if (m)
        disb200::k_fp64_peak<true><<<blocks, th, 0, st>>>(out, n, 1.0, 1.0000000001);
      else
        disb200::k_fp64_peak<false><<<blocks, th, 0, st>>>(out, n, 1.0, 1e-9);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double g = ops / (ms * 1e-3) / 1e9;
      if (rep > 0 && g > best[m]) best[m] = g;  // rep 0 warms up
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  *dadd_gops = best[0];
  *dmul_gops = best[1];
  return cudaGetLastError() == cudaSuccess ? DIS_OK : DIS_ERR_CUDA;
}

extern "C" DIS_API int dis_selftest_div(const double* n, const double* d, double* fast,
                                        double* ieee, size_t count, void* stream) {
  disb200::k_selftest_div<<<148 * 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, d, fast, ieee, count);
  return cudaGetLastError() == cudaSuccess ? DIS_OK : DIS_ERR_CUDA;
}
