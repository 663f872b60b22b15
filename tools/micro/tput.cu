// Microbenchmark: FP64 / FP32 / INT throughput per SM (many warps, independent chains).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void k(T* out, int n, T a, T b) {
  T x0 = a + threadIdx.x, x1 = a * 2, x2 = a * 3, x3 = a * 4, x4 = b, x5 = b * 2, x6 = b * 3, x7 = b * 4;
  for (int i = 0; i < n; ++i) {
    x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
    x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void kadd(double* out, int n, double a, double b) {
  double x0 = a + threadIdx.x, x1 = a * 2, x2 = a * 3, x3 = a * 4, x4 = b, x5 = b * 2, x6 = b * 3, x7 = b * 4;
  for (int i = 0; i < n; ++i) {
    x0 = x0 + b; x1 = x1 + b; x2 = x2 + b; x3 = x3 + b; x4 = x4 + a; x5 = x5 + a; x6 = x6 + a; x7 = x7 + a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* od; float* of; cudaMalloc(&od, 1 << 26); cudaMalloc(&of, 1 << 26);
  int n = 20000, blocks = sms * 4, th = 256;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k<double><<<blocks, th>>>(od, n, 0.999999, 1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * th * n * 8;
    printf("DFMA: %.2f Tops/s = %.1f per SM per clk (clk %d MHz)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    cudaEventRecord(e0); kadd<<<blocks, th>>>(od, n, 0.999999, 1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DADD: %.2f Tops/s = %.1f per SM per clk\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
    cudaEventRecord(e0); k<float><<<blocks, th>>>(of, n, 0.999999f, 1e-7f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA: %.2f Tops/s = %.1f per SM per clk\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
  }
  return 0;
}
