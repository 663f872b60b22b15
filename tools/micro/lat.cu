// Microbenchmark: dependent-chain latencies of FP64 ops and LDS on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  sm[threadIdx.x & 63] = a;
  __syncthreads();
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + y; x = x + y; x = x + y; x = x + y; }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { x = __fma_rn(x, y, a); x = __fma_rn(x, y, a); x = __fma_rn(x, y, a); x = __fma_rn(x, y, a); }
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  long long t3 = clock64();
  int idx = (int)x & 63;
  for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = ((int)v + i) & 63; x += v; }
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) { x = x / (y + i); }
  long long t5 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
  int n = 1000;
  k<<<1, 32>>>(o, c, 1.0000001, 1e-9, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0000001, 1e-9, n); cudaDeviceSynchronize();
  printf("DADD dep latency %.1f clk\n", c[0] / (4.0 * n));
  printf("DFMA dep latency %.1f clk\n", c[1] / (4.0 * n));
  printf("RCP64 dep latency %.1f clk\n", c[2] / (1.0 * n));
  printf("LDS+F2I+DADD chain %.1f clk\n", c[3] / (1.0 * n));
  printf("DDIV dep latency %.1f clk\n", c[4] / (1.0 * n));
  return 0;
}
