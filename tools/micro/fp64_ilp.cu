// Microbenchmark: FP64 issue rate of ONE warp with k independent DADD chains
// (and of 1..4 warps per SM partition), no FMA.
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void k(double* out, long long* cyc, double a, int n) {
  double x[K];
#pragma unroll
  for (int i = 0; i < K; ++i) x[i] = a + i;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = __dadd_rn(x[i], a);
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = __dmul_rn(x[i], a);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int K>
void run(int warps) {
  double* o; long long* c;
  cudaMalloc(&o, 1 << 20); cudaMallocManaged(&c, 1024);
  int n = 2000;
  k<K><<<1, 32 * warps>>>(o, c, 1.0000001, n); cudaDeviceSynchronize();
  k<K><<<1, 32 * warps>>>(o, c, 1.0000001, n); cudaDeviceSynchronize();
  double per = (double)c[0] / (2.0 * K * n);
  printf("chains=%d warps=%d: %.2f cycles per warp-DP-instruction (per warp), %.2f per SM\n", K, warps, per, per / warps);
  cudaFree(o); cudaFree(c);
}
int main() {
  for (int w : {1, 2, 4, 8}) { run<1>(w); run<4>(w); run<8>(w); run<16>(w); }
  return 0;
}
