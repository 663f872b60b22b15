// upsample.cu — upsample_flow (core.py:178-190) by the pyramid factor k
// (DisParams.downscale, 2 on the benchmark configs):
//   out(x, y) = k * bilinear_map(flow, x / k, y / k)  (numpy bilinear form)
// applied level by level (_upscale_to_full, pipeline.py:129-133), plus the
// planar -> (H, W, 2) interleave of the final field.  HBM-bound gathers.
#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

// bilinear_map (core.py:154-170) of u and v at output pixel (x, y): one
// clamp/floor/fraction setup, then the numpy formula for each component
__device__ __forceinline__ void upsample_px(const double* __restrict__ U,
                                            const double* __restrict__ V, int W, int H, int x,
                                            int y, double k, double& u, double& v) {
  double xs = (double)x / k;
  double ys = (double)y / k;
  xs = xs > W - 1.0 ? W - 1.0 : xs;
  ys = ys > H - 1.0 ? H - 1.0 : ys;
  const int x0 = (int)xs, y0 = (int)ys;  // xs, ys >= 0: floor
  const int x1 = x0 + 1 < W - 1 ? x0 + 1 : W - 1;
  const int y1 = y0 + 1 < H - 1 ? y0 + 1 : H - 1;
  const double fx = xs - (double)x0, fy = ys - (double)y0;
  const double gx = 1.0 - fx, gy = 1.0 - fy;
  const size_t r0 = (size_t)y0 * W, r1 = (size_t)y1 * W;
  const double ut = __ldg(U + r0 + x0) * gx + __ldg(U + r0 + x1) * fx;
  const double ub = __ldg(U + r1 + x0) * gx + __ldg(U + r1 + x1) * fx;
  const double vt = __ldg(V + r0 + x0) * gx + __ldg(V + r0 + x1) * fx;
  const double vb = __ldg(V + r1 + x0) * gx + __ldg(V + r1 + x1) * fx;
  u = (ut * gy + ub * fy) * k;
  v = (vt * gy + vb * fy) * k;
}

// Two horizontally adjacent output pixels per thread (x = 2i, 2i + 1 share
// their source columns through L1); the interleaved final field is written
// as one 32-byte streaming store per thread.  KC = the factor at compile
// time (2: x / 2.0 is the exact multiplication by 0.5; a runtime factor
// costs an IEEE division per coordinate), 0 = the runtime factor kr.
template <int KC>
__global__ void __launch_bounds__(256) k_upsample(const double* __restrict__ iu,
                                                  const double* __restrict__ iv, int W, int H,
                                                  double* __restrict__ ou,
                                                  double* __restrict__ ov,
                                                  double* __restrict__ oi, int Wn, int Hn,
                                                  double kr) {
  const double k = KC > 0 ? (double)KC : kr;
  const int b = blockIdx.z;
  const int x = 2 * (blockIdx.x * 32 + (threadIdx.x & 31));
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= Wn || y >= Hn) return;
  const size_t plane = (size_t)W * H;
  const double* U = iu + b * plane;
  const double* V = iv + b * plane;
  const size_t g = ((size_t)b * Hn + y) * Wn + x;
  double u0, v0;
  upsample_px(U, V, W, H, x, y, k, u0, v0);
  if (x + 1 < Wn) {
    double u1, v1;
    upsample_px(U, V, W, H, x + 1, y, k, u1, v1);
    if (oi) {
      double* d = oi + 2 * g;
      if ((reinterpret_cast<uintptr_t>(d) & 31) == 0) {  // streamed: not re-read
        asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(d), "d"(u0), "d"(v0),
                     "d"(u1), "d"(v1)
                     : "memory");
      } else {
        __stcs(reinterpret_cast<double2*>(oi) + g, make_double2(u0, v0));
        __stcs(reinterpret_cast<double2*>(oi) + g + 1, make_double2(u1, v1));
      }
    } else {
      ou[g] = u0;
      ov[g] = v0;
      ou[g + 1] = u1;
      ov[g + 1] = v1;
    }
  } else if (oi) {
    __stcs(reinterpret_cast<double2*>(oi) + g, make_double2(u0, v0));
  } else {
    ou[g] = u0;
    ov[g] = v0;
  }
}

__global__ void __launch_bounds__(256) k_interleave(const double* __restrict__ u,
                                                    const double* __restrict__ v, size_t n,
                                                    double* __restrict__ out) {
  for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (size_t)gridDim.x * blockDim.x)
    reinterpret_cast<double2*>(out)[g] = make_double2(u[g], v[g]);
}

static unsigned blocks_for(size_t n) {
  size_t b = (n + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

void launch_upsample(const double* iu, const double* iv, int B, int W, int H, double* ou,
                     double* ov, double* out_interleaved, int Wn, int Hn, int factor,
                     cudaStream_t st) {
  prof_begin(KC_UPSAMPLE, st);
  dim3 g((unsigned)((Wn + 63) / 64), (unsigned)((Hn + 7) / 8), (unsigned)B);
  if (factor == 2)
    k_upsample<2><<<g, 256, 0, st>>>(iu, iv, W, H, ou, ov, out_interleaved, Wn, Hn, 2.0);
  else
    k_upsample<0><<<g, 256, 0, st>>>(iu, iv, W, H, ou, ov, out_interleaved, Wn, Hn,
                                     (double)factor);
  prof_end(KC_UPSAMPLE, st);
  note_launch();
}

void launch_interleave(const double* u, const double* v, int B, int W, int H, double* out,
                       cudaStream_t st) {
  const size_t n = (size_t)B * W * H;
  prof_begin(KC_UPSAMPLE, st);
  k_interleave<<<blocks_for(n), 256, 0, st>>>(u, v, n, out);
  prof_end(KC_UPSAMPLE, st);
  note_launch();
}

// the flow rounded to float32 (round to nearest even, numpy's astype) for
// the host path's half-size copy-out; n doubles, n even
__global__ void __launch_bounds__(256) k_flow_to_f32(const double2* __restrict__ in,
                                                     float2* __restrict__ out, size_t n2) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
       i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = in[i];
    out[i] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
  }
}

void launch_flow_to_f32(const double* in, float* out, size_t n, cudaStream_t st) {
  prof_begin(KC_UPSAMPLE, st);
  k_flow_to_f32<<<blocks_for(n / 2), 256, 0, st>>>(reinterpret_cast<const double2*>(in),
                                                    reinterpret_cast<float2*>(out), n / 2);
  prof_end(KC_UPSAMPLE, st);
  note_launch();
}

}  // namespace disb200
