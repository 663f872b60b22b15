// upsample.cu — upsample_flow (core.py:178-190) by the factor 2:
//   out(x, y) = 2 * bilinear_map(flow, x / 2, y / 2)  (numpy bilinear form)
// applied level by level (_upscale_to_full, pipeline.py:129-133), plus the
// planar -> (H, W, 2) interleave of the final field.  HBM-bound gathers.
#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

__global__ void __launch_bounds__(256) k_upsample(const double* __restrict__ iu,
                                                  const double* __restrict__ iv, int B, int W,
                                                  int H, double* __restrict__ ou,
                                                  double* __restrict__ ov,
                                                  double* __restrict__ oi, int Wn, int Hn) {
  const size_t nplane = (size_t)Wn * Hn;
  const size_t n = (size_t)B * nplane;
  const size_t plane = (size_t)W * H;
  for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(g / nplane);
    const size_t p = g - (size_t)b * nplane;
    const int y = (int)(p / Wn);
    const int x = (int)(p - (size_t)y * Wn);
    const double xs = (double)x / 2.0;
    const double ys = (double)y / 2.0;
    const double u = bilin_np(iu + b * plane, W, H, xs, ys) * 2.0;
    const double v = bilin_np(iv + b * plane, W, H, xs, ys) * 2.0;
    if (oi) {
      reinterpret_cast<double2*>(oi)[g] = make_double2(u, v);
    } else {
      ou[g] = u;
      ov[g] = v;
    }
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
                     double* ov, double* out_interleaved, int Wn, int Hn, cudaStream_t st) {
  const size_t n = (size_t)B * Wn * Hn;
  prof_begin(KC_UPSAMPLE, st);
  k_upsample<<<blocks_for(n), 256, 0, st>>>(iu, iv, B, W, H, ou, ov, out_interleaved, Wn, Hn);
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

}  // namespace disb200
