// compose.cu — compose_flows (pipeline.py:186-199), the frame-chaining
// operator: out(x) = ab(x) + bc(x + ab(x)), bc sampled with the numpy
// bilinear_map formula (core.py:154-170).  One thread per pixel; the fields
// are interleaved (H, W, 2) float64 like the reference's arrays, so each
// pixel reads ab as one 16-byte load and each bilinear corner of bc as one
// 16-byte load carrying both components.  HBM-bound: 16 B (ab) + 16 B (out)
// per pixel streamed, the bc gather mostly hits L1/L2 for smooth ab.
#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

__global__ void __launch_bounds__(256) k_compose(const double2* __restrict__ ab,
                                                 const double2* __restrict__ bc, int W, int H,
                                                 double2* __restrict__ out) {
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= W || y >= H) return;
  const size_t plane = (size_t)W * H;
  const size_t g = (size_t)b * plane + (size_t)y * W + x;
  const double2 f = __ldcs(ab + g);
  // px = gx + ab_u, py = gy + ab_v (pipeline.py:194-195); bilinear_map's
  // np.clip / np.floor / x1 = min(x0 + 1, w - 1) (core.py:159-166); a NaN
  // coordinate is mapped to 0 (bilin_np)
  double px = (double)x + f.x;
  double py = (double)y + f.y;
  px = !(px >= 0.0) ? 0.0 : px;
  px = px > W - 1.0 ? W - 1.0 : px;
  py = !(py >= 0.0) ? 0.0 : py;
  py = py > H - 1.0 ? H - 1.0 : py;
  const int x0 = (int)floor(px), y0 = (int)floor(py);
  const int x1 = x0 + 1 < W - 1 ? x0 + 1 : W - 1;
  const int y1 = y0 + 1 < H - 1 ? y0 + 1 : H - 1;
  const double fx = px - (double)x0, fy = py - (double)y0;
  const double gx = 1.0 - fx, gy = 1.0 - fy;
  const double2* B = bc + (size_t)b * plane;
  const double2 i00 = __ldg(B + (size_t)y0 * W + x0), i01 = __ldg(B + (size_t)y0 * W + x1);
  const double2 i10 = __ldg(B + (size_t)y1 * W + x0), i11 = __ldg(B + (size_t)y1 * W + x1);
  // top = img[y0,x0]*(1-fx) + img[y0,x1]*fx; bot = ...; top*(1-fy) + bot*fy
  const double tu = i00.x * gx + i01.x * fx, bu = i10.x * gx + i11.x * fx;
  const double tv = i00.y * gx + i01.y * fx, bv = i10.y * gx + i11.y * fx;
  __stcs(out + g, make_double2(f.x + (tu * gy + bu * fy), f.y + (tv * gy + bv * fy)));
}

void launch_compose(const double* ab, const double* bc, int B, int H, int W, double* out,
                    cudaStream_t st) {
  prof_begin(KC_UPSAMPLE, st);
  dim3 g((unsigned)((W + 31) / 32), (unsigned)((H + 7) / 8), (unsigned)B);
  k_compose<<<g, 256, 0, st>>>(reinterpret_cast<const double2*>(ab),
                               reinterpret_cast<const double2*>(bc), W, H,
                               reinterpret_cast<double2*>(out));
  prof_end(KC_UPSAMPLE, st);
  note_launch();
}

}  // namespace disb200
