// pyramid.cu — image pyramid + gradient rasters (reference core.py:65-128,
// variational.py:168-171).
//
//   level 0     = the frame converted to float64 (as_image, core.py:65-72)
//   level s > 0 = 2x2 box mean of level s-1, ((a+b)+(c+d))/4, dims floored
//                 (_box_downsample, core.py:88-98)
//   gx, gy      = central differences [-0.5, 0, 0.5] with one-sided borders
//                 (image_gradients, core.py:75-85), only at the levels the
//                 flow path reads (finest..coarsest; Appendix A.9: the
//                 reference computes the others but never reads them)
//   dd          = gradients of gx and gy (gxx, gxy, gyx, gyy) for the
//                 variational stage (_second_derivatives,
//                 variational.py:168-171), evaluated from the image with the
//                 same border rules, so they are bit-identical.
//
// All rasters row-major float64; HBM-bound elementwise/stencil kernels, one
// thread per output pixel, rows read coalesced.
#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

template <typename T>
__device__ __forceinline__ double to_f64(T v) {
  return (double)v;
}

__device__ __forceinline__ bool finite_f64(double v) { return isfinite(v); }

// level 0 (convert) from the frames; also the finiteness check of as_image
template <typename T>
__global__ void k_level0(const T* __restrict__ frames, int B, int H, int W,
                         double* __restrict__ out, uint32_t* status) {
  size_t n = (size_t)B * H * W;
  bool bad = false;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    double v = to_f64(frames[i]);
    bad |= !finite_f64(v);
    if (out) out[i] = v;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) set_status(status, DIS_STATUS_NONFINITE_INPUT);
}

// level 1 straight from the frames (no float64 level-0 copy needed when the
// finest scale is >= 1): ((a+b)+(c+d))/4 of the converted pixels
template <typename T>
__global__ void k_level1_from_frames(const T* __restrict__ frames, int B, int H, int W,
                                     double* __restrict__ out) {
  int Ho = H / 2, Wo = W / 2;
  size_t n = (size_t)B * Ho * Wo;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    int X = (int)(i % Wo);
    size_t t = i / Wo;
    int Y = (int)(t % Ho);
    int b = (int)(t / Ho);
    const T* r0 = frames + ((size_t)b * H + 2 * Y) * W + 2 * X;
    const T* r1 = r0 + W;
    double a = to_f64(r0[0]), bb = to_f64(r0[1]), c = to_f64(r1[0]), d = to_f64(r1[1]);
    out[i] = ((a + bb) + (c + d)) / 4.0;
  }
}

// level s from level s-1 (both float64 row-major)
// two output pixels per thread: each input row pair read as one 32-byte
// load per row when aligned, the outputs as one 16-byte store
__global__ void k_downsample(const double* __restrict__ in, int B, int H, int W,
                             double* __restrict__ out) {
  const int Ho = H / 2, Wo = W / 2;
  const int Wp = (Wo + 1) / 2;  // output pairs per row
  const size_t n = (size_t)B * Ho * Wp;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int Xp = (int)(i % Wp);
    const size_t t = i / Wp;
    const int Y = (int)(t % Ho);
    const int b = (int)(t / Ho);
    const int X = 2 * Xp;
    const double* r0 = in + ((size_t)b * H + 2 * Y) * W + 2 * X;
    const double* r1 = r0 + W;
    const size_t o = ((size_t)b * Ho + Y) * Wo + X;
    if (X + 1 < Wo) {
      double a[4], c[4];
      if (((reinterpret_cast<uintptr_t>(r0) | reinterpret_cast<uintptr_t>(r1)) & 31) == 0) {
        asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
            : "=d"(a[0]), "=d"(a[1]), "=d"(a[2]), "=d"(a[3]) : "l"(r0));
        asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
            : "=d"(c[0]), "=d"(c[1]), "=d"(c[2]), "=d"(c[3]) : "l"(r1));
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q] = r0[q];
          c[q] = r1[q];
        }
      }
      const double o0 = ((a[0] + a[1]) + (c[0] + c[1])) / 4.0;
      const double o1 = ((a[2] + a[3]) + (c[2] + c[3])) / 4.0;
      if ((o & 1) == 0) {
        *reinterpret_cast<double2*>(out + o) = make_double2(o0, o1);
      } else {
        out[o] = o0;
        out[o + 1] = o1;
      }
    } else {
      const double a = r0[0], bb = r0[1], c = r1[0], d = r1[1];
      out[o] = ((a + bb) + (c + d)) / 4.0;
    }
  }
}

// gradient of a raster along x / y with the reference's border rules
struct RowGrad {
  const double* img;
  int W, H;
  __device__ __forceinline__ double v(int x, int y) const { return img[(size_t)y * W + x]; }
  __device__ __forceinline__ double gx(int x, int y) const {
    if (x == 0) return 0.5 * (v(1, y) - v(0, y));
    if (x == W - 1) return 0.5 * (v(W - 1, y) - v(W - 2, y));
    return 0.5 * (v(x + 1, y) - v(x - 1, y));
  }
  __device__ __forceinline__ double gy(int x, int y) const {
    if (y == 0) return 0.5 * (v(x, 1) - v(x, 0));
    if (y == H - 1) return 0.5 * (v(x, H - 1) - v(x, H - 2));
    return 0.5 * (v(x, y + 1) - v(x, y - 1));
  }
  // x-gradient of gx, y-gradient of gx, x-gradient of gy, y-gradient of gy
  __device__ __forceinline__ double gxx(int x, int y) const {
    if (x == 0) return 0.5 * (gx(1, y) - gx(0, y));
    if (x == W - 1) return 0.5 * (gx(W - 1, y) - gx(W - 2, y));
    return 0.5 * (gx(x + 1, y) - gx(x - 1, y));
  }
  __device__ __forceinline__ double gxy(int x, int y) const {
    if (y == 0) return 0.5 * (gx(x, 1) - gx(x, 0));
    if (y == H - 1) return 0.5 * (gx(x, H - 1) - gx(x, H - 2));
    return 0.5 * (gx(x, y + 1) - gx(x, y - 1));
  }
  __device__ __forceinline__ double gyx(int x, int y) const {
    if (x == 0) return 0.5 * (gy(1, y) - gy(0, y));
    if (x == W - 1) return 0.5 * (gy(W - 1, y) - gy(W - 2, y));
    return 0.5 * (gy(x + 1, y) - gy(x - 1, y));
  }
  __device__ __forceinline__ double gyy(int x, int y) const {
    if (y == 0) return 0.5 * (gy(x, 1) - gy(x, 0));
    if (y == H - 1) return 0.5 * (gy(x, H - 1) - gy(x, H - 2));
    return 0.5 * (gy(x, y + 1) - gy(x, y - 1));
  }
};

__global__ void k_gradients(const double* __restrict__ img, int B, int H, int W,
                            double* __restrict__ gx, double* __restrict__ gy,
                            double* __restrict__ dd) {
  size_t plane = (size_t)H * W;
  size_t n = (size_t)B * plane;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    int b = (int)(i / plane);
    size_t p = i - (size_t)b * plane;
    int y = (int)(p / W);
    int x = (int)(p - (size_t)y * W);
    RowGrad g{img + (size_t)b * plane, W, H};
    if (gx) gx[i] = g.gx(x, y);
    if (gy) gy[i] = g.gy(x, y);
    if (dd) {
      double* d = dd + (size_t)b * 4 * plane + p;
      d[0] = g.gxx(x, y);
      d[plane] = g.gxy(x, y);
      d[2 * plane] = g.gyx(x, y);
      d[3 * plane] = g.gyy(x, y);
    }
  }
}

// Tiled gradients: a 32 x 16 output tile per block.  The level image is
// read once (tile + 2-pixel halo) into shared memory, gx / gy are evaluated
// once for the tile + 1-pixel halo, the second derivatives come from those;
// all outputs are written coalesced.  Identical arithmetic to RowGrad (the
// border rules use global coordinates; halo cells outside the level are
// never read for an in-level output).
constexpr int kGTX = 32, kGTY = 16;
__global__ void __launch_bounds__(256) k_gradients_tile(const double* __restrict__ img_all, int H,
                                                        int W, double* __restrict__ gx_all,
                                                        double* __restrict__ gy_all,
                                                        double* __restrict__ dd_all) {
  __shared__ double I[kGTY + 4][kGTX + 4];
  __shared__ double GX[kGTY + 2][kGTX + 2];
  __shared__ double GY[kGTY + 2][kGTX + 2];
  const int b = blockIdx.z;
  const int X0 = blockIdx.x * kGTX, Y0 = blockIdx.y * kGTY;
  const size_t plane = (size_t)W * H;
  const double* img = img_all + b * plane;
  const int tid = threadIdx.x;
  for (int i = tid; i < (kGTY + 4) * (kGTX + 4); i += 256) {
    const int ly = i / (kGTX + 4), lx = i - ly * (kGTX + 4);
    int gy = Y0 - 2 + ly, gx = X0 - 2 + lx;
    gy = gy < 0 ? 0 : (gy > H - 1 ? H - 1 : gy);
    gx = gx < 0 ? 0 : (gx > W - 1 ? W - 1 : gx);
    I[ly][lx] = __ldg(img + (size_t)gy * W + gx);
  }
  __syncthreads();
  // gx, gy on the tile + 1 halo (local (ly, lx) <-> image (Y0-1+ly, X0-1+lx))
  for (int i = tid; i < (kGTY + 2) * (kGTX + 2); i += 256) {
    const int ly = i / (kGTX + 2), lx = i - ly * (kGTX + 2);
    const int y = Y0 - 1 + ly, x = X0 - 1 + lx;
    const int cy = ly + 1, cx = lx + 1;  // in I
    double g;
    if (x <= 0)
      g = 0.5 * (I[cy][cx + 1] - I[cy][cx]);
    else if (x >= W - 1)
      g = 0.5 * (I[cy][cx] - I[cy][cx - 1]);
    else
      g = 0.5 * (I[cy][cx + 1] - I[cy][cx - 1]);
    GX[ly][lx] = g;
    if (y <= 0)
      g = 0.5 * (I[cy + 1][cx] - I[cy][cx]);
    else if (y >= H - 1)
      g = 0.5 * (I[cy][cx] - I[cy - 1][cx]);
    else
      g = 0.5 * (I[cy + 1][cx] - I[cy - 1][cx]);
    GY[ly][lx] = g;
  }
  __syncthreads();
  for (int i = tid; i < kGTY * kGTX; i += 256) {
    const int ly = i / kGTX, lx = i - ly * kGTX;
    const int y = Y0 + ly, x = X0 + lx;
    if (y >= H || x >= W) continue;
    const int cy = ly + 1, cx = lx + 1;  // in GX / GY
    const size_t o = b * plane + (size_t)y * W + x;
    if (gx_all) gx_all[o] = GX[cy][cx];
    if (gy_all) gy_all[o] = GY[cy][cx];
    if (dd_all) {
      double gxx, gxy, gyx, gyy;
      if (x == 0) {
        gxx = 0.5 * (GX[cy][cx + 1] - GX[cy][cx]);
        gyx = 0.5 * (GY[cy][cx + 1] - GY[cy][cx]);
      } else if (x == W - 1) {
        gxx = 0.5 * (GX[cy][cx] - GX[cy][cx - 1]);
        gyx = 0.5 * (GY[cy][cx] - GY[cy][cx - 1]);
      } else {
        gxx = 0.5 * (GX[cy][cx + 1] - GX[cy][cx - 1]);
        gyx = 0.5 * (GY[cy][cx + 1] - GY[cy][cx - 1]);
      }
      if (y == 0) {
        gxy = 0.5 * (GX[cy + 1][cx] - GX[cy][cx]);
        gyy = 0.5 * (GY[cy + 1][cx] - GY[cy][cx]);
      } else if (y == H - 1) {
        gxy = 0.5 * (GX[cy][cx] - GX[cy - 1][cx]);
        gyy = 0.5 * (GY[cy][cx] - GY[cy - 1][cx]);
      } else {
        gxy = 0.5 * (GX[cy + 1][cx] - GX[cy - 1][cx]);
        gyy = 0.5 * (GY[cy + 1][cx] - GY[cy - 1][cx]);
      }
      double* d = dd_all + b * 4 * plane + (size_t)y * W + x;
      d[0] = gxx;
      d[plane] = gxy;
      d[2 * plane] = gyx;
      d[3 * plane] = gyy;
    }
  }
}

// gx / gy only (no second derivatives): two horizontally adjacent pixels per
// thread, the image_gradients stencil (core.py:75-85) read straight from the
// level (rows coalesced, the vertical neighbours hit L1/L2), gx and gy
// written as 16-byte stores when the pair is 16-byte aligned
__global__ void __launch_bounds__(256) k_gradients_xy(const double* __restrict__ img_all, int H,
                                                      int W, double* __restrict__ gx_all,
                                                      double* __restrict__ gy_all) {
  const int b = blockIdx.z;
  const int x = 2 * (blockIdx.x * 32 + (threadIdx.x & 31));
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= W || y >= H) return;
  const size_t plane = (size_t)W * H;
  const double* row = img_all + b * plane + (size_t)y * W;
  const double* up = img_all + b * plane + (size_t)(y > 0 ? y - 1 : 0) * W;
  const double* dn = img_all + b * plane + (size_t)(y < H - 1 ? y + 1 : H - 1) * W;
  const size_t o = b * plane + (size_t)y * W + x;
  // clamped indices = the one-sided border forms (x = 0: f[1] - f[0], ...)
  auto gxv = [&](int xx) {
    const int xm = xx > 0 ? xx - 1 : 0, xp = xx < W - 1 ? xx + 1 : W - 1;
    return 0.5 * (__ldg(row + xp) - __ldg(row + xm));
  };
  auto gyv = [&](int xx) { return 0.5 * (__ldg(dn + xx) - __ldg(up + xx)); };
  if (x + 1 < W && (o & 1) == 0) {
    if (gx_all)
      *reinterpret_cast<double2*>(gx_all + o) = make_double2(gxv(x), gxv(x + 1));
    if (gy_all)
      *reinterpret_cast<double2*>(gy_all + o) = make_double2(gyv(x), gyv(x + 1));
  } else {
    for (int q = 0; q < 2 && x + q < W; ++q) {
      if (gx_all) gx_all[o + q] = gxv(x + q);
      if (gy_all) gy_all[o + q] = gyv(x + q);
    }
  }
}

// level 1 straight from the frames + the finiteness check of every input
// pixel (as_image, core.py:65-72), one pass over the frames; two output
// pixels (four input columns) per thread, 16-byte output stores
template <typename T>
__device__ __forceinline__ void load4(const T* p, double* v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) v[q] = to_f64(p[q]);
}
template <>
__device__ __forceinline__ void load4<float>(const float* p, double* v) {
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = f.x;
    v[1] = f.y;
    v[2] = f.z;
    v[3] = f.w;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = (double)p[q];
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_level1_checked(const T* __restrict__ frames, int H,
                                                        int W, double* __restrict__ out,
                                                        uint32_t* status) {
  const int Ho = H / 2, Wo = W / 2;
  const int b = blockIdx.z;
  const int X = 2 * (blockIdx.x * 32 + (threadIdx.x & 31));  // first of my two outputs
  const int Y = blockIdx.y * 8 + (threadIdx.x >> 5);
  bool bad = false;
  if (X < Wo && Y < Ho) {
    const T* r0 = frames + ((size_t)b * H + 2 * Y) * W + 2 * X;
    const T* r1 = r0 + W;
    const size_t o = ((size_t)b * Ho + Y) * Wo + X;
    if (X + 1 < Wo) {
      double t[4], u[4];
      load4<T>(r0, t);
      load4<T>(r1, u);
      bad = !(isfinite(t[0]) && isfinite(t[1]) && isfinite(t[2]) && isfinite(t[3]) &&
              isfinite(u[0]) && isfinite(u[1]) && isfinite(u[2]) && isfinite(u[3]));
      const double o0 = ((t[0] + t[1]) + (u[0] + u[1])) / 4.0;
      const double o1 = ((t[2] + t[3]) + (u[2] + u[3])) / 4.0;
      if ((o & 1) == 0) {
        *reinterpret_cast<double2*>(out + o) = make_double2(o0, o1);
      } else {
        out[o] = o0;
        out[o + 1] = o1;
      }
    } else {
      const double a = to_f64(r0[0]), bb = to_f64(r0[1]), c = to_f64(r1[0]), d = to_f64(r1[1]);
      bad = !(isfinite(a) && isfinite(bb) && isfinite(c) && isfinite(d));
      out[o] = ((a + bb) + (c + d)) / 4.0;
    }
  }
  // the pixels no 2x2 block covers (odd last column / row)
  const bool last_pair = X <= Wo - 1 && Wo - 1 <= X + 1;  // holds output column Wo - 1
  if ((W & 1) && last_pair && Y < H / 2) {
    bad |= !isfinite(to_f64(frames[((size_t)b * H + 2 * Y) * W + W - 1]));
    bad |= !isfinite(to_f64(frames[((size_t)b * H + 2 * Y + 1) * W + W - 1]));
  }
  if ((H & 1) && Y == Ho - 1) {
    for (int q = 0; q < 2; ++q) {
      const int Xq = X + q;
      if (Xq >= W / 2) break;
      bad |= !isfinite(to_f64(frames[((size_t)b * H + H - 1) * W + 2 * Xq]));
      bad |= !isfinite(to_f64(frames[((size_t)b * H + H - 1) * W + 2 * Xq + 1]));
      if ((W & 1) && Xq == Wo - 1) bad |= !isfinite(to_f64(frames[((size_t)b * H + H - 1) * W + W - 1]));
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) set_status(status, DIS_STATUS_NONFINITE_INPUT);
}

static inline int grid_for(size_t n, int threads) {
  size_t blocks = (n + threads - 1) / threads;
  size_t cap = 148 * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

template <typename T>
static void launch_pyramid_t(const T* frames, int B, int H, int W, int coarsest,
                             double* const* img, double* const* gx, double* const* gy,
                             double* const* dd, uint32_t* status, cudaStream_t st) {
  const int TH = 256;
  prof_begin(KC_PYRAMID, st);
  int h = H, w = W;
  if (img[0] != nullptr || coarsest == 0) {
    // level 0 stored (finest scale 0): convert + check, then box-mean chain
    const size_t n0 = (size_t)B * H * W;
    k_level0<T><<<grid_for(n0, TH), TH, 0, st>>>(frames, B, H, W, img[0], status);
    note_launch();
  }
  for (int s = 1; s <= coarsest; ++s) {
    const int ho = h / 2, wo = w / 2;
    if (s == 1 && img[0] == nullptr) {
      dim3 g((unsigned)((wo + 63) / 64), (unsigned)((ho + 7) / 8), (unsigned)B);
      k_level1_checked<T><<<g, TH, 0, st>>>(frames, H, W, img[1], status);
    } else {
      k_downsample<<<grid_for((size_t)B * ho * ((wo + 1) / 2), TH), TH, 0, st>>>(img[s - 1], B,
                                                                                 h, w, img[s]);
    }
    note_launch();
    h = ho;
    w = wo;
  }
  h = H;
  w = W;
  for (int s = 0; s <= coarsest; ++s) {
    if (gx[s] || gy[s] || (dd && dd[s])) {
      dim3 g((unsigned)((w + kGTX - 1) / kGTX), (unsigned)((h + kGTY - 1) / kGTY), (unsigned)B);
      if (dd && dd[s]) {
        k_gradients_tile<<<g, 256, 0, st>>>(img[s], h, w, gx[s], gy[s], dd[s]);
      } else {
        dim3 g2((unsigned)((w + 63) / 64), (unsigned)((h + 7) / 8), (unsigned)B);
        k_gradients_xy<<<g2, 256, 0, st>>>(img[s], h, w, gx[s], gy[s]);
      }
      note_launch();
    }
    h /= 2;
    w /= 2;
  }
  prof_end(KC_PYRAMID, st);
}

void launch_pyramid(const void* frames, int dtype, int B, int H, int W, int coarsest,
                    double* const* img, double* const* gx, double* const* gy,
                    double* const* dd, uint32_t* status, cudaStream_t st) {
  switch (dtype) {
    case DIS_DTYPE_F32:
      launch_pyramid_t((const float*)frames, B, H, W, coarsest, img, gx, gy, dd, status, st);
      break;
    case DIS_DTYPE_F64:
      launch_pyramid_t((const double*)frames, B, H, W, coarsest, img, gx, gy, dd, status, st);
      break;
    default:
      launch_pyramid_t((const uint8_t*)frames, B, H, W, coarsest, img, gx, gy, dd, status,
                       st);
      break;
  }
}

}  // namespace disb200
