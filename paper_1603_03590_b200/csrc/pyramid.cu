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

// numpy's pairwise_sum of n contiguous values (the inner loop of np.add's
// reduction, numpy/_core/src/umath/loops_utils.h.src) for n <= 128: n < 8
// sequential from 0.0; else eight strided accumulators combined
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the remainder
template <typename T>
__device__ __forceinline__ double np_pairwise_sum(const T* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += to_f64(a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = to_f64(a[j]);
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += to_f64(a[i + j]);
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += to_f64(a[i]);
  return res;
}

// _box_downsample by a factor k != 2 (core.py:88-98):
// crop.reshape(h, k, w, k).mean(axis=(1, 3)) = (sum over the k block rows,
// in order from 0, of each row's pairwise sum) / (k*k) — numpy 2.3's order,
// pinned by tests/test_downscale.py against the reference (k = 3, 4, 8, 9).
// T = the frame type for level 1 from the frames, double otherwise.
template <typename T>
__global__ void __launch_bounds__(256) k_downsample_k(const T* __restrict__ in, int B, int H,
                                                      int W, int k, double* __restrict__ out) {
  const int Ho = H / k, Wo = W / k;
  const size_t n = (size_t)B * Ho * Wo;
  const double kk = (double)k * (double)k;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int X = (int)(i % Wo);
    const size_t t = i / Wo;
    const int Y = (int)(t % Ho);
    const int b = (int)(t / Ho);
    const T* blk = in + ((size_t)b * H + (size_t)k * Y) * W + (size_t)k * X;
    double acc = 0.0;
    for (int r = 0; r < k; ++r) acc += np_pairwise_sum(blk + (size_t)r * W, k);
    out[i] = acc / kk;
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

// ---------------------------------------------------------------------------
// Fused pyramid (the flow path; no second derivatives): two launches for both
// frames of a batch instead of a convert / downsample / gradient chain per
// level and frame.
//
// k_pyr_tile: one block per kPTX x kPTY tile of the BASE level L0 (level 1
// built straight from the frames when the finest scale is >= 1, else level
// 0): the tile plus a one-pixel halo (clamped coordinates = the reference's
// one-sided borders) is formed in shared memory, the base image and its
// gradients are written, and every coarser level whose 2^k-aligned pixels
// fall inside the tile (box means are local to the tile) is reduced in
// shared memory and written — levels L0+1 .. L0+5 from one read of the
// frames.  The finiteness check of as_image covers every frame pixel.
// k_pyr_grad: the gradients of the coarser levels, all levels and both
// frames in one launch (their images are L2-resident by then).
// ---------------------------------------------------------------------------
constexpr int kPTX = 64, kPTY = 32;
constexpr int kPTLevels = 5;  // halvings inside one tile (kPTY = 2^5)

struct PyrArgs {
  const void* frames[2];
  int B, H, W;    // frames
  int L0;         // base level: 0 or 1
  int smax;       // deepest level reduced in the tile kernel
  int g0, g1;     // gradient levels handled by k_pyr_grad: [g0, g1]
  int Ws[32], Hs[32];
  double* img[2][32];
  double* gx[2][32];
  double* gy[2][32];
  uint32_t* status;
};

template <typename T>
__global__ void __launch_bounds__(256) k_pyr_tile(PyrArgs a) {
  __shared__ double base[kPTY + 2][kPTX + 2];
  __shared__ double lv[2][kPTY / 2][kPTX / 2];
  const int z = blockIdx.z;
  const int f = z / a.B, b = z - f * a.B;
  const int W = a.W, H = a.H;
  const T* __restrict__ fr = static_cast<const T*>(a.frames[f]) + (size_t)b * H * W;
  const int L0 = a.L0;
  const int Wb = a.Ws[L0], Hb = a.Hs[L0];
  const int X0 = blockIdx.x * kPTX, Y0 = blockIdx.y * kPTY;
  bool bad = false;
  // ---- 1. base tile + halo (clamped coordinates) ----
  for (int i = threadIdx.x; i < (kPTY + 2) * (kPTX + 2); i += 256) {
    const int ly = i / (kPTX + 2), lx = i - ly * (kPTX + 2);
    const int uy = Y0 - 1 + ly, ux = X0 - 1 + lx;
    const int by = uy < 0 ? 0 : (uy > Hb - 1 ? Hb - 1 : uy);
    const int bx = ux < 0 ? 0 : (ux > Wb - 1 ? Wb - 1 : ux);
    const bool core = uy == by && ux == bx && ly >= 1 && ly <= kPTY && lx >= 1 && lx <= kPTX;
    double v;
    if (L0 == 0) {
      v = to_f64(fr[(size_t)by * W + bx]);
      if (core) bad |= !isfinite(v);
    } else {  // _box_downsample of the converted frame: ((a+b)+(c+d))/4
      const T* r0 = fr + (size_t)(2 * by) * W + 2 * bx;
      const T* r1 = r0 + W;
      const double p00 = to_f64(r0[0]), p01 = to_f64(r0[1]);
      const double p10 = to_f64(r1[0]), p11 = to_f64(r1[1]);
      if (core) bad |= !(isfinite(p00) && isfinite(p01) && isfinite(p10) && isfinite(p11));
      v = ((p00 + p01) + (p10 + p11)) / 4.0;
    }
    base[ly][lx] = v;
  }
  if (L0 == 1) {  // frame pixels no 2x2 block covers: the odd last column / row
    const bool right = X0 + kPTX >= Wb, bottom = Y0 + kPTY >= Hb;
    if ((W & 1) && right)
      for (int r = threadIdx.x; r < 2 * kPTY; r += 256) {
        const int yy = 2 * Y0 + r;
        if (yy < 2 * Hb) bad |= !isfinite(to_f64(fr[(size_t)yy * W + W - 1]));
      }
    if ((H & 1) && bottom) {
      for (int c = threadIdx.x; c < 2 * kPTX; c += 256) {
        const int xx = 2 * X0 + c;
        if (xx < 2 * Wb) bad |= !isfinite(to_f64(fr[(size_t)(H - 1) * W + xx]));
      }
      if ((W & 1) && right && threadIdx.x == 0)
        bad |= !isfinite(to_f64(fr[(size_t)(H - 1) * W + W - 1]));
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    set_status(a.status, DIS_STATUS_NONFINITE_INPUT);
  __syncthreads();
  // ---- 2. base image + gradients (image_gradients, clamped = one-sided) ----
  {
    double* __restrict__ oimg = a.img[f][L0];
    double* __restrict__ ogx = a.gx[f][L0];
    double* __restrict__ ogy = a.gy[f][L0];
    const size_t plane = (size_t)Wb * Hb;
    for (int i = threadIdx.x; i < kPTY * (kPTX / 2); i += 256) {
      const int ly = i / (kPTX / 2), lx = 2 * (i - ly * (kPTX / 2));
      const int y = Y0 + ly, x = X0 + lx;
      if (y >= Hb || x >= Wb) continue;
      const size_t o = (size_t)b * plane + (size_t)y * Wb + x;
      const int cy = ly + 1, cx = lx + 1;
      const double i0 = base[cy][cx], i1 = base[cy][cx + 1];
      const double gx0 = 0.5 * (base[cy][cx + 1] - base[cy][cx - 1]);
      const double gx1 = 0.5 * (base[cy][cx + 2] - base[cy][cx]);
      const double gy0 = 0.5 * (base[cy + 1][cx] - base[cy - 1][cx]);
      const double gy1 = 0.5 * (base[cy + 1][cx + 1] - base[cy - 1][cx + 1]);
      if (x + 1 < Wb && (o & 1) == 0) {
        if (oimg) *reinterpret_cast<double2*>(oimg + o) = make_double2(i0, i1);
        if (ogx) *reinterpret_cast<double2*>(ogx + o) = make_double2(gx0, gx1);
        if (ogy) *reinterpret_cast<double2*>(ogy + o) = make_double2(gy0, gy1);
      } else {
        if (oimg) oimg[o] = i0;
        if (ogx) ogx[o] = gx0;
        if (ogy) ogy[o] = gy0;
        if (x + 1 < Wb) {
          if (oimg) oimg[o + 1] = i1;
          if (ogx) ogx[o + 1] = gx1;
          if (ogy) ogy[o + 1] = gy1;
        }
      }
    }
  }
  // ---- 3. coarser levels reduced in shared memory ----
  for (int s = L0 + 1; s <= a.smax; ++s) {
    const int k = s - L0;  // halvings from the base
    const int tw = kPTX >> k, th = kPTY >> k;
    const int Xs = X0 >> k, Ys = Y0 >> k;
    const int Wsl = a.Ws[s], Hsl = a.Hs[s];
    double* __restrict__ oimg = a.img[f][s];
    double(*dst)[kPTX / 2] = lv[(k - 1) & 1];
    double(*src)[kPTX / 2] = lv[k & 1];
    for (int i = threadIdx.x; i < tw * th; i += 256) {
      const int ly = i / tw, lx = i - ly * tw;
      double p00, p01, p10, p11;
      if (k == 1) {
        p00 = base[2 * ly + 1][2 * lx + 1];
        p01 = base[2 * ly + 1][2 * lx + 2];
        p10 = base[2 * ly + 2][2 * lx + 1];
        p11 = base[2 * ly + 2][2 * lx + 2];
      } else {
        p00 = src[2 * ly][2 * lx];
        p01 = src[2 * ly][2 * lx + 1];
        p10 = src[2 * ly + 1][2 * lx];
        p11 = src[2 * ly + 1][2 * lx + 1];
      }
      const double v = ((p00 + p01) + (p10 + p11)) / 4.0;
      dst[ly][lx] = v;
      const int y = Ys + ly, x = Xs + lx;
      if (y < Hsl && x < Wsl) oimg[(size_t)b * Wsl * Hsl + (size_t)y * Wsl + x] = v;
    }
    __syncthreads();
  }
}

// gradients of levels [g0, g1] of both frames: blockIdx.y = level - g0,
// blockIdx.z = frame * B + pair; 64 x 8 outputs per block (k_gradients_xy)
__global__ void __launch_bounds__(256) k_pyr_grad(PyrArgs a) {
  const int s = a.g0 + (int)blockIdx.y;
  const int z = blockIdx.z;
  const int f = z / a.B, b = z - f * a.B;
  double* __restrict__ ogx = a.gx[f][s];
  double* __restrict__ ogy = a.gy[f][s];
  if (!ogx && !ogy) return;
  const int W = a.Ws[s], H = a.Hs[s];
  const int tx = (W + 63) / 64;
  const int tile = blockIdx.x;
  if (tile >= tx * ((H + 7) / 8)) return;
  const int ty = tile / tx;
  const int x = 2 * ((tile - ty * tx) * 32 + (threadIdx.x & 31));
  const int y = ty * 8 + (threadIdx.x >> 5);
  if (x >= W || y >= H) return;
  const size_t plane = (size_t)W * H;
  const double* img = a.img[f][s] + b * plane;
  const double* row = img + (size_t)y * W;
  const double* up = img + (size_t)(y > 0 ? y - 1 : 0) * W;
  const double* dn = img + (size_t)(y < H - 1 ? y + 1 : H - 1) * W;
  const size_t o = b * plane + (size_t)y * W + x;
  auto gxv = [&](int xx) {
    const int xm = xx > 0 ? xx - 1 : 0, xp = xx < W - 1 ? xx + 1 : W - 1;
    return 0.5 * (row[xp] - row[xm]);
  };
  auto gyv = [&](int xx) { return 0.5 * (dn[xx] - up[xx]); };
  if (x + 1 < W && (o & 1) == 0) {
    if (ogx) *reinterpret_cast<double2*>(ogx + o) = make_double2(gxv(x), gxv(x + 1));
    if (ogy) *reinterpret_cast<double2*>(ogy + o) = make_double2(gyv(x), gyv(x + 1));
  } else {
    for (int q = 0; q < 2 && x + q < W; ++q) {
      if (ogx) ogx[o + q] = gxv(x + q);
      if (ogy) ogy[o + q] = gyv(x + q);
    }
  }
}

template <typename T>
static void launch_pyramid_fused_t(PyrArgs& a, int nf, int coarsest, cudaStream_t st) {
  prof_begin(KC_PYRAMID, st);
  const int L0 = a.L0;
  a.smax = L0 + kPTLevels < coarsest ? L0 + kPTLevels : coarsest;
  dim3 g((unsigned)((a.Ws[L0] + kPTX - 1) / kPTX), (unsigned)((a.Hs[L0] + kPTY - 1) / kPTY),
         (unsigned)(nf * a.B));
  k_pyr_tile<T><<<g, 256, 0, st>>>(a);
  note_launch();
  // levels deeper than one tile's halvings: box means level by level
  for (int s = a.smax + 1; s <= coarsest; ++s) {
    for (int f = 0; f < nf; ++f) {
      const int ho = a.Hs[s], wo = a.Ws[s];
      k_downsample<<<grid_for((size_t)a.B * ho * ((wo + 1) / 2), 256), 256, 0, st>>>(
          a.img[f][s - 1], a.B, a.Hs[s - 1], a.Ws[s - 1], a.img[f][s]);
      note_launch();
    }
  }
  a.g0 = L0 + 1;
  a.g1 = coarsest;
  int tiles = 0;
  bool any = false;
  for (int s = a.g0; s <= a.g1; ++s) {
    const int t = ((a.Ws[s] + 63) / 64) * ((a.Hs[s] + 7) / 8);
    tiles = t > tiles ? t : tiles;
    for (int f = 0; f < nf; ++f) any |= a.gx[f][s] || a.gy[f][s];
  }
  if (any) {
    dim3 gg((unsigned)tiles, (unsigned)(a.g1 - a.g0 + 1), (unsigned)(nf * a.B));
    k_pyr_grad<<<gg, 256, 0, st>>>(a);
    note_launch();
  }
  prof_end(KC_PYRAMID, st);
}

// pyramid factor k != 2: a box-mean launch per level and frame (the first
// from the frames, after a finiteness pass over them when level 0 is not
// stored), then every level's gradients in one launch
template <typename T>
static void launch_pyramid_k_t(PyrArgs& a, int nf, int coarsest, int k, cudaStream_t st) {
  prof_begin(KC_PYRAMID, st);
  const int TH = 256;
  for (int f = 0; f < nf; ++f) {
    const T* fr = static_cast<const T*>(a.frames[f]);
    const size_t n0 = (size_t)a.B * a.H * a.W;
    k_level0<T><<<grid_for(n0, TH), TH, 0, st>>>(fr, a.B, a.H, a.W, a.img[f][0], a.status);
    note_launch();
    for (int s = 1; s <= coarsest; ++s) {
      const size_t n = (size_t)a.B * a.Hs[s] * a.Ws[s];
      if (s == 1 && a.img[f][0] == nullptr)
        k_downsample_k<T><<<grid_for(n, TH), TH, 0, st>>>(fr, a.B, a.H, a.W, k, a.img[f][1]);
      else
        k_downsample_k<double><<<grid_for(n, TH), TH, 0, st>>>(a.img[f][s - 1], a.B,
                                                               a.Hs[s - 1], a.Ws[s - 1], k,
                                                               a.img[f][s]);
      note_launch();
    }
  }
  a.g0 = a.L0;
  a.g1 = coarsest;
  int tiles = 0;
  bool any = false;
  for (int s = a.g0; s <= a.g1; ++s) {
    const int t = ((a.Ws[s] + 63) / 64) * ((a.Hs[s] + 7) / 8);
    tiles = t > tiles ? t : tiles;
    for (int f = 0; f < nf; ++f) any |= a.gx[f][s] || a.gy[f][s];
  }
  if (any) {
    dim3 gg((unsigned)tiles, (unsigned)(a.g1 - a.g0 + 1), (unsigned)(nf * a.B));
    k_pyr_grad<<<gg, 256, 0, st>>>(a);
    note_launch();
  }
  prof_end(KC_PYRAMID, st);
}

// both frames (f2 may be null: one frame); img[f][s] needed for s >= L0
// (L0 = 0 when img[f][0] is requested, else 1); gx/gy where non-null
void launch_pyramid_pair(const void* f1, const void* f2, int dtype, int B, int H, int W,
                         int coarsest, int downscale, double* const (*img)[32],
                         double* const (*gx)[32], double* const (*gy)[32], uint32_t* status,
                         cudaStream_t st) {
  PyrArgs a{};
  const int nf = f2 ? 2 : 1;
  a.frames[0] = f1;
  a.frames[1] = f2;
  a.B = B;
  a.H = H;
  a.W = W;
  a.L0 = (img[0][0] != nullptr || coarsest == 0) ? 0 : 1;
  const int k = downscale;
  for (int s = 0; s <= coarsest && s < 32; ++s) {
    a.Ws[s] = s ? a.Ws[s - 1] / k : W;
    a.Hs[s] = s ? a.Hs[s - 1] / k : H;
    for (int f = 0; f < nf; ++f) {
      a.img[f][s] = img[f][s];
      a.gx[f][s] = gx[f][s];
      a.gy[f][s] = gy[f][s];
    }
  }
  a.status = status;
  if (k != 2) {
    switch (dtype) {
      case DIS_DTYPE_F32:
        launch_pyramid_k_t<float>(a, nf, coarsest, k, st);
        break;
      case DIS_DTYPE_F64:
        launch_pyramid_k_t<double>(a, nf, coarsest, k, st);
        break;
      default:
        launch_pyramid_k_t<uint8_t>(a, nf, coarsest, k, st);
        break;
    }
    return;
  }
  switch (dtype) {
    case DIS_DTYPE_F32:
      launch_pyramid_fused_t<float>(a, nf, coarsest, st);
      break;
    case DIS_DTYPE_F64:
      launch_pyramid_fused_t<double>(a, nf, coarsest, st);
      break;
    default:
      launch_pyramid_fused_t<uint8_t>(a, nf, coarsest, st);
      break;
  }
}

template <typename T>
static void launch_pyramid_t(const T* frames, int B, int H, int W, int coarsest, int k,
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
  if (k != 2 && img[0] == nullptr && coarsest > 0) {  // finiteness pass over the frames
    k_level0<T><<<grid_for((size_t)B * H * W, TH), TH, 0, st>>>(frames, B, H, W, nullptr,
                                                                status);
    note_launch();
  }
  int hl[32], wl[32];
  hl[0] = H;
  wl[0] = W;
  for (int s = 1; s <= coarsest; ++s) {
    const int ho = h / k, wo = w / k;
    hl[s] = ho;
    wl[s] = wo;
    if (k != 2) {
      if (s == 1 && img[0] == nullptr)
        k_downsample_k<T><<<grid_for((size_t)B * ho * wo, TH), TH, 0, st>>>(frames, B, h, w, k,
                                                                            img[1]);
      else
        k_downsample_k<double><<<grid_for((size_t)B * ho * wo, TH), TH, 0, st>>>(
            img[s - 1], B, h, w, k, img[s]);
    } else if (s == 1 && img[0] == nullptr) {
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
  for (int s = 0; s <= coarsest; ++s) {
    h = hl[s];
    w = wl[s];
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
  }
  prof_end(KC_PYRAMID, st);
}

void launch_pyramid(const void* frames, int dtype, int B, int H, int W, int coarsest,
                    int downscale, double* const* img, double* const* gx, double* const* gy,
                    double* const* dd, uint32_t* status, cudaStream_t st) {
  bool want_dd = false;
  for (int s = 0; s <= coarsest; ++s) want_dd |= dd && dd[s];
  if (!want_dd && coarsest < 32) {
    double* im[1][32] = {};
    double* x[1][32] = {};
    double* y[1][32] = {};
    for (int s = 0; s <= coarsest; ++s) {
      im[0][s] = img[s];
      x[0][s] = gx ? gx[s] : nullptr;
      y[0][s] = gy ? gy[s] : nullptr;
    }
    launch_pyramid_pair(frames, nullptr, dtype, B, H, W, coarsest, downscale, im, x, y, status,
                        st);
    return;
  }
  switch (dtype) {
    case DIS_DTYPE_F32:
      launch_pyramid_t((const float*)frames, B, H, W, coarsest, downscale, img, gx, gy, dd,
                       status, st);
      break;
    case DIS_DTYPE_F64:
      launch_pyramid_t((const double*)frames, B, H, W, coarsest, downscale, img, gx, gy, dd,
                       status, st);
      break;
    default:
      launch_pyramid_t((const uint8_t*)frames, B, H, W, coarsest, downscale, img, gx, gy, dd,
                       status, st);
      break;
  }
}

}  // namespace disb200
