// stage_search.cu — the reference's inverse-search and initialisation stage
// functions on materialised per-patch arrays (the operator layer the
// reference's tests and stage-level callers use; the flow path itself runs
// the fused kernels of patch_search.cu):
//
//   k_precompute_set : precompute_patch_set (inverse_search.py:306-341) —
//                      _patch_precompute (75-98) at arbitrary real window
//                      origins (bilinear samples via _bilin) +
//                      _condition_hessians (255-276)
//   k_optimize_set   : optimize_patch_set (344-371) — _patch_optimize
//                      (113-189) per patch from its init_displacement
//   k_window_stats   : refresh_patch_stats (374-387) — _window_stats (227-248)
//   k_init_patches   : init_patches (densification.py:82-95)
//   k_reset_outliers : reset_outliers (densification.py:98-107)
//
// One thread per patch; every sum in the reference's order, float64, no FMA
// contraction (-fmad=false), IEEE division — bit-identical to the reference.
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

__global__ void __launch_bounds__(128)
    k_precompute_set(const double* __restrict__ img, const double* __restrict__ gx,
                     const double* __restrict__ gy, int W, int H, const double* __restrict__ xs,
                     const double* __restrict__ ys, int n, int ps, int horizontal,
                     double* __restrict__ tmpl, double* __restrict__ sdx,
                     double* __restrict__ sdy, double* __restrict__ mean_t,
                     double* __restrict__ hess, double* __restrict__ hinv,
                     uint8_t* __restrict__ valid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int nn = ps * ps;
  const double x0 = xs[i], y0 = ys[i];
  double tsum = 0.0, h00 = 0.0, h01 = 0.0, h11 = 0.0;
  size_t k = (size_t)i * nn;
  for (int oy = 0; oy < ps; ++oy) {
    const double py = y0 + oy;
    for (int ox = 0; ox < ps; ++ox, ++k) {
      const double px = x0 + ox;
      const double t = bilin_nb(img, W, H, px, py);
      const double gxv = bilin_nb(gx, W, H, px, py);
      const double gyv = bilin_nb(gy, W, H, px, py);
      tmpl[k] = t;
      sdx[k] = gxv;
      sdy[k] = gyv;
      tsum += t;
      h00 += gxv * gxv;
      h01 += gxv * gyv;
      h11 += gyv * gyv;
    }
  }
  mean_t[i] = tsum / (double)nn;
  hess[3 * i] = h00;
  hess[3 * i + 1] = h01;
  hess[3 * i + 2] = h11;
  if (horizontal) {  // horizontal_only (inverse_search.py:259-264)
    const bool v = h00 > 1e-6;
    hinv[3 * i] = v ? 1.0 / h00 : 0.0;
    hinv[3 * i + 1] = 0.0;
    hinv[3 * i + 2] = 0.0;
    valid[i] = v;
    return;
  }
  const double tr = h00 + h11;
  const double det = h00 * h11 - h01 * h01;
  const double q = 0.25 * tr * tr;
  const double rel = isnan(q) ? q : (1.0 > q ? 1.0 : q);  // np.maximum propagates NaN
  const double arg = tr * tr - 4.0 * det;
  const double disc = sqrt(isnan(arg) ? arg : (arg > 0.0 ? arg : 0.0));
  const double lmin = 0.5 * (tr - disc);
  const double lmax = 0.5 * (tr + disc);
  const bool v = (det > 1e-6 * rel) && (lmin > 0.0) && (lmax <= 1e6 * lmin);
  hinv[3 * i] = v ? h11 / det : 0.0;
  hinv[3 * i + 1] = v ? -h01 / det : 0.0;
  hinv[3 * i + 2] = v ? h00 / det : 0.0;
  valid[i] = v;
}

// one window evaluation of _patch_optimize (inverse_search.py:130-152)
__device__ __forceinline__ void eval_window(const double* __restrict__ q, int W, int H, int ps,
                                            double bx, double by, const double* __restrict__ t,
                                            const double* __restrict__ sx,
                                            const double* __restrict__ sy, double mean_t,
                                            bool mean_norm, int code, double hb, double& off,
                                            double& ssd, double& mar, double& b0, double& b1) {
  const int nn = ps * ps;
  double wsum = 0.0;
  for (int oy = 0; oy < ps; ++oy)
    for (int ox = 0; ox < ps; ++ox) wsum += bilin_nb(q, W, H, bx + ox, by + oy);
  off = mean_norm ? wsum / (double)nn - mean_t : 0.0;
  ssd = 0.0;
  mar = 0.0;
  b0 = 0.0;
  b1 = 0.0;
  int k = 0;
  for (int oy = 0; oy < ps; ++oy)
    for (int ox = 0; ox < ps; ++ox, ++k) {
      const double e = bilin_nb(q, W, H, bx + ox, by + oy) - off - t[k];
      mar += fabs(e);
      const double et = transform_residual(e, code, hb);
      ssd += et * et;
      b0 += sx[k] * et;
      b1 += sy[k] * et;
    }
  mar /= (double)nn;
}

__global__ void __launch_bounds__(128)
    k_optimize_set(const double* __restrict__ qry, int W, int H, const double* __restrict__ xs,
                   const double* __restrict__ ys, int n, int ps, const double* __restrict__ tmpl,
                   const double* __restrict__ sdx, const double* __restrict__ sdy,
                   const double* __restrict__ hinv, const double* __restrict__ mean_t,
                   const uint8_t* __restrict__ valid, const double* __restrict__ init,
                   int iters, int mean_norm, int code, double hb, double* __restrict__ disp,
                   double* __restrict__ offset, double* __restrict__ mar_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int nn = ps * ps;
  const double* t = tmpl + (size_t)i * nn;
  const double* sx = sdx + (size_t)i * nn;
  const double* sy = sdy + (size_t)i * nn;
  const double x0 = xs[i], y0 = ys[i];
  const double i00 = hinv[3 * i], i01 = hinv[3 * i + 1], i11 = hinv[3 * i + 2];
  const double u0 = init[2 * i], v0 = init[2 * i + 1];
  double u = u0, v = v0;
  double prev_ssd = 1e300, prev_u = u, prev_v = v, prev_off = 0.0, prev_mar = 0.0;
  bool stop = !valid[i];
  int k = 0;
  double off, ssd, mar, b0, b1;
  for (;;) {
    eval_window(qry, W, H, ps, x0 + u, y0 + v, t, sx, sy, mean_t[i], mean_norm != 0, code, hb,
                off, ssd, mar, b0, b1);
    if (ssd > prev_ssd) {  // the step made things worse: keep the previous iterate
      u = prev_u;
      v = prev_v;
      off = prev_off;
      mar = prev_mar;
      break;
    }
    if (stop || k >= iters) break;
    prev_ssd = ssd;
    prev_u = u;
    prev_v = v;
    prev_off = off;
    prev_mar = mar;
    const double du = i00 * b0 + i01 * b1;
    const double dv = i01 * b0 + i11 * b1;
    u -= du;
    v -= dv;
    k += 1;
    if (sqrt(du * du + dv * dv) < 1e-2) stop = true;  // CONVERGENCE_STEP
    const double cx = x0 + u + 0.5 * ps;
    const double cy = y0 + v + 0.5 * ps;
    if (cx < (double)(-W) || cx > 2.0 * W || cy < (double)(-H) || cy > 2.0 * H) {
      u = u0;  // runaway displacement: back to the initialisation
      v = v0;
      prev_ssd = 1e300;
      stop = true;
    }
  }
  disp[2 * i] = u;
  disp[2 * i + 1] = v;
  offset[i] = off;
  mar_out[i] = mar;
}

__global__ void __launch_bounds__(128)
    k_window_stats(const double* __restrict__ qry, int W, int H, const double* __restrict__ xs,
                   const double* __restrict__ ys, int n, int ps, const double* __restrict__ tmpl,
                   const double* __restrict__ mean_t, const uint8_t* __restrict__ sel,
                   const double* __restrict__ disp, int mean_norm, double* __restrict__ offset,
                   double* __restrict__ mar_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !sel[i]) return;
  const int nn = ps * ps;
  const double bx = xs[i] + disp[2 * i], by = ys[i] + disp[2 * i + 1];
  double wsum = 0.0;
  for (int oy = 0; oy < ps; ++oy)
    for (int ox = 0; ox < ps; ++ox) wsum += bilin_nb(qry, W, H, bx + ox, by + oy);
  const double off = mean_norm ? wsum / (double)nn - mean_t[i] : 0.0;
  double mar = 0.0;
  const double* t = tmpl + (size_t)i * nn;
  int k = 0;
  for (int oy = 0; oy < ps; ++oy)
    for (int ox = 0; ox < ps; ++ox, ++k)
      mar += fabs(bilin_nb(qry, W, H, bx + ox, by + oy) - off - t[k]);
  offset[i] = off;
  mar_out[i] = mar / (double)nn;
}

// init_patches: coarser field (Hc x Wc x 2, interleaved like the reference's
// (H, W, 2) array) at centre / k, times k; zeros without a coarser field
__global__ void __launch_bounds__(128)
    k_init_patches(const double* __restrict__ coarse, int Wc, int Hc,
                   const double* __restrict__ centers, int n, int ds,
                   double* __restrict__ init) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!coarse) {
    init[2 * i] = 0.0;
    init[2 * i + 1] = 0.0;
    return;
  }
  const double k = (double)ds;
  double x = centers[2 * i] / k, y = centers[2 * i + 1] / k;
  // bilinear_map (core.py:154-170) on the interleaved components
  x = !(x >= 0.0) ? 0.0 : (x > Wc - 1.0 ? Wc - 1.0 : x);
  y = !(y >= 0.0) ? 0.0 : (y > Hc - 1.0 ? Hc - 1.0 : y);
  const int x0 = (int)floor(x), y0 = (int)floor(y);
  const int x1 = x0 + 1 < Wc - 1 ? x0 + 1 : Wc - 1;
  const int y1 = y0 + 1 < Hc - 1 ? y0 + 1 : Hc - 1;
  const double fx = x - (double)x0, fy = y - (double)y0;
  for (int c = 0; c < 2; ++c) {
    const double i00 = coarse[2 * ((size_t)y0 * Wc + x0) + c];
    const double i01 = coarse[2 * ((size_t)y0 * Wc + x1) + c];
    const double i10 = coarse[2 * ((size_t)y1 * Wc + x0) + c];
    const double i11 = coarse[2 * ((size_t)y1 * Wc + x1) + c];
    const double top = i00 * (1.0 - fx) + i01 * fx;
    const double bot = i10 * (1.0 - fx) + i11 * fx;
    init[2 * i + c] = (top * (1.0 - fy) + bot * fy) * k;
  }
}

// np.hypot(du, dv) > ps decided for a correctly rounded hypot
// (patch_search.cu)
__device__ __forceinline__ bool hypot_gt_stage(double a, double b, int ps) {
  if (!(isfinite(a) && isfinite(b))) return isinf(a) || isinf(b);
  double p1 = a * a, e1 = fma(a, a, -p1);
  double p2 = b * b, e2 = fma(b, b, -p2);
  double s = p1 + p2;
  double bv = s - p1;
  double es = (p1 - (s - bv)) + (p2 - bv);
  double lo = es + (e1 + e2);
  double dps = (double)ps;
  double ulp = nextafter(dps, DBL_MAX) - dps;
  double t_hi = dps * dps;
  double t_lo = dps * ulp + 0.25 * ulp * ulp;
  return (s - t_hi) + (lo - t_lo) > 0.0;
}

__global__ void __launch_bounds__(128)
    k_reset_outliers(const double* __restrict__ disp, const double* __restrict__ init, int n,
                     int ps, double* __restrict__ out, uint8_t* __restrict__ was_reset) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double u = disp[2 * i], v = disp[2 * i + 1];
  const double iu = init[2 * i], iv = init[2 * i + 1];
  const bool bad = hypot_gt_stage(u - iu, v - iv, ps);
  out[2 * i] = bad ? iu : u;
  out[2 * i + 1] = bad ? iv : v;
  if (was_reset) was_reset[i] = bad;
}

static unsigned nblk(int n) { return (unsigned)((n + 127) / 128 > 0 ? (n + 127) / 128 : 1); }

void launch_precompute_set(const double* img, const double* gx, const double* gy, int W, int H,
                           const double* xs, const double* ys, int n, int ps, int horizontal,
                           double* tmpl, double* sdx, double* sdy, double* mean_t, double* hess,
                           double* hinv, uint8_t* valid, cudaStream_t st) {
  k_precompute_set<<<nblk(n), 128, 0, st>>>(img, gx, gy, W, H, xs, ys, n, ps, horizontal, tmpl,
                                            sdx, sdy, mean_t, hess, hinv, valid);
  note_launch();
}

void launch_optimize_set(const double* qry, int W, int H, const double* xs, const double* ys,
                         int n, int ps, const double* tmpl, const double* sdx, const double* sdy,
                         const double* hinv, const double* mean_t, const uint8_t* valid,
                         const double* init, int iters, int mean_norm, int code, double hb,
                         double* disp, double* offset, double* mar, cudaStream_t st) {
  k_optimize_set<<<nblk(n), 128, 0, st>>>(qry, W, H, xs, ys, n, ps, tmpl, sdx, sdy, hinv, mean_t,
                                          valid, init, iters, mean_norm, code, hb, disp, offset,
                                          mar);
  note_launch();
}

void launch_window_stats(const double* qry, int W, int H, const double* xs, const double* ys,
                         int n, int ps, const double* tmpl, const double* mean_t,
                         const uint8_t* sel, const double* disp, int mean_norm, double* offset,
                         double* mar, cudaStream_t st) {
  k_window_stats<<<nblk(n), 128, 0, st>>>(qry, W, H, xs, ys, n, ps, tmpl, mean_t, sel, disp,
                                          mean_norm, offset, mar);
  note_launch();
}

void launch_init_patches(const double* coarse, int Wc, int Hc, const double* centers, int n,
                         int ds, double* init, cudaStream_t st) {
  k_init_patches<<<nblk(n), 128, 0, st>>>(coarse, Wc, Hc, centers, n, ds, init);
  note_launch();
}

void launch_reset_outliers(const double* disp, const double* init, int n, int ps, double* out,
                           uint8_t* was_reset, cudaStream_t st) {
  k_reset_outliers<<<nblk(n), 128, 0, st>>>(disp, init, n, ps, out, was_reset);
  note_launch();
}

}  // namespace disb200
