// patch_search.cu — per-scale inverse patch search (one pyramid level, a
// batch of pairs): the whole of _ScaleState.search (pipeline.py:54-82)
//
//   init_patches         densification.py:82-95   (numpy bilinear_map form)
//   _patch_precompute    inverse_search.py:75-98  (template, S', Hessian)
//   _condition_hessians  inverse_search.py:255-276
//   _patch_optimize      inverse_search.py:113-189 (inverse-compositional
//                        Gauss-Newton, mean normalisation, rollback, early
//                        exit, runaway guard)
//   reset_outliers       densification.py:98-107
//   refresh_patch_stats  inverse_search.py:374-387 / _window_stats 227-248
//
// Mapping: one thread per (pair, patch).  The exact-parity requirement
// (c2 is chaotic, a warp-tree reduction moves its flow by
// 3.8e-2 px) forces each patch's sums to run sequentially in the reference's
// row-major order, so a patch is a thread, not a warp.
//
// Template/steepest-descent samples sit at integer coordinates, where the
// reference's _bilin returns the pixel itself; they are read straight from
// the level (never materialised — the reference's (P, ps^2, 3) arrays are
// 168 MB for c2).  Only mean_t and the conditioned H^-1 are per-patch state.
//
// "Refresh" after an outlier reset re-evaluates the window at u_init with the
// same loop order as the first Gauss-Newton evaluation, which is also at
// u_init — so the kernel keeps the first evaluation's (offset, residual)
// instead of a second pass (bit-identical).
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

// _transform_residual, inverse_search.py:61-72
__device__ __forceinline__ double transform_residual(double e, int code, double b) {
  if (code == DIS_NORM_L1) {
    double r = sqrt(fabs(e));
    return e >= 0.0 ? r : -r;
  }
  if (code == DIS_NORM_HUBER) {
    if (fabs(e) < b) return e;
    double r = sqrt(2.0 * b * fabs(e) - b * b);
    return e >= 0.0 ? r : -r;
  }
  return e;
}

// reset_outliers' test np.hypot(du, dv) > ps (densification.py:104),
// decided exactly for a correctly rounded hypot: sqrt(a^2 + b^2) compared
// with the rounding midpoint ps + ulp(ps)/2 in double-double.  (glibc's
// hypot is faithful, not correctly rounded; the two can only disagree when
// |delta| lies within one ulp of ps.)
__device__ __forceinline__ bool hypot_gt(double a, double b, int ps) {
  if (!(isfinite(a) && isfinite(b))) return isinf(a) || isinf(b);  // hypot(inf, nan) = inf
  double p1 = a * a, e1 = fma(a, a, -p1);
  double p2 = b * b, e2 = fma(b, b, -p2);
  double s = p1 + p2;
  double bv = s - p1;
  double es = (p1 - (s - bv)) + (p2 - bv);
  double lo = es + (e1 + e2);
  double dps = (double)ps;
  double ulp = nextafter(dps, DBL_MAX) - dps;
  double t_hi = dps * dps;                  // exact for ps < 2^26
  double t_lo = dps * ulp + 0.25 * ulp * ulp;  // exact (powers of two times ps)
  return (s - t_hi) + (lo - t_lo) > 0.0;
}

__global__ void __launch_bounds__(128) k_patch_search(SearchArgs a) {
  const int nx = a.ax.n;
  const int P = nx * a.ay.n;
  const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (size_t)a.B * P) return;
  const int b = (int)(gid / P);
  const int i = (int)(gid - (size_t)b * P);
  const int iy = i / nx;
  const int ix = i - iy * nx;
  const int ps = a.ps, W = a.W, H = a.H;
  const int x0i = a.ax.origin(ix);
  const int y0i = a.ay.origin(iy);
  const double x0 = (double)x0i;
  const double y0 = (double)y0i;
  const size_t plane = (size_t)W * H;
  const double* __restrict__ ref = a.ref + b * plane;
  const double* __restrict__ rgx = a.rgx + b * plane;
  const double* __restrict__ rgy = a.rgy + b * plane;
  const double* __restrict__ qry = a.qry + b * plane;

  // ---- init_patches (densification.py:82-95) ----
  double u0 = 0.0, v0 = 0.0;
  if (a.cu) {
    const size_t cplane = (size_t)a.Wc * a.Hc;
    const double half = 0.5 * ps;
    const double xs = (x0 + half) / 2.0;
    const double ys = (y0 + half) / 2.0;
    u0 = bilin_np(a.cu + b * cplane, a.Wc, a.Hc, xs, ys) * 2.0;
    v0 = bilin_np(a.cv + b * cplane, a.Wc, a.Hc, xs, ys) * 2.0;
  }

  // ---- _patch_precompute (inverse_search.py:75-98) ----
  double tsum = 0.0, h00 = 0.0, h01 = 0.0, h11 = 0.0;
  for (int oy = 0; oy < ps; ++oy) {
    const size_t row = (size_t)(y0i + oy) * W + x0i;
    for (int ox = 0; ox < ps; ++ox) {
      const double t = __ldg(ref + row + ox);
      const double gxv = __ldg(rgx + row + ox);
      const double gyv = __ldg(rgy + row + ox);
      tsum += t;
      h00 += gxv * gxv;
      h01 += gxv * gyv;
      h11 += gyv * gyv;
    }
  }
  const double dn = (double)(ps * ps);
  const double mean_t = exact_div_pos(tsum, dn);

  // ---- _condition_hessians (inverse_search.py:255-276) ----
  const double tr = h00 + h11;
  const double det = h00 * h11 - h01 * h01;
  const double q = 0.25 * tr * tr;
  const double rel = isnan(q) ? q : (1.0 > q ? 1.0 : q);
  const double arg = tr * tr - 4.0 * det;
  const double disc = sqrt(isnan(arg) ? arg : (arg > 0.0 ? arg : 0.0));
  const double lmin = 0.5 * (tr - disc);
  const double lmax = 0.5 * (tr + disc);
  const bool valid = (det > 1e-6 * rel) && (lmin > 0.0) && (lmax <= 1e6 * lmin);
  const double i00 = valid ? h11 / det : 0.0;
  const double i01 = valid ? -h01 / det : 0.0;
  const double i11 = valid ? h00 / det : 0.0;

  // ---- _patch_optimize (inverse_search.py:113-189) ----
  double u = u0, v = v0;
  double prev_ssd = 1e300, prev_u = u, prev_v = v, prev_off = 0.0, prev_mar = 0.0;
  bool stop_after_eval = !valid;
  int k = 0;
  double off = 0.0, mar = 0.0, off0 = 0.0, mar0 = 0.0;
  int evals = 0;
  const int code = a.code;
  const double hb = a.hb;
  for (;;) {
    const double bx = x0 + u;
    const double by = y0 + v;
    double wsum = 0.0;
    for (int oy = 0; oy < ps; ++oy)
      for (int ox = 0; ox < ps; ++ox) wsum += bilin_nb(qry, W, H, bx + ox, by + oy);
    off = a.mean_norm ? exact_div_pos(wsum, dn) - mean_t : 0.0;
    double ssd = 0.0, b0 = 0.0, b1 = 0.0;
    mar = 0.0;
    for (int oy = 0; oy < ps; ++oy) {
      const size_t row = (size_t)(y0i + oy) * W + x0i;
      for (int ox = 0; ox < ps; ++ox) {
        const double val = bilin_nb(qry, W, H, bx + ox, by + oy);
        const double e = val - off - __ldg(ref + row + ox);
        mar += fabs(e);
        const double et = transform_residual(e, code, hb);
        ssd += et * et;
        b0 += __ldg(rgx + row + ox) * et;
        b1 += __ldg(rgy + row + ox) * et;
      }
    }
    mar = exact_div_pos(mar, dn);
    if (evals == 0) {
      off0 = off;
      mar0 = mar;
    }
    ++evals;
    if (ssd > prev_ssd) {
      u = prev_u;
      v = prev_v;
      off = prev_off;
      mar = prev_mar;
      break;
    }
    if (stop_after_eval || k >= a.iters) break;
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
    if (sqrt(du * du + dv * dv) < 1e-2) stop_after_eval = true;
    const double cx = x0 + u + 0.5 * ps;
    const double cy = y0 + v + 0.5 * ps;
    if (cx < (double)(-W) || cx > 2.0 * W || cy < (double)(-H) || cy > 2.0 * H) {
      u = u0;
      v = v0;
      prev_ssd = 1e300;
      stop_after_eval = true;
    }
  }

  // ---- reset_outliers + refresh_patch_stats ----
  if (hypot_gt(u - u0, v - v0, ps)) {
    u = u0;
    v = v0;
    off = a.mean_norm ? off0 : 0.0;
    mar = mar0;
  }

  const size_t o = (size_t)b * P + i;
  a.out_u[o] = u;
  a.out_v[o] = v;
  a.out_off[o] = off;
  if (a.out_mar) a.out_mar[o] = mar;
  if (a.out_iu) a.out_iu[o] = u0;
  if (a.out_iv) a.out_iv[o] = v0;
  if (a.out_valid) a.out_valid[o] = valid ? 1 : 0;
  if (a.out_evals) a.out_evals[o] = evals;
}

void launch_patch_search(const SearchArgs& a, cudaStream_t st) {
  const size_t n = (size_t)a.B * a.ax.n * a.ay.n;
  const int TH = 128;
  const unsigned blocks = (unsigned)((n + TH - 1) / TH);
  prof_begin(KC_SEARCH, st);
  k_patch_search<<<blocks, TH, 0, st>>>(a);
  prof_end(KC_SEARCH, st);
  note_launch();
}

}  // namespace disb200
