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
#include <cstdlib>

#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

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

// 256-bit read-only load of 4 doubles (32-byte aligned address)
__device__ __forceinline__ void ldg256(const double* p, double* v) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
      : "l"(p));
}

// N consecutive doubles p[0 .. N-1] (8-byte aligned p) as 256-bit loads from
// the 32-byte aligned address at or below p, shifted into place by the
// lane's offset o = (p / 8) mod 4 with two select levels
template <int N>
__device__ __forceinline__ void load_run256(const double* p, double* s) {
  constexpr int NV = (N + 3 + 3) / 4;
  const unsigned o = (unsigned)(((uintptr_t)p >> 3) & 3u);
  const double* pa = p - o;
  double v[4 * NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) ldg256(pa + 4 * q, v + 4 * q);
  double w[N + 1];
#pragma unroll
  for (int i = 0; i <= N; ++i) w[i] = (o & 2u) ? v[i + 2] : v[i];
#pragma unroll
  for (int c = 0; c < N; ++c) s[c] = (o & 1u) ? w[c + 1] : w[c];
}

// ---------------------------------------------------------------------------
// Stage 1 — per-patch prep (one thread per patch): init_patches,
// _patch_precompute and _condition_hessians.  Writes the kPrep record the
// Gauss-Newton stage needs; resets the GN work counter.
// ---------------------------------------------------------------------------
// Lane kernel work distribution: block b owns the contiguous patch range
// [b N / nb, (b+1) N / nb) and its warps refill their pools from it in
// order, so the 8 warps of an SM work on neighbouring grid rows and share
// their template and window rows in L1 (a global queue scatters an SM's
// warps over 8 distant regions: L1 hit rate 47 %); a block whose range is
// used up steals pools from the following blocks' ranges.
#ifndef DIS_GN_PREFETCH
#define DIS_GN_PREFETCH 0  // experiments: prefetch the template rows into L1
#endif
#ifndef DIS_GN_RANGES
#define DIS_GN_RANGES 0  // lane kernel: per-block patch ranges (0: one global queue)
#endif
#ifndef DIS_GN_CARVEOUT
#define DIS_GN_CARVEOUT -1  // experiments: the lane kernel's shared-memory carveout (%)
#endif
constexpr int kStragglers = 10;  // lane kernel: see SearchArgs::stragglers
constexpr int kRangeCounters = 4;     // counter[4 ..]: consumed patches per block range
constexpr int kMaxGnBlocks = 1024;

enum PrepField { PR_U0 = 0, PR_V0, PR_MEAN, PR_I00, PR_I01, PR_I11, PR_VALID, kPrep };

__global__ void __launch_bounds__(128) k_patch_prep(SearchArgs a, double* __restrict__ prep,
                                                     unsigned* counter) {
  const int nx = a.ax.n;
  const int P = nx * a.ay.n;
  const size_t N = (size_t)a.B * P;
  const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid == 0) {
    counter[0] = 0u;  // work queue
    counter[1] = 0u;  // parked patches
    counter[2] = 0u;  // parked-patch queue
  }
  // the lane kernel's per-block range counters
  for (size_t i = gid; i < kMaxGnBlocks; i += (size_t)gridDim.x * blockDim.x)
    counter[kRangeCounters + i] = 0u;
  if (gid >= N) return;
  const int b = (int)(gid / P);
  const int i = (int)(gid - (size_t)b * P);
  const int iy = i / nx;
  const int ix = i - iy * nx;
  const int ps = a.ps, W = a.W, H = a.H;
  const int x0i = a.ax.origin(ix);
  const int y0i = a.ay.origin(iy);
  const size_t plane = (size_t)W * H;
  const double* __restrict__ ref = a.ref + b * plane;
  const double* __restrict__ rgx = a.rgx + b * plane;
  const double* __restrict__ rgy = a.rgy + b * plane;

  // ---- init_patches (densification.py:82-95) ----
  double u0 = 0.0, v0 = 0.0;
  if (a.cu) {
    const size_t cplane = (size_t)a.Wc * a.Hc;
    const double half = 0.5 * ps;
    const double k = (double)a.ds;
    // (/ 2 is the exact multiplication by 0.5: no IEEE division for the usual factor)
    const double xs = a.ds == 2 ? ((double)x0i + half) * 0.5 : ((double)x0i + half) / k;
    const double ys = a.ds == 2 ? ((double)y0i + half) * 0.5 : ((double)y0i + half) / k;
    u0 = bilin_np(a.cu + b * cplane, a.Wc, a.Hc, xs, ys) * k;
    v0 = bilin_np(a.cv + b * cplane, a.Wc, a.Hc, xs, ys) * k;
  }

  // ---- _patch_precompute (inverse_search.py:75-98) ----
  // samples at integer coordinates: the reference's _bilin returns the pixel
  double tsum = 0.0, h00 = 0.0, h01 = 0.0, h11 = 0.0;
  auto add = [&](double t, double gxv, double gyv) {
    tsum += t;
    h00 += gxv * gxv;
    h01 += gxv * gyv;
    h11 += gyv * gyv;
  };
  // rows 32-byte aligned (element offset and pitch multiples of 4, e.g. grid
  // spacing 4): 256-bit loads, one sector per lane per load
  const size_t off0 = (size_t)b * plane + (size_t)y0i * W + x0i;
  // the common patch sizes with compile-time loops (all rows' loads in
  // flight ahead of the sequential sums)
  auto rows_fixed = [&](auto psc) {
    constexpr int PSc = decltype(psc)::value;
    if (((off0 | (size_t)W) & 3) == 0) {
#pragma unroll
      for (int oy = 0; oy < PSc; ++oy) {
        const size_t row = (size_t)(y0i + oy) * W + x0i;
#pragma unroll
        for (int ox = 0; ox < PSc; ox += 4) {
          double t[4], gx4[4], gy4[4];
          ldg256(ref + row + ox, t);
          ldg256(rgx + row + ox, gx4);
          ldg256(rgy + row + ox, gy4);
#pragma unroll
          for (int q = 0; q < 4; ++q) add(t[q], gx4[q], gy4[q]);
        }
      }
    } else {
#pragma unroll
      for (int oy = 0; oy < PSc; ++oy) {
        const size_t row = (size_t)(y0i + oy) * W + x0i;
#pragma unroll
        for (int ox = 0; ox < PSc; ++ox)
          add(__ldg(ref + row + ox), __ldg(rgx + row + ox), __ldg(rgy + row + ox));
      }
    }
  };
  if (ps == 8) {
    rows_fixed(std::integral_constant<int, 8>{});
  } else if (ps == 12) {
    rows_fixed(std::integral_constant<int, 12>{});
  } else if ((ps & 3) == 0 && ((off0 | (size_t)W) & 3) == 0) {
    for (int oy = 0; oy < ps; ++oy) {
      const size_t row = (size_t)(y0i + oy) * W + x0i;
      for (int ox = 0; ox < ps; ox += 4) {
        double t[4], gx4[4], gy4[4];
        ldg256(ref + row + ox, t);
        ldg256(rgx + row + ox, gx4);
        ldg256(rgy + row + ox, gy4);
#pragma unroll
        for (int q = 0; q < 4; ++q) add(t[q], gx4[q], gy4[q]);
      }
    }
  } else {
    for (int oy = 0; oy < ps; ++oy) {
      const size_t row = (size_t)(y0i + oy) * W + x0i;
      for (int ox = 0; ox < ps; ++ox)
        add(__ldg(ref + row + ox), __ldg(rgx + row + ox), __ldg(rgy + row + ox));
    }
  }
  const double dn = (double)(ps * ps);
  const double mean_t = exact_div_pos(tsum, dn);

  // ---- _condition_hessians (inverse_search.py:255-276) ----
  if (a.horizontal) {  // horizontal_only (259-264): valid = h00 > 1e-6, hinv = [1/h00, 0, 0]
    const bool hv = h00 > 1e-6;
    prep[PR_U0 * N + gid] = u0;
    prep[PR_V0 * N + gid] = v0;
    prep[PR_MEAN * N + gid] = mean_t;
    prep[PR_I00 * N + gid] = hv ? 1.0 / h00 : 0.0;
    prep[PR_I01 * N + gid] = 0.0;
    prep[PR_I11 * N + gid] = 0.0;
    prep[PR_VALID * N + gid] = hv ? 1.0 : 0.0;
    if (a.out_iu) a.out_iu[gid] = u0;
    if (a.out_iv) a.out_iv[gid] = v0;
    if (a.out_valid) a.out_valid[gid] = hv ? 1 : 0;
    return;
  }
  const double tr = h00 + h11;
  const double det = h00 * h11 - h01 * h01;
  const double q = 0.25 * tr * tr;
  const double rel = isnan(q) ? q : (1.0 > q ? 1.0 : q);
  const double arg = tr * tr - 4.0 * det;
  const double disc = sqrt(isnan(arg) ? arg : (arg > 0.0 ? arg : 0.0));
  const double lmin = 0.5 * (tr - disc);
  const double lmax = 0.5 * (tr + disc);
  const bool valid = (det > 1e-6 * rel) && (lmin > 0.0) && (lmax <= 1e6 * lmin);
  prep[PR_U0 * N + gid] = u0;
  prep[PR_V0 * N + gid] = v0;
  prep[PR_MEAN * N + gid] = mean_t;
  prep[PR_I00 * N + gid] = valid ? h11 / det : 0.0;
  prep[PR_I01 * N + gid] = valid ? -h01 / det : 0.0;
  prep[PR_I11 * N + gid] = valid ? h00 / det : 0.0;
  prep[PR_VALID * N + gid] = valid ? 1.0 : 0.0;
  if (a.out_iu) a.out_iu[gid] = u0;
  if (a.out_iv) a.out_iv[gid] = v0;
  if (a.out_valid) a.out_valid[gid] = valid ? 1 : 0;
}

// ---------------------------------------------------------------------------
// Stage 2 — inverse-compositional Gauss-Newton (_patch_optimize,
// inverse_search.py:113-189) + reset_outliers + refresh.
//
// Persistent lanes pulling patches from a work queue (warp-aggregated
// atomicAdd on a counter): a lane whose patch exits early (rollback,
// convergence) takes the next patch instead of idling until the slowest lane
// of its warp is done (mean 3-5.5 window evaluations, p99 up
// to 22).  Which lane computes which patch never affects a patch's result.
//
// One window evaluation = the reference's two passes over the ps x ps
// samples (sum for the mean offset; then residuals, SSD and the steepest
// descent products), sequential in row-major order.  Each sample's
// coordinate is (bx + ox, by + oy): its clamp, integer part and fraction
// depend on ox alone or oy alone, so they are computed once per column /
// row of the window (bit-identical to clamping every sample).
// ---------------------------------------------------------------------------
struct Axis1 {
  int i0, i1;
  double f;
};
__device__ __forceinline__ Axis1 axis_sample(double c, int n) {
  if (!(c >= 0.0))
    c = 0.0;
  else if (c > n - 1.0)
    c = n - 1.0;
  Axis1 a;
  a.i0 = (int)c;
  a.i1 = a.i0 + 1 > n - 1 ? n - 1 : a.i0 + 1;
  a.f = c - (double)a.i0;
  return a;
}

#ifndef DIS_GN_POOL
#define DIS_GN_POOL 64
#endif
constexpr unsigned kPool = DIS_GN_POOL;  // patches per warp-pool refill
constexpr int kSpillStride = 16;  // doubles per parked patch state

struct Lane {
  int pid;  // patch (b * P + i) or -1
  int b, x0i, y0i;
  double u, v, u0, v0, prev_ssd, prev_u, prev_v, prev_off, prev_mar, off0, mar0;
  double mean_t, i00, i01, i11;
  int k, evals;
  bool stop;
};

__device__ __forceinline__ void lane_start(Lane& L, const SearchArgs& a,
                                           const double* __restrict__ prep, unsigned N, int P,
                                           int nx, unsigned g) {
  L.pid = (int)g;
  L.b = (int)(g / (unsigned)P);
  const int i = (int)(g - (unsigned)L.b * (unsigned)P);
  const int iy = i / nx;
  L.x0i = a.ax.origin(i - iy * nx);
  L.y0i = a.ay.origin(iy);
  L.u0 = prep[PR_U0 * (size_t)N + g];
  L.v0 = prep[PR_V0 * (size_t)N + g];
  L.mean_t = prep[PR_MEAN * (size_t)N + g];
  L.i00 = prep[PR_I00 * (size_t)N + g];
  L.i01 = prep[PR_I01 * (size_t)N + g];
  L.i11 = prep[PR_I11 * (size_t)N + g];
  L.stop = !(prep[PR_VALID * (size_t)N + g] != 0.0);
  L.u = L.u0;
  L.v = L.v0;
  L.prev_ssd = 1e300;
  L.prev_u = L.u;
  L.prev_v = L.v;
  L.prev_off = 0.0;
  L.prev_mar = 0.0;
  L.k = 0;
  L.evals = 0;
}

// park / resume the dynamic part of a lane's state (prep fields are reloaded)
__device__ __forceinline__ void lane_park(const Lane& L, double* e) {
  e[0] = (double)L.pid;
  e[1] = L.u;
  e[2] = L.v;
  e[3] = L.prev_ssd;
  e[4] = L.prev_u;
  e[5] = L.prev_v;
  e[6] = L.prev_off;
  e[7] = L.prev_mar;
  e[8] = L.off0;
  e[9] = L.mar0;
  e[10] = (double)L.k;
  e[11] = (double)L.evals;
  e[12] = L.stop ? 1.0 : 0.0;
}
__device__ __forceinline__ void lane_resume(Lane& L, const SearchArgs& a,
                                            const double* __restrict__ prep, unsigned N, int P,
                                            int nx, const double* e) {
  lane_start(L, a, prep, N, P, nx, (unsigned)e[0]);
  L.u = e[1];
  L.v = e[2];
  L.prev_ssd = e[3];
  L.prev_u = e[4];
  L.prev_v = e[5];
  L.prev_off = e[6];
  L.prev_mar = e[7];
  L.off0 = e[8];
  L.mar0 = e[9];
  L.k = (int)e[10];
  L.evals = (int)e[11];
  L.stop = e[12] != 0.0;
}

// Gauss-Newton bookkeeping after one window evaluation
// (inverse_search.py:153-188) + reset_outliers / refresh on exit.  Returns
// true (and writes the patch's outputs) when the patch is finished.
__device__ __forceinline__ bool gn_update(Lane& L, const SearchArgs& a, int ps, double off,
                                          double ssd, double b0, double b1, double mar,
                                          bool writer = true) {
  const double x0 = (double)L.x0i, y0 = (double)L.y0i;
  const int W = a.W, H = a.H;
  if (L.evals == 0) {
    L.off0 = off;
    L.mar0 = mar;
  }
  ++L.evals;
  bool finished = false;
  double u = L.u, v = L.v;
  if (ssd > L.prev_ssd) {
    u = L.prev_u;
    v = L.prev_v;
    off = L.prev_off;
    mar = L.prev_mar;
    finished = true;
  } else if (L.stop || L.k >= a.iters) {
    finished = true;
  } else {
    L.prev_ssd = ssd;
    L.prev_u = u;
    L.prev_v = v;
    L.prev_off = off;
    L.prev_mar = mar;
    const double du = L.i00 * b0 + L.i01 * b1;
    const double dv = L.i01 * b0 + L.i11 * b1;
    u -= du;
    v -= dv;
    L.k += 1;
    if (sqrt(du * du + dv * dv) < 1e-2) L.stop = true;
    const double cx = x0 + u + 0.5 * ps;
    const double cy = y0 + v + 0.5 * ps;
    if (cx < (double)(-W) || cx > 2.0 * W || cy < (double)(-H) || cy > 2.0 * H) {
      u = L.u0;
      v = L.v0;
      L.prev_ssd = 1e300;
      L.stop = true;
    }
    L.u = u;
    L.v = v;
  }
  if (finished) {
    if (hypot_gt(u - L.u0, v - L.v0, ps)) {
      u = L.u0;
      v = L.v0;
      off = a.mean_norm ? L.off0 : 0.0;
      mar = L.mar0;
    }
    if (writer) {
      const size_t o = (size_t)L.pid;
      a.out_u[o] = u;
      a.out_v[o] = v;
      a.out_off[o] = off;
      if (a.out_mar) a.out_mar[o] = mar;
      if (a.out_evals) a.out_evals[o] = L.evals;
      if (a.census) {
        atomicAdd(a.census, (unsigned long long)L.evals);
        atomicAdd(a.census + 1, 1ull);
      }
    }
    L.pid = -1;
  }
  return finished;
}

// bilinear sample from four pixels, the reference's _bilin arithmetic
__device__ __forceinline__ double seg_sample(double i00, double i01, double i10, double i11,
                                             double fx, double fy) {
  const double a = i00 + fx * (i01 - i00);
  const double bb = i10 + fx * (i11 - i10);
  return a + fy * (bb - a);
}

// Is the window at (bx, by) "regular": its ps sample columns (rows) are ps
// consecutive pixels xbase.. (ybase..) with their right (lower) neighbours?
// Then each sample's bilinear operands are segment entries c, c+1 of the
// rows ybase.. ybase+ps.  The lane kernel reads the query level from a copy
// with a replicated border of kQPad pixels (k_pad_query): P[Y][X] = I[clamp(Y)][clamp(X)].  A window
// is then "regular" whenever its samples' integer parts are consecutive in
// padded coordinates, clamped or not, and the clamped samples come out as
// the reference's: where _bilin clamps a coordinate (inverse_search.py:
// 38-45) its two operands along that axis are the same replicated pixel, so
// the interpolant is p + f*(p - p) = p + (+0) for the reference's f = 0 and
// for any other f (the fractions are still taken from the clamped
// coordinate).  The reference forms p + 0*(q - p) with q its unclamped
// neighbour, which differs only in the sign of an exactly-zero sample; a
// sample enters only sums started at +0.0 (which stay +0 under either zero)
// and e = val - off - t, whose sign of zero is squared, absolute-valued or
// multiplied into such a sum — so every output is bit-identical.  Only
// windows reaching more than kQPad pixels past the level still park.
constexpr int kQPad = 16;
__host__ __device__ constexpr int qpad_pitch(int W) { return (W + 2 * kQPad + 4 + 3) & ~3; }
__host__ __device__ constexpr int qpad_rows(int H) { return H + 2 * kQPad; }

__global__ void __launch_bounds__(256) k_pad_query(const double* __restrict__ src, int W, int H,
                                                   double* __restrict__ dst, int pitch) {
  const int b = blockIdx.z;
  const int Y = blockIdx.y;
  const int y = min(max(Y - kQPad, 0), H - 1);
  const double* __restrict__ s = src + ((size_t)b * H + y) * W;
  double2* __restrict__ d =
      reinterpret_cast<double2*>(dst + ((size_t)b * qpad_rows(H) + Y) * pitch);
  for (int X2 = blockIdx.x * blockDim.x + threadIdx.x; X2 < pitch / 2;
       X2 += gridDim.x * blockDim.x) {
    const int x0 = min(max(2 * X2 - kQPad, 0), W - 1);
    const int x1 = min(max(2 * X2 + 1 - kQPad, 0), W - 1);
    d[X2] = make_double2(__ldg(s + x0), __ldg(s + x1));
  }
}

// sample coordinate c's fraction with the reference's clamping (0 where
// _bilin clamps, c - floor(c) elsewhere) and its floor
__device__ __forceinline__ double clamped_frac(double c, double fl, int n) {
  return (c < 0.0 || c > n - 1.0) ? 0.0 : c - fl;
}

template <int PS>
__device__ __forceinline__ bool window_regular_pad(double bx, double by, int W, int H,
                                                   double* FX, int& xbase, int& ybase) {
  if (!(bx >= (double)(-kQPad) && bx < (double)(W - 1 + kQPad - PS) &&
        by >= (double)(-kQPad) && by < (double)(H - 1 + kQPad - PS)))
    return false;  // (also NaN)
  const double flx = floor(bx), fly = floor(by);
  xbase = (int)flx;
  ybase = (int)fly;
  bool regular = true;
#pragma unroll
  for (int o = 0; o < PS; ++o) {
    const double cx = bx + o, cy = by + o;
    const double fx = floor(cx), fy = floor(cy);
    regular = regular && fx - flx == (double)o && fy - fly == (double)o;
    FX[o] = clamped_frac(cx, fx, W);
  }
  return regular;
}

// One window evaluation (the reference's two passes, inverse_search.py:
// 130-152) for a regular window: rows loaded once each as contiguous
// segments with immediate-offset loads, one row ahead of the arithmetic (the
// next row's loads are in flight while this row is interpolated).  Sample
// (oy, c) is _bilin's a + fy*(b - a) with a = row(oy)[c] + fx_c*(row(oy)[c+1]
// - row(oy)[c]) and b the same expression on row oy+1; since fx_c depends on
// the column alone, b of row oy IS a of row oy+1 (same operands, same
// operations), so each row's horizontal interpolants are computed once and
// carried down.  CODE is the residual norm (_transform_residual).
template <int PS, int CODE, int UNR>
__device__ __forceinline__ void eval_regular(const double* __restrict__ qry,
                                             const double* __restrict__ ref,
                                             const double* __restrict__ rgx,
                                             const double* __restrict__ rgy, int W, int H,
                                             int Wq, int x0i, int y0i, double by,
                                             const double* FX, int xbase, int ybase,
                                             double mean_t, bool mean_norm,
                                             double hb, bool tmpl128, bool tmpl256, double& off,
                                             double& ssd, double& b0, double& b1, double& mar) {
  constexpr int S1 = PS + 1;
  constexpr bool kPre = PS <= 8;  // one-row-ahead loads (register budget)
  const double dn = (double)(PS * PS);
  // row oy of the window: elements idx .. idx + PS, idx = (ybase + oy)W + xbase,
  // read as 256-bit loads from the 32-byte aligned element at or below idx
  // (one sector per lane per load instead of one per element) and shifted
  // into place by the lane's offset o = idx mod 4 (two select levels)
  auto load_row = [&](ptrdiff_t idx, double* s) {
    if (PS > 12) {  // (wider rows: the shift registers cost more than the loads save;
                    // measured at 12: c4's patch search 46.8 -> 39.0 ms)
#pragma unroll
      for (int c = 0; c < S1; ++c) s[c] = __ldg(qry + idx + c);
      return;
    }
    load_run256<S1>(qry + idx, s);
  };
  double wsum = 0.0;
#if DIS_GN_PREFETCH & 2
  {  // all window rows into L1 at once (their misses overlap)
    const double* wp = qry + (ptrdiff_t)ybase * Wq + xbase;
#pragma unroll
    for (int oy = 0; oy <= PS; ++oy) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(wp));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(wp + PS));
      wp += Wq;
    }
  }
#endif
#if DIS_GN_PREFETCH & 1
  {  // the template rows pass 2 reads: into L1 while pass 1 runs
    const double* tp = ref + (size_t)y0i * W + x0i;
    const double* xp = rgx + (size_t)y0i * W + x0i;
    const double* yp = rgy + (size_t)y0i * W + x0i;
#pragma unroll
    for (int oy = 0; oy < PS; ++oy) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(tp + PS - 1));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(xp + PS - 1));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(yp + PS - 1));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(tp));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(xp));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(yp));
      tp += W;
      xp += W;
      yp += W;
    }
  }
#endif
  {
    ptrdiff_t idx = (ptrdiff_t)ybase * Wq + xbase;
    double A[PS], s1[S1], s2[kPre ? S1 : 1];
    load_row(idx, s1);
    if (kPre) {
      idx += Wq;
      load_row(idx, s2);
    }
#pragma unroll
    for (int c = 0; c < PS; ++c) A[c] = s1[c] + FX[c] * (s1[c + 1] - s1[c]);
#pragma unroll (UNR)
    for (int oy = 0; oy < PS; ++oy) {
      if (kPre) {
#pragma unroll
        for (int c = 0; c < S1; ++c) s1[c] = s2[c];
        if (oy + 1 < PS) {  // row oy + 2 in flight during this row's arithmetic
          idx += Wq;
          load_row(idx, s2);
        }
      } else {
        idx += Wq;
        load_row(idx, s1);
      }
      const double fy = axis_sample(by + oy, H).f;
#pragma unroll
      for (int ox = 0; ox < PS; ++ox) {
        const double Bv = s1[ox] + FX[ox] * (s1[ox + 1] - s1[ox]);
        wsum += A[ox] + fy * (Bv - A[ox]);
        A[ox] = Bv;
      }
    }
  }
  off = mean_norm ? exact_div_pos(wsum, dn) - mean_t : 0.0;
  ssd = 0.0;
  b0 = 0.0;
  b1 = 0.0;
  mar = 0.0;
  auto accumulate = [&](double val, double t, double gxv, double gyv) {
    const double e = val - off - t;
    mar += fabs(e);
    const double et = transform_residual(e, CODE, hb);
    ssd += et * et;
    b0 += gxv * et;
    b1 += gyv * et;
  };
  {
    ptrdiff_t idx = (ptrdiff_t)ybase * Wq + xbase;
    double A[PS], s1[S1], s2[kPre ? S1 : 1];
    load_row(idx, s1);
    if (kPre) {
      idx += Wq;
      load_row(idx, s2);
    }
#pragma unroll
    for (int c = 0; c < PS; ++c) A[c] = s1[c] + FX[c] * (s1[c + 1] - s1[c]);
    const double* tr = ref + (size_t)y0i * W + x0i;
    const double* gxr = rgx + (size_t)y0i * W + x0i;
    const double* gyr = rgy + (size_t)y0i * W + x0i;
#pragma unroll (UNR)
    for (int oy = 0; oy < PS; ++oy) {
      if (kPre) {
#pragma unroll
        for (int c = 0; c < S1; ++c) s1[c] = s2[c];
        if (oy + 1 < PS) {
          idx += Wq;
          load_row(idx, s2);
        }
      } else {
        idx += Wq;
        load_row(idx, s1);
      }
      const double fy = axis_sample(by + oy, H).f;
      if (tmpl256) {  // template rows 32-byte aligned across the warp
#pragma unroll
        for (int ox = 0; ox < PS; ox += 4) {
          double t[4], gx[4], gy[4];
          ldg256(tr + ox, t);
          ldg256(gxr + ox, gx);
          ldg256(gyr + ox, gy);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double Bv = s1[ox + q] + FX[ox + q] * (s1[ox + q + 1] - s1[ox + q]);
            accumulate(A[ox + q] + fy * (Bv - A[ox + q]), t[q], gx[q], gy[q]);
            A[ox + q] = Bv;
          }
        }
      } else if (tmpl128) {
#pragma unroll
        for (int ox = 0; ox < PS; ox += 2) {
          const double2 t = __ldg(reinterpret_cast<const double2*>(tr + ox));
          const double2 gx = __ldg(reinterpret_cast<const double2*>(gxr + ox));
          const double2 gy = __ldg(reinterpret_cast<const double2*>(gyr + ox));
          const double B0 = s1[ox] + FX[ox] * (s1[ox + 1] - s1[ox]);
          accumulate(A[ox] + fy * (B0 - A[ox]), t.x, gx.x, gy.x);
          A[ox] = B0;
          const double B1 = s1[ox + 1] + FX[ox + 1] * (s1[ox + 2] - s1[ox + 1]);
          accumulate(A[ox + 1] + fy * (B1 - A[ox + 1]), t.y, gx.y, gy.y);
          A[ox + 1] = B1;
        }
      } else {
#pragma unroll
        for (int ox = 0; ox < PS; ++ox) {
          const double Bv = s1[ox] + FX[ox] * (s1[ox + 1] - s1[ox]);
          accumulate(A[ox] + fy * (Bv - A[ox]), __ldg(tr + ox), __ldg(gxr + ox),
                     __ldg(gyr + ox));
          A[ox] = Bv;
        }
      }
      tr += W;
      gxr += W;
      gyr += W;
    }
  }
  mar = exact_div_pos(mar, dn);
}

// 8-pixel patches, template rows 32-byte aligned: the same evaluation with the
// window's samples kept in registers between the passes (pass 2 reads them
// back instead of reloading and re-interpolating the window rows) and pass
// 2's template rows loaded one row ahead of their arithmetic (their load
// latency was 60 % of the kernel's long-scoreboard stalls).  Same values,
// same sums in the same order: bit-identical to eval_regular.
template <int CODE>
__device__ __forceinline__ void eval_regular8_t256(
    const double* __restrict__ qry, const double* __restrict__ ref,
    const double* __restrict__ rgx, const double* __restrict__ rgy, int W, int H, int Wq,
    int x0i, int y0i, double by, const double* FX, int xbase, int ybase, double mean_t,
    bool mean_norm, double hb, double& off, double& ssd, double& b0, double& b1, double& mar) {
  constexpr int PS = 8, S1 = PS + 1;
  const double dn = (double)(PS * PS);
  double V[PS * PS];
  double wsum = 0.0;
  {
    ptrdiff_t idx = (ptrdiff_t)ybase * Wq + xbase;
    double A[PS], s1[S1], s2[S1];
    load_run256<S1>(qry + idx, s1);
    idx += Wq;
    load_run256<S1>(qry + idx, s2);
#pragma unroll
    for (int c = 0; c < PS; ++c) A[c] = s1[c] + FX[c] * (s1[c + 1] - s1[c]);
#pragma unroll
    for (int oy = 0; oy < PS; ++oy) {
#pragma unroll
      for (int c = 0; c < S1; ++c) s1[c] = s2[c];
      if (oy + 1 < PS) {
        idx += Wq;
        load_run256<S1>(qry + idx, s2);
      }
      const double fy = axis_sample(by + oy, H).f;
#pragma unroll
      for (int ox = 0; ox < PS; ++ox) {
        const double Bv = s1[ox] + FX[ox] * (s1[ox + 1] - s1[ox]);
        V[oy * PS + ox] = A[ox] + fy * (Bv - A[ox]);
        wsum += V[oy * PS + ox];
        A[ox] = Bv;
      }
    }
  }
  const double* tr = ref + (size_t)y0i * W + x0i;
  const double* gxr = rgx + (size_t)y0i * W + x0i;
  const double* gyr = rgy + (size_t)y0i * W + x0i;
  double T[2][3][PS];  // template rows oy (arithmetic) and oy + 1 (in flight)
  auto load_t = [&](int oy, double (*t)[PS]) {
#pragma unroll
    for (int ox = 0; ox < PS; ox += 4) {
      ldg256(tr + (size_t)oy * W + ox, t[0] + ox);
      ldg256(gxr + (size_t)oy * W + ox, t[1] + ox);
      ldg256(gyr + (size_t)oy * W + ox, t[2] + ox);
    }
  };
  load_t(0, T[0]);
  off = mean_norm ? exact_div_pos(wsum, dn) - mean_t : 0.0;
  ssd = 0.0;
  b0 = 0.0;
  b1 = 0.0;
  mar = 0.0;
#pragma unroll
  for (int oy = 0; oy < PS; ++oy) {
    if (oy + 1 < PS) load_t(oy + 1, T[(oy + 1) & 1]);
#pragma unroll
    for (int ox = 0; ox < PS; ++ox) {
      const double e = V[oy * PS + ox] - off - T[oy & 1][0][ox];
      mar += fabs(e);
      const double et = transform_residual(e, CODE, hb);
      ssd += et * et;
      b0 += T[oy & 1][1][ox] * et;
      b1 += T[oy & 1][2][ox] * et;
    }
  }
  mar = exact_div_pos(mar, dn);
}

// One window evaluation for any window and patch size: every sample gathers
// its own four pixels with the reference's clamping.
__device__ __forceinline__ void eval_general(const double* __restrict__ qry,
                                             const double* __restrict__ ref,
                                             const double* __restrict__ rgx,
                                             const double* __restrict__ rgy, int W, int H,
                                             int ps, int x0i, int y0i, double bx, double by,
                                             double mean_t, bool mean_norm, int code, double hb,
                                             double& off, double& ssd, double& b0, double& b1,
                                             double& mar) {
  const double dn = (double)(ps * ps);
  double wsum = 0.0;
  for (int oy = 0; oy < ps; ++oy) {
    const Axis1 ay = axis_sample(by + oy, H);
    const double* r0 = qry + (size_t)ay.i0 * W;
    const double* r1 = qry + (size_t)ay.i1 * W;
    for (int ox = 0; ox < ps; ++ox) {
      const Axis1 ax = axis_sample(bx + ox, W);
      wsum += seg_sample(__ldg(r0 + ax.i0), __ldg(r0 + ax.i1), __ldg(r1 + ax.i0),
                         __ldg(r1 + ax.i1), ax.f, ay.f);
    }
  }
  off = mean_norm ? exact_div_pos(wsum, dn) - mean_t : 0.0;
  ssd = 0.0;
  b0 = 0.0;
  b1 = 0.0;
  mar = 0.0;
  for (int oy = 0; oy < ps; ++oy) {
    const Axis1 ay = axis_sample(by + oy, H);
    const double* r0 = qry + (size_t)ay.i0 * W;
    const double* r1 = qry + (size_t)ay.i1 * W;
    const size_t row = (size_t)(y0i + oy) * W + x0i;
    for (int ox = 0; ox < ps; ++ox) {
      const Axis1 ax = axis_sample(bx + ox, W);
      const double val = seg_sample(__ldg(r0 + ax.i0), __ldg(r0 + ax.i1), __ldg(r1 + ax.i0),
                                    __ldg(r1 + ax.i1), ax.f, ay.f);
      const double e = val - off - __ldg(ref + row + ox);
      mar += fabs(e);
      const double et = transform_residual(e, code, hb);
      ssd += et * et;
      b0 += __ldg(rgx + row + ox) * et;
      b1 += __ldg(rgy + row + ox) * et;
    }
  }
  mar = exact_div_pos(mar, dn);
}

// Fine levels: one lane per patch, regular windows only.  Lanes refill from
// a warp pool of consecutive patches (one grid-row segment, so neighbouring
// lanes read the same image rows and share L1 lines).  A patch whose next
// window is not regular is parked (state to the spill list) and finished by
// k_patch_gn_general — this keeps the warp on one code path.
// Blocks per SM (MINB) and the row loops' unroll: 8px patches run one
// 256-lane block per SM with the rows fully unrolled (no register rotation
// of the prefetched rows and interpolants; 238 registers; c1 1.50 -> 1.37
// ms against 2 blocks with rolled loops).  12px patches: one block with the
// rows unrolled by 2 on levels up to 1 Mpixel (c2 8.1 -> 7.5 ms), two blocks
// with rolled rows on larger ones (better at c4's 1920x1080 level, whose
// gathers miss L1 more often).
template <int PS, int CODE, int MINB>
__global__ void __launch_bounds__(256, MINB) k_patch_gn(SearchArgs a,
                                                     const double* __restrict__ prep,
                                                     unsigned* counter, double* spill,
                                                     unsigned* spill_count) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int nx = a.ax.n;
  const int P = nx * a.ay.n;
  const unsigned N = (unsigned)(a.B * P);
  const int W = a.W, H = a.H;
  const size_t plane = (size_t)W * H;
  const int Wq = a.qp_pitch;
  const size_t qplane = (size_t)qpad_rows(H) * Wq;
  const bool mean_norm = a.mean_norm != 0;
  // the lane's Gauss-Newton state lives in shared memory (touched a few
  // times per window evaluation): the registers go to the window rows
  __shared__ Lane lanes[256];
  Lane& L = lanes[threadIdx.x];
  L.pid = -1;
  bool done = false;
  bool drained = false;  // warp-uniform: the work queue had nothing left for this warp
  unsigned pool_next = 0, pool_end = 0;  // warp-uniform
  // block ranges (see kRangeCounters); victim = the range refills come from
  const unsigned nb = gridDim.x;
  unsigned victim = blockIdx.x, tried = 0;
  auto range_start = [&](unsigned v) {
    return (unsigned)(((unsigned long long)N * v) / nb);
  };
  for (;;) {
    const bool need = !done && L.pid < 0;
    unsigned mask = __ballot_sync(FULL, need);
    unsigned g = 0xffffffffu;
    while (mask) {
      if (pool_next >= pool_end) {
        bool got = false;
        while (tried < nb) {  // own range first, then the following blocks'
          const unsigned rs = range_start(victim);
          unsigned re = range_start(victim + 1);
          unsigned base = 0;
          if (lane == 0)
            base = DIS_GN_RANGES ? rs + atomicAdd(counter + kRangeCounters + victim, kPool)
                                 : atomicAdd(counter, kPool);
          if (!DIS_GN_RANGES) re = N;
          base = __shfl_sync(FULL, base, 0);
          if (base < re) {
            pool_next = base;
            pool_end = base + kPool < re ? base + kPool : re;
            got = true;
            break;
          }
          tried = DIS_GN_RANGES ? tried + 1 : nb;
          victim = victim + 1 == nb ? 0 : victim + 1;
        }
        if (!got) {
          drained = true;
          break;
        }
      }
      const unsigned avail = pool_end - pool_next;
      const unsigned rank = (unsigned)__popc(mask & ((1u << lane) - 1u));
      const bool mine = ((mask >> lane) & 1u) && rank < avail;
      if (mine) g = pool_next + rank;
      const unsigned took = __ballot_sync(FULL, mine);
      pool_next += (unsigned)__popc(took);
      mask &= ~took;
    }
    if (need) {
      if (g == 0xffffffffu)
        done = true;
      else
        lane_start(L, a, prep, N, P, nx, g);
    }
    if (__all_sync(FULL, done)) break;
    // Stragglers: with the queue empty, a warp whose last few patches keep
    // iterating (mean 3-5.5 evaluations, p99 22) runs at a
    // few lanes of 32 and one evaluation of its serial chain takes as long
    // as ever.  Such a warp parks its running patches (the same exact
    // park/resume as the irregular windows: the state is complete between
    // evaluations) for the lane-group kernel, whose 8 / 16 lanes per patch
    // finish an evaluation several times sooner and spread over all SMs.
    if (drained && a.stragglers > 0) {
      const unsigned act = __ballot_sync(FULL, !done);
      if (__popc(act) <= a.stragglers) {
        if (!done) {
          const unsigned slot = atomicAdd(spill_count, 1u);
          lane_park(L, spill + (size_t)slot * kSpillStride);
        }
        break;
      }
    }
    if (done) continue;

    const double bx = (double)L.x0i + L.u, by = (double)L.y0i + L.v;
    double FX[PS];
    int xbase, ybase;
    if (!window_regular_pad<PS>(bx, by, W, H, FX, xbase, ybase)) {
      const unsigned slot = atomicAdd(spill_count, 1u);
      lane_park(L, spill + (size_t)slot * kSpillStride);
      L.pid = -1;
      continue;
    }
    const size_t po = (size_t)L.b * plane;
    // template rows at (y0i + oy) W + x0i of the pair's rasters: 16 / 32-byte
    // aligned when the element offset and the row pitch are even / multiples of 4
    const size_t toff = po + (size_t)L.y0i * W + L.x0i;
    const unsigned am = __activemask();
    const bool tmpl128 = (PS & 1) == 0 && __all_sync(am, ((toff | (size_t)W) & 1) == 0);
    const bool tmpl256 = (PS & 3) == 0 && __all_sync(am, ((toff | (size_t)W) & 3) == 0);
    // the pair's padded query level, at its pixel (0, 0)
    const double* qp = a.qpad + (size_t)L.b * qplane + (size_t)kQPad * Wq + kQPad;
    double off, ssd, b0, b1, mar;
    if (PS == 8 && tmpl256)
      eval_regular8_t256<CODE>(qp, a.ref + po, a.rgx + po, a.rgy + po, W, H, Wq, L.x0i, L.y0i,
                               by, FX, xbase, ybase, L.mean_t, mean_norm, a.hb, off, ssd, b0,
                               b1, mar);
    else
      eval_regular<PS, CODE, (PS == 8 ? PS : (MINB == 1 ? 2 : 1))>(
          qp, a.ref + po, a.rgx + po, a.rgy + po, W, H, Wq, L.x0i, L.y0i, by, FX, xbase, ybase,
          L.mean_t, mean_norm, a.hb, tmpl128, tmpl256, off, ssd, b0, b1, mar);
    gn_update(L, a, PS, off, ssd, b0, b1, mar);
  }
}

// Any patch size / parked patches: one lane per patch, general windows.
// from_spill = true: resume the parked patches k_patch_gn left behind;
// false: run every patch of the level from its start (patch sizes without a
// specialised fast kernel).
__global__ void __launch_bounds__(128) k_patch_gn_general(SearchArgs a,
                                                          const double* __restrict__ prep,
                                                          const double* __restrict__ spill,
                                                          const unsigned* spill_count,
                                                          bool from_spill) {
  const int nx = a.ax.n;
  const int P = nx * a.ay.n;
  const unsigned N = (unsigned)(a.B * P);
  const unsigned count = from_spill ? *spill_count : N;
  const int W = a.W, H = a.H;
  const size_t plane = (size_t)W * H;
  const bool mean_norm = a.mean_norm != 0;
  for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < count;
       idx += gridDim.x * blockDim.x) {
    Lane L;
    if (from_spill)
      lane_resume(L, a, prep, N, P, nx, spill + (size_t)idx * kSpillStride);
    else
      lane_start(L, a, prep, N, P, nx, idx);
    const size_t po = (size_t)L.b * plane;
    for (;;) {
      double off, ssd, b0, b1, mar;
      eval_general(a.qry + po, a.ref + po, a.rgx + po, a.rgy + po, W, H, a.ps, L.x0i, L.y0i,
                   (double)L.x0i + L.u, (double)L.y0i + L.v, L.mean_t, mean_norm, a.code, a.hb,
                   off, ssd, b0, b1, mar);
      if (gn_update(L, a, a.ps, off, ssd, b0, b1, mar)) break;
    }
  }
}

// ---------------------------------------------------------------------------
// Stage 2, coarse levels — the same Gauss-Newton loop with a GROUP of G lanes
// per patch (lane r owns window row r).  Small levels have too few patches to
// fill the GPU, so a lane-per-patch kernel is bound by one lane's serial
// latency (two passes x ps rows of loads and sums).  Here the rows' loads and
// bilinear samples run in parallel; the reference's row-major sums stay
// exactly sequential: row r's lane adds its ps values to the running sums it
// receives from row r-1's lane (warp shuffle), so every sum is formed in the
// same order as the reference's loop.  All lanes of a group hold the same
// patch state and apply the same update.
// ---------------------------------------------------------------------------
// (3 blocks per SM for 8px patches: 168 registers, measured best; 12px
// patches keep the compiler's choice)
template <int PS, int G, int CODE>
__global__ void __launch_bounds__(128, PS == 8 ? 3 : 1) k_patch_gn_group(SearchArgs a,
                                                         const double* __restrict__ prep,
                                                         unsigned* counter,
                                                         const double* __restrict__ spill,
                                                         const unsigned* spill_count,
                                                         bool from_spill) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int r = lane & (G - 1);  // my window row
  const int gbase = lane - r;
  const int nx = a.ax.n;
  const int P = nx * a.ay.n;
  const unsigned N = (unsigned)(a.B * P);
  const unsigned limit = from_spill ? *spill_count : N;
  unsigned* queue = from_spill ? counter + 2 : counter;
  const int W = a.W, H = a.H;
  const size_t plane = (size_t)W * H;
  const bool mean_norm = a.mean_norm != 0;
  const double dn = (double)(PS * PS);
  const int rr_row = r < PS ? r : PS - 1;
  // my window row's template samples and gradients, constant per patch:
  // loaded once per patch (not once per evaluation), lane-minor layout
  __shared__ double2 Ts[3 * PS / 2][128];
  Lane L;
  L.pid = -1;
  L.b = L.x0i = L.y0i = 0;  // an idle group evaluates a harmless in-bounds window
  L.u = L.v = 0.0;
  bool done = false;
  for (;;) {
    // ---- fetch (one patch per group; the group's lane 0 asks) ----
    const bool need = !done && L.pid < 0;
    const unsigned mask = __ballot_sync(FULL, need && r == 0);
    if (mask) {
      const int leader = __ffs(mask) - 1;
      unsigned base = 0;
      if (lane == leader) base = atomicAdd(queue, (unsigned)__popc(mask));
      base = __shfl_sync(FULL, base, leader);
      const unsigned g = base + (unsigned)__popc(mask & ((1u << gbase) - 1u));
      if (need) {
        if (g >= limit)
          done = true;
        else if (from_spill)
          lane_resume(L, a, prep, N, P, nx, spill + (size_t)g * kSpillStride);
        else
          lane_start(L, a, prep, N, P, nx, g);
        if (!done) {  // my template row of the new patch -> shared memory
          const size_t trow = (size_t)L.b * plane + (size_t)(L.y0i + rr_row) * W + L.x0i;
#pragma unroll
          for (int c = 0; c < PS; c += 2) {
            Ts[c / 2][threadIdx.x] = make_double2(__ldg(a.ref + trow + c), __ldg(a.ref + trow + c + 1));
            Ts[PS / 2 + c / 2][threadIdx.x] =
                make_double2(__ldg(a.rgx + trow + c), __ldg(a.rgx + trow + c + 1));
            Ts[PS + c / 2][threadIdx.x] =
                make_double2(__ldg(a.rgy + trow + c), __ldg(a.rgy + trow + c + 1));
          }
        }
      }
    }
    if (__all_sync(FULL, done)) break;
    const bool live = !done;  // whole group agrees

    // ---- window evaluation: my row's samples ----
    const size_t po = (size_t)(live ? L.b : 0) * plane;
    const double* __restrict__ qry = a.qry + po;
    const double bx = (double)L.x0i + L.u, by = (double)L.y0i + L.v;
    double FX[PS];
    int xbase = 0;
    bool regx = true;
#pragma unroll
    for (int o = 0; o < PS; ++o) {
      const Axis1 ax = axis_sample(bx + o, W);
      if (o == 0) xbase = ax.i0;
      regx = regx && ax.i0 == xbase + o && ax.i1 == ax.i0 + 1;
      FX[o] = ax.f;
    }
    const Axis1 ay = axis_sample(by + rr_row, H);
    double val[PS];
    if (regx) {
      const double* r0 = qry + (size_t)ay.i0 * W + xbase;
      const double* r1 = qry + (size_t)ay.i1 * W + xbase;
      double s0[PS + 1], s1[PS + 1];
      if (PS <= 12) {
        load_run256<PS + 1>(r0, s0);
        load_run256<PS + 1>(r1, s1);
      } else {
#pragma unroll
        for (int c = 0; c <= PS; ++c) {
          s0[c] = __ldg(r0 + c);
          s1[c] = __ldg(r1 + c);
        }
      }
#pragma unroll
      for (int c = 0; c < PS; ++c)
        val[c] = seg_sample(s0[c], s0[c + 1], s1[c], s1[c + 1], FX[c], ay.f);
    } else {
      const double* r0 = qry + (size_t)ay.i0 * W;
      const double* r1 = qry + (size_t)ay.i1 * W;
#pragma unroll
      for (int c = 0; c < PS; ++c) {
        const Axis1 ax = axis_sample(bx + c, W);
        val[c] = seg_sample(__ldg(r0 + ax.i0), __ldg(r0 + ax.i1), __ldg(r1 + ax.i0),
                            __ldg(r1 + ax.i1), ax.f, ay.f);
      }
    }
    // pass 1: wsum over rows in order (row rr's lane continues the chain)
    double wsum = 0.0;
#pragma unroll
    for (int rr = 0; rr < PS; ++rr) {
      double acc = wsum;
#pragma unroll
      for (int c = 0; c < PS; ++c) acc += val[c];
      wsum = __shfl_sync(FULL, acc, gbase + rr);
    }
    const double off = mean_norm ? exact_div_pos(wsum, dn) - L.mean_t : 0.0;
    // pass 2: the addends of my row, then the four sums in row order
    double EA[PS], E2[PS], EX[PS], EY[PS];
    auto addends = [&](int c, double t, double gxv, double gyv) {
      const double e = val[c] - off - t;
      EA[c] = fabs(e);
      const double et = transform_residual(e, CODE, a.hb);
      E2[c] = et * et;
      EX[c] = gxv * et;
      EY[c] = gyv * et;
    };
#pragma unroll
    for (int c = 0; c < PS; c += 2) {
      const double2 t = Ts[c / 2][threadIdx.x];
      const double2 gx2 = Ts[PS / 2 + c / 2][threadIdx.x];
      const double2 gy2 = Ts[PS + c / 2][threadIdx.x];
      addends(c, t.x, gx2.x, gy2.x);
      addends(c + 1, t.y, gx2.y, gy2.y);
    }
    double mar = 0.0, ssd = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int rr = 0; rr < PS; ++rr) {
      double am = mar, as = ssd, a0 = b0, a1 = b1;
#pragma unroll
      for (int c = 0; c < PS; ++c) {
        am += EA[c];
        as += E2[c];
        a0 += EX[c];
        a1 += EY[c];
      }
      mar = __shfl_sync(FULL, am, gbase + rr);
      ssd = __shfl_sync(FULL, as, gbase + rr);
      b0 = __shfl_sync(FULL, a0, gbase + rr);
      b1 = __shfl_sync(FULL, a1, gbase + rr);
    }
    mar = exact_div_pos(mar, dn);
    if (!live) continue;
    // ---- Gauss-Newton update (replicated in the group; lane 0 writes) ----
    gn_update(L, a, PS, off, ssd, b0, b1, mar, r == 0);
  }
}

template <int PS, int G, int CODE>
static void launch_gn_group_code(const SearchArgs& a, const double* prep, unsigned* counter,
                                 size_t n, cudaStream_t st, const double* spill,
                                 const unsigned* spill_count, bool from_spill) {
  static int caps[kMaxDevices];
  int& cap = caps[current_device()];
  if (!cap) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_patch_gn_group<PS, G, CODE>, 128,
                                                  0);
    cap = (per_sm > 0 ? per_sm : 1) * device_sm_count();
  }
  const size_t need = (n * G + 127) / 128;
  int blocks = (int)(need < (size_t)cap ? need : (size_t)cap);
  if (blocks < 1) blocks = 1;
  k_patch_gn_group<PS, G, CODE><<<blocks, 128, 0, st>>>(a, prep, counter, spill, spill_count,
                                                         from_spill);
}

template <int PS, int G>
static void launch_gn_group(const SearchArgs& a, const double* prep, unsigned* counter,
                            size_t n, cudaStream_t st, const double* spill = nullptr,
                            const unsigned* spill_count = nullptr, bool from_spill = false) {
  if (a.code == DIS_NORM_L1)
    launch_gn_group_code<PS, G, DIS_NORM_L1>(a, prep, counter, n, st, spill, spill_count,
                                             from_spill);
  else if (a.code == DIS_NORM_HUBER)
    launch_gn_group_code<PS, G, DIS_NORM_HUBER>(a, prep, counter, n, st, spill, spill_count,
                                                from_spill);
  else
    launch_gn_group_code<PS, G, DIS_NORM_L2>(a, prep, counter, n, st, spill, spill_count,
                                             from_spill);
}

template <int PS, int CODE, int MINB>
static void launch_gn_lane_minb(const SearchArgs& a, const double* prep, unsigned* counter,
                                double* spill, unsigned* spill_count, size_t n, int sms,
                                cudaStream_t st) {
  static int per_sms[kMaxDevices];
  int& per_sm = per_sms[current_device()];
  if (!per_sm) {
#if DIS_GN_CARVEOUT >= 0
    cudaFuncSetAttribute(k_patch_gn<PS, CODE, MINB>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, DIS_GN_CARVEOUT);
#endif
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_patch_gn<PS, CODE, MINB>, 256, 0);
    if (per_sm < 1) per_sm = 1;
  }
  size_t blocks = (size_t)per_sm * sms;
  if (blocks > (size_t)kMaxGnBlocks) blocks = kMaxGnBlocks;
  const size_t need = (n + 255) / 256;
  if (blocks > need) blocks = need;
  k_patch_gn<PS, CODE, MINB>
      <<<(unsigned)blocks, 256, 0, st>>>(a, prep, counter, spill, spill_count);
}

template <int PS, int CODE>
static void launch_gn_lane_code(const SearchArgs& a, const double* prep, unsigned* counter,
                                double* spill, unsigned* spill_count, size_t n, int sms,
                                cudaStream_t st) {
  if constexpr (PS == 12) {
    if ((size_t)a.W * a.H > ((size_t)1 << 20)) {
      launch_gn_lane_minb<PS, CODE, 2>(a, prep, counter, spill, spill_count, n, sms, st);
      return;
    }
  }
  launch_gn_lane_minb<PS, CODE, 1>(a, prep, counter, spill, spill_count, n, sms, st);
}

template <int PS>
static void launch_gn_lane(const SearchArgs& a, const double* prep, unsigned* counter,
                           double* spill, unsigned* spill_count, size_t n, cudaStream_t st) {
  const int sms = device_sm_count();
  if (a.code == DIS_NORM_L1)
    launch_gn_lane_code<PS, DIS_NORM_L1>(a, prep, counter, spill, spill_count, n, sms, st);
  else if (a.code == DIS_NORM_HUBER)
    launch_gn_lane_code<PS, DIS_NORM_HUBER>(a, prep, counter, spill, spill_count, n, sms, st);
  else
    launch_gn_lane_code<PS, DIS_NORM_L2>(a, prep, counter, spill, spill_count, n, sms, st);
}

// lane-group kernel up to ~2 (8px) / ~4 (12px) waves of group lanes; above, the
// lane kernel (measured: c1's 256x109 level, 105k patches, is 0.03 ms faster
// on the 8px lane kernel; c2's 256x109 level is faster on the group kernel)
constexpr size_t kGroupLanes8 = (size_t)148 * 2048 * 2;
constexpr size_t kGroupLanes12 = (size_t)148 * 2048 * 4;

static size_t search_state_bytes(int B, int P) {
  return (((size_t)(kPrep + kSpillStride) * B * P) * sizeof(double) +
          (kRangeCounters + kMaxGnBlocks) * sizeof(unsigned) + 255) & ~size_t(255);
}

size_t patch_search_scratch_bytes(int B, int P, int W, int H) {
  return search_state_bytes(B, P) + (size_t)B * qpad_rows(H) * qpad_pitch(W) * sizeof(double);
}

void launch_patch_search(const SearchArgs& a, void* scratch, cudaStream_t st) {
  const size_t n = (size_t)a.B * a.ax.n * a.ay.n;
  double* prep = static_cast<double*>(scratch);
  double* spill = prep + (size_t)kPrep * n;
  unsigned* counter = reinterpret_cast<unsigned*>(spill + (size_t)kSpillStride * n);
  unsigned* spill_count = counter + 1;
  prof_begin(KC_SEARCH, st);
  const int TH = 128;
  k_patch_prep<<<(unsigned)((n + TH - 1) / TH), TH, 0, st>>>(a, prep, counter);
  note_launch();
  static const size_t forced = [] {
    const char* e = getenv("DIS_GROUP_LANES");  // experiments only
    return e ? (size_t)atoll(e) : 0;
  }();
  const size_t glanes = forced ? forced : (a.ps == 8 ? kGroupLanes8 : kGroupLanes12);
  // coarse levels (few patches): a group of lanes per patch; fine levels: a
  // lane per patch (+ the general kernel for the parked, irregular windows)
  const bool group = (a.ps == 8 && n * 8 <= glanes) || (a.ps == 12 && n * 16 <= glanes);
  if (group) {
    if (a.ps == 8)
      launch_gn_group<8, 8>(a, prep, counter, n, st);
    else
      launch_gn_group<12, 16>(a, prep, counter, n, st);
    note_launch();
  } else if (a.ps == 8 || a.ps == 12) {
    // the query level with its replicated border (see kQPad)
    SearchArgs al = a;
    static const int stragglers = [] {
      const char* e = getenv("DIS_GN_STRAGGLERS");  // experiments only
      return e ? atoi(e) : kStragglers;
    }();
    al.stragglers = stragglers;
    double* qpad = reinterpret_cast<double*>(static_cast<char*>(scratch) +
                                             search_state_bytes(a.B, a.ax.n * a.ay.n));
    al.qpad = qpad;
    al.qp_pitch = qpad_pitch(a.W);
    {
      const int half = al.qp_pitch / 2;
      const unsigned bx = (unsigned)((half + 255) / 256);
      k_pad_query<<<dim3(bx, (unsigned)qpad_rows(a.H), (unsigned)a.B), 256, 0, st>>>(
          a.qry, a.W, a.H, qpad, al.qp_pitch);
      note_launch();
    }
    if (a.ps == 8)
      launch_gn_lane<8>(al, prep, counter, spill, spill_count, n, st);
    else
      launch_gn_lane<12>(al, prep, counter, spill, spill_count, n, st);
    note_launch();
    // parked (irregular-window) patches: a lane group per patch
    if (a.ps == 8)
      launch_gn_group<8, 8>(a, prep, counter, n, st, spill, spill_count, true);
    else
      launch_gn_group<12, 16>(a, prep, counter, n, st, spill, spill_count, true);
    note_launch();
  } else {
    size_t blocks = (n + 127) / 128;
    k_patch_gn_general<<<(unsigned)blocks, 128, 0, st>>>(a, prep, spill, spill_count, false);
    note_launch();
  }
  prof_end(KC_SEARCH, st);
}

}  // namespace disb200
