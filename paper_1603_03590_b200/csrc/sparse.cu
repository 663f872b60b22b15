// sparse.cu — sparse correspondences (sparse_correspondences, pipeline.py:
// 230-287): displacements at seed locations only.
//
//   k_sparse_chain  : _sparse_chain (pipeline.py:202-227) — one thread per
//                     seed carries its own patch down the scales: window
//                     origin clip(seed/2^s - ps/2, 0, dim - ps) (a real
//                     coordinate, so the template, S' and Hessian are
//                     bilinear samples, _patch_precompute inverse_search.py:
//                     75-98), _condition_hessians, then _patch_optimize
//                     (113-189) from 0 at the coarsest scale or 2x the
//                     previous scale's displacement; no outlier reset.
//   k_sparse_sample : densified mode — the finest computed scale's dense
//                     field (unrefined, _dense_scales refine=False) sampled
//                     with bilinear_map at seed / 2^sf, times 2^sf.
//
// Seeds are few and independent, so a seed is a thread and its ps^2
// template/gradient samples live in a per-seed slice of the workspace.
#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

__global__ void __launch_bounds__(128) k_sparse_chain(SparseChainArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n || !a.valid[i]) return;
  const int ps = a.ps, nn = ps * ps;
  double* tmpl = a.scratch + (size_t)i * 3 * nn;
  double* sdx = tmpl + nn;
  double* sdy = sdx + nn;
  const double sx = a.seeds[2 * i], sy = a.seeds[2 * i + 1];
  double u = 0.0, v = 0.0;
  const double kd = (double)a.ds;
  double scale = 1.0;  // params.downscale ** s (pipeline.py:213), exact
  for (int s = 0; s < a.coarsest; ++s) scale *= kd;
  for (int s = a.coarsest; s >= a.finest; --s, scale /= kd) {
    const int W = a.W[s], H = a.H[s];
    const double* __restrict__ img = a.img[s];
    const double* __restrict__ gx = a.gx[s];
    const double* __restrict__ gy = a.gy[s];
    const double* __restrict__ q = a.qry[s];
    // pipeline.py:215-218
    double x0 = sx / scale - 0.5 * ps;
    double y0 = sy / scale - 0.5 * ps;
    x0 = x0 < 0.0 ? 0.0 : x0;
    x0 = x0 > (double)(W - ps) ? (double)(W - ps) : x0;
    y0 = y0 < 0.0 ? 0.0 : y0;
    y0 = y0 > (double)(H - ps) ? (double)(H - ps) : y0;
    // _patch_precompute (inverse_search.py:75-98)
    double tsum = 0.0, h00 = 0.0, h01 = 0.0, h11 = 0.0;
    int k = 0;
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
    const double mean_t = tsum / (double)nn;
    // _condition_hessians (inverse_search.py:266-276)
    const double tr = h00 + h11;
    const double det = h00 * h11 - h01 * h01;
    const double qq = 0.25 * tr * tr;
    const double rel = isnan(qq) ? qq : (1.0 > qq ? 1.0 : qq);
    const double arg = tr * tr - 4.0 * det;
    const double disc = sqrt(isnan(arg) ? arg : (arg > 0.0 ? arg : 0.0));
    const double lmin = 0.5 * (tr - disc);
    const double lmax = 0.5 * (tr + disc);
    const bool valid = (det > 1e-6 * rel) && (lmin > 0.0) && (lmax <= 1e6 * lmin);
    const double i00 = valid ? h11 / det : 0.0;
    const double i01 = valid ? -h01 / det : 0.0;
    const double i11 = valid ? h00 / det : 0.0;
    // _patch_optimize (inverse_search.py:113-189)
    const double u0 = s == a.coarsest ? 0.0 : u * kd;  // init_displacement * downscale
    const double v0 = s == a.coarsest ? 0.0 : v * kd;
    u = u0;
    v = v0;
    double prev_ssd = 1e300, prev_u = u, prev_v = v;
    bool stop = !valid;
    int it = 0;
    for (;;) {
      const double bx = x0 + u, by = y0 + v;
      double wsum = 0.0;
      for (int oy = 0; oy < ps; ++oy)
        for (int ox = 0; ox < ps; ++ox) wsum += bilin_nb(q, W, H, bx + ox, by + oy);
      const double off = a.mean_norm ? wsum / (double)nn - mean_t : 0.0;
      double ssd = 0.0, b0 = 0.0, b1 = 0.0;
      k = 0;
      for (int oy = 0; oy < ps; ++oy)
        for (int ox = 0; ox < ps; ++ox, ++k) {
          const double e = bilin_nb(q, W, H, bx + ox, by + oy) - off - tmpl[k];
          const double et = transform_residual(e, a.code, a.hb);
          ssd += et * et;
          b0 += sdx[k] * et;
          b1 += sdy[k] * et;
        }
      if (ssd > prev_ssd) {
        u = prev_u;
        v = prev_v;
        break;
      }
      if (stop || it >= a.iters) break;
      prev_ssd = ssd;
      prev_u = u;
      prev_v = v;
      const double du = i00 * b0 + i01 * b1;
      const double dv = i01 * b0 + i11 * b1;
      u -= du;
      v -= dv;
      it += 1;
      if (sqrt(du * du + dv * dv) < 1e-2) stop = true;
      const double cx = x0 + u + 0.5 * ps;
      const double cy = y0 + v + 0.5 * ps;
      if (cx < (double)(-W) || cx > 2.0 * W || cy < (double)(-H) || cy > 2.0 * H) {
        u = u0;
        v = v0;
        prev_ssd = 1e300;
        stop = true;
      }
    }
  }
  double f = 1.0;  // params.downscale ** finest_scale (pipeline.py:231)
  for (int s = 0; s < a.finest; ++s) f *= kd;
  a.out[2 * i] = u * f;
  a.out[2 * i + 1] = v * f;
}

__global__ void __launch_bounds__(128) k_sparse_sample(const double* __restrict__ fu,
                                                       const double* __restrict__ fv, int W,
                                                       int H, double scale,
                                                       const double* __restrict__ seeds,
                                                       const uint8_t* __restrict__ valid, int n,
                                                       double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !valid[i]) return;
  const double gx = seeds[2 * i] / scale, gy = seeds[2 * i + 1] / scale;
  out[2 * i] = bilin_np(fu, W, H, gx, gy) * scale;
  out[2 * i + 1] = bilin_np(fv, W, H, gx, gy) * scale;
}

void launch_sparse_chain(const SparseChainArgs& a, cudaStream_t st) {
  k_sparse_chain<<<(a.n + 127) / 128, 128, 0, st>>>(a);
  note_launch();
}

void launch_sparse_sample(const double* fu, const double* fv, int W, int H, double scale,
                          const double* seeds, const uint8_t* valid, int n, double* out,
                          cudaStream_t st) {
  k_sparse_sample<<<(n + 127) / 128, 128, 0, st>>>(fu, fv, W, H, scale, seeds, valid, n, out);
  note_launch();
}

}  // namespace disb200
