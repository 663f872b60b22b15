// variational.cu — variational refinement of one level (refine,
// variational.py:220-275) for a batch of pairs.
//
// Per outer (fixed-point) iteration:
//   k_tensor_assemble : _tensor_fields (variational.py:36-88) fused with
//                       _assemble_system (91-121); the 12 tensor entries never
//                       reach HBM.  Writes the 8-value SOR record of every
//                       pixel (u, v, m00, m01, m11, r0, r1, ws) in the skewed
//                       layout [(x + y) * H + y].
//   k_sor<S>          : theta_vi in-place lexicographic SOR sweeps
//                       (_sor_sweeps, variational.py:124-165) + the update
//                       u += du, v += dv (266-267) + the finiteness check.
//
// Exact lexicographic SOR on a GPU — the systolic wavefront.
// The reference sweeps row-major in place: pixel (x, y) in sweep t reads its
// left/up neighbours from sweep t and its right/down neighbours from sweep
// t-1.  Processing pixel (x, y) of sweep t at step k = x + y + 2t respects
// every one of those dependencies (bit-identical), and at
// a fixed step row y holds exactly one pixel per sweep, x = k - y - 2t.  So
// one THREAD OWNS ONE ROW and carries all sweeps at once:
//   left  (x-1, y, t)   = this thread's own sweep-t value from step k-1
//   right (x+1, y, t-1) = this thread's own sweep-(t-1) value from step k-1
//   own   (x,   y, t-1) = this thread's sweep-(t-1) value from step k-2
//   up    (x, y-1, t)   = lane y-1's sweep-t value from step k-1 (shuffle)
//   down  (x, y+1, t-1) = lane y+1's sweep-(t-1) value from step k-1 (shuffle)
// Sweeps are processed in decreasing t inside a step so every read sees the
// previous step's value; warp boundaries exchange through shared memory with
// one __syncthreads per step.  All values stay in registers; the static
// per-pixel record is read from the skewed layout, where the pixels of one
// step (an anti-diagonal) are contiguous: coalesced.
//
// Neighbour terms use U_q = fl(u_q + du_q) exactly as the reference's
// `u[y, x-1] + du[y, x-1]`; the last sweep's U is the updated flow.
#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

constexpr int kRecords = 8;  // u v m00 m01 m11 r0 r1 ws
constexpr int kMaxSweepsPerPass = 8;

size_t refine_scratch_doubles(int B, int W, int H) {
  const size_t Ls = (size_t)(W + H - 1) * H;
  return (size_t)(kRecords + 2) * B * Ls;  // + du/dv carry for > 8 sweeps
}

__global__ void __launch_bounds__(256) k_tensor_assemble(RefineArgs a, size_t Ls) {
  const int W = a.W, H = a.H;
  const int y = blockIdx.x * 32 + threadIdx.x;
  const int d = blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.z;
  const int x = d - y;
  if (y >= H || x < 0 || x >= W) return;
  const size_t plane = (size_t)W * H;
  const size_t p = (size_t)y * W + x;
  const double* __restrict__ u = a.fu + b * plane;
  const double* __restrict__ v = a.fv + b * plane;
  const double* __restrict__ ref = a.ref + b * plane;
  const double* __restrict__ rgx = a.rgx + b * plane;
  const double* __restrict__ rgy = a.rgy + b * plane;
  const double* __restrict__ rdd = a.rdd + b * 4 * plane;
  const double* __restrict__ qry = a.qry + b * plane;
  const double* __restrict__ qgx = a.qgx + b * plane;
  const double* __restrict__ qgy = a.qgy + b * plane;
  const double* __restrict__ qdd = a.qdd + b * 4 * plane;

  const double up_ = u[p], vp_ = v[p];
  // ---- _tensor_fields (variational.py:36-88) ----
  double t0xx = 0.0, t0xy = 0.0, t0xz = 0.0, t0yy = 0.0, t0yz = 0.0, t0zz = 0.0;
  double tgxx = 0.0, tgxy = 0.0, tgxz = 0.0, tgyy = 0.0, tgyz = 0.0, tgzz = 0.0;
  const double wxp = x + up_;
  const double wyp = y + vp_;
  if (!(x == 0 || x == W - 1 || y == 0 || y == H - 1 || wxp < 0.0 || wxp > W - 1.0 ||
        wyp < 0.0 || wyp > H - 1.0)) {
    const double iw = bilin_nb(qry, W, H, wxp, wyp);
    const double gxw = bilin_nb(qgx, W, H, wxp, wyp);
    const double gyw = bilin_nb(qgy, W, H, wxp, wyp);
    const double rgxp = rgx[p], rgyp = rgy[p];
    const double ix = 0.5 * (rgxp + gxw);
    const double iy = 0.5 * (rgyp + gyw);
    const double iz = iw - ref[p];
    const double b0 = 1.0 / (ix * ix + iy * iy + 0.01);
    t0xx = b0 * ix * ix;
    t0xy = b0 * ix * iy;
    t0xz = b0 * ix * iz;
    t0yy = b0 * iy * iy;
    t0yz = b0 * iy * iz;
    t0zz = b0 * iz * iz;
    const double ixx = 0.5 * (rdd[p] + bilin_nb(qdd, W, H, wxp, wyp));
    const double ixy = 0.5 * (rdd[plane + p] + bilin_nb(qdd + plane, W, H, wxp, wyp));
    const double ixz = gxw - rgxp;
    const double iyx = 0.5 * (rdd[2 * plane + p] + bilin_nb(qdd + 2 * plane, W, H, wxp, wyp));
    const double iyy = 0.5 * (rdd[3 * plane + p] + bilin_nb(qdd + 3 * plane, W, H, wxp, wyp));
    const double iyz = gyw - rgyp;
    const double bx = 1.0 / (ixx * ixx + ixy * ixy + 0.01);
    const double by = 1.0 / (iyx * iyx + iyy * iyy + 0.01);
    tgxx = bx * ixx * ixx + by * iyx * iyx;
    tgxy = bx * ixx * ixy + by * iyx * iyy;
    tgxz = bx * ixx * ixz + by * iyx * iyz;
    tgyy = bx * ixy * ixy + by * iyy * iyy;
    tgyz = bx * ixy * ixz + by * iyy * iyz;
    tgzz = bx * ixz * ixz + by * iyz * iyz;
  }
  // ---- _assemble_system (variational.py:91-121) ----
  const double eps2 = a.eps * a.eps;
  const double psi_i = 0.5 / sqrt(t0zz + eps2);
  const double psi_g = 0.5 / sqrt(tgzz + eps2);
  const double wi = a.delta * psi_i;
  const double wg = a.gamma * psi_g;
  const double m00 = wi * t0xx + wg * tgxx;
  const double m01 = wi * t0xy + wg * tgxy;
  const double m11 = wi * t0yy + wg * tgyy;
  const double r0 = -(wi * t0xz + wg * tgxz);
  const double r1 = -(wi * t0yz + wg * tgyz);
  const int xm = x > 0 ? x - 1 : 0;
  const int xp = x < W - 1 ? x + 1 : W - 1;
  const int ym = y > 0 ? y - 1 : 0;
  const int yp = y < H - 1 ? y + 1 : H - 1;
  const double ux = 0.5 * (u[(size_t)y * W + xp] - u[(size_t)y * W + xm]);
  const double uy = 0.5 * (u[(size_t)yp * W + x] - u[(size_t)ym * W + x]);
  const double vx = 0.5 * (v[(size_t)y * W + xp] - v[(size_t)y * W + xm]);
  const double vy = 0.5 * (v[(size_t)yp * W + x] - v[(size_t)ym * W + x]);
  const double grad2 = ux * ux + uy * uy + vx * vx + vy * vy;
  const double ws = a.alpha * 0.5 / sqrt(grad2 + eps2);

  const size_t s = (size_t)d * H + y;
  double* rec = a.rec;
  const size_t B = (size_t)a.B;
  rec[(0 * B + b) * Ls + s] = up_;
  rec[(1 * B + b) * Ls + s] = vp_;
  rec[(2 * B + b) * Ls + s] = m00;
  rec[(3 * B + b) * Ls + s] = m01;
  rec[(4 * B + b) * Ls + s] = m11;
  rec[(5 * B + b) * Ls + s] = r0;
  rec[(6 * B + b) * Ls + s] = r1;
  rec[(7 * B + b) * Ls + s] = ws;
}

constexpr unsigned kFull = 0xffffffffu;

template <int S>
__global__ void __launch_bounds__(576) k_sor(const double* __restrict__ rec, int B, int W,
                                             int H, size_t Ls, double omega,
                                             const double* du_in, const double* dv_in,
                                             double* du_out, double* dv_out,
                                             double* __restrict__ fu,
                                             double* __restrict__ fv, uint32_t* status) {
  const int b = blockIdx.x;
  const int y = threadIdx.x;
  const int lane = y & 31;
  const int warp = y >> 5;
  const int nwarps = blockDim.x >> 5;
  const bool row_ok = y < H;
  const double* __restrict__ Ru = rec + (size_t)(0 * B + b) * Ls;
  const double* __restrict__ Rv = rec + (size_t)(1 * B + b) * Ls;
  const double* __restrict__ Rm00 = rec + (size_t)(2 * B + b) * Ls;
  const double* __restrict__ Rm01 = rec + (size_t)(3 * B + b) * Ls;
  const double* __restrict__ Rm11 = rec + (size_t)(4 * B + b) * Ls;
  const double* __restrict__ Rr0 = rec + (size_t)(5 * B + b) * Ls;
  const double* __restrict__ Rr1 = rec + (size_t)(6 * B + b) * Ls;
  const double* __restrict__ Rws = rec + (size_t)(7 * B + b) * Ls;
  const double* Dui = du_in ? du_in + (size_t)b * Ls : nullptr;  // may alias du_out
  const double* Dvi = dv_in ? dv_in + (size_t)b * Ls : nullptr;
  const double om1 = 1.0 - omega;

  // [parity][warp][0 = lane 0 (top), 1 = lane 31 (bottom)][sweep][U, V, ws]
  __shared__ double xch[2][18][2][S][3];

  double lU[S], lV[S], lW[S], ldu[S], ldv[S], pdu[S], pdv[S];
#pragma unroll
  for (int t = 0; t < S; ++t) {
    lU[t] = lV[t] = lW[t] = ldu[t] = ldv[t] = pdu[t] = pdv[t] = 0.0;
  }
  bool bad = false;
  const int nsteps = W + H - 1 + 2 * (S - 1);
  for (int k = 0; k < nsteps; ++k) {
    const int rd = (k & 1) ^ 1;
#pragma unroll
    for (int t = S - 1; t >= 0; --t) {
      const int x = k - y - 2 * t;
      double upU = __shfl_up_sync(kFull, lU[t], 1);
      double upV = __shfl_up_sync(kFull, lV[t], 1);
      double upW = __shfl_up_sync(kFull, lW[t], 1);
      double dnU = 0.0, dnV = 0.0, dnW = 0.0;
      if (t > 0) {
        dnU = __shfl_down_sync(kFull, lU[t - 1], 1);
        dnV = __shfl_down_sync(kFull, lV[t - 1], 1);
        dnW = __shfl_down_sync(kFull, lW[t - 1], 1);
      }
      if (!row_ok) continue;
      if (x >= 0 && x < W) {
        if (lane == 0 && warp > 0) {
          upU = xch[rd][warp - 1][1][t][0];
          upV = xch[rd][warp - 1][1][t][1];
          upW = xch[rd][warp - 1][1][t][2];
        }
        if (t > 0 && lane == 31 && warp < nwarps - 1) {
          dnU = xch[rd][warp + 1][0][t - 1][0];
          dnV = xch[rd][warp + 1][0][t - 1][1];
          dnW = xch[rd][warp + 1][0][t - 1][2];
        }
        const size_t idx = (size_t)(x + y) * H + y;
        const double uc = Ru[idx], vc = Rv[idx], wp = Rws[idx];
        double sw = 0.0, su = 0.0, sv = 0.0;
        if (x > 0) {
          const double wq = 0.5 * (wp + lW[t]);
          sw += wq;
          su += wq * (lU[t] - uc);
          sv += wq * (lV[t] - vc);
        }
        if (x < W - 1) {
          double rU, rV, rW;
          if (t > 0) {
            rU = lU[t - 1];
            rV = lV[t - 1];
            rW = lW[t - 1];
          } else {
            const size_t q = idx + H;
            rU = Ru[q] + (Dui ? Dui[q] : 0.0);
            rV = Rv[q] + (Dvi ? Dvi[q] : 0.0);
            rW = Rws[q];
          }
          const double wq = 0.5 * (wp + rW);
          sw += wq;
          su += wq * (rU - uc);
          sv += wq * (rV - vc);
        }
        if (y > 0) {
          const double wq = 0.5 * (wp + upW);
          sw += wq;
          su += wq * (upU - uc);
          sv += wq * (upV - vc);
        }
        if (y < H - 1) {
          if (t == 0) {
            const size_t q = idx + H + 1;
            dnU = Ru[q] + (Dui ? Dui[q] : 0.0);
            dnV = Rv[q] + (Dvi ? Dvi[q] : 0.0);
            dnW = Rws[q];
          }
          const double wq = 0.5 * (wp + dnW);
          sw += wq;
          su += wq * (dnU - uc);
          sv += wq * (dnV - vc);
        }
        double du, dv;
        if (t > 0) {
          du = pdu[t - 1];
          dv = pdv[t - 1];
        } else {
          du = Dui ? Dui[idx] : 0.0;
          dv = Dvi ? Dvi[idx] : 0.0;
        }
        const double den_u = Rm00[idx] + sw;
        const double m01 = Rm01[idx];
        if (den_u > 1e-12) {
          const double val = (Rr0[idx] + su - m01 * dv) / den_u;
          du = om1 * du + omega * val;
        }
        const double den_v = Rm11[idx] + sw;
        if (den_v > 1e-12) {
          const double val = (Rr1[idx] + sv - m01 * du) / den_v;
          dv = om1 * dv + omega * val;
        }
        pdu[t] = ldu[t];
        pdv[t] = ldv[t];
        ldu[t] = du;
        ldv[t] = dv;
        lU[t] = uc + du;
        lV[t] = vc + dv;
        lW[t] = wp;
        if (t == S - 1) {
          if (du_out) {
            du_out[(size_t)b * Ls + idx] = du;
            dv_out[(size_t)b * Ls + idx] = dv;
          }
          if (fu) {
            const size_t o = (size_t)b * W * H + (size_t)y * W + x;
            fu[o] = lU[t];
            fv[o] = lV[t];
            bad |= !(isfinite(lU[t]) && isfinite(lV[t]));
          }
        }
      } else if (x == W) {
        pdu[t] = ldu[t];
        pdv[t] = ldv[t];
      }
    }
    if (row_ok && (lane == 0 || lane == 31)) {
      const int side = lane == 31 ? 1 : 0;
#pragma unroll
      for (int t = 0; t < S; ++t) {
        xch[k & 1][warp][side][t][0] = lU[t];
        xch[k & 1][warp][side][t][1] = lV[t];
        xch[k & 1][warp][side][t][2] = lW[t];
      }
    }
    __syncthreads();
  }
  if (bad) set_status(status, DIS_STATUS_NONFINITE_FLOW);
}

template <int S>
static void launch_sor_t(const RefineArgs& a, size_t Ls, const double* dui, const double* dvi,
                         double* duo, double* dvo, bool final_pass, cudaStream_t st) {
  const int threads = (a.H + 31) / 32 * 32;
  k_sor<S><<<a.B, threads, 0, st>>>(a.rec, a.B, a.W, a.H, Ls, a.omega, dui, dvi, duo, dvo,
                                     final_pass ? a.fu : nullptr, final_pass ? a.fv : nullptr,
                                     a.status);
}

static void launch_sor(const RefineArgs& a, size_t Ls, int S, const double* dui,
                       const double* dvi, double* duo, double* dvo, bool final_pass,
                       cudaStream_t st) {
  switch (S) {
#define DIS_SOR_CASE(n) \
  case n:               \
    launch_sor_t<n>(a, Ls, dui, dvi, duo, dvo, final_pass, st); \
    break;
    DIS_SOR_CASE(1)
    DIS_SOR_CASE(2)
    DIS_SOR_CASE(3)
    DIS_SOR_CASE(4)
    DIS_SOR_CASE(5)
    DIS_SOR_CASE(6)
    DIS_SOR_CASE(7)
    DIS_SOR_CASE(8)
#undef DIS_SOR_CASE
    default:
      break;
  }
}

int launch_refine(const RefineArgs& a, cudaStream_t st) {
  if (a.H > 576) return DIS_ERR_VALUE;  // one CTA owns all rows of a level (see header)
  const size_t Ls = (size_t)(a.W + a.H - 1) * a.H;
  double* carry_u = a.rec + (size_t)kRecords * a.B * Ls;
  double* carry_v = carry_u + (size_t)a.B * Ls;
  dim3 tb(32, 8);
  dim3 tg((a.H + 31) / 32, (a.W + a.H - 1 + 7) / 8, a.B);
  for (int it = 0; it < a.outer; ++it) {
    prof_begin(KC_TENSOR, st);
    k_tensor_assemble<<<tg, tb, 0, st>>>(a, Ls);
    prof_end(KC_TENSOR, st);
    note_launch();
    int left = a.sweeps;
    bool first = true;
    while (left > 0) {
      const int S = left > kMaxSweepsPerPass ? kMaxSweepsPerPass : left;
      left -= S;
      const bool last = left == 0;
      // chained passes carry du/dv through the skewed carry buffers; a pass
      // may read and write the same buffer only at the same pixel, which it
      // reads (t = 0) before it writes (t = S - 1, two steps later or more)
      prof_begin(KC_SOR, st);
      launch_sor(a, Ls, S, first ? nullptr : carry_u, first ? nullptr : carry_v,
                 last ? nullptr : carry_u, last ? nullptr : carry_v, last, st);
      prof_end(KC_SOR, st);
      note_launch();
      first = false;
    }
  }
  return DIS_OK;
}

}  // namespace disb200
