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
constexpr int kLookahead = 3;  // diagonals prefetched ahead of the wavefront

enum RecField { F_U = 0, F_V, F_M00, F_M01, F_M11, F_R0, F_R1, F_WS };

template <int S>
__host__ __device__ constexpr int ring_slots() {
  // slots in use at step k: diagonals k - 2(S-1) .. k + 1, plus the ones in
  // flight up to k + kLookahead
  return kLookahead + 2 * S - 1;
}

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// The wavefront SOR kernel (see the file header).  RING = true stages the
// records of the live diagonals in a shared-memory ring filled by cp.async
// kLookahead steps ahead (levels up to ~290 rows); RING = false reads them
// from global memory (L1/L2).  All sweeps of a step are evaluated
// branch-free (selects), so their independent dependency chains interleave.
template <int S, bool RING>
__global__ void __launch_bounds__(RING ? 320 : 576) k_sor(const double* __restrict__ rec, int B, int W,
                                             int H, size_t Ls, double omega,
                                             const double* du_in, const double* dv_in,
                                             double* du_out, double* dv_out,
                                             double* __restrict__ fu,
                                             double* __restrict__ fv, uint32_t* status) {
  extern __shared__ double smem[];
  constexpr int R = ring_slots<S>();
  const int b = blockIdx.x;
  const int y = threadIdx.x;
  const int Hp = blockDim.x;
  const int lane = y & 31;
  const int warp = y >> 5;
  const int nwarps = Hp >> 5;
  const bool row_ok = y < H;
  const int ymc = y > 0 ? y - 1 : 0;               // clamped up row
  const int ypc = y < H - 1 ? y + 1 : H - 1;       // clamped down row
  const int ndiag = W + H - 1;
  double* ring = smem;
  double* xch = smem + (RING ? (size_t)R * 8 * Hp : 0);  // [2][nwarps][2][S][2]
  const double* __restrict__ base = rec + (size_t)b * Ls;
  const size_t fstride = (size_t)B * Ls;  // distance between record fields
  const double* Dui = du_in ? du_in + (size_t)b * Ls : nullptr;  // may alias du_out
  const double* Dvi = dv_in ? dv_in + (size_t)b * Ls : nullptr;
  const double om1 = 1.0 - omega;

  // record field f of pixel (j - yy, yy) on diagonal j (0 <= j < ndiag)
  auto rv = [&](int f, int j, int yy) -> double {
    if (RING) return ring[((size_t)(j % R) * 8 + f) * Hp + yy];
    return __ldg(base + f * fstride + (size_t)j * H + yy);
  };
  auto issue = [&](int j) {
    const int x = j - y;
    if (row_ok && x >= 0 && x < W) {
      const size_t g = (size_t)j * H + y;
      double* dst = ring + (size_t)(j % R) * 8 * Hp + y;
#pragma unroll
      for (int f = 0; f < 8; ++f) cp_async8(dst + (size_t)f * Hp, base + f * fstride + g);
    }
  };

  if (RING) {
#pragma unroll
    for (int j = 0; j < kLookahead; ++j) {
      issue(j);
      cp_async_commit();
    }
    cp_async_wait<kLookahead - 2>();
    __syncthreads();
  }

  double lU[S], lV[S], lW[S], ldu[S], ldv[S], pdu[S], pdv[S];
#pragma unroll
  for (int t = 0; t < S; ++t) lU[t] = lV[t] = lW[t] = ldu[t] = ldv[t] = pdu[t] = pdv[t] = 0.0;
  bool bad = false;
  const int nsteps = ndiag + 2 * (S - 1);
  for (int k = 0; k < nsteps; ++k) {
    if (RING) {
      issue(k + kLookahead);
      cp_async_commit();
    }
    const int rd = (k & 1) ^ 1;
#pragma unroll
    for (int t = S - 1; t >= 0; --t) {
      const int j = k - 2 * t;           // diagonal of this sweep's pixel
      const int x = j - y;
      const bool act = row_ok && x >= 0 && x < W;
      const int jc = j < 0 ? 0 : (j > ndiag - 1 ? ndiag - 1 : j);
      const int jm = jc > 0 ? jc - 1 : 0;
      const int jp = jc < ndiag - 1 ? jc + 1 : ndiag - 1;
      // previous-step values of the neighbours (warp-synchronous)
      double upU = __shfl_up_sync(kFull, lU[t], 1);
      double upV = __shfl_up_sync(kFull, lV[t], 1);
      double dnU = 0.0, dnV = 0.0;
      if (t > 0) {
        dnU = __shfl_down_sync(kFull, lU[t - 1], 1);
        dnV = __shfl_down_sync(kFull, lV[t - 1], 1);
      }
      if (lane == 0 && warp > 0) {
        const double* xs = xch + ((((size_t)rd * nwarps + warp - 1) * 2 + 1) * S + t) * 2;
        upU = xs[0];
        upV = xs[1];
      }
      if (t > 0 && lane == 31 && warp < nwarps - 1) {
        const double* xs = xch + ((((size_t)rd * nwarps + warp + 1) * 2 + 0) * S + t - 1) * 2;
        dnU = xs[0];
        dnV = xs[1];
      }
      const double uc = rv(F_U, jc, y), vc = rv(F_V, jc, y), wp = rv(F_WS, jc, y);
      const double m00 = rv(F_M00, jc, y), m01 = rv(F_M01, jc, y), m11 = rv(F_M11, jc, y);
      const double r0 = rv(F_R0, jc, y), r1 = rv(F_R1, jc, y);
      const double upW = rv(F_WS, jm, ymc);
      const double dnW = rv(F_WS, jp, ypc);
      double rU, rV, rW;
      if (t > 0) {
        rU = lU[t - 1];
        rV = lV[t - 1];
        rW = lW[t - 1];
      } else {
        rU = rv(F_U, jp, y) + (Dui ? Dui[(size_t)jp * H + y] : 0.0);
        rV = rv(F_V, jp, y) + (Dvi ? Dvi[(size_t)jp * H + y] : 0.0);
        rW = rv(F_WS, jp, y);
        dnU = rv(F_U, jp, ypc) + (Dui ? Dui[(size_t)jp * H + ypc] : 0.0);
        dnV = rv(F_V, jp, ypc) + (Dvi ? Dvi[(size_t)jp * H + ypc] : 0.0);
      }
      const bool hasL = x > 0, hasR = x < W - 1, hasU = y > 0, hasD = y < H - 1;
      double sw = 0.0, su = 0.0, sv = 0.0, wq;
      wq = 0.5 * (wp + lW[t]);
      sw = hasL ? sw + wq : sw;
      su = hasL ? su + wq * (lU[t] - uc) : su;
      sv = hasL ? sv + wq * (lV[t] - vc) : sv;
      wq = 0.5 * (wp + rW);
      sw = hasR ? sw + wq : sw;
      su = hasR ? su + wq * (rU - uc) : su;
      sv = hasR ? sv + wq * (rV - vc) : sv;
      wq = 0.5 * (wp + upW);
      sw = hasU ? sw + wq : sw;
      su = hasU ? su + wq * (upU - uc) : su;
      sv = hasU ? sv + wq * (upV - vc) : sv;
      wq = 0.5 * (wp + dnW);
      sw = hasD ? sw + wq : sw;
      su = hasD ? su + wq * (dnU - uc) : su;
      sv = hasD ? sv + wq * (dnV - vc) : sv;
      double du, dv;
      if (t > 0) {
        du = pdu[t - 1];
        dv = pdv[t - 1];
      } else {
        du = Dui ? Dui[(size_t)jc * H + y] : 0.0;
        dv = Dvi ? Dvi[(size_t)jc * H + y] : 0.0;
      }
      const double den_u = m00 + sw;
      const double nu = om1 * du + omega * ((r0 + su - m01 * dv) / den_u);
      du = den_u > 1e-12 ? nu : du;
      const double den_v = m11 + sw;
      const double nv = om1 * dv + omega * ((r1 + sv - m01 * du) / den_v);
      dv = den_v > 1e-12 ? nv : dv;
      const double U = uc + du, V = vc + dv;
      const bool shiftp = row_ok && x >= 0 && x <= W;
      pdu[t] = shiftp ? ldu[t] : pdu[t];
      pdv[t] = shiftp ? ldv[t] : pdv[t];
      ldu[t] = act ? du : ldu[t];
      ldv[t] = act ? dv : ldv[t];
      lU[t] = act ? U : lU[t];
      lV[t] = act ? V : lV[t];
      lW[t] = act ? wp : lW[t];
      if (t == S - 1 && act) {
        if (du_out) {
          du_out[(size_t)b * Ls + (size_t)j * H + y] = du;
          dv_out[(size_t)b * Ls + (size_t)j * H + y] = dv;
        }
        if (fu) {
          const size_t o = (size_t)b * W * H + (size_t)y * W + x;
          fu[o] = U;
          fv[o] = V;
          bad |= !(isfinite(U) && isfinite(V));
        }
      }
    }
    if (row_ok && (lane == 0 || lane == 31)) {
      double* xs = xch + (((size_t)(k & 1) * nwarps + warp) * 2 + (lane == 31 ? 1 : 0)) * S * 2;
#pragma unroll
      for (int t = 0; t < S; ++t) {
        xs[2 * t] = lU[t];
        xs[2 * t + 1] = lV[t];
      }
    }
    if (RING) cp_async_wait<kLookahead - 2>();
    __syncthreads();
  }
  if (bad) set_status(status, DIS_STATUS_NONFINITE_FLOW);
}

template <int S>
static size_t sor_smem_bytes(int threads, bool ring) {
  const size_t xch = (size_t)2 * (threads / 32) * 2 * S * 2 * sizeof(double);
  return xch + (ring ? (size_t)ring_slots<S>() * 8 * threads * sizeof(double) : 0);
}

constexpr size_t kMaxSmem = 227 * 1024;

template <int S>
static void launch_sor_t(const RefineArgs& a, size_t Ls, const double* dui, const double* dvi,
                         double* duo, double* dvo, bool final_pass, cudaStream_t st) {
  const int threads = (a.H + 31) / 32 * 32;
  const bool ring = threads <= 320 && sor_smem_bytes<S>(threads, true) <= kMaxSmem;
  const size_t smem = sor_smem_bytes<S>(threads, ring);
  double* fu = final_pass ? a.fu : nullptr;
  double* fv = final_pass ? a.fv : nullptr;
  if (ring) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_sor<S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kMaxSmem);
      attr = true;
    }
    k_sor<S, true><<<a.B, threads, smem, st>>>(a.rec, a.B, a.W, a.H, Ls, a.omega, dui, dvi,
                                               duo, dvo, fu, fv, a.status);
  } else {
    k_sor<S, false><<<a.B, threads, smem, st>>>(a.rec, a.B, a.W, a.H, Ls, a.omega, dui, dvi,
                                                duo, dvo, fu, fv, a.status);
  }
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
