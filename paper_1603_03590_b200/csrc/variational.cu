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
constexpr int kPitch = 9;      // doubles per ring row: 8 fields + 1 pad (72 B, conflict-free LDS.64)
constexpr int kMaxRowsPerCta = 256;

enum RecField { F_U = 0, F_V, F_M00, F_M01, F_M11, F_R0, F_R1, F_WS };

template <int S>
__host__ __device__ constexpr int ring_slots() {
  // live at step k: diagonals k - 2(S-1) - 1 (last sweep's up-neighbour) .. k + 1,
  // plus the ones in flight up to k + kLookahead
  return kLookahead + 2 * S;
}

__device__ __forceinline__ void cp_async8(unsigned smem_dst, const double* gsrc, unsigned src_bytes) {
  // src_bytes = 0 zero-fills the 8 destination bytes
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_dst), "l"(gsrc),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// store a double into the shared memory of CTA `rank` of this cluster
__device__ __forceinline__ void st_cluster(const double* local, unsigned rank, double v) {
  unsigned a = (unsigned)__cvta_generic_to_shared(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(ra), "d"(v) : "memory");
}

// The wavefront SOR kernel (see the file header).
//
// A pair's rows are split over a cluster of C CTAs (C = gridDim-cluster size,
// 1..8); CTA c owns rows [c*Hc, c*Hc + Hc), one thread per row.  The records
// of the live diagonals sit in a shared-memory ring [slot][row][kPitch]
// filled by cp.async kLookahead steps ahead, including one halo row above
// and below the CTA's band; entries of pixels outside the level are
// zero-filled, so a sweep that is not active on its row (before its start
// or after its end) computes finite garbage that is never stored — the
// per-sweep state then needs no selects.  Boundary rows of the band exchange
// their U, V with the neighbouring CTAs through distributed shared memory;
// one (cluster) barrier per step.
template <int S>
__global__ void __launch_bounds__(kMaxRowsPerCta, 1)
    k_sor(const double* __restrict__ rec, int B, int W, int H, int Hc, size_t Ls, double omega,
          const double* du_in, const double* dv_in, double* du_out, double* dv_out,
          double* __restrict__ fu, double* __restrict__ fv, uint32_t* status) {
  extern __shared__ double smem[];
  constexpr int R = ring_slots<S>();
  const int C = (int)(gridDim.x / (unsigned)B) > 0 ? (int)(gridDim.x / (unsigned)B) : 1;
  const int c = C > 1 ? (int)cluster_rank() : 0;
  const int b = blockIdx.x / C;
  const int ty = threadIdx.x;
  const int Hp = blockDim.x;
  const int y0 = c * Hc;
  const int y = y0 + ty;
  const int nrows = min(Hc, H - y0);  // rows this CTA owns
  const int lane = ty & 31;
  const int warp = ty >> 5;
  const int nwarps = Hp >> 5;
  const bool row_ok = ty < nrows;
  const int ndiag = W + H - 1;
  const int slot_rows = Hp + 2;                 // + halo above and below
  double* ring = smem;                          // [R][slot_rows][kPitch]
  double* xch = ring + (size_t)R * slot_rows * kPitch;   // [2][nwarps][2][S][2]
  double* cxin = xch + (size_t)2 * nwarps * 2 * S * 2;   // [2][2][S][2]: 0 from above, 1 from below
  const double* __restrict__ base = rec + (size_t)b * Ls;
  const size_t fstride = (size_t)B * Ls;
  const double* Dui = du_in ? du_in + (size_t)b * Ls : nullptr;  // may alias du_out
  const double* Dvi = dv_in ? dv_in + (size_t)b * Ls : nullptr;
  const double om1 = 1.0 - omega;
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
  const unsigned slot_bytes = (unsigned)(slot_rows * kPitch * 8);

  // load ring row r (image row y0 - 1 + r) of diagonal j
  auto load_row = [&](int j, int r) {
    const int yy = y0 - 1 + r;
    const int x = j - yy;
    const bool ok = yy >= 0 && yy < H && x >= 0 && x < W;
    const size_t g = ok ? (size_t)j * H + yy : 0;
    const unsigned dst = ring_s + (unsigned)(j % R) * slot_bytes + (unsigned)(r * kPitch * 8);
#pragma unroll
    for (int f = 0; f < 8; ++f) cp_async8(dst + 8 * f, base + f * fstride + g, ok ? 8u : 0u);
  };
  auto issue = [&](int j) {
    if (j >= ndiag) return;
    load_row(j, ty + 1);
    if (ty == 0) load_row(j, 0);
    if (ty == Hp - 1) load_row(j, Hp + 1);
  };

  {  // exchange buffers start finite (they feed inactive sweeps at step 0)
    const int nx = 2 * nwarps * 2 * S * 2 + 2 * 2 * S * 2;
    for (int i = ty; i < nx; i += Hp) xch[i] = 0.0;
  }
#pragma unroll
  for (int j = 0; j < kLookahead; ++j) {
    issue(j);
    cp_async_commit();
  }
  cp_async_wait<kLookahead - 2>();
  if (C > 1) {
    cluster_arrive();
    cluster_wait();
  } else {
    __syncthreads();
  }

  double lU[S], lV[S], lW[S], ldu[S], ldv[S], pdu[S], pdv[S];
#pragma unroll
  for (int t = 0; t < S; ++t) lU[t] = lV[t] = lW[t] = ldu[t] = ldv[t] = pdu[t] = pdv[t] = 0.0;
  const bool hasU = y > 0, hasD = y < H - 1;
  const bool top_row = ty == 0 && c > 0;                   // gets "up" from CTA c-1
  const bool bot_row = ty == nrows - 1 && c < C - 1;       // gets "down" from CTA c+1
  bool bad = false;
  const int nsteps = ndiag + 2 * (S - 1);
  int slot0 = 0;  // (k) mod R
  for (int k = 0; k < nsteps; ++k) {
    issue(k + kLookahead);
    cp_async_commit();
    const int rd = (k & 1) ^ 1;
#pragma unroll
    for (int t = S - 1; t >= 0; --t) {
      const int j = k - 2 * t;
      const int x = j - y;
      // ring addresses of this sweep's pixel row (slot of diagonal j) and of
      // the neighbouring diagonals j-1 / j+1
      int sj = slot0 - 2 * t;
      sj += sj < 0 ? R : 0;
      sj += sj < 0 ? R : 0;
      const int sm = sj == 0 ? R - 1 : sj - 1;
      const int sp = sj == R - 1 ? 0 : sj + 1;
      const double* rp = ring + (size_t)sj * slot_rows * kPitch + (size_t)(ty + 1) * kPitch;
      const double* rm = ring + (size_t)sm * slot_rows * kPitch + (size_t)(ty + 1) * kPitch;
      const double* rn = ring + (size_t)sp * slot_rows * kPitch + (size_t)(ty + 1) * kPitch;
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
      if (top_row) {
        const double* xs = cxin + (((size_t)rd * 2 + 0) * S + t) * 2;
        upU = xs[0];
        upV = xs[1];
      }
      if (t > 0 && bot_row) {
        const double* xs = cxin + (((size_t)rd * 2 + 1) * S + t - 1) * 2;
        dnU = xs[0];
        dnV = xs[1];
      }
      const double uc = rp[F_U], vc = rp[F_V], wp = rp[F_WS];
      const double m00 = rp[F_M00], m01 = rp[F_M01], m11 = rp[F_M11];
      const double r0 = rp[F_R0], r1 = rp[F_R1];
      const double upW = rm[F_WS - kPitch];   // (x, y-1): diagonal j-1, row above
      const double dnW = rn[F_WS + kPitch];   // (x, y+1): diagonal j+1, row below
      double rU, rV, rW;
      if (t > 0) {
        rU = lU[t - 1];
        rV = lV[t - 1];
        rW = lW[t - 1];
      } else {
        const int jp = j + 1;
        const bool okp = jp >= 0 && jp < ndiag;
        const size_t gq = okp ? (size_t)jp * H + y : 0;
        const size_t gd = okp && hasD ? (size_t)jp * H + y + 1 : 0;
        rU = rn[F_U] + (Dui ? Dui[gq] : 0.0);
        rV = rn[F_V] + (Dvi ? Dvi[gq] : 0.0);
        rW = rn[F_WS];
        dnU = rn[F_U + kPitch] + (Dui ? Dui[gd] : 0.0);
        dnV = rn[F_V + kPitch] + (Dvi ? Dvi[gd] : 0.0);
      }
      // absent neighbours (borders) contribute wq = +0 times a finite value:
      // adding an exact zero leaves the reference's partial sums unchanged
      const double wqL = x > 0 ? 0.5 * (wp + lW[t]) : 0.0;
      const double wqR = x < W - 1 ? 0.5 * (wp + rW) : 0.0;
      const double wqU = hasU ? 0.5 * (wp + upW) : 0.0;
      const double wqD = hasD ? 0.5 * (wp + dnW) : 0.0;
      const double sw = (((0.0 + wqL) + wqR) + wqU) + wqD;
      const double su = (((0.0 + wqL * (lU[t] - uc)) + wqR * (rU - uc)) + wqU * (upU - uc)) +
                        wqD * (dnU - uc);
      const double sv = (((0.0 + wqL * (lV[t] - vc)) + wqR * (rV - vc)) + wqU * (upV - vc)) +
                        wqD * (dnV - vc);
      double du, dv;
      if (t > 0) {
        du = pdu[t - 1];
        dv = pdv[t - 1];
      } else {
        const bool ok = j >= 0 && j < ndiag;
        du = Dui ? Dui[ok ? (size_t)j * H + y : 0] : 0.0;
        dv = Dvi ? Dvi[ok ? (size_t)j * H + y : 0] : 0.0;
      }
      const double den_u = m00 + sw;
      const double nu = om1 * du + omega * ((r0 + su - m01 * dv) / den_u);
      du = den_u > 1e-12 ? nu : du;
      const double den_v = m11 + sw;
      const double nv = om1 * dv + omega * ((r1 + sv - m01 * du) / den_v);
      dv = den_v > 1e-12 ? nv : dv;
      const double U = uc + du, V = vc + dv;
      pdu[t] = ldu[t];
      pdv[t] = ldv[t];
      ldu[t] = du;
      ldv[t] = dv;
      lU[t] = U;
      lV[t] = V;
      lW[t] = wp;
      if (t == S - 1 && row_ok && x >= 0 && x < W) {
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
    // publish boundary rows for the next step
    if (lane == 0 || lane == 31) {
      double* xs = xch + (((size_t)(k & 1) * nwarps + warp) * 2 + (lane == 31 ? 1 : 0)) * S * 2;
#pragma unroll
      for (int t = 0; t < S; ++t) {
        xs[2 * t] = lU[t];
        xs[2 * t + 1] = lV[t];
      }
    }
    if (C > 1) {
      if (ty == 0 && c > 0) {  // my first row -> CTA c-1's "from below"
        double* xs = cxin + (((size_t)(k & 1) * 2 + 1) * S) * 2;
#pragma unroll
        for (int t = 0; t < S; ++t) {
          st_cluster(xs + 2 * t, c - 1, lU[t]);
          st_cluster(xs + 2 * t + 1, c - 1, lV[t]);
        }
      }
      if (ty == nrows - 1 && c < C - 1) {  // my last row -> CTA c+1's "from above"
        double* xs = cxin + (((size_t)(k & 1) * 2 + 0) * S) * 2;
#pragma unroll
        for (int t = 0; t < S; ++t) {
          st_cluster(xs + 2 * t, c + 1, lU[t]);
          st_cluster(xs + 2 * t + 1, c + 1, lV[t]);
        }
      }
    }
    cp_async_wait<kLookahead - 2>();
    if (C > 1) {
      cluster_arrive();
      cluster_wait();
    } else {
      __syncthreads();
    }
    slot0 = slot0 == R - 1 ? 0 : slot0 + 1;
  }
  if (bad) set_status(status, DIS_STATUS_NONFINITE_FLOW);
}

template <int S>
static size_t sor_smem_bytes(int threads) {
  const size_t ring = (size_t)ring_slots<S>() * (threads + 2) * kPitch * sizeof(double);
  const size_t xch = (size_t)2 * (threads / 32) * 2 * S * 2 * sizeof(double);
  const size_t cx = (size_t)2 * 2 * S * 2 * sizeof(double);
  return ring + xch + cx;
}

constexpr size_t kMaxSmem = 227 * 1024;

// rows-per-CTA split: enough CTAs per pair to keep every band <= 256 rows and
// its ring in shared memory, and, for small batches, to spread a pair over
// several SMs (the step rate of one band is bound by its SM's FP64 pipe).
template <int S>
static int choose_cluster(int B, int H) {
  int C = 1;
  while (C < 8 && ((H + C - 1) / C > kMaxRowsPerCta ||
                   sor_smem_bytes<S>(((H + C - 1) / C + 31) / 32 * 32) > kMaxSmem))
    ++C;
  while (C < 8 && B * (C + 1) <= 148 && (H + C) / (C + 1) >= 64) ++C;
  return C;
}

template <int S>
static int launch_sor_t(const RefineArgs& a, size_t Ls, const double* dui, const double* dvi,
                        double* duo, double* dvo, bool final_pass, cudaStream_t st) {
  const int C = choose_cluster<S>(a.B, a.H);
  const int Hc = (a.H + C - 1) / C;
  const int threads = (Hc + 31) / 32 * 32;
  const size_t smem = sor_smem_bytes<S>(threads);
  if (threads > kMaxRowsPerCta || smem > kMaxSmem) return DIS_ERR_VALUE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sor<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
    cudaFuncSetAttribute(k_sor<S>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.B * C));
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = (unsigned)C;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  double* fu = final_pass ? a.fu : nullptr;
  double* fv = final_pass ? a.fv : nullptr;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_sor<S>, (const double*)a.rec, a.B, a.W, a.H, Hc,
                                     Ls, a.omega, dui, dvi, duo, dvo, fu, fv, a.status);
  return e == cudaSuccess ? DIS_OK : DIS_ERR_CUDA;
}

static int launch_sor(const RefineArgs& a, size_t Ls, int S, const double* dui,
                      const double* dvi, double* duo, double* dvo, bool final_pass,
                      cudaStream_t st) {
  switch (S) {
#define DIS_SOR_CASE(n) \
  case n:               \
    return launch_sor_t<n>(a, Ls, dui, dvi, duo, dvo, final_pass, st);
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
      return DIS_ERR_VALUE;
  }
}

int launch_refine(const RefineArgs& a, cudaStream_t st) {
  if (a.H > 8 * kMaxRowsPerCta) return DIS_ERR_VALUE;  // at most 8 CTAs per pair
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
      int rc = launch_sor(a, Ls, S, first ? nullptr : carry_u, first ? nullptr : carry_v,
                          last ? nullptr : carry_u, last ? nullptr : carry_v, last, st);
      prof_end(KC_SOR, st);
      if (rc) return rc;
      note_launch();
      first = false;
    }
  }
  return DIS_OK;
}

}  // namespace disb200
