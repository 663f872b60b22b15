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
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

constexpr int kRecords = 8;  // u v m00 m01 m11 r0 r1 ws
constexpr int kMaxSweepsPerPass = 8;

size_t refine_scratch_doubles(int B, int W, int H) {
  const size_t Ls = (size_t)(W + H - 1) * H;
  return (size_t)(kRecords + 2) * B * Ls;  // + du/dv carry for > 8 sweeps
}

// Tile of kTTX x kTTY pixels per block: the record of each pixel is computed
// with row-major (coalesced) reads, staged in shared memory, then written to
// the skewed layout one diagonal run at a time (contiguous y on a diagonal).
constexpr int kTTX = 32, kTTY = 16;

__device__ __forceinline__ void pixel_record(const RefineArgs& a, int b, int x, int y,
                                             double* r) {
  const int W = a.W, H = a.H;
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
  const int xm = x > 0 ? x - 1 : 0;
  const int xp = x < W - 1 ? x + 1 : W - 1;
  const int ym = y > 0 ? y - 1 : 0;
  const int yp = y < H - 1 ? y + 1 : H - 1;
  const double ux = 0.5 * (u[(size_t)y * W + xp] - u[(size_t)y * W + xm]);
  const double uy = 0.5 * (u[(size_t)yp * W + x] - u[(size_t)ym * W + x]);
  const double vx = 0.5 * (v[(size_t)y * W + xp] - v[(size_t)y * W + xm]);
  const double vy = 0.5 * (v[(size_t)yp * W + x] - v[(size_t)ym * W + x]);
  const double grad2 = ux * ux + uy * uy + vx * vx + vy * vy;
  r[0] = up_;
  r[1] = vp_;
  r[2] = wi * t0xx + wg * tgxx;        // m00
  r[3] = wi * t0xy + wg * tgxy;        // m01
  r[4] = wi * t0yy + wg * tgyy;        // m11
  r[5] = -(wi * t0xz + wg * tgxz);     // r0
  r[6] = -(wi * t0yz + wg * tgyz);     // r1
  r[7] = a.alpha * 0.5 / sqrt(grad2 + eps2);  // ws
}

__global__ void __launch_bounds__(256, 3) k_tensor_assemble(RefineArgs a, size_t Ls) {
  __shared__ double rs[kRecords][kTTY][kTTX + 1];
  const int W = a.W, H = a.H;
  const int b = blockIdx.z;
  const int X0 = blockIdx.x * kTTX, Y0 = blockIdx.y * kTTY;
  const int lx = threadIdx.x & 31;
  for (int ly = threadIdx.x >> 5; ly < kTTY; ly += 8) {
    const int x = X0 + lx, y = Y0 + ly;
    if (x < W && y < H) {
      double r[kRecords];
      pixel_record(a, b, x, y, r);
#pragma unroll
      for (int f = 0; f < kRecords; ++f) rs[f][ly][lx] = r[f];
    }
  }
  __syncthreads();
  // write diagonal runs: diagonal d = X0 + Y0 + dd, rows y with x = d - y in
  // the tile -> contiguous [d*H + y] in every record field
  const size_t B = (size_t)a.B;
  const int ndd = kTTX + kTTY - 1;
  for (int i = threadIdx.x; i < kRecords * ndd * kTTY; i += 256) {
    const int ly = i % kTTY;
    const int rest = i / kTTY;
    const int dd = rest % ndd;
    const int f = rest / ndd;
    const int lxx = dd - ly;
    const int x = X0 + lxx, y = Y0 + ly;
    if (lxx < 0 || lxx >= kTTX || x >= W || y >= H) continue;
    const size_t d = (size_t)(x + y);
    a.rec[(f * B + b) * Ls + d * H + y] = rs[f][ly][lxx];
  }
}

constexpr int kLookahead = 8;  // diagonals prefetched ahead of the wavefront (covers HBM latency)
constexpr int kPitch = 9;      // doubles per ring row: 8 fields + 1 pad (72 B, conflict-free LDS.64)
constexpr int kMaxBandRows = 128;  // rows (threads per sweep) of one CTA's band

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

// mbarrier helpers (band-boundary signalling between the CTAs of a cluster)
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(unsigned bar_local, unsigned rank) {
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(bar_local), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(ra)
               : "memory");
}
// st.async of (x, y) into CTA `rank`'s shared memory at local-equivalent
// address a; completion is counted (16 bytes) on that CTA's mbarrier bar
__device__ __forceinline__ void st_async2(unsigned a, unsigned bar, unsigned rank, double x,
                                          double y) {
  unsigned ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(bar), "r"(rank));
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
          ra),
      "d"(x), "d"(y), "r"(rb)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// The wavefront SOR kernel (see the file header).
//
// Thread (sweep t, row group g) owns RT consecutive rows of a band and, at
// step k, computes pixel x = k - y - 2t of each of them (all on diagonal
// j = k - 2t).  Its rows are independent within a step (every neighbour
// value is from an earlier step), so a thread carries RT independent update
// chains.  A pair's rows are split over a cluster of C CTAs (1..16); CTA c
// owns the band [c*Hc, c*Hc + Hc).  Shared memory holds
//   ring[R][Hp+2][kPitch] : records of the live diagonals (+ one halo row
//                           above and below the band), filled by cp.async
//                           kLookahead steps ahead; entries outside the
//                           level are zero-filled
//   xuv[2][S][Hp+2][2]    : U, V produced at the last two steps
//   xd [3][S][Hp+2][2]    : du, dv of the last three steps (own previous)
// Neighbours of (x, y, t): left = own registers (step k-1); up = the
// thread's own row above (registers, step k-1) or xuv[k-1][t][y-1] for its
// first row; right = xuv[k-1][t-1][y]; down = xuv[k-1][t-1][y+1]; own
// previous du/dv = xd[k-2][t-1][y]; for t = 0 the initial values come from
// the ring (du = 0, or the carried du of a chained pass).  The band's
// boundary rows write their U, V straight into the neighbouring CTA's halo
// rows of xuv (distributed shared memory) and signal it with a remote
// mbarrier arrive; the consumer waits on its local mbarrier — neighbour to
// neighbour, no cluster-wide barrier per step.  A thread whose pixel is
// outside the level computes finite garbage from zero-filled entries and
// never stores it, so no selects are needed.
// explicit shared-space accesses (32-bit addresses; keeps the compiler
// from re-deriving generic->shared windows every step)
__device__ __forceinline__ double lds(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts2(unsigned a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void lds2(unsigned a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}

template <int S, int RT, bool HZ>
__global__ void __launch_bounds__(S * kMaxBandRows / RT, 1)
    k_sor(const double* __restrict__ rec, int B, int W, int H, int Hc, size_t Ls, double omega,
          const double* du_in, const double* dv_in, double* du_out, double* dv_out,
          double* __restrict__ fu, double* __restrict__ fv, uint32_t* status) {
  extern __shared__ double smem[];
  constexpr int R = ring_slots<S>();
  constexpr int kFieldsPerThread = (8 + S - 1) / S;
  constexpr unsigned kRowB = kPitch * 8;  // ring row bytes
  const int C = (int)(gridDim.x / (unsigned)B) > 0 ? (int)(gridDim.x / (unsigned)B) : 1;
  const int c = C > 1 ? (int)cluster_rank() : 0;
  const int b = blockIdx.x / C;
  const int TS = blockDim.x / S;          // threads per sweep
  const int Hp = TS * RT;                 // band rows (padded)
  const int t = threadIdx.x / TS;         // sweep
  const int tg = threadIdx.x - t * TS;    // row group
  const int y0 = c * Hc;
  const int ty0 = tg * RT;                // first band row of this thread
  const int nrows = min(Hc, H - y0);
  const int ndiag = W + H - 1;
  const int rows = Hp + 2;  // + halo above and below
  const unsigned slot_bytes = (unsigned)rows * kRowB;
  double* ring = smem;                                // [R][rows][kPitch]
  double* xuvp = ring + (size_t)R * rows * kPitch;   // [2][S][rows][2]
  double* xdp = xuvp + (size_t)2 * S * rows * 2;     // [3][S][rows][2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xdp + (size_t)3 * S * rows * 2);
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
  const unsigned ring_end = ring_s + (unsigned)R * slot_bytes;
  const unsigned xuv_s = (unsigned)__cvta_generic_to_shared(xuvp);
  const unsigned xd_s = (unsigned)__cvta_generic_to_shared(xdp);
  const unsigned uv_par_b = (unsigned)(S * rows * 16);  // one parity of xuv, bytes
  const unsigned d_ph_b = (unsigned)(S * rows * 16);    // one phase of xd, bytes
  // mbarriers [above p0, above p1, below p0, below p1]: one per direction and
  // step parity, so a barrier's phase n is step 2n + p and a neighbour (at
  // most one step ahead) can never overrun a phase its consumer still waits on
  const unsigned bar_above = (unsigned)__cvta_generic_to_shared(bars);
  const unsigned bar_below = bar_above + 16;
  const double* __restrict__ base = rec + (size_t)b * Ls;
  const size_t fstride = (size_t)B * Ls;
  const double* Dui = du_in ? du_in + (size_t)b * Ls : nullptr;  // may alias du_out
  const double* Dvi = dv_in ? dv_in + (size_t)b * Ls : nullptr;
  const double om1 = 1.0 - omega;

  // cp.async of this thread's record fields (t, t+S, ...) of one ring row
  auto fetch = [&](unsigned dst, const double* src, bool ok) {
    const double* g = ok ? src : base;
#pragma unroll
    for (int i = 0; i < kFieldsPerThread; ++i) {
      const int f = t + i * S;
      if (f < 8) cp_async8(dst + 8 * f, g + f * fstride, ok ? 8u : 0u);
    }
  };

  {  // ring + exchange buffers start at zero (idle threads read them)
    const int nx = R * rows * kPitch + (2 + 3) * S * rows * 2;
    for (int i = threadIdx.x; i < nx; i += blockDim.x) ring[i] = 0.0;
  }
  if (threadIdx.x == 0 && C > 1) {
    // one local arrive (the consumer's expect_tx) per phase; the neighbour's
    // S st.async (16 bytes each) complete the phase's transaction count
    mbar_init(bar_above, 1);
    mbar_init(bar_above + 8, 1);
    mbar_init(bar_below, 1);
    mbar_init(bar_below + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  int jn = 0;
  unsigned sin_s = ring_s;
  const double* gsrc = base + y0 + ty0;  // &record[jn * H + y0 + ty0]
  const unsigned my_ring_row = (unsigned)(ty0 + 1) * kRowB;
  auto issue_next = [&]() {
    if (jn < ndiag) {
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int yy = y0 + ty0 + i;
        const int x = jn - yy;
        fetch(sin_s + my_ring_row + i * kRowB, gsrc + i, yy < H && x >= 0 && x < W);
      }
      if (tg == 0) fetch(sin_s, gsrc - 1, y0 > 0 && jn - (y0 - 1) >= 0 && jn - (y0 - 1) < W);
      if (tg == TS - 1) {
        const int yy = y0 + Hp;
        fetch(sin_s + (unsigned)(Hp + 1) * kRowB, gsrc + RT, yy < H && jn - yy >= 0 &&
                                                                 jn - yy < W);
      }
    }
    cp_async_commit();
    ++jn;
    gsrc += H;
    sin_s += slot_bytes;
    if (sin_s == ring_end) sin_s = ring_s;
  };
  for (int j = 0; j < kLookahead; ++j) issue_next();
  cp_async_wait<kLookahead - 2>();
  if (C > 1) {  // barriers initialised everywhere before any remote arrive
    cluster_arrive();
    cluster_wait();
  } else {
    __syncthreads();
  }

  double lU[RT], lV[RT], lW[RT];  // each row's previous pixel (left neighbour / up of next row)
#pragma unroll
  for (int i = 0; i < RT; ++i) lU[i] = lV[i] = lW[i] = 0.0;
  bool bad = false;
  const int nsteps = ndiag + 2 * (S - 1);
  // ring slot address of diagonal j = k - 2t (rotates by one slot per step)
  unsigned a_j = ring_s + (unsigned)(((-2 * t) % R + R) % R) * slot_bytes;
  // exchange-buffer offsets of (t, my first row) and (t-1, my first row)
  const unsigned uv_me = (unsigned)((t * rows + ty0 + 1) * 16);
  const unsigned uv_prev = (unsigned)(((t > 0 ? t - 1 : 0) * rows + ty0 + 1) * 16);
  unsigned uv_r = xuv_s + uv_par_b, uv_w = xuv_s;  // parity of step k-1 / step k
  unsigned d_w = xd_s, d_r = xd_s + d_ph_b;       // phase k mod 3 / (k-2) mod 3
  const unsigned d_end = xd_s + 3 * d_ph_b;
  const size_t fplane = (size_t)W * H;
  // band-boundary roles
  const bool first_owner = C > 1 && c > 0 && tg == 0;                  // needs "up" of row 0
  const int last_ty = nrows - 1;
  const bool last_owner = C > 1 && c < C - 1 && ty0 <= last_ty && last_ty < ty0 + RT;
  int xk = -y0 - ty0 - 2 * t;  // x of my first row at step k
  for (int k = 0; k < nsteps; ++k, ++xk) {
    if (C > 1) {
      // post this step's expected halo bytes (phase k>>1 of barrier k&1; the
      // barrier's previous phase, step k-2, completed before step k-1 began)
      if (first_owner && t == 0) mbar_expect_tx(bar_above + (unsigned)(k & 1) * 8u, 16u * S);
      if (last_owner && t == 0) mbar_expect_tx(bar_below + (unsigned)(k & 1) * 8u, 16u * S);
      if (k > 0) {  // halo values of step k-1 from the neighbouring bands
        const unsigned sel = (unsigned)((k - 1) & 1) * 8u;
        const unsigned par = (unsigned)(((k - 1) >> 1) & 1);
        if (first_owner) mbar_wait_parity(bar_above + sel, par);
        // every boundary-row thread waits (t = 0 does not read the halo, but
        // its next write into the neighbour's halo must not overtake the
        // neighbour's read of the previous one)
        if (last_owner) mbar_wait_parity(bar_below + sel, par);
      }
    }
    issue_next();
    const int j = k - 2 * t;
    const unsigned a_m = (a_j == ring_s ? ring_end : a_j) - slot_bytes;
    const unsigned a_p = a_j + slot_bytes == ring_end ? ring_s : a_j + slot_bytes;
    const unsigned rp0 = a_j + my_ring_row;          // (x, y) of my first row
    const unsigned rm0 = a_m + my_ring_row - kRowB;  // (x, y-1)
    const unsigned rn0 = a_p + my_ring_row;          // (x+1, y); + kRowB: (x, y+1)
    double nU[RT], nV[RT], mU[RT], mV[RT], dU[RT], dV[RT], ucA[RT], vcA[RT], wpA[RT],
        m01A[RT], den_uA[RT], den_vA[RT], r1svA[RT];
    // Phase A (all rows, straight-line): neighbour values, weights, the four
    // sums and the u numerator.  Decreasing i: the "up" value of row i is
    // row i-1's step k-1 value (registers).
#pragma unroll
    for (int i = RT - 1; i >= 0; --i) {
      const int y = y0 + ty0 + i;
      const int x = xk - i;
      const bool hasU = y > 0, hasD = y < H - 1;
      const unsigned rp = rp0 + i * kRowB, rm = rm0 + i * kRowB, rn = rn0 + i * kRowB;
      const double uc = lds(rp + 8 * F_U), vc = lds(rp + 8 * F_V), wp = lds(rp + 8 * F_WS);
      const double m00 = lds(rp + 8 * F_M00), m01 = lds(rp + 8 * F_M01);
      const double m11 = lds(rp + 8 * F_M11);
      const double r0 = lds(rp + 8 * F_R0), r1 = lds(rp + 8 * F_R1);
      double upU, upV;
      if (i > 0) {  // row above is mine: its value from step k-1 (not yet updated)
        upU = lU[i - 1];
        upV = lV[i - 1];
      } else {
        lds2(uv_r + uv_me - 16, upU, upV);
      }
      const double upW = lds(rm + 8 * F_WS);
      const double rW = lds(rn + 8 * F_WS);
      const double dnW = lds(rn + kRowB + 8 * F_WS);
      double rU, rV, dnU, dnV, du, dv;
      if (t > 0) {
        lds2(uv_r + uv_prev + 16 * i, rU, rV);
        lds2(uv_r + uv_prev + 16 * (i + 1), dnU, dnV);
        lds2(d_r + uv_prev + 16 * i, du, dv);
      } else if (Dui) {  // chained pass: the carried du/dv of the previous sweeps
        const int jp = j + 1;
        const bool okp = jp >= 0 && jp < ndiag;
        const bool ok = j >= 0 && j < ndiag && y < H;
        const int yc = y < H ? y : H - 1;
        rU = lds(rn + 8 * F_U) + Dui[okp ? (size_t)jp * H + yc : 0];
        rV = lds(rn + 8 * F_V) + Dvi[okp ? (size_t)jp * H + yc : 0];
        dnU = lds(rn + kRowB + 8 * F_U) + Dui[okp && hasD ? (size_t)jp * H + yc + 1 : 0];
        dnV = lds(rn + kRowB + 8 * F_V) + Dvi[okp && hasD ? (size_t)jp * H + yc + 1 : 0];
        du = Dui[ok ? (size_t)j * H + y : 0];
        dv = Dvi[ok ? (size_t)j * H + y : 0];
      } else {
        rU = lds(rn + 8 * F_U) + 0.0;  // u + du with du = 0 (reference: u[q] + du[q])
        rV = lds(rn + 8 * F_V) + 0.0;
        dnU = lds(rn + kRowB + 8 * F_U) + 0.0;
        dnV = lds(rn + kRowB + 8 * F_V) + 0.0;
        du = 0.0;
        dv = 0.0;
      }
      // absent neighbours (borders) contribute wq = +0 times a finite value:
      // adding an exact zero leaves the reference's partial sums unchanged
      const double wqL = x > 0 ? 0.5 * (wp + lW[i]) : 0.0;
      const double wqR = x < W - 1 ? 0.5 * (wp + rW) : 0.0;
      const double wqU = hasU ? 0.5 * (wp + upW) : 0.0;
      const double wqD = hasD ? 0.5 * (wp + dnW) : 0.0;
      const double sw = (((0.0 + wqL) + wqR) + wqU) + wqD;
      const double su = (((0.0 + wqL * (lU[i] - uc)) + wqR * (rU - uc)) + wqU * (upU - uc)) +
                        wqD * (dnU - uc);
      const double sv = (((0.0 + wqL * (lV[i] - vc)) + wqR * (rV - vc)) + wqU * (upV - vc)) +
                        wqD * (dnV - vc);
      ucA[i] = uc;
      vcA[i] = vc;
      wpA[i] = wp;
      m01A[i] = m01;
      den_uA[i] = m00 + sw;
      den_vA[i] = m11 + sw;
      r1svA[i] = r1 + sv;
      dU[i] = du;
      dV[i] = dv;
      nU[i] = r0 + su - m01 * dv;
    }
    // Phase B: u quotients (straight-line fast division; rare IEEE fallback;
    // quotients of rows with den <= 1e-12 are discarded, whatever they are)
    bool slow = false;
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      slow = slow | ((den_uA[i] > 1e-12) & !div_fast_ok(nU[i], den_uA[i]));
      mU[i] = div_fast_rn(nU[i], den_uA[i]);
    }
    if (slow) {
#pragma unroll
      for (int i = 0; i < RT; ++i) mU[i] = exact_div_pos(nU[i], den_uA[i]);
    }
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      const double q = nU[i] == 0.0 ? nU[i] : mU[i];
      const double nu = om1 * dU[i] + omega * q;
      dU[i] = den_uA[i] > 1e-12 ? nu : dU[i];
      nV[i] = r1svA[i] - m01A[i] * dU[i];
    }
    // Phase C: v quotients (none in stereo mode: horizontal_only skips the
    // dv update, variational.py:161)
    if (!HZ) {
      slow = false;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        slow = slow | ((den_vA[i] > 1e-12) & !div_fast_ok(nV[i], den_vA[i]));
        mV[i] = div_fast_rn(nV[i], den_vA[i]);
      }
      if (slow) {
#pragma unroll
        for (int i = 0; i < RT; ++i) mV[i] = exact_div_pos(nV[i], den_vA[i]);
      }
    }
    // Phase D: updates, exchange stores, halo, output
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      const int ty = ty0 + i;
      const int y = y0 + ty;
      const int x = xk - i;
      double dv = dV[i];
      if (!HZ) {
        const double q = nV[i] == 0.0 ? nV[i] : mV[i];
        const double nv = om1 * dV[i] + omega * q;
        dv = den_vA[i] > 1e-12 ? nv : dV[i];
      }
      const double du = dU[i];
      const double U = ucA[i] + du, V = vcA[i] + dv;
      lU[i] = U;
      lV[i] = V;
      lW[i] = wpA[i];
      if (ty < nrows) {  // padding rows never store: row nrows+1 is the halo
        sts2(uv_w + uv_me + 16 * i, U, V);
        sts2(d_w + uv_me + 16 * i, du, dv);
      }
      if (C > 1) {
        if (ty == 0 && c > 0)  // band's first row -> CTA c-1's row below its band
          st_async2(uv_w + (unsigned)((t * rows + Hc + 1) * 16), bar_below + (unsigned)(k & 1) * 8u,
                    c - 1, U, V);
        if (ty == last_ty && c < C - 1)  // band's last row -> CTA c+1's row above its band
          st_async2(uv_w + (unsigned)(t * rows * 16), bar_above + (unsigned)(k & 1) * 8u, c + 1,
                    U, V);
      }
      if (t == S - 1 && ty < nrows && x >= 0 && x < W) {
        if (du_out) {
          du_out[(size_t)b * Ls + (size_t)j * H + y] = du;
          dv_out[(size_t)b * Ls + (size_t)j * H + y] = dv;
        }
        if (fu) {
          const size_t oo = (size_t)b * fplane + (size_t)y * W + x;
          fu[oo] = U;
          fv[oo] = V;
          bad |= !(isfinite(U) && isfinite(V));
        }
      }
    }
    cp_async_wait<kLookahead - 2>();
    __syncthreads();
    a_j = a_p;
    const unsigned tu = uv_r;
    uv_r = uv_w;
    uv_w = tu;
    d_w += d_ph_b;  // phases k mod 3 and (k-2) mod 3 both advance by one
    if (d_w == d_end) d_w = xd_s;
    d_r += d_ph_b;
    if (d_r == d_end) d_r = xd_s;
  }
  if (C > 1) {  // no CTA may exit while a neighbour can still write into it
    cluster_arrive();
    cluster_wait();
  }
  if (bad) set_status(status, DIS_STATUS_NONFINITE_FLOW);
}

template <int S>
static size_t sor_smem_bytes(int hp) {
  const size_t rows = (size_t)hp + 2;
  return ((size_t)ring_slots<S>() * rows * kPitch + (size_t)(2 + 3) * S * rows * 2) *
             sizeof(double) +
         4 * sizeof(uint64_t);
}

// rows per thread (RT): a thread carries RT independent row updates per
// step; fewer rows per thread = more warps to hide latency.
static int sor_rows_per_thread() {
  static const int rt = [] {
    const char* e = getenv("DIS_SOR_RT");  // experiments only
    const int v = e ? atoi(e) : 1;
    return (v == 1 || v == 2 || v == 4) ? v : 1;
  }();
  return rt;
}

constexpr size_t kMaxSmem = 227 * 1024;

// rows-per-CTA split: enough CTAs per pair to keep every band <= 256 rows and
// its ring in shared memory, and, for small batches, to spread a pair over
// several SMs (the step rate of one band is bound by its SM's FP64 pipe).
template <int S>
static int choose_cluster(int B, int H, int RT) {
  static const int forced = [] {
    const char* e = getenv("DIS_SOR_CLUSTER");  // experiments only
    return e ? atoi(e) : 0;
  }();
  if (forced > 0) return forced;
  const int q = 32 * RT;
  auto hp = [&](int C) { return ((H + C - 1) / C + q - 1) / q * q; };
  int C = 1;
  while (C < 16 && (hp(C) > kMaxBandRows || hp(C) / RT * S > S * kMaxBandRows / RT ||
                    sor_smem_bytes<S>(hp(C)) > kMaxSmem))
    ++C;
  // a band's step time scales with its rows: while the batch leaves SMs idle,
  // split the rows further (bands of >= 32 rows; the st.async halo exchange
  // costs ~0.15 us per step)
  static const int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  while (C < 16 && B * (C + 1) <= sms && (H + C) / (C + 1) >= 32) ++C;
  return C;
}

template <int S, int RT, bool HZ>
static int launch_sor_rt(const RefineArgs& a, size_t Ls, const double* dui, const double* dvi,
                         double* duo, double* dvo, bool final_pass, cudaStream_t st) {
  const int C = choose_cluster<S>(a.B, a.H, RT);
  const int Hc = (a.H + C - 1) / C;
  const int q = 32 * RT;
  const int hp = (Hc + q - 1) / q * q;
  const int threads = hp / RT * S;
  const size_t smem = sor_smem_bytes<S>(hp);
  if (hp > kMaxBandRows || smem > kMaxSmem) return DIS_ERR_VALUE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sor<S, RT, HZ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kMaxSmem);
    cudaFuncSetAttribute(k_sor<S, RT, HZ>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_sor<S, RT, HZ>, (const double*)a.rec, a.B, a.W, a.H,
                                     Hc, Ls, a.omega, dui, dvi, duo, dvo, fu, fv, a.status);
  return e == cudaSuccess ? DIS_OK : DIS_ERR_CUDA;
}

template <int S>
static int launch_sor_t(const RefineArgs& a, size_t Ls, const double* dui, const double* dvi,
                        double* duo, double* dvo, bool final_pass, cudaStream_t st) {
  // stereo (horizontal_only): one row per thread
  if (a.horizontal) return launch_sor_rt<S, 1, true>(a, Ls, dui, dvi, duo, dvo, final_pass, st);
  // more than 5 sweeps: the per-row shared memory grows, keep one row per thread
  const int rt = S > 5 ? 1 : sor_rows_per_thread();
  if (rt == 4) return launch_sor_rt<S, 4, false>(a, Ls, dui, dvi, duo, dvo, final_pass, st);
  if (rt == 2) return launch_sor_rt<S, 2, false>(a, Ls, dui, dvi, duo, dvo, final_pass, st);
  return launch_sor_rt<S, 1, false>(a, Ls, dui, dvi, duo, dvo, final_pass, st);
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
  if (a.H > 2048) return DIS_ERR_VALUE;  // at most 8 CTAs of <= 256 rows per pair
  const size_t Ls = (size_t)(a.W + a.H - 1) * a.H;
  double* carry_u = a.rec + (size_t)kRecords * a.B * Ls;
  double* carry_v = carry_u + (size_t)a.B * Ls;
  dim3 tb(256);
  dim3 tg((a.W + kTTX - 1) / kTTX, (a.H + kTTY - 1) / kTTY, a.B);
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
