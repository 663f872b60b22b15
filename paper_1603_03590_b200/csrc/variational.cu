// variational.cu — variational refinement of one level (refine,
// variational.py:220-275) for a batch of pairs.
//
// Per outer (fixed-point) iteration:
//   k_tensor_assemble : _tensor_fields (variational.py:36-88) fused with
//                       _assemble_system (91-121); the 12 tensor entries never
//                       reach HBM.  It also folds in everything of the SOR
//                       update (124-165) that does not change during the
//                       sweeps: the four neighbour weights wq = 0.5 (wp + ws_q)
//                       (+0 for an absent neighbour), sw = (((0 + wqL) + wqR)
//                       + wqU) + wqD and the denominators den_u = m00 + sw,
//                       den_v = m11 + sw — the same operations in the same
//                       order, so bit-identical, computed once instead of
//                       once per sweep.  Writes one 96-byte SOR record per
//                       pixel (u, v, m01, r0, r1, den_u, den_v, rcp_u, wqR,
//                       wqU, wqD, rcp_v) as six 16-byte chunks (rcp_* = the
//                       denominators' refined reciprocals) in the skewed,
//                       chunk-major layout [x + y][chunk][y]: one chunk of a
//                       whole anti-diagonal is one contiguous run, so a band
//                       of a diagonal is six bulk copies.
//   k_sor<S, HZ, P>   : theta_vi in-place lexicographic SOR sweeps
//                       (_sor_sweeps, variational.py:124-165) + the update
//                       u += du, v += dv (266-267) + the finiteness check.
//
// Exact lexicographic SOR on a GPU — the systolic wavefront.
// The reference sweeps row-major in place: pixel (x, y) in sweep t reads its
// left/up neighbours from sweep t and its right/down neighbours from sweep
// t-1.  Processing pixel (x, y) of sweep t at step k = x + y + 2t respects
// every one of those dependencies (bit-identical), and at
// a fixed step row y holds exactly one pixel per sweep, x = k - y - 2t.  A
// thread owns one row and a group of P consecutive sweeps; all rows of a
// band step together with one barrier per step (see k_sor below).
//
// Neighbour terms use U_q = fl(u_q + du_q) exactly as the reference's
// `u[y, x-1] + du[y, x-1]`; the last sweep's U is the updated flow.
#include <cuda.h>  // CUtensorMap (the encode entry point comes from the runtime)

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

// SOR record (doubles); 96 bytes = 6 chunks of 16 bytes.  RCPU/RCPV are the
// denominators' refined reciprocals (rcp_refined); the left weight is not
// stored: wq(x, x-1) == wq(x-1, x), the right weight of the previous pixel.
enum RecField {
  F_U = 0, F_V, F_M01, F_R0, F_R1, F_DENU, F_DENV, F_RCPU, F_WR, F_WU, F_WD, F_RCPV, kRec
};
constexpr int kChunks = kRec / 2;  // 16-byte chunks per record
constexpr int kMaxSweepsPerPass = 8;


size_t refine_scratch_doubles(int B, int W, int H) {
  const size_t Ls = (size_t)(W + H - 1) * H;
  // records + du/dv carry for > 8 sweeps
  return (size_t)(kRec + 2) * B * Ls;
}

// Tile of kTTX x kTTY pixels per block (one pixel per thread).
constexpr int kTTX = 32, kTTY = 8;

// image_gradients (core.py:75-85) of raster f at one pixel, computed on the
// fly: the one-sided border forms are the central form with the index
// clamped, 0.5 * (f[x+1] - f[x-1]) -> 0.5 * (f[1] - f[0]) at x = 0 and
// 0.5 * (f[W-1] - f[W-2]) at x = W-1 (W, H >= 2).  Used for the second
// derivatives _second_derivatives (variational.py:168-171) = the gradients
// of the gradient rasters, so they never go through HBM.
__device__ __forceinline__ double dx_at(const double* __restrict__ f, int W, int x, int y) {
  const int xm = x > 0 ? x - 1 : 0, xp = x < W - 1 ? x + 1 : W - 1;
  const size_t row = (size_t)y * W;
  return 0.5 * (__ldg(f + row + xp) - __ldg(f + row + xm));
}
__device__ __forceinline__ double dy_at(const double* __restrict__ f, int W, int H, int x, int y) {
  const int ym = y > 0 ? y - 1 : 0, yp = y < H - 1 ? y + 1 : H - 1;
  return 0.5 * (__ldg(f + (size_t)yp * W + x) - __ldg(f + (size_t)ym * W + x));
}

// _bilin (inverse_search.py:34-58) set-up shared by every raster sampled at
// the same warped coordinate (clamp, truncate, fractions)
struct BilinAt {
  int x0, x1, y0, y1;
  double fx, fy;
};
__device__ __forceinline__ BilinAt bilin_at(int W, int H, double x, double y) {
  if (!(x >= 0.0))
    x = 0.0;
  else if (x > W - 1.0)
    x = W - 1.0;
  if (!(y >= 0.0))
    y = 0.0;
  else if (y > H - 1.0)
    y = H - 1.0;
  BilinAt b;
  b.x0 = (int)x;
  b.y0 = (int)y;
  b.x1 = b.x0 + 1 > W - 1 ? W - 1 : b.x0 + 1;
  b.y1 = b.y0 + 1 > H - 1 ? H - 1 : b.y0 + 1;
  b.fx = x - (double)b.x0;
  b.fy = y - (double)b.y0;
  return b;
}
__device__ __forceinline__ double bilin_mix(const BilinAt& b, double i00, double i01, double i10,
                                            double i11) {
  const double a = i00 + b.fx * (i01 - i00);
  const double bb = i10 + b.fx * (i11 - i10);
  return a + b.fy * (bb - a);
}
__device__ __forceinline__ double bilin_raster(const double* __restrict__ f, int W,
                                               const BilinAt& b) {
  const double* r0 = f + (size_t)b.y0 * W;
  const double* r1 = f + (size_t)b.y1 * W;
  return bilin_mix(b, __ldg(r0 + b.x0), __ldg(r0 + b.x1), __ldg(r1 + b.x0), __ldg(r1 + b.x1));
}

// _tensor_fields (variational.py:36-88) + the system part of _assemble_system
// (91-118) at one pixel: u, v, m00, m01, m11, r0, r1.  The second
// derivatives of both levels (and their bilinear samples at the warped
// position) are formed from the gradient rasters on the fly.
// (up_, vp_: the pixel's flow, loaded by the caller)
__device__ __forceinline__ void pixel_system(const RefineArgs& a, int b, int x, int y,
                                             double up_, double vp_, double* r) {
  const int W = a.W, H = a.H;
  const size_t plane = (size_t)W * H;
  const size_t p = (size_t)y * W + x;
  const double* __restrict__ ref = a.ref + b * plane;
  const double* __restrict__ rgx = a.rgx + b * plane;
  const double* __restrict__ rgy = a.rgy + b * plane;
  const double* __restrict__ qry = a.qry + b * plane;
  const double* __restrict__ qgx = a.qgx + b * plane;
  const double* __restrict__ qgy = a.qgy + b * plane;

  double t0xx = 0.0, t0xy = 0.0, t0xz = 0.0, t0yy = 0.0, t0yz = 0.0, t0zz = 0.0;
  double tgxx = 0.0, tgxy = 0.0, tgxz = 0.0, tgyy = 0.0, tgyz = 0.0, tgzz = 0.0;
  const double wxp = x + up_;
  const double wyp = y + vp_;
  if (!(x == 0 || x == W - 1 || y == 0 || y == H - 1 || wxp < 0.0 || wxp > W - 1.0 ||
        wyp < 0.0 || wyp > H - 1.0)) {
    const BilinAt bl = bilin_at(W, H, wxp, wyp);
    const double iw = bilin_raster(qry, W, bl);
    // a query gradient raster at the warped position, with its two second
    // derivatives there: bilin_mix of dx_at / dy_at at the four corners.
    // The corners' central differences share their operands, so the 16
    // differences read 12 distinct pixels: rows y0, y1 at columns xL, x0,
    // x1, xR and rows yT, yB at columns x0, x1 (xL = max(x0-1, 0), xR =
    // min(x1+1, W-1), ...; at a clamped corner x1 == x0 the difference at
    // x1 is the one at x0, as dx_at's own clamping gives).  Same operands,
    // same operations: bit-identical to calling dx_at / dy_at per corner.
    const int xL = bl.x0 > 0 ? bl.x0 - 1 : 0, xR = bl.x1 < W - 1 ? bl.x1 + 1 : W - 1;
    const int yT = bl.y0 > 0 ? bl.y0 - 1 : 0, yB = bl.y1 < H - 1 ? bl.y1 + 1 : H - 1;
    const bool cx = bl.x1 == bl.x0, cy = bl.y1 == bl.y0;
    auto grad_at = [&](const double* __restrict__ f, double& fw, double& fxx, double& fxy) {
      const double* r0 = f + (size_t)bl.y0 * W;
      const double* r1 = f + (size_t)bl.y1 * W;
      const double* rT = f + (size_t)yT * W;
      const double* rB = f + (size_t)yB * W;
      const double a0L = __ldg(r0 + xL), a00 = __ldg(r0 + bl.x0), a01 = __ldg(r0 + bl.x1),
                   a0R = __ldg(r0 + xR);
      const double a1L = __ldg(r1 + xL), a10 = __ldg(r1 + bl.x0), a11 = __ldg(r1 + bl.x1),
                   a1R = __ldg(r1 + xR);
      const double aT0 = __ldg(rT + bl.x0), aT1 = __ldg(rT + bl.x1);
      const double aB0 = __ldg(rB + bl.x0), aB1 = __ldg(rB + bl.x1);
      fw = bilin_mix(bl, a00, a01, a10, a11);
      fxx = bilin_mix(bl, 0.5 * (a01 - a0L), 0.5 * (a0R - (cx ? a0L : a00)),
                      0.5 * (a11 - a1L), 0.5 * (a1R - (cx ? a1L : a10)));
      fxy = bilin_mix(bl, 0.5 * (a10 - aT0), 0.5 * (a11 - aT1), 0.5 * (aB0 - (cy ? aT0 : a00)),
                      0.5 * (aB1 - (cy ? aT1 : a01)));
    };
    double gxw, qxx, qxy, gyw, qyx, qyy;
    grad_at(qgx, gxw, qxx, qxy);
    grad_at(qgy, gyw, qyx, qyy);
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
    const double ixx = 0.5 * (dx_at(rgx, W, x, y) + qxx);
    const double ixy = 0.5 * (dy_at(rgx, W, H, x, y) + qxy);
    const double ixz = gxw - rgxp;
    const double iyx = 0.5 * (dx_at(rgy, W, x, y) + qyx);
    const double iyy = 0.5 * (dy_at(rgy, W, H, x, y) + qyy);
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
  const double eps2 = a.eps * a.eps;
  const double psi_i = 0.5 / sqrt(t0zz + eps2);
  const double psi_g = 0.5 / sqrt(tgzz + eps2);
  const double wi = a.delta * psi_i;
  const double wg = a.gamma * psi_g;
  r[0] = up_;
  r[1] = vp_;
  r[2] = wi * t0xx + wg * tgxx;     // m00
  r[3] = wi * t0xy + wg * tgxy;     // m01
  r[4] = wi * t0yy + wg * tgyy;     // m11
  r[5] = -(wi * t0xz + wg * tgxz);  // r0
  r[6] = -(wi * t0yz + wg * tgyz);  // r1
}

// the smoothness weight of _assemble_system (variational.py:113-121) from
// the flow at the pixel's four neighbours (clamped to the level like
// image_gradients' one-sided forms: (x+1, x-1) -> (1, 0) at x = 0)
__device__ __forceinline__ double pixel_ws(const RefineArgs& a, double2 l, double2 r, double2 t,
                                          double2 d) {
  const double ux = 0.5 * (r.x - l.x);
  const double uy = 0.5 * (d.x - t.x);
  const double vx = 0.5 * (r.y - l.y);
  const double vy = 0.5 * (d.y - t.y);
  const double grad2 = ux * ux + uy * uy + vx * vx + vy * vy;
  const double eps2 = a.eps * a.eps;
  return a.alpha * 0.5 / sqrt(grad2 + eps2);
}

// One block per kTTX x kTTY tile: the smoothness weights of the tile plus a
// one-pixel ring (the neighbours' ws), then each pixel's record (system +
// static SOR terms) staged in shared memory and written out as contiguous
// diagonal runs of 96-byte records (16-byte stores, coalesced).
// 4 blocks per SM (64 registers): the gathers are latency-bound; measured
// 3 -> 4 blocks: c1 0.62 -> 0.57 ms, c3 10.7 -> 9.7 ms (5 blocks spill)
__global__ void __launch_bounds__(256, 4) k_tensor_assemble(RefineArgs a, size_t Ls) {
  constexpr int HX = kTTX + 2, HY = kTTY + 2;
  constexpr int FX = kTTX + 4, FY = kTTY + 4;
  constexpr int kPad = kChunks + 1;  // 7 x 16 B per staged record: conflict-free writes
  __shared__ double ws_t[HY][HX];
  __shared__ double2 uv_t[FY][FX];  // the flow with a 2-pixel ring, clamped to the level
  __shared__ double2 rs[kTTY * kTTX][kPad];
  const int W = a.W, H = a.H;
  const int b = blockIdx.z;
  const int X0 = blockIdx.x * kTTX, Y0 = blockIdx.y * kTTY;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int x = X0 + lx, y = Y0 + ly;
  const bool inside = x < W && y < H;
  // the pixel's flow first: its loads are in flight while the flow tile's
  // are issued, and the system's warped gathers need only it (one memory
  // latency fewer on each thread's chain than tile -> barrier -> system)
  double up_ = 0.0, vp_ = 0.0;
  if (inside) {
    const size_t p = (size_t)b * W * H + (size_t)y * W + x;
    up_ = a.fu[p];
    vp_ = a.fv[p];
  }
  {  // flow tile: each pixel read once (the ring's smoothness weights read
     // their four neighbours from here instead of 8 gathers each)
    const double* __restrict__ u = a.fu + (size_t)b * W * H;
    const double* __restrict__ v = a.fv + (size_t)b * W * H;
    for (int i = threadIdx.x; i < FX * FY; i += 256) {
      const int fy = i / FX, fx = i - fy * FX;
      const int xx = min(max(X0 - 2 + fx, 0), W - 1), yy = min(max(Y0 - 2 + fy, 0), H - 1);
      const size_t q = (size_t)yy * W + xx;
      uv_t[fy][fx] = make_double2(u[q], v[q]);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HX * HY; i += 256) {
    const int hy = i / HX, hx = i - hy * HX;
    const int xx = X0 - 1 + hx, yy = Y0 - 1 + hy;
    ws_t[hy][hx] = (xx >= 0 && xx < W && yy >= 0 && yy < H)
                       ? pixel_ws(a, uv_t[hy + 1][hx], uv_t[hy + 1][hx + 2], uv_t[hy][hx + 1],
                                  uv_t[hy + 2][hx + 1])
                       : 0.0;
  }
  double r[7];
  if (inside) pixel_system(a, b, x, y, up_, vp_, r);
  __syncthreads();
  {
    if (inside) {
      // _sor_sweeps' static part (variational.py:133-158): absent neighbours
      // give wq = +0, and adding +0 to the non-negative partial sum sw
      // leaves it unchanged
      const double wp = ws_t[ly + 1][lx + 1];
      const double wqL = x > 0 ? 0.5 * (wp + ws_t[ly + 1][lx]) : 0.0;
      const double wqR = x < W - 1 ? 0.5 * (wp + ws_t[ly + 1][lx + 2]) : 0.0;
      const double wqU = y > 0 ? 0.5 * (wp + ws_t[ly][lx + 1]) : 0.0;
      const double wqD = y < H - 1 ? 0.5 * (wp + ws_t[ly + 2][lx + 1]) : 0.0;
      const double sw = (((0.0 + wqL) + wqR) + wqU) + wqD;
      double2* o = rs[threadIdx.x];
      o[0] = make_double2(r[0], r[1]);       // u, v
      o[1] = make_double2(r[3], r[5]);       // m01, r0
      o[2] = make_double2(r[6], r[2] + sw);  // r1, den_u = m00 + sw
      const double den_u = r[2] + sw, den_v = r[4] + sw;
      // the reciprocals carry the SOR's fast-division flag in their sign:
      // both denominators in the fast path's exact range -> the positive
      // refined reciprocals, else -1 (the SOR then divides exactly)
      const bool dfast = den_fast_ok(den_u) && den_fast_ok(den_v);
      o[3] = make_double2(den_v, dfast ? rcp_refined(den_u) : -1.0);  // den_v = m11 + sw
      o[4] = make_double2(wqR, wqU);
      o[5] = make_double2(wqD, dfast ? rcp_refined(den_v) : -1.0);
    }
  }
  __syncthreads();
  // diagonal runs: diagonal d = X0 + Y0 + dd holds tile rows ly with
  // lx = dd - ly in the tile; chunk c of those records is the contiguous run
  // [(d * kChunks + c) * H + y] of the layout.  Lane -> (row ly = lane % 8,
  // slot = lane / 8); the warp's four slots take consecutive (diagonal,
  // chunk) pairs, so 8 lanes write one 128-byte run.
  static_assert(kTTY == 8, "one 8-lane group per diagonal run");
  constexpr int ndd = kTTX + kTTY - 1;
  constexpr int npairs = ndd * kChunks;
  double2* __restrict__ out = reinterpret_cast<double2*>(a.rec + (size_t)b * Ls * kRec);
  const int wy = threadIdx.x & 7;
  const int oy = Y0 + wy;
  if (oy < H) {
    // (diagonal, chunk) pair m = dd * kChunks + c of the tile: its global run
    // starts at ((X0 + Y0) * kChunks + m) * H — linear in m, so the output
    // pointer advances by a constant; dd and c step by 32 = 5 * kChunks + 2
    static_assert(kChunks == 6, "pair stepping below");
    const int m0 = threadIdx.x >> 3;
    int dd = m0 / kChunks;
    int c = m0 - dd * kChunks;
    const unsigned xlim = (unsigned)min(kTTX, W - X0);  // tile columns inside the level
    double2* __restrict__ o = out + ((size_t)(X0 + Y0) * kChunks + m0) * H + oy;
    const double2* src = &rs[wy * kTTX][0] + (dd - wy) * kPad + c;
    const size_t ostep = (size_t)32 * H;
#pragma unroll 2
    for (int m = m0; m < npairs; m += 32) {
      if ((unsigned)(dd - wy) < xlim) *o = *src;
      o += ostep;
      c += 2;
      dd += 5;
      src += 5 * kPad + 2;
      if (c >= kChunks) {
        c -= kChunks;
        dd += 1;
        src += kPad - kChunks;
      }
    }
  }
}

#ifndef DIS_SOR_LOOKAHEAD
#define DIS_SOR_LOOKAHEAD 5
#endif
constexpr int kLookahead = DIS_SOR_LOOKAHEAD;  // diagonals fetched ahead of sweep 0
constexpr int kMaxBandRows = 128;  // rows (threads per sweep) of one CTA's band
// ring rows of a band of hc rows: the band + the row below (sweep 0's down
// neighbour of the band's last row), rounded to 4 (a ring slot of 6 chunks x
// rows x 16 B is then a multiple of 128 bytes, the TMA destination
// alignment); the TMA box holds 2 * rows <= 256 doubles.  A 128-row band
// (levels of 2033..2048 rows: 16 bands) has no room for the row below in
// the box: its u, v come as a second 16-byte box into a 128-byte slot beside
// the ring ("below mode").
__host__ __device__ constexpr bool sor_below_mode(int hc) { return hc + 1 > 128; }
__host__ __device__ constexpr int sor_ring_rows(int hc) {
  return sor_below_mode(hc) ? ((hc + 3) & ~3) : ((hc + 1 + 3) & ~3);
}
constexpr int kBelowSlot = 128;  // below mode: bytes after a ring slot for the row below

template <int S>
__host__ __device__ constexpr int ring_slots() {
  // live at step k: diagonals k - 2(S-1) (last sweep) .. k + 1 (sweep 0's right
  // and down neighbours), plus the fills in flight up to k + kLookahead
  return 2 * (S - 1) + 1 + kLookahead;
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
// mbarrier helpers (band-boundary signalling between the CTAs of a cluster)
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
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
// explicit shared-space accesses (32-bit addresses)
__device__ __forceinline__ void sts2(unsigned a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void lds2(unsigned a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}

__device__ __forceinline__ void mbar_wait_parity_cta(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// The wavefront SOR kernel.
//
// Thread (g, r) owns band row y = y0 + r and a group of P consecutive sweeps
// t = gP .. gP+P-1 (the last group may hold fewer), and computes, at step k,
// the pixels x_t = k - y - 2t of its sweeps (diagonals j = k - 2t;
// independent within the step, so their chains interleave).  A pair's rows
// are split over a cluster of C CTAs (1..16); CTA c owns the band
// [c*Hc, c*Hc + Hc), padded to Hp rows (a multiple of 32).  Inside a group
// three of the five neighbour terms come from the thread's own registers:
//   left  (x-1, y) of sweep t   = my sweep-t value of step k-1
//   right (x+1, y) of sweep t-1 = my sweep-(t-1) value of step k-1
//   self du of sweep t-1        = my sweep-(t-1) du of step k-2
//   up    (x, y-1) of sweep t   = row r-1's sweep-t value of step k-1 (xuv)
//   down  (x, y+1) of sweep t-1 = row r+1's sweep-(t-1) value of step k-1 (xuv)
// A group's first sweep takes right from xuv and self du from xd (written
// by the previous group's last sweep two steps before); sweep 0's right,
// down and self terms are the records' u, v (+ du = 0, or the carried du of
// a chained pass).  The left weight is the previous pixel's right weight
// (same operands, commutative add) and the denominators' reciprocals come
// refined in the record, so an update is operation for operation the
// reference's: su, sv in its neighbour order, then the two divisions.
// Shared memory:
//   ring[R][6][rb] x 16 B   : the 96-byte records of the live diagonals (band
//                             rows + the row below, sweep 0's down
//                             neighbour; rb = sor_ring_rows), chunk-major
//                             like the global layout: one diagonal = one
//                             TMA box (cp.async.bulk.tensor) issued by the
//                             producer warp kLookahead steps ahead,
//                             completion counted on the slot's mbarrier
//   xuv[2][S][Hp+2] x 16 B  : U, V of the last two steps (+ halo rows above
//                             and below the band)
//   xd [3][G-1][Hp] x 16 B  : group-boundary du, dv of the last three steps
// The band's boundary rows write their U, V straight into the neighbouring
// CTA's halo rows (distributed shared memory, st.async counted on that
// CTA's mbarrier).
//
// Idle pixels (outside the level: ramp-up/down of the wavefront, rows past
// the band) publish U = V = 0 and a zero right weight (their ring slots are
// zero-filled past the last row and hold no record where x is outside
// [0, W): masked); a valid pixel's absent neighbour enters its sums as
// +0 * 0.  A warp whose pixels are all idle skips the arithmetic (and
// publishes zeros).
template <int S, bool HZ, int P>
__global__ void __launch_bounds__(((S + P - 1) / P) * kMaxBandRows + 32, 1)
    k_sor(const double* __restrict__ rec, int B, int W, int H, int Hc, size_t Ls,
               double omega, const double* du_in, const double* dv_in, double* du_out,
               double* dv_out, double* __restrict__ fu, double* __restrict__ fv,
               uint32_t* status, const __grid_constant__ CUtensorMap tmap,
               const __grid_constant__ CUtensorMap tmap_below) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int R = ring_slots<S>();
  constexpr int G = (S + P - 1) / P;       // sweep groups
  constexpr int PL = S - (G - 1) * P;      // sweeps of the last group
  const int C = (int)(gridDim.x / (unsigned)B) > 0 ? (int)(gridDim.x / (unsigned)B) : 1;
  const int c = C > 1 ? (int)cluster_rank() : 0;
  const int b = blockIdx.x / C;
  const int Hp = ((int)blockDim.x - 32) / G;  // band rows (padded); + one producer warp
  const bool producer = threadIdx.x >= (unsigned)(G * Hp);  // ring fill, no pixels
  const int g = producer ? 0 : (int)threadIdx.x / Hp;
  const int r = producer ? Hp : (int)threadIdx.x - g * Hp;
  const int t0 = g * P;  // my first sweep
  const int y0 = c * Hc;
  const int y = y0 + r;
  const int nrows = min(Hc, H - y0);
  const int ndiag = W + H - 1;
  const int rrows = sor_ring_rows(Hc);  // ring rows
  const int xrows = Hp + 2;  // exchange rows
  const bool below = sor_below_mode(Hc);  // the row below has its own 16 bytes
  const unsigned below_off = (unsigned)(kChunks * rrows * 16);  // (after the slot's chunks)
  const unsigned slot_bytes = below_off + (below ? (unsigned)kBelowSlot : 0u);
  // (opaque: the compiler otherwise rebuilds the shared-window address from
  // SR_CgaCtaId, an S2R on every step's ring wrap)
  unsigned ring_s_v = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("" : "+r"(ring_s_v));
  const unsigned ring_s = ring_s_v;
  const unsigned ring_end = ring_s + (unsigned)R * slot_bytes;
  const unsigned xuv_s = ring_end;
  const unsigned xd_s = xuv_s + (unsigned)(2 * S * xrows * 16);
  const unsigned d_ph_b = (unsigned)((G > 1 ? G - 1 : 1) * Hp * 16);  // one xd phase
  const unsigned bar_above = xd_s + 3 * d_ph_b;  // 8-byte aligned
  const unsigned bar_below = bar_above + 16;
  const unsigned bar_ring = bar_above + 32;  // [R] slot-fill barriers
  const double* Dui = du_in ? du_in + (size_t)b * Ls : nullptr;  // may alias du_out
  const double* Dvi = dv_in ? dv_in + (size_t)b * Ls : nullptr;
  const double om1 = 1.0 - omega;

  {  // ring + exchange buffers start at zero
    const unsigned nz = (bar_above - ring_s) / 16u;  // 16-byte entries
    for (unsigned i = threadIdx.x; i < nz; i += blockDim.x) sts2(ring_s + 16 * i, 0.0, 0.0);
  }
  if (threadIdx.x == 0) {
    if (C > 1) {
      mbar_init(bar_above, 1);
      mbar_init(bar_above + 8, 1);
      mbar_init(bar_below, 1);
      mbar_init(bar_below + 8, 1);
    }
    for (int i = 0; i < R; ++i) mbar_init(bar_ring + 8u * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ring fill (producer warp): diagonal jn -> slot jn % R, one TMA box per
  // diagonal issued by one thread (the per-chunk bulk copies it replaces
  // cost ~800 cycles of issue per diagonal, on the small levels' critical
  // path: 0.66 -> 0.57 us per step).
  const unsigned lane = threadIdx.x & 31;
  int jn = 0;
  unsigned sin_s = ring_s, sin_bar = bar_ring;
  auto issue_next = [&]() {
    // the box [2 * rrows doubles of rows y0 ..][6 chunks] of diagonal jn:
    // rows past the level are zero-filled by the TMA unit, the diagonal's
    // slots of pixels outside the level (x = jn - y outside [0, W)) hold
    // whatever the record array holds there (masked by the compute warps)
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sin_bar),
                   "r"(below_off + (below ? 16u : 0u))
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(sin_s),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(2 * y0), "r"(0), "r"(b * ndiag + jn),
          "r"(sin_bar)
          : "memory");
      if (below)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(sin_s + below_off),
            "l"(reinterpret_cast<uint64_t>(&tmap_below)), "r"(2 * (y0 + Hc)), "r"(0),
            "r"(b * ndiag + jn), "r"(sin_bar)
            : "memory");
    }
    ++jn;
    sin_s += slot_bytes;
    sin_bar += 8;
    if (sin_s == ring_end) {
      sin_s = ring_s;
      sin_bar = bar_ring;
    }
  };
  // slot readiness: fill n of slot s (diagonal s + nR) completes phase n
  auto wait_diag = [&](int j) {
    if (j >= 0 && j < jn)
      mbar_wait_parity_cta(bar_ring + 8u * (unsigned)(j % R), (unsigned)((j / R) & 1));
  };
  const bool filler = threadIdx.x == (unsigned)(G * Hp);  // lane 0 of the producer warp
  if (producer) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the start-up clear
    for (int j = 0; j < kLookahead; ++j) issue_next();
    if (filler) {
      wait_diag(0);
      wait_diag(1);
    }
  }
  if (C > 1) {  // barriers initialised everywhere before any remote arrive
    cluster_arrive();
    cluster_wait();
  } else {
    __syncthreads();
  }
  const int nsteps = ndiag + 2 * (S - 1);
  // my values of the last two steps, per sweep of my group
  double Up[P], Vp[P], Dp[P], DVp[P], Dp2[P], DVp2[P], WRp[P], Un[P], Vn[P], Dn[P], DVn[P],
      WRn[P];
#pragma unroll
  for (int i = 0; i < P; ++i) Up[i] = Vp[i] = Dp[i] = DVp[i] = Dp2[i] = DVp2[i] = WRp[i] = 0.0;
  bool bad = false;
  unsigned a_k = ring_s;  // slot of diagonal k
  const unsigned rrow = (unsigned)(r * 16);
  // sweep 0's down neighbour in the next diagonal's slot: ring row r + 1, or
  // (below mode, the band's last row) the row-below area
  const unsigned dn_off = below && r == Hc - 1 ? below_off : rrow + 16;
  const unsigned cstride = (unsigned)(rrows * 16);
  const unsigned xstride = (unsigned)(xrows * 16);
  unsigned uv_r = xuv_s + (unsigned)S * xstride, uv_w = xuv_s;  // step k-1 / step k
  unsigned d_w = xd_s, d_r = xd_s + d_ph_b;  // xd phase k mod 3 / (k-2) mod 3
  const unsigned d_end = xd_s + 3 * d_ph_b;
  const size_t fplane = (size_t)W * H;
  const int last_r = nrows - 1;
  const int wr0 = r & ~31;  // first row of my warp
  const bool first_owner = C > 1 && c > 0 && r == 0 && !producer;
  const bool last_owner = C > 1 && c < C - 1 && r == last_r && !producer;
  const bool live_warp = !producer && wr0 < nrows;
  const int nt = g == G - 1 ? PL : P;  // my sweeps (warp-uniform)

  // one step of my group's NT sweeps (NT = P, or PL for the last group)
  auto step = [&](auto ntc, int k, unsigned a_p) {
    constexpr int NT = decltype(ntc)::value;
    // warp-uniform: any of my warp's pixels inside the level in any of my
    // sweeps?  (lane 0 holds the warp's largest x; sweep t's x is k - y - 2t)
    const int xw0 = k - y0 - wr0 - 2 * t0;
    if (!(live_warp && xw0 >= 0 && xw0 - 2 * (NT - 1) < W + 31)) {
#pragma unroll
      for (int i = 0; i < NT; ++i) Un[i] = Vn[i] = Dn[i] = DVn[i] = WRn[i] = 0.0;
      return;
    }
    // my first sweep's right / down neighbours and own du
    double rUf, rVf, dnUf, dnVf, duf = 0.0, dvf = 0.0;
    if (g == 0) {  // sweep 0: the records (+ the carried du of a chained pass)
      lds2(a_p + rrow, rUf, rVf);
      // (below mode, the band's last row: the row below has its own slot)
      lds2(a_p + dn_off, dnUf, dnVf);
      if (Dui) {
        const int j = k;
        const bool hasD = y < H - 1;
        const int jp = j + 1;
        const bool okp = jp >= 0 && jp < ndiag;
        const bool ok = j >= 0 && j < ndiag && y < H;
        const int yc = y < H ? y : H - 1;
        rUf = rUf + Dui[okp ? (size_t)jp * H + yc : 0];
        rVf = rVf + Dvi[okp ? (size_t)jp * H + yc : 0];
        dnUf = dnUf + Dui[okp && hasD ? (size_t)jp * H + yc + 1 : 0];
        dnVf = dnVf + Dvi[okp && hasD ? (size_t)jp * H + yc + 1 : 0];
        duf = Dui[ok ? (size_t)j * H + y : 0];
        dvf = Dvi[ok ? (size_t)j * H + y : 0];
      } else {
        rUf = rUf + 0.0;  // the reference's u[q] + du[q]
        rVf = rVf + 0.0;
        dnUf = dnUf + 0.0;
        dnVf = dnVf + 0.0;
      }
      if (!(k - y + 1 < W)) {  // right neighbour outside the level:
        rUf = 0.0;                              // its ring slot is not a record
        rVf = 0.0;
      }
    } else {  // the previous group's last sweep (exchange buffers)
      lds2(uv_r + (unsigned)(t0 - 1) * xstride + rrow + 16, rUf, rVf);
      lds2(uv_r + (unsigned)(t0 - 1) * xstride + rrow + 32, dnUf, dnVf);
      lds2(d_r + (unsigned)((g - 1) * Hp * 16) + rrow, duf, dvf);
    }
    // all my sweeps' pixels, branch-free (independent chains interleave);
    // idle pixels see zero records and never update.  The rare operands
    // outside the fast division's exact range are redone after each pass.
    double uc[NT], vc[NT], m01[NT], r1[NT], den_u[NT], den_v[NT], rcp_v[NT], sv[NT], du[NT],
        dv[NT], q[NT], nn[NT];
    bool dfast[NT], slow[NT], valid[NT];
    bool any_slow = false;
    // slot of my first sweep's diagonal k - 2 t0 (mod R)
    unsigned a_f = a_k - (unsigned)(2 * t0) * slot_bytes;
    if ((int)(a_k - ring_s) < 2 * t0 * (int)slot_bytes) a_f += (unsigned)R * slot_bytes;
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const int t = t0 + i;
      unsigned a_j = a_f - (unsigned)(2 * i) * slot_bytes;  // slot of k - 2t
      if (i > 0 && (int)(a_f - ring_s) < 2 * i * (int)slot_bytes) a_j += (unsigned)R * slot_bytes;
      double r0, rcp_u, wqR, wqU, wqD;
      lds2(a_j + rrow, uc[i], vc[i]);
      lds2(a_j + cstride + rrow, m01[i], r0);
      lds2(a_j + 2 * cstride + rrow, r1[i], den_u[i]);
      lds2(a_j + 3 * cstride + rrow, den_v[i], rcp_u);
      lds2(a_j + 4 * cstride + rrow, wqR, wqU);
      lds2(a_j + 5 * cstride + rrow, wqD, rcp_v[i]);
      const double wqL = WRp[i];  // the previous pixel's right weight
      // pixel inside the level (TMA ring: other slots are not records)
      valid[i] = (unsigned)(k - y - 2 * t) < (unsigned)W && r < nrows;
      WRn[i] = wqR;
      dfast[i] = rcp_u > 0.0;  // (tensor_assemble: -1 when not both in range)
      double upU, upV, rU, rV, dnU, dnV;
      lds2(uv_r + (unsigned)t * xstride + rrow, upU, upV);  // exchange row r = band row r-1
      if (i > 0) {
        rU = Up[i - 1];
        rV = Vp[i - 1];
        lds2(uv_r + (unsigned)(t - 1) * xstride + rrow + 32, dnU, dnV);  // band row r+1
        du[i] = Dp2[i - 1];
        dv[i] = DVp2[i - 1];
      } else {
        rU = rUf;
        rV = rVf;
        dnU = dnUf;
        dnV = dnVf;
        du[i] = duf;
        dv[i] = dvf;
      }
      const double cu = uc[i], cv = vc[i];
      const double su = (((0.0 + wqL * (Up[i] - cu)) + wqR * (rU - cu)) + wqU * (upU - cu)) +
                        wqD * (dnU - cu);
      sv[i] = (((0.0 + wqL * (Vp[i] - cv)) + wqR * (rV - cv)) + wqU * (upV - cv)) +
              wqD * (dnV - cv);
      nn[i] = r0 + su - m01[i] * dv[i];
      q[i] = div_by_rcp(nn[i], den_u[i], rcp_u);
      slow[i] = valid[i] && (den_u[i] > 1e-12) && !(dfast[i] && num_fast_ok(nn[i]));
      any_slow |= slow[i];
    }
    if (any_slow) {
#pragma unroll
      for (int i = 0; i < NT; ++i)
        if (slow[i]) q[i] = exact_div_pos(nn[i], den_u[i]);
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const double qq = nn[i] == 0.0 ? nn[i] : q[i];
      const double nu = om1 * du[i] + omega * qq;
      du[i] = den_u[i] > 1e-12 ? nu : du[i];
    }
    if (!HZ) {
      any_slow = false;
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        nn[i] = r1[i] + sv[i] - m01[i] * du[i];
        q[i] = div_by_rcp(nn[i], den_v[i], rcp_v[i]);
        slow[i] = valid[i] && (den_v[i] > 1e-12) && !(dfast[i] && num_fast_ok(nn[i]));
        any_slow |= slow[i];
      }
      if (any_slow) {
#pragma unroll
        for (int i = 0; i < NT; ++i)
          if (slow[i]) q[i] = exact_div_pos(nn[i], den_v[i]);
      }
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        const double qq = nn[i] == 0.0 ? nn[i] : q[i];
        const double nv = om1 * dv[i] + omega * qq;
        dv[i] = den_v[i] > 1e-12 ? nv : dv[i];
      }
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      // pixels outside the level publish U = V = 0 and a zero right weight
      // (what valid neighbours read; their du, dv only reach the same
      // pixel's later sweeps, which are outside the level too)
      Un[i] = valid[i] ? uc[i] + du[i] : 0.0;
      Vn[i] = valid[i] ? vc[i] + dv[i] : 0.0;
      Dn[i] = du[i];
      DVn[i] = dv[i];
      WRn[i] = valid[i] ? WRn[i] : 0.0;
    }
  };

  for (int k = 0; k < nsteps; ++k) {
    if (first_owner) {
      if (g == 0) mbar_expect_tx(bar_above + (unsigned)(k & 1) * 8u, 16u * S);
      if (k > 0)
        mbar_wait_parity(bar_above + (unsigned)((k - 1) & 1) * 8u, (unsigned)(((k - 1) >> 1) & 1));
    }
    if (last_owner) {
      if (g == 0) mbar_expect_tx(bar_below + (unsigned)(k & 1) * 8u, 16u * S);
      if (k > 0)
        mbar_wait_parity(bar_below + (unsigned)((k - 1) & 1) * 8u, (unsigned)(((k - 1) >> 1) & 1));
    }
    if (producer) issue_next();
    const unsigned a_p = a_k + slot_bytes == ring_end ? ring_s : a_k + slot_bytes;  // k + 1
    if (PL == P || nt == P)
      step(std::integral_constant<int, P>{}, k, a_p);
    else
      step(std::integral_constant<int, PL>{}, k, a_p);
    // ---- exchange, halo, output ----
    if (!producer && r < nrows) {  // padding rows never store
#pragma unroll
      for (int i = 0; i < P; ++i)
        if (i < nt) sts2(uv_w + (unsigned)(t0 + i) * xstride + rrow + 16, Un[i], Vn[i]);
    }
    if (G > 1 && !producer && g < G - 1)  // my last sweep's du for the next group
      sts2(d_w + (unsigned)(g * Hp * 16) + rrow, Dn[P - 1], DVn[P - 1]);
    if (first_owner) {  // band's first row -> CTA c-1's row below its band
#pragma unroll
      for (int i = 0; i < P; ++i)
        if (i < nt)
          st_async2(uv_w + (unsigned)(t0 + i) * xstride + (unsigned)((Hc + 1) * 16),
                    bar_below + (unsigned)(k & 1) * 8u, c - 1, Un[i], Vn[i]);
    }
    if (last_owner) {  // band's last row -> CTA c+1's row above its band
#pragma unroll
      for (int i = 0; i < P; ++i)
        if (i < nt)
          st_async2(uv_w + (unsigned)(t0 + i) * xstride, bar_above + (unsigned)(k & 1) * 8u,
                    c + 1, Un[i], Vn[i]);
    }
    if (!producer && g == G - 1) {  // the last sweep's pixel: outputs
      const int x = k - y - 2 * (S - 1);
      const int j = k - 2 * (S - 1);
      if (r < nrows && x >= 0 && x < W) {
        const double uo = Un[PL - 1], vo = Vn[PL - 1];
        if (du_out) {
          du_out[(size_t)b * Ls + (size_t)j * H + y] = Dn[PL - 1];
          dv_out[(size_t)b * Ls + (size_t)j * H + y] = DVn[PL - 1];
        }
        if (fu) {
          const size_t oo = (size_t)b * fplane + (size_t)y * W + x;
          fu[oo] = uo;
          fv[oo] = vo;
          bad |= !(isfinite(uo) && isfinite(vo));
        }
      }
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
      Up[i] = Un[i];
      Vp[i] = Vn[i];
      WRp[i] = WRn[i];
      Dp2[i] = Dp[i];
      DVp2[i] = DVp[i];
      Dp[i] = Dn[i];
      DVp[i] = DVn[i];
    }
    if (filler) wait_diag(k + 2);  // sweep 0 reads k+1 and k+2 next step
    __syncthreads();
    a_k = a_p;
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
static int sor_group_size(int hc, int ctas) {
  static const int forced = [] {
    const char* e = getenv("DIS_SOR_P");  // experiments only
    const int v = e ? atoi(e) : 0;
    return v == 1 || v == 2 ? v : (v > 2 ? S : 0);
  }();
  // two sweeps per thread (half the threads, two independent chains each)
  // where the step is issue-bound: tall bands or more CTAs than SMs
  // (measured: 218-row levels 1.075 -> 1.015 us/step, c3's 60-row bands
  // over 2304 CTAs 0.979 -> 0.937); one sweep per thread on the small,
  // latency-bound levels (13-row level 0.557 vs 0.608 us/step)
  const int p = forced ? forced : ((hc >= 96 || ctas > device_sm_count()) ? 2 : 1);
  return p < S ? p : S;
}

// dynamic shared memory of a band of hc rows padded to hp (the kernel's
// carve-out: ring slots of sor_ring_rows(hc) rows (+ the below-mode slot),
// exchange rows, group-boundary du phases, barriers).  Exact, so two CTAs
// of small bands still fit one SM (a 49-row band at P = 1 needs 93 KB; the
// hp + 4 row bound it replaces came to 116 KB and cost c2's 1024x436 level
// its second CTA per SM: 1.67 -> 2.35 ms)
template <int S>
static size_t sor_rows_smem_bytes(int hc, int hp, int P = 1) {
  const int G = (S + P - 1) / P;
  const size_t rrows = (size_t)sor_ring_rows(hc), xrows = (size_t)hp + 2;
  const size_t slot = kChunks * rrows * 16 + (sor_below_mode(hc) ? (size_t)kBelowSlot : 0);
  return (size_t)ring_slots<S>() * slot + (size_t)2 * S * xrows * 16 +
         (size_t)3 * (G > 1 ? G - 1 : 1) * hp * 16 + (4 + ring_slots<S>()) * sizeof(uint64_t);
}

constexpr size_t kMaxSmem = 227 * 1024;

template <int S>
static int choose_cluster(int B, int H) {
  static const int forced = [] {
    const char* e = getenv("DIS_SOR_CLUSTER");  // experiments only
    return e ? atoi(e) : 0;
  }();
  if (forced > 0) return forced;
  auto hp = [&](int C) { return ((H + C - 1) / C + 31) / 32 * 32; };
  const int max_rows = kMaxBandRows;
  int C = 1;
  while (C < 16 && ((H + C - 1) / C > max_rows || hp(C) > kMaxBandRows ||
                    sor_rows_smem_bytes<S>((H + C - 1) / C, hp(C)) > kMaxSmem))
    ++C;
  const int sms = device_sm_count();
  // while the batch leaves SMs idle, split the rows further (bands of >= 32
  // rows; the st.async halo exchange costs ~0.15 us per step)
  while (C < 16 && B * (C + 1) <= sms && (H + C) / (C + 1) >= 32) ++C;
  // several waves of CTAs: 64-row bands (two CTAs per SM, whose steps
  // interleave) when they pad no more rows (c3's 540-row level: 9
  // bands of 60 rows run 12 % faster than 5 of 108)
  if (B * C > sms) {
    const int C64 = (H + 63) / 64;
    if (C64 <= 16 && (long)C64 * 64 <= (long)C * hp(C) &&
        sor_rows_smem_bytes<S>((H + C64 - 1) / C64, 64) * 2 <= kMaxSmem)
      C = C64;
  }
  return C;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time dependency on libcuda)
static bool encode_tensor_map(CUtensorMap* m, CUtensorMapDataType dt, cuuint32_t rank,
                              void* addr, const cuuint64_t* dims, const cuuint64_t* strides,
                              const cuuint32_t* box, const cuuint32_t* estr) {
  using EncFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncFn>(f);
  }();
  if (!fn) return false;
  return fn(m, dt, rank, addr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int S, bool HZ>
static int launch_sor_t(const RefineArgs& a, size_t Ls, const double* dui, const double* dvi,
                        double* duo, double* dvo, bool final_pass, cudaStream_t st) {
  int C = choose_cluster<S>(a.B, a.H);
  while (C > 1 && (C - 1) * ((a.H + C - 1) / C) >= a.H) --C;  // no empty band (forced sizes)
  const int Hc = (a.H + C - 1) / C;
  const int hp = (Hc + 31) / 32 * 32;
  const int P = sor_group_size<S>(Hc, a.B * C);
  const int G = (S + P - 1) / P;
  const int threads = hp * G + 32;  // + the producer warp
  const size_t smem = sor_rows_smem_bytes<S>(Hc, hp, P);
  if (hp > kMaxBandRows || smem > kMaxSmem) return DIS_ERR_VALUE;
  using KFn = void (*)(const double*, int, int, int, int, size_t, double, const double*,
                       const double*, double*, double*, double*, double*, uint32_t*,
                       const CUtensorMap, const CUtensorMap);
  CUtensorMap tmap, tmap_below;
  std::memset(&tmap, 0, sizeof(tmap));
  std::memset(&tmap_below, 0, sizeof(tmap_below));
  {
    // the record array as [B * (W + H - 1) diagonals][6 chunks][2H doubles];
    // box = one band's ring rows of one diagonal (tmap) / the u, v of one
    // row (tmap_below: the row below the band)
    if (sor_ring_rows(Hc) > kMaxBandRows) return DIS_ERR_VALUE;
    const cuuint64_t dims[3] = {(cuuint64_t)2 * a.H, (cuuint64_t)kChunks,
                                (cuuint64_t)a.B * (a.W + a.H - 1)};
    const cuuint64_t strides[2] = {(cuuint64_t)2 * a.H * sizeof(double),
                                   (cuuint64_t)kChunks * 2 * a.H * sizeof(double)};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * sor_ring_rows(Hc)), (cuuint32_t)kChunks, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const cuuint32_t box_below[3] = {2, 1, 1};
    if (!encode_tensor_map(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)a.rec, dims, strides,
                           box, estr) ||
        !encode_tensor_map(&tmap_below, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)a.rec, dims,
                           strides, box_below, estr))
      return DIS_ERR_CUDA;
  }
  KFn kfn = k_sor<S, HZ, S>;
  if (P == 1)
    kfn = k_sor<S, HZ, 1>;
  else if (P == 2)
    kfn = k_sor<S, HZ, (S >= 2 ? 2 : 1)>;
  // function attributes are per device and kernel: set them once for each
  // (device, group size) used
  static bool attr[kMaxDevices][3];
  const int dev = current_device();
  const int pi = P == 1 ? 0 : (P == 2 ? 1 : 2);
  if (!attr[dev][pi]) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
    cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr[dev][pi] = true;
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, (const double*)a.rec, a.B, a.W, a.H, Hc, Ls, a.omega, dui,
                                     dvi, duo, dvo, fu, fv, a.status, tmap, tmap_below);
  return e == cudaSuccess ? DIS_OK : DIS_ERR_CUDA;
}

static int launch_sor(const RefineArgs& a, size_t Ls, int S, const double* dui,
                      const double* dvi, double* duo, double* dvo, bool final_pass,
                      cudaStream_t st) {
  switch (S) {
#define DIS_SOR_CASE(n)                                                                 \
  case n:                                                                               \
    return a.horizontal ? launch_sor_t<n, true>(a, Ls, dui, dvi, duo, dvo, final_pass, st) \
                        : launch_sor_t<n, false>(a, Ls, dui, dvi, duo, dvo, final_pass, st);
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
  if (a.H > 2048) return DIS_ERR_VALUE;  // at most 16 CTAs of <= 128 rows per pair
  const size_t Ls = (size_t)(a.W + a.H - 1) * a.H;
  double* carry_u = a.rec + (size_t)kRec * a.B * Ls;
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
