// densify.cu — patch-weighted densification (densify, densification.py:173-191;
// _accumulate_forward 110-128; Eq. 3 of the paper).
//
// The reference scatters every patch's ps x ps window into accumulators in
// ascending patch index.  Here every pixel GATHERS the patches covering it,
// visiting them in ascending (grid row, grid column) order — the same
// ascending patch index — so each pixel's sums are formed in the reference's
// order: bit-identical, deterministic, no atomics.
//
// Covering grid rows of pixel y: regular origins j*spacing in
// [y - ps + 1, y] (j in [ceil((y-ps+1)/sp), floor(y/sp)] clamped to the
// regular range), then the edge-clamped last origin when it covers y.  The
// clamped origin is both the largest index and the largest coordinate, so
// the visiting order is ascending.
#include "common.cuh"
#include "kernels.cuh"

namespace disb200 {

// the densification weight 1 / max(1, |d|) (densification.py:122-123): the
// divisor is >= 1, so div_fast_rn is exact up to 2^400 (den_fast_ok); IEEE
// division beyond (only for absurd residuals)
__device__ __forceinline__ double inv_weight(double ad) {
  const double den = ad > 1.0 ? ad : 1.0;
  return den < 0x1p400 ? div_fast_rn(1.0, den) : 1.0 / den;
}

struct Cover {
  int j0, j1;   // regular origins j0..j1 (inclusive; empty if j1 < j0)
  bool extra;   // the clamped last origin covers too
};

// floor(v / spacing) for 0 <= v < 2^20 / spacing: (v * magic) >> 20 with
// magic = ceil(2^20 / spacing) (exact in that range)
__device__ __forceinline__ int div_sp(int v, unsigned magic) {
  return (int)(((unsigned long long)(unsigned)v * magic) >> 20);
}

__device__ __forceinline__ Cover cover_range(const GridAxis& ax, int ps, int y, unsigned magic) {
  Cover c;
  const int lo = y - ps + 1;
  const int j0 = lo <= 0 ? 0 : div_sp(lo + ax.spacing - 1, magic);
  int j1 = div_sp(y, magic);
  if (j1 > ax.nreg - 1) j1 = ax.nreg - 1;
  if (j1 < j0) j1 = j0 - 1;  // no regular origin covers y
  c.j0 = j0;
  c.j1 = j1;
  c.extra = (ax.n > ax.nreg) && (ax.last <= y) && (y < ax.last + ps);
  return c;
}

// one thread per pixel (2D tiles of 32 x 8): covering patches in ascending
// (grid row, grid column) order = the reference's ascending patch index
__global__ void __launch_bounds__(256) k_densify(const double* __restrict__ ref_all,
                                                 const double* __restrict__ qry_all, int W,
                                                 int H, GridAxis ax, GridAxis ay, int ps,
                                                 unsigned magic, const double* __restrict__ pu,
                                                 const double* __restrict__ pv,
                                                 const double* __restrict__ poff,
                                                 double* __restrict__ fu, double* __restrict__ fv,
                                                 uint32_t* status) {
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  bool bad = false;
  if (x < W && y < H) {
    const size_t plane = (size_t)W * H;
    const int nx = ax.n;
    const int P = nx * ay.n;
    const size_t p = (size_t)y * W + x;
    const double* __restrict__ ref = ref_all + b * plane;
    const double* __restrict__ qry = qry_all + b * plane;
    const double* __restrict__ u_ = pu + (size_t)b * P;
    const double* __restrict__ v_ = pv + (size_t)b * P;
    const double* __restrict__ o_ = poff + (size_t)b * P;
    const double r = __ldg(ref + p);
    const Cover cy = cover_range(ay, ps, y, magic);
    const Cover cx = cover_range(ax, ps, x, magic);
    double acc_u = 0.0, acc_v = 0.0, acc_w = 0.0;
    const int ny_cov = (cy.j1 - cy.j0 + 1) + (cy.extra ? 1 : 0);
    const int nx_cov = (cx.j1 - cx.j0 + 1) + (cx.extra ? 1 : 0);
    for (int a = 0; a < ny_cov; ++a) {
      const int iy = (cy.j0 + a <= cy.j1) ? cy.j0 + a : ay.n - 1;
      for (int c = 0; c < nx_cov; ++c) {
        const int ix = (cx.j0 + c <= cx.j1) ? cx.j0 + c : nx - 1;
        const int i = iy * nx + ix;
        const double u = __ldg(u_ + i);
        const double v = __ldg(v_ + i);
        const double off = __ldg(o_ + i);
        const double d = bilin_nb(qry, W, H, (double)x + u, (double)y + v) - off - r;
        const double ad = fabs(d);
        const double wgt = inv_weight(ad);
        acc_u += wgt * u;
        acc_v += wgt * v;
        acc_w += wgt;
      }
    }
    bad = !(acc_w > 0.0);
    fu[b * plane + p] = exact_div_pos(acc_u, acc_w);  // acc_w > 0 (else flagged)
    fv[b * plane + p] = exact_div_pos(acc_v, acc_w);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) set_status(status, DIS_STATUS_COVERAGE);
}

// ---------------------------------------------------------------------------
// Bidirectional densification (densify_bidirectional, densification.py:
// 194-234): forward patches gathered as above, plus the backward patches
// (found on the query frame) whose window, displaced by their non-integer
// displacement, contains the pixel (_accumulate_backward 131-153), summed in
// ascending backward-patch index into separate accumulators.
//
// Backward windows land anywhere, so they are binned first: every patch
// adds itself to the kBT x kBT tiles its window box touches (counts, scan,
// fill — the fill order within a tile is arbitrary), and the densify kernel
// sorts each tile's list by patch index in shared memory before gathering,
// so the per-pixel sums are formed in the reference's order: deterministic
// whatever order the atomics ran in.  A tile whose list exceeds the shared
// memory capacity falls back to scanning all patches of its pair in order.
// ---------------------------------------------------------------------------
constexpr int kBT = 16;          // bin tile edge (pixels)
constexpr int kBinCap = 2048;    // sorted candidates held in shared memory per tile

struct BwdBox {
  int x_lo, x_hi, y_lo, y_hi;  // inclusive; empty when lo > hi
};

// _accumulate_backward's window (densification.py:141-147): x_lo =
// max(0, int(ceil(sx))), x_hi = min(w - 1, int(ceil(sx + ps)) - 1), same for
// y, sx = x_start + ub.  Evaluated in double and clamped before the integer
// conversion (identical for every finite displacement; a non-finite one
// gives an empty box).
__device__ __forceinline__ BwdBox bwd_box(double x0, double y0, double ub, double vb, int ps,
                                          int W, int H) {
  BwdBox b;
  const double sx = x0 + ub, sy = y0 + vb;
  double xl = ceil(sx), xh = ceil(sx + (double)ps) - 1.0;
  double yl = ceil(sy), yh = ceil(sy + (double)ps) - 1.0;
  if (!(isfinite(sx) && isfinite(sy))) {
    b.x_lo = b.y_lo = 1;
    b.x_hi = b.y_hi = 0;
    return b;
  }
  xl = xl < 0.0 ? 0.0 : (xl > (double)W ? (double)W : xl);
  yl = yl < 0.0 ? 0.0 : (yl > (double)H ? (double)H : yl);
  xh = xh > W - 1.0 ? W - 1.0 : (xh < -1.0 ? -1.0 : xh);
  yh = yh > H - 1.0 ? H - 1.0 : (yh < -1.0 ? -1.0 : yh);
  b.x_lo = (int)xl;
  b.x_hi = (int)xh;
  b.y_lo = (int)yl;
  b.y_hi = (int)yh;
  return b;
}

__device__ __forceinline__ BwdBox patch_box(const GridAxis& ax, const GridAxis& ay, int j,
                                            double ub, double vb, int ps, int W, int H) {
  const int iy = j / ax.n;
  const int ix = j - iy * ax.n;
  return bwd_box((double)ax.origin(ix), (double)ay.origin(iy), ub, vb, ps, W, H);
}

struct BinArgs {
  GridAxis ax, ay;
  int ps, W, H, B, P;
  int ntx, nty;        // tiles per pair
  int max_tiles;       // bins one patch can touch
  const double* pu;    // the binned (backward) patch set
  const double* pv;
  int* count;          // [B][nt]
  int* fill;           // [B][nt]
  int* start;          // [B][nt] (exclusive scan of count)
  int* entries;        // [B][P * max_tiles]
};

// pass 0: count, pass 1: fill
template <int PASS>
__global__ void __launch_bounds__(256) k_bin_patches(BinArgs a) {
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (size_t)a.B * a.P) return;
  const int b = (int)(g / (size_t)a.P);
  const int j = (int)(g - (size_t)b * a.P);
  const BwdBox bx = patch_box(a.ax, a.ay, j, a.pu[g], a.pv[g], a.ps, a.W, a.H);
  if (bx.x_lo > bx.x_hi || bx.y_lo > bx.y_hi) return;
  const int nt = a.ntx * a.nty;
  for (int ty = bx.y_lo / kBT; ty <= bx.y_hi / kBT; ++ty)
    for (int tx = bx.x_lo / kBT; tx <= bx.x_hi / kBT; ++tx) {
      const int t = b * nt + ty * a.ntx + tx;
      if (PASS == 0) {
        atomicAdd(&a.count[t], 1);
      } else {
        const int slot = atomicAdd(&a.fill[t], 1);
        a.entries[(size_t)b * a.P * a.max_tiles + a.start[t] + slot] = j;
      }
    }
}

// per pair: exclusive scan of the tile counts (one block of 1024 threads)
__global__ void __launch_bounds__(1024) k_bin_scan(BinArgs a) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int b = blockIdx.x;
  const int nt = a.ntx * a.nty;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nt; base += 1024) {
    const int t = base + threadIdx.x;
    const int c = t < nt ? a.count[b * nt + t] : 0;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;  // inclusive
    }
    __syncthreads();
    const int excl = carry + (wid ? warp_tot[wid - 1] : 0) + x - c;
    if (t < nt) {
      a.start[b * nt + t] = excl;
      a.fill[b * nt + t] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + c;
    __syncthreads();
  }
}

// One block per (tile, pair), one thread per pixel of the kBT x kBT tile.
__global__ void __launch_bounds__(kBT * kBT) k_densify_bidir(
    const double* __restrict__ ref_all, const double* __restrict__ qry_all, int W, int H,
    GridAxis ax, GridAxis ay, int ps, unsigned magic, const double* __restrict__ fu_p,
    const double* __restrict__ fv_p, const double* __restrict__ foff_p,
    const double* __restrict__ bu_p, const double* __restrict__ bv_p,
    const double* __restrict__ boff_p, BinArgs bin, double* __restrict__ fu,
    double* __restrict__ fv, uint32_t* status) {
  __shared__ int s_key[kBinCap];
  __shared__ int s_sorted[kBinCap];
  __shared__ double s_ub[256], s_vb[256], s_off[256];
  __shared__ int4 s_box[256];
  const int b = blockIdx.z;
  const int tx = blockIdx.x, ty = blockIdx.y;
  const int x = tx * kBT + (threadIdx.x % kBT);
  const int y = ty * kBT + (threadIdx.x / kBT);
  const bool inside = x < W && y < H;
  const size_t plane = (size_t)W * H;
  const int P = ax.n * ay.n;
  const double* __restrict__ ref = ref_all + b * plane;
  const double* __restrict__ qry = qry_all + b * plane;
  const size_t p = (size_t)y * W + x;

  // ---- forward sums (as k_densify) ----
  double acc_u = 0.0, acc_v = 0.0, acc_w = 0.0, r = 0.0;
  if (inside) {
    const double* __restrict__ u_ = fu_p + (size_t)b * P;
    const double* __restrict__ v_ = fv_p + (size_t)b * P;
    const double* __restrict__ o_ = foff_p + (size_t)b * P;
    r = __ldg(ref + p);
    const Cover cy = cover_range(ay, ps, y, magic);
    const Cover cx = cover_range(ax, ps, x, magic);
    const int ny_cov = (cy.j1 - cy.j0 + 1) + (cy.extra ? 1 : 0);
    const int nx_cov = (cx.j1 - cx.j0 + 1) + (cx.extra ? 1 : 0);
    for (int a = 0; a < ny_cov; ++a) {
      const int iy = (cy.j0 + a <= cy.j1) ? cy.j0 + a : ay.n - 1;
      for (int c = 0; c < nx_cov; ++c) {
        const int ix = (cx.j0 + c <= cx.j1) ? cx.j0 + c : ax.n - 1;
        const int i = iy * ax.n + ix;
        const double u = __ldg(u_ + i);
        const double v = __ldg(v_ + i);
        const double off = __ldg(o_ + i);
        const double d = bilin_nb(qry, W, H, (double)x + u, (double)y + v) - off - r;
        const double ad = fabs(d);
        const double wgt = inv_weight(ad);
        acc_u += wgt * u;
        acc_v += wgt * v;
        acc_w += wgt;
      }
    }
  }

  // ---- backward sums over this tile's candidates, ascending index ----
  const int nt = bin.ntx * bin.nty;
  const int t = b * nt + ty * bin.ntx + tx;
  const int n = bin.count[t];
  const int* __restrict__ list = bin.entries + (size_t)b * P * bin.max_tiles + bin.start[t];
  const double* __restrict__ bu_ = bu_p + (size_t)b * P;
  const double* __restrict__ bv_ = bv_p + (size_t)b * P;
  const double* __restrict__ bo_ = boff_p + (size_t)b * P;
  double b_u = 0.0, b_v = 0.0, b_w = 0.0;
  const bool binned = n <= kBinCap;
  if (binned) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_key[i] = list[i];
    __syncthreads();
    // rank sort (keys are distinct patch indices)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int k = s_key[i];
      int rank = 0;
      for (int m = 0; m < n; ++m) rank += s_key[m] < k;
      s_sorted[rank] = k;
    }
    __syncthreads();
  }
  const int total = binned ? n : P;  // overflow: every patch of the pair, in order
  for (int base = 0; base < total; base += 256) {
    const int m = base + (int)threadIdx.x;
    if (m < total) {
      const int j = binned ? s_sorted[m] : m;
      const double ub = __ldg(bu_ + j), vb = __ldg(bv_ + j);
      const BwdBox bx = patch_box(ax, ay, j, ub, vb, ps, W, H);
      s_ub[threadIdx.x] = ub;
      s_vb[threadIdx.x] = vb;
      s_off[threadIdx.x] = __ldg(bo_ + j);
      s_box[threadIdx.x] = make_int4(bx.x_lo, bx.x_hi, bx.y_lo, bx.y_hi);
    }
    __syncthreads();
    const int cnt = total - base < 256 ? total - base : 256;
    if (inside) {
      for (int k = 0; k < cnt; ++k) {
        const int4 bx = s_box[k];
        if (x < bx.x || x > bx.y || y < bx.z || y > bx.w) continue;
        const double ub = s_ub[k], vb = s_vb[k];
        const double d = r - s_off[k] - bilin_nb(qry, W, H, (double)x - ub, (double)y - vb);
        const double ad = fabs(d);
        const double wgt = inv_weight(ad);
        b_u += wgt * (-ub);
        b_v += wgt * (-vb);
        b_w += wgt;
      }
    }
    __syncthreads();
  }

  bool bad = false;
  if (inside) {
    bad = !(acc_w > 0.0);
    double tw = acc_w + b_w;
    if (tw == 0.0) {  // densification.py:226-230 (unreachable with coverage)
      tw = acc_w;
      b_u = 0.0;
      b_v = 0.0;
    }
    fu[b * plane + p] = exact_div_pos(acc_u + b_u, tw);
    fv[b * plane + p] = exact_div_pos(acc_v + b_v, tw);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    set_status(status, DIS_STATUS_COVERAGE);
}

size_t bidir_scratch_bytes(int B, int W, int H, int P, int ps) {
  const size_t nt = (size_t)((W + kBT - 1) / kBT) * ((H + kBT - 1) / kBT);
  const int per_axis = (ps + 1 + kBT - 1) / kBT + 1;
  return (3 * (size_t)B * nt + (size_t)B * P * per_axis * per_axis) * sizeof(int) + 256;
}

void launch_densify_bidir(const double* ref, const double* qry, int B, int W, int H,
                          GridAxis ax, GridAxis ay, int ps, const double* fu_p,
                          const double* fv_p, const double* foff_p, const double* bu_p,
                          const double* bv_p, const double* boff_p, double* fu, double* fv,
                          void* scratch, uint32_t* status, cudaStream_t st) {
  const unsigned magic = (unsigned)(((1u << 20) + ax.spacing - 1) / ax.spacing);
  BinArgs a;
  a.ax = ax;
  a.ay = ay;
  a.ps = ps;
  a.W = W;
  a.H = H;
  a.B = B;
  a.P = ax.n * ay.n;
  a.ntx = (W + kBT - 1) / kBT;
  a.nty = (H + kBT - 1) / kBT;
  const int per_axis = (ps + 1 + kBT - 1) / kBT + 1;
  a.max_tiles = per_axis * per_axis;
  a.pu = bu_p;
  a.pv = bv_p;
  const size_t nt = (size_t)a.ntx * a.nty;
  a.count = static_cast<int*>(scratch);
  a.fill = a.count + (size_t)B * nt;
  a.start = a.fill + (size_t)B * nt;
  a.entries = a.start + (size_t)B * nt;
  prof_begin(KC_DENSIFY, st);
  cudaMemsetAsync(a.count, 0, (size_t)B * nt * sizeof(int), st);
  const size_t n = (size_t)B * a.P;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  k_bin_patches<0><<<blocks, 256, 0, st>>>(a);
  k_bin_scan<<<B, 1024, 0, st>>>(a);
  k_bin_patches<1><<<blocks, 256, 0, st>>>(a);
  dim3 g((unsigned)a.ntx, (unsigned)a.nty, (unsigned)B);
  k_densify_bidir<<<g, kBT * kBT, 0, st>>>(ref, qry, W, H, ax, ay, ps, magic, fu_p, fv_p,
                                           foff_p, bu_p, bv_p, boff_p, a, fu, fv, status);
  prof_end(KC_DENSIFY, st);
  note_launch(4);
}

void launch_densify(const double* ref, const double* qry, int B, int W, int H, GridAxis ax,
                    GridAxis ay, int ps, const double* pu, const double* pv,
                    const double* poff, double* fu, double* fv, uint32_t* status,
                    cudaStream_t st) {
  const unsigned magic = (unsigned)(((1u << 20) + ax.spacing - 1) / ax.spacing);
  dim3 g((unsigned)((W + 31) / 32), (unsigned)((H + 7) / 8), (unsigned)B);
  prof_begin(KC_DENSIFY, st);
  k_densify<<<g, 256, 0, st>>>(ref, qry, W, H, ax, ay, ps, magic, pu, pv, poff, fu, fv, status);
  prof_end(KC_DENSIFY, st);
  note_launch();
}

}  // namespace disb200
