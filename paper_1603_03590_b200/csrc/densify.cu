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
        const double wgt = 1.0 / (ad > 1.0 ? ad : 1.0);
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
