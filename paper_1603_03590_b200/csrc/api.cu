// api.cu — the C ABI (include/dis_b200.h): parameter validation, workspace
// planning and the coarse-to-fine host loop (dis_flow / _dense_scales /
// _upscale_to_full, pipeline.py:85-163) enqueueing the sm_100a kernels on one
// stream.  Nothing on the flow path allocates device memory (only the
// bench-only evaluation census owns two counters); nothing synchronizes except
// the explicitly synchronous *_host / dis_read_status entry points.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

using namespace disb200;

// ---- instrumentation --------------------------------------------------------
// Launch counter: every kernel launch made by this library bumps it;
// dis_flow_batch resets it, so dis_last_launch_count() is the number of our
// kernels one batch enqueued.
// Profiler: when enabled, a CUDA event pair is recorded around every stage
// launch on the launching stream; dis_profile_read() resolves them (after the
// stream has completed) into per-class totals.
namespace {
std::atomic<long long> g_launches{0};
std::mutex g_prof_mu;
bool g_prof_on = false;
struct EvPair {
  cudaEvent_t a, b;
  int cls, level;
};
struct LogEntry {
  int cls, level;
  double ms;
};
std::vector<EvPair> g_prof_pending;
std::vector<LogEntry> g_prof_log;  // every resolved launch since the last reset, in order
int g_prof_level = -1;              // pyramid level of the launches being enqueued
std::vector<cudaEvent_t> g_prof_free;
cudaEvent_t g_prof_open[KC_COUNT];
double g_prof_ms[KC_COUNT];
long long g_prof_n[KC_COUNT];

cudaEvent_t prof_event() {
  if (!g_prof_free.empty()) {
    cudaEvent_t e = g_prof_free.back();
    g_prof_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

namespace disb200 {
void note_launch(int n) { g_launches += n; }

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 ? 0 : d % kMaxDevices;
}

int device_sm_count() {
  static std::atomic<int> sms[kMaxDevices];
  const int d = current_device();
  int n = sms[d].load(std::memory_order_relaxed);
  if (n <= 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (n <= 0) n = 148;
    sms[d].store(n, std::memory_order_relaxed);
  }
  return n;
}

// evaluation census: while enabled, the Gauss-Newton kernels add each
// finished patch's window-evaluation count to census[0] and 1 to census[1]
// (bench.py's FP64 roofline of the patch search; not used when timing)
unsigned long long* g_census = nullptr;
bool g_census_on = false;
unsigned long long* census_counters() { return g_census_on ? g_census : nullptr; }
void prof_begin(int cls, cudaStream_t st) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on) return;
  cudaEvent_t e = prof_event();
  cudaEventRecord(e, st);
  g_prof_open[cls] = e;
}
void prof_level(int level) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_level = level;
}
void prof_end(int cls, cudaStream_t st) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on || !g_prof_open[cls]) return;
  cudaEvent_t e = prof_event();
  cudaEventRecord(e, st);
  g_prof_pending.push_back({g_prof_open[cls], e, cls, g_prof_level});
  g_prof_open[cls] = nullptr;
}
}  // namespace disb200

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_cuda(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DIS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
  return DIS_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- workspace plan -------------------------------------------------------
struct Plan {
  int B, H, W, ss, sf, ps, ds;
  bool var;
  int hs[32], ws[32];
  GridAxis ax[32], ay[32];
  size_t off_status;
  size_t off_img[2][32], off_gx[2][32], off_gy[2][32], off_dd[2][32];
  size_t off_pu[32], off_pv[32], off_poff[32];
  size_t off_fu[32], off_fv[32];
  bool bidir;
  size_t off_bpu[32], off_bpv[32], off_bpoff[32];  // backward patches (bidirectional)
  size_t off_bfu[32], off_bfv[32];                 // backward dense flows
  size_t off_bin;                                  // backward-window bins
  size_t off_rec;
  size_t off_search;
  size_t total;
};

constexpr size_t kNone = ~size_t(0);

size_t take(size_t& cur, size_t bytes) {
  size_t o = (cur + 255) & ~size_t(255);
  cur = o + bytes;
  return o;
}

void make_plan(const dis_params_t* p, int B, int H, int W, Plan* pl) {
  pl->B = B;
  pl->H = H;
  pl->W = W;
  pl->ss = p->coarsest_scale;
  pl->sf = p->finest_scale;
  pl->ps = p->patch_size;
  pl->var = p->variational != 0;
  pl->bidir = p->bidirectional != 0;
  pl->ds = p->downscale;
  const int sp = grid_spacing(p->patch_size, p->overlap);
  for (int s = 0; s <= pl->ss; ++s) {  // floor(dim / k^s) (core.py:88-98 per level)
    pl->hs[s] = s ? pl->hs[s - 1] / pl->ds : H;
    pl->ws[s] = s ? pl->ws[s - 1] / pl->ds : W;
    if (s >= pl->sf) {
      pl->ax[s] = make_axis(pl->ws[s], pl->ps, sp);
      pl->ay[s] = make_axis(pl->hs[s], pl->ps, sp);
    }
  }
  size_t cur = 0;
  pl->off_status = take(cur, 256);
  const size_t d = sizeof(double);
  for (int f = 0; f < 2; ++f)
    for (int s = 0; s <= pl->ss; ++s) {
      const size_t n = (size_t)B * pl->hs[s] * pl->ws[s];
      const bool need_img = s >= 1 || pl->sf == 0;
      pl->off_img[f][s] = need_img ? take(cur, n * d) : kNone;
      const bool used = s >= pl->sf;
      pl->off_gx[f][s] = used ? take(cur, n * d) : kNone;
      pl->off_gy[f][s] = used ? take(cur, n * d) : kNone;
      // second derivatives are formed on the fly by the refinement
      pl->off_dd[f][s] = kNone;
    }
  for (int s = pl->sf; s <= pl->ss; ++s) {
    const size_t P = (size_t)B * pl->ax[s].n * pl->ay[s].n;
    pl->off_pu[s] = take(cur, P * d);
    pl->off_pv[s] = take(cur, P * d);
    pl->off_poff[s] = take(cur, P * d);
  }
  for (int s = 1; s <= pl->ss; ++s) {  // dense flow of levels >= 1 (level 0 -> output)
    const size_t n = (size_t)B * pl->hs[s] * pl->ws[s];
    pl->off_fu[s] = take(cur, n * d);
    pl->off_fv[s] = take(cur, n * d);
  }
  pl->off_fu[0] = pl->off_fv[0] = kNone;
  if (pl->sf == 0) {  // full-resolution dense flow before interleaving
    const size_t n = (size_t)B * H * W;
    pl->off_fu[0] = take(cur, n * d);
    pl->off_fv[0] = take(cur, n * d);
  }
  pl->off_bin = kNone;
  for (int s = 0; s < 32; ++s)
    pl->off_bpu[s] = pl->off_bpv[s] = pl->off_bpoff[s] = pl->off_bfu[s] = pl->off_bfv[s] = kNone;
  if (pl->bidir) {
    size_t mx = 0;
    for (int s = pl->sf; s <= pl->ss; ++s) {
      const int P = pl->ax[s].n * pl->ay[s].n;
      const size_t Pb = (size_t)B * P;
      pl->off_bpu[s] = take(cur, Pb * d);
      pl->off_bpv[s] = take(cur, Pb * d);
      pl->off_bpoff[s] = take(cur, Pb * d);
      const size_t n = (size_t)B * pl->hs[s] * pl->ws[s];
      pl->off_bfu[s] = take(cur, n * d);
      pl->off_bfv[s] = take(cur, n * d);
      size_t r = bidir_scratch_bytes(B, pl->ws[s], pl->hs[s], P, pl->ps);
      if (r > mx) mx = r;
    }
    pl->off_bin = take(cur, mx);
  }
  {
    size_t mx = 0;
    for (int s = pl->sf; s <= pl->ss; ++s) {
      size_t r = patch_search_scratch_bytes(B, pl->ax[s].n * pl->ay[s].n, pl->ws[s], pl->hs[s]);
      if (r > mx) mx = r;
    }
    pl->off_search = take(cur, mx);
  }
  pl->off_rec = kNone;
  if (pl->var) {
    size_t mx = 0;
    for (int s = pl->sf; s <= pl->ss; ++s) {
      size_t r = refine_scratch_doubles(B, pl->ws[s], pl->hs[s]);
      if (r > mx) mx = r;
    }
    pl->off_rec = take(cur, mx * d);
  }
  pl->total = (cur + 255) & ~size_t(255);
}

template <typename T>
T* at(void* base, size_t off) {
  return off == kNone ? nullptr : reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

// validation mirroring dis_flow's checks (pipeline.py:150-163; core.py:65-72,
// 106-128; pipeline.py:30-41)
int check_dims(const dis_params_t* p, int B, int H, int W) {
  if (B < 1) return fail(DIS_ERR_VALUE, "batch must hold at least one pair, got %d", B);
  if (H < 1 || W < 1)
    return fail(DIS_ERR_VALUE, "image must be 2D and non-empty, got shape (%d, %d)", H, W);
  if (H < 2 || W < 2) return fail(DIS_ERR_VALUE, "image must be at least 2x2");
  int hc = H, wc = W;
  for (int s = 1; s <= p->coarsest_scale; ++s) {
    hc /= p->downscale;
    wc /= p->downscale;
    if (hc < 2 || wc < 2)
      return fail(DIS_ERR_VALUE,
                  "downsampled level would be %dx%d; levels below 2 pixels per axis are not "
                  "representable",
                  wc, hc);
  }
  if (wc < p->patch_size || hc < p->patch_size)
    return fail(DIS_ERR_VALUE,
                "coarsest level %dx%d cannot hold a %dpx patch; lower coarsest_scale", wc, hc,
                p->patch_size);
  int hf = H;
  for (int s = 1; s <= p->finest_scale; ++s) hf /= p->downscale;
  if (p->variational && hf > 2048)
    return fail(DIS_ERR_VALUE,
                "variational refinement of a level taller than 2048 rows is not supported by "
                "this build (level %d is %d rows)",
                p->finest_scale, hf);
  return DIS_OK;
}

// one direction's _ScaleState.search (pipeline.py:54-82) on level s
void search_scale(const Plan& pl, const dis_params_t* p, void* ws, int s, int dir, bool stereo,
                  const double* coarse_u, const double* coarse_v, int wc, int hc,
                  double* pu, double* pv, double* poff, cudaStream_t st) {
  SearchArgs a{};
  a.ref = at<double>(ws, pl.off_img[dir][s]);
  a.rgx = at<double>(ws, pl.off_gx[dir][s]);
  a.rgy = at<double>(ws, pl.off_gy[dir][s]);
  a.qry = at<double>(ws, pl.off_img[1 - dir][s]);
  a.B = pl.B;
  a.W = pl.ws[s];
  a.H = pl.hs[s];
  a.cu = coarse_u;
  a.cv = coarse_v;
  a.Wc = wc;
  a.Hc = hc;
  a.ax = pl.ax[s];
  a.ay = pl.ay[s];
  a.ps = pl.ps;
  a.iters = p->iterations;
  a.mean_norm = p->use_mean_normalization;
  a.code = p->residual_norm;
  a.hb = p->huber_b;
  a.ds = p->downscale;
  a.out_u = pu;
  a.out_v = pv;
  a.out_off = poff;
  a.census = census_counters();
  a.horizontal = stereo ? 1 : 0;
  launch_patch_search(a, at<char>(ws, pl.off_search), st);
}

// refine (variational.py:220-275) of one direction's field on level s
int refine_scale(const Plan& pl, const dis_params_t* p, void* ws, int s, int dir, bool stereo,
                 double* fu, double* fv, cudaStream_t st) {
  RefineArgs r{};
  r.ref = at<double>(ws, pl.off_img[dir][s]);
  r.rgx = at<double>(ws, pl.off_gx[dir][s]);
  r.rgy = at<double>(ws, pl.off_gy[dir][s]);
  r.qry = at<double>(ws, pl.off_img[1 - dir][s]);
  r.qgx = at<double>(ws, pl.off_gx[1 - dir][s]);
  r.qgy = at<double>(ws, pl.off_gy[1 - dir][s]);
  r.B = pl.B;
  r.W = pl.ws[s];
  r.H = pl.hs[s];
  r.delta = p->var_intensity_weight;
  r.gamma = p->var_gradient_weight;
  r.alpha = p->var_smoothness_weight;
  r.eps = p->var_penalizer_eps;
  r.omega = p->var_sor_omega;
  r.sweeps = p->var_inner_sor_iters;
  r.outer = p->outer_iters_fixed > 0 ? p->outer_iters_fixed : s + 1;
  r.horizontal = stereo ? 1 : 0;
  r.fu = fu;
  r.fv = fv;
  r.rec = at<double>(ws, pl.off_rec);
  r.status = at<uint32_t>(ws, pl.off_status);
  int rc = launch_refine(r, st);
  if (rc) return fail(rc, "refine: level %d (%dx%d) unsupported", s, pl.ws[s], pl.hs[s]);
  return DIS_OK;
}

// _dense_scales (pipeline.py:85-126) + _upscale_to_full (129-133)
int run_pipeline(const Plan& pl, const dis_params_t* p, double* out, void* ws, cudaStream_t st,
                 bool stereo, bool upscale = true) {
  uint32_t* status = at<uint32_t>(ws, pl.off_status);
  double* prev_u = nullptr;
  double* prev_v = nullptr;
  double* bprev_u = nullptr;  // backward state's flow (bidirectional)
  double* bprev_v = nullptr;
  int prev_w = 0, prev_h = 0;
  for (int s = pl.ss; s >= pl.sf; --s) {
    prof_level(s);
    const int h = pl.hs[s], w = pl.ws[s];
    double* ref = at<double>(ws, pl.off_img[0][s]);
    double* qry = at<double>(ws, pl.off_img[1][s]);
    double* pu = at<double>(ws, pl.off_pu[s]);
    double* pv = at<double>(ws, pl.off_pv[s]);
    double* poff = at<double>(ws, pl.off_poff[s]);
    search_scale(pl, p, ws, s, 0, stereo, prev_u, prev_v, prev_w, prev_h, pu, pv, poff, st);
    double* fu = at<double>(ws, pl.off_fu[s]);
    double* fv = at<double>(ws, pl.off_fv[s]);
    double* bfu = nullptr;
    double* bfv = nullptr;
    if (!pl.bidir) {
      launch_densify(ref, qry, pl.B, w, h, pl.ax[s], pl.ay[s], pl.ps, pu, pv, poff, fu, fv,
                     status, st);
    } else {
      double* bpu = at<double>(ws, pl.off_bpu[s]);
      double* bpv = at<double>(ws, pl.off_bpv[s]);
      double* bpoff = at<double>(ws, pl.off_bpoff[s]);
      search_scale(pl, p, ws, s, 1, stereo, bprev_u, bprev_v, prev_w, prev_h, bpu, bpv, bpoff,
                   st);
      bfu = at<double>(ws, pl.off_bfu[s]);
      bfv = at<double>(ws, pl.off_bfv[s]);
      void* bins = at<char>(ws, pl.off_bin);
      // densification.py:194-234, both directions (pipeline.py:102-113)
      launch_densify_bidir(ref, qry, pl.B, w, h, pl.ax[s], pl.ay[s], pl.ps, pu, pv, poff, bpu,
                           bpv, bpoff, fu, fv, bins, status, st);
      launch_densify_bidir(qry, ref, pl.B, w, h, pl.ax[s], pl.ay[s], pl.ps, bpu, bpv, bpoff, pu,
                           pv, poff, bfu, bfv, bins, status, st);
    }
    if (pl.var) {
      int rc = refine_scale(pl, p, ws, s, 0, stereo, fu, fv, st);
      if (rc) return rc;
      if (pl.bidir) {
        rc = refine_scale(pl, p, ws, s, 1, stereo, bfu, bfv, st);
        if (rc) return rc;
      }
    }
    prev_u = fu;
    prev_v = fv;
    bprev_u = bfu;
    bprev_v = bfv;
    prev_w = w;
    prev_h = h;
  }
  prof_level(-1);
  if (!upscale) return check_cuda("dense_scales");  // the finest scale's field stays in ws
  // _upscale_to_full (pipeline.py:129-133)
  if (pl.sf == 0) {
    launch_interleave(prev_u, prev_v, pl.B, pl.W, pl.H, out, st);
  } else {
    for (int s = pl.sf; s > 0; --s) {
      const int hn = pl.hs[s - 1], wn = pl.ws[s - 1];
      if (s - 1 == 0) {
        launch_upsample(prev_u, prev_v, pl.B, prev_w, prev_h, nullptr, nullptr, out, wn, hn,
                        pl.ds, st);
      } else {
        double* nu = at<double>(ws, pl.off_fu[s - 1]);
        double* nv = at<double>(ws, pl.off_fv[s - 1]);
        launch_upsample(prev_u, prev_v, pl.B, prev_w, prev_h, nu, nv, nullptr, wn, hn, pl.ds,
                        st);
        prev_u = nu;
        prev_v = nv;
        prev_w = wn;
        prev_h = hn;
      }
    }
  }
  return check_cuda("dis_flow_batch");
}

void build_pyramids(const Plan& pl, const void* f1, const void* f2, int dtype, void* ws,
                    cudaStream_t st) {
  uint32_t* status = at<uint32_t>(ws, pl.off_status);
  double* img[2][32] = {};
  double* gx[2][32] = {};
  double* gy[2][32] = {};
  for (int f = 0; f < 2; ++f)
    for (int s = 0; s <= pl.ss; ++s) {
      img[f][s] = at<double>(ws, pl.off_img[f][s]);
      gx[f][s] = at<double>(ws, pl.off_gx[f][s]);
      gy[f][s] = at<double>(ws, pl.off_gy[f][s]);
    }
  launch_pyramid_pair(f1, f2, dtype, pl.B, pl.H, pl.W, pl.ss, pl.ds, img, gx, gy, status, st);
}

size_t dtype_size(int dtype) {
  return dtype == DIS_DTYPE_F32 ? 4 : dtype == DIS_DTYPE_F64 ? 8 : 1;
}

}  // namespace

extern "C" {

const char* dis_last_error(void) { return g_last_error.c_str(); }

long long dis_last_launch_count(void) { return g_launches.load(); }

void dis_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = on != 0;
}

void dis_profile_reset(void) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& p : g_prof_pending) {
    g_prof_free.push_back(p.a);
    g_prof_free.push_back(p.b);
  }
  g_prof_pending.clear();
  g_prof_log.clear();
  for (int c = 0; c < KC_COUNT; ++c) {
    g_prof_ms[c] = 0.0;
    g_prof_n[c] = 0;
    g_prof_open[c] = nullptr;
  }
}

int dis_census_enable(int32_t on) {
  if (on && !g_census) {
    if (cudaMalloc(&g_census, 2 * sizeof(unsigned long long)) != cudaSuccess)
      return fail(DIS_ERR_CUDA, "census: cudaMalloc failed");
  }
  if (on && cudaMemset(g_census, 0, 2 * sizeof(unsigned long long)) != cudaSuccess)
    return fail(DIS_ERR_CUDA, "census: cudaMemset failed");
  g_census_on = on != 0;
  return DIS_OK;
}

int dis_census_read(long long* evals_out, long long* patches_out) {
  unsigned long long h[2] = {0, 0};
  if (g_census && cudaMemcpy(h, g_census, sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(DIS_ERR_CUDA, "census: cudaMemcpy failed");
  *evals_out = (long long)h[0];
  *patches_out = (long long)h[1];
  return DIS_OK;
}

int dis_profile_read(double* ms_out, int64_t* count_out, int32_t n_classes) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& p : g_prof_pending) {
    cudaError_t e = cudaEventSynchronize(p.b);
    if (e != cudaSuccess) return fail(DIS_ERR_CUDA, "profile: %s", cudaGetErrorString(e));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    g_prof_ms[p.cls] += ms;
    g_prof_n[p.cls] += 1;
    g_prof_log.push_back({p.cls, p.level, (double)ms});
    g_prof_free.push_back(p.a);
    g_prof_free.push_back(p.b);
  }
  g_prof_pending.clear();
  for (int c = 0; c < n_classes && c < KC_COUNT; ++c) {
    ms_out[c] = g_prof_ms[c];
    count_out[c] = g_prof_n[c];
  }
  return DIS_OK;
}
int32_t dis_profile_log(int32_t* cls_out, int32_t* level_out, double* ms_out, int32_t max) {
  double ms[KC_COUNT];
  int64_t n[KC_COUNT];
  int rc = dis_profile_read(ms, n, KC_COUNT);  // resolves the pending events
  if (rc) return rc;
  std::lock_guard<std::mutex> g(g_prof_mu);
  const int32_t cnt = (int32_t)g_prof_log.size();
  for (int32_t i = 0; i < cnt && i < max; ++i) {
    if (cls_out) cls_out[i] = g_prof_log[i].cls;
    if (level_out) level_out[i] = g_prof_log[i].level;
    if (ms_out) ms_out[i] = g_prof_log[i].ms;
  }
  return cnt;
}

int32_t dis_abi_version(void) { return DIS_B200_ABI_VERSION; }

void dis_params_default(dis_params_t* p) {
  std::memset(p, 0, sizeof *p);
  p->patch_size = 8;
  p->iterations = 12;
  p->finest_scale = 3;
  p->coarsest_scale = 5;
  p->downscale = 2;
  p->use_mean_normalization = 1;
  p->use_densification = 1;
  p->residual_norm = DIS_NORM_L2;
  p->overlap = 0.40;
  p->huber_b = 1.0;
  p->variational = 1;
  p->var_inner_sor_iters = 5;
  p->var_intensity_weight = 5.0;
  p->var_gradient_weight = 10.0;
  p->var_smoothness_weight = 10.0;
  p->var_penalizer_eps = 0.001;
  p->var_sor_omega = 1.6;
  p->outer_iters_fixed = 0;
}

int dis_params_validate(const dis_params_t* p) {
  if (!p) return fail(DIS_ERR_PARAMETER, "params is NULL");
  if (p->patch_size < 2) return fail(DIS_ERR_PARAMETER, "patch_size must be >= 2");
  if (!(p->overlap >= 0.0 && p->overlap < 1.0))
    return fail(DIS_ERR_PARAMETER, "overlap must lie in [0, 1)");
  if (p->iterations < 1) return fail(DIS_ERR_PARAMETER, "iterations must be >= 1");
  if (p->finest_scale < 0 || p->coarsest_scale < p->finest_scale)
    return fail(DIS_ERR_PARAMETER, "need 0 <= finest_scale <= coarsest_scale");
  if (p->coarsest_scale > 30) return fail(DIS_ERR_PARAMETER, "coarsest_scale too large");
  if (p->downscale < 2) return fail(DIS_ERR_PARAMETER, "downscale must be an integer >= 2");
  if (p->downscale > 128)
    return fail(DIS_ERR_PARAMETER, "this path implements downscale factors up to 128");
  if (p->residual_norm < 0 || p->residual_norm > 2)
    return fail(DIS_ERR_PARAMETER, "residual_norm must be one of ('l2', 'l1', 'huber')");
  if (p->residual_norm == DIS_NORM_HUBER && !(p->huber_b > 0))
    return fail(DIS_ERR_PARAMETER, "huber_b must be > 0");
  if (p->mode != 0 && p->mode != 1) return fail(DIS_ERR_PARAMETER, "mode must be 'flow' or 'stereo'");
  if (p->mode == 1 && p->bidirectional)
    return fail(DIS_ERR_PARAMETER, "bidirectional matching is not defined for stereo mode");
  if (p->variational) {
    if (p->var_intensity_weight < 0 || p->var_gradient_weight < 0 ||
        p->var_smoothness_weight < 0)
      return fail(DIS_ERR_PARAMETER, "variational weights must be >= 0");
    if (p->var_inner_sor_iters < 1) return fail(DIS_ERR_PARAMETER, "inner_sor_iters must be >= 1");
    if (!(p->var_penalizer_eps > 0)) return fail(DIS_ERR_PARAMETER, "penalizer_eps must be > 0");
    if (!(p->var_sor_omega > 0.0 && p->var_sor_omega < 2.0))
      return fail(DIS_ERR_PARAMETER, "sor_omega must lie in (0, 2)");
  }
  return DIS_OK;
}

size_t dis_workspace_bytes(int32_t B, int32_t H, int32_t W, const dis_params_t* p) {
  if (dis_params_validate(p) || check_dims(p, B, H, W)) return 0;
  Plan pl;
  make_plan(p, B, H, W, &pl);
  return pl.total;
}

// ---- host-buffer path: chunked, multi-stream pipeline -----------------------
// The batch is cut into nchunks chunks, each with its own slice of the
// workspace and its own internal stream: chunk i's host->device copy, its
// kernels and its device->host copy are stream-ordered, different chunks
// overlap (the two copy directions run on separate copy engines, concurrently
// with the kernels of other chunks).
namespace {
constexpr int kHostChunksMax = 16;

// Chunk schedule of the host-buffer pipeline.  The device->host copy of the
// float64 flow is the bottleneck (2x the input bytes, one copy engine per
// direction), and it can only start once the first chunk is computed, so the
// first chunks are small (1, 1, 2, 4 pairs: a short exposed head) and the rest
// are large enough for efficient kernels (up to 8 pairs); every chunk runs on
// its own stream, so chunk i's copies overlap the kernels of the others.
struct ChunkPlan {
  int n = 0;
  int first[kHostChunksMax + 1];  // chunk c holds pairs [first[c], first[c+1])
  int bmax = 0;
};
ChunkPlan host_chunks(int B) {
  static const int forced = [] {
    const char* e = getenv("DIS_HOST_CHUNKS");  // experiments only: equal chunks
    return e ? atoi(e) : 0;
  }();
  ChunkPlan p;
  std::vector<int> sz;
  if (forced > 0) {
    const int n = forced < kHostChunksMax ? (forced < B ? forced : B) : kHostChunksMax;
    const int bc = (B + n - 1) / n;
    for (int left = B; left > 0; left -= bc) sz.push_back(left < bc ? left : bc);
  } else {
    const int ramp[] = {1, 1, 2, 4};
    const int big = 8;
    int left = B;
    for (int r : ramp) {
      if (left <= 0) break;
      const int t = r < left ? r : left;
      sz.push_back(t);
      left -= t;
    }
    int slots = kHostChunksMax - (int)sz.size();
    while (left > 0) {  // the rest in chunks of ~big pairs, within the stream budget
      int t = (left + slots - 1) / slots;
      t = t < big ? (left < big ? left : big) : t;
      sz.push_back(t);
      left -= t;
      --slots;
    }
  }
  p.n = (int)sz.size();
  p.first[0] = 0;
  for (int c = 0; c < p.n; ++c) {
    p.first[c + 1] = p.first[c] + sz[c];
    p.bmax = sz[c] > p.bmax ? sz[c] : p.bmax;
  }
  return p;
}

size_t host_chunk_bytes(int Bc, int H, int W, int dtype, const dis_params_t* p) {
  size_t base = dis_workspace_bytes(Bc, H, W, p);
  if (!base) return 0;
  size_t cur = base;
  const size_t frames = (size_t)Bc * H * W * dtype_size(dtype);
  take(cur, frames);
  take(cur, frames);
  take(cur, (size_t)Bc * H * W * 2 * sizeof(double));
  return (cur + 255) & ~size_t(255);
}

struct HostStreams {
  int dev = -1;
  cudaStream_t s[kHostChunksMax] = {};  // per-chunk kernels
  cudaStream_t in = nullptr, out = nullptr;  // the copies, in chunk order
  cudaStream_t cap = nullptr;  // graph capture origin (never the legacy stream)
  cudaEvent_t start = nullptr, done[kHostChunksMax] = {};
  cudaEvent_t landed[kHostChunksMax] = {}, computed[kHostChunksMax] = {};
};
std::mutex g_host_mu;
HostStreams g_host[16];
// The chunks' status words of a host-buffer call land in a small pinned
// array owned by the library (one per workspace address), copied on the
// out stream behind each chunk's flow: finishing a call then needs no
// device read of its own (a blocking 4-byte copy would queue behind the
// flow copies of another call in flight).
struct HostStatus {
  const void* ws;
  uint32_t* pinned;
};
std::vector<HostStatus> g_host_status;  // guarded by g_host_mu
uint32_t* host_status_for(const void* ws, bool create) {
  for (const HostStatus& h : g_host_status)
    if (h.ws == ws) return h.pinned;
  if (!create) return nullptr;
  uint32_t* pinned = nullptr;
  if (cudaHostAlloc(reinterpret_cast<void**>(&pinned), kHostChunksMax * sizeof(uint32_t),
                    cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  std::memset(pinned, 0, kHostChunksMax * sizeof(uint32_t));
  g_host_status.push_back({ws, pinned});
  return pinned;
}
}  // namespace

size_t dis_host_workspace_bytes(int32_t B, int32_t H, int32_t W, int32_t dtype,
                                const dis_params_t* p) {
  if (B < 1) return 0;
  const ChunkPlan cp = host_chunks(B);
  const size_t per = host_chunk_bytes(cp.bmax, H, W, dtype, p);
  return per ? per * cp.n : 0;
}

}  // extern "C"

namespace {
// dis_flow / dis_stereo on a batch (pipeline.py:150-183): validation, pyramids,
// _dense_scales, _upscale_to_full — all enqueued on `stream`.
int flow_batch_impl(const void* frame1, const void* frame2, int32_t dtype, int32_t B, int32_t H,
                    int32_t W, const dis_params_t* p, double* flow_out, void* workspace,
                    size_t workspace_bytes, void* stream, bool stereo) {
  int rc = dis_params_validate(p);
  if (rc) return rc;
  // dis_flow_on_pyramids rejects stereo-mode parameters (pipeline.py:141-142);
  // dis_stereo takes either mode (pipeline.py:172-180)
  if (!stereo && p->mode == 1)
    return fail(DIS_ERR_VALUE, "use dis_stereo for stereo-mode parameters");
  if (dtype < 0 || dtype > 2) return fail(DIS_ERR_VALUE, "unsupported frame dtype %d", dtype);
  rc = check_dims(p, B, H, W);
  if (rc) return rc;
  Plan pl;
  make_plan(p, B, H, W, &pl);
  if (workspace_bytes < pl.total)
    return fail(DIS_ERR_WORKSPACE, "workspace holds %zu bytes, need %zu", workspace_bytes,
                pl.total);
  cudaStream_t st = as_stream(stream);
  g_launches = 0;
  cudaMemsetAsync(at<char>(workspace, pl.off_status), 0, 256, st);
  build_pyramids(pl, frame1, frame2, dtype, workspace, st);
  rc = check_cuda("pyramid");
  if (rc) return rc;
  return run_pipeline(pl, p, flow_out, workspace, st, stereo);
}

int host_batch_impl(const void* host_frame1, const void* host_frame2, int32_t dtype, int32_t B,
                    int32_t H, int32_t W, const dis_params_t* p, double* host_flow_out,
                    void* workspace, size_t workspace_bytes, void* stream, bool stereo,
                    bool wait = true, bool f32 = false);
int host_batch_finish(const void* workspace, int32_t B, int32_t H, int32_t W, int32_t dtype,
                      const dis_params_t* p, void* stream);
}  // namespace

extern "C" {

int dis_flow_batch(const void* frame1, const void* frame2, int32_t dtype, int32_t B, int32_t H,
                   int32_t W, const dis_params_t* p, double* flow_out, void* workspace,
                   size_t workspace_bytes, void* stream) {
  return flow_batch_impl(frame1, frame2, dtype, B, H, W, p, flow_out, workspace,
                         workspace_bytes, stream, false);
}

int dis_flow_batch_levels(const double* const* img1, const double* const* gx1,
                          const double* const* gy1, const double* const* img2,
                          const double* const* gx2, const double* const* gy2, int32_t B,
                          int32_t H, int32_t W, const dis_params_t* p, double* flow_out,
                          void* workspace, size_t workspace_bytes, void* stream) {
  int rc = dis_params_validate(p);
  if (rc) return rc;
  if (p->mode == 1) return fail(DIS_ERR_VALUE, "use dis_stereo for stereo-mode parameters");
  rc = check_dims(p, B, H, W);
  if (rc) return rc;
  Plan pl;
  make_plan(p, B, H, W, &pl);
  if (workspace_bytes < pl.total)
    return fail(DIS_ERR_WORKSPACE, "workspace holds %zu bytes, need %zu", workspace_bytes,
                pl.total);
  cudaStream_t st = as_stream(stream);
  g_launches = 0;
  cudaMemsetAsync(at<char>(workspace, pl.off_status), 0, 256, st);
  // the levels this parameter set reads (images of levels >= 1 or the finest,
  // gradients of levels >= finest) into the workspace's pyramid slots
  const double* const* src[2][3] = {{img1, gx1, gy1}, {img2, gx2, gy2}};
  for (int f = 0; f < 2; ++f)
    for (int s = 0; s <= pl.ss; ++s) {
      const size_t bytes = (size_t)B * pl.hs[s] * pl.ws[s] * sizeof(double);
      const size_t offs[3] = {pl.off_img[f][s], pl.off_gx[f][s], pl.off_gy[f][s]};
      for (int k = 0; k < 3; ++k) {
        if (offs[k] == kNone) continue;
        if (!src[f][k] || !src[f][k][s])
          return fail(DIS_ERR_VALUE, "pyramid %d level %d: missing %s raster", f + 1, s,
                      k == 0 ? "image" : (k == 1 ? "grad_x" : "grad_y"));
        cudaMemcpyAsync(at<char>(workspace, offs[k]), src[f][k][s], bytes,
                        cudaMemcpyDeviceToDevice, st);
      }
    }
  rc = check_cuda("dis_flow_batch_levels");
  if (rc) return rc;
  return run_pipeline(pl, p, flow_out, workspace, st, false);
}

int dis_stereo_batch(const void* left, const void* right, int32_t dtype, int32_t B, int32_t H,
                     int32_t W, const dis_params_t* p, double* flow_out, void* workspace,
                     size_t workspace_bytes, void* stream) {
  return flow_batch_impl(left, right, dtype, B, H, W, p, flow_out, workspace, workspace_bytes,
                         stream, true);
}

int dis_read_status(const void* workspace, uint32_t* status_out, void* stream) {
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemcpyAsync(status_out, workspace, sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(DIS_ERR_CUDA, "dis_read_status: %s", cudaGetErrorString(e));
  return DIS_OK;
}

int dis_status_to_error(uint32_t status) {
  if (status & DIS_STATUS_NONFINITE_INPUT)
    return fail(DIS_ERR_VALUE, "image contains non-finite values");
  if (status & DIS_STATUS_COVERAGE)
    return fail(DIS_ERR_COVERAGE, "pixel without a contributing patch; grid coverage broken");
  if (status & DIS_STATUS_NONFINITE_FLOW)
    return fail(DIS_ERR_NONFINITE, "variational refinement produced a non-finite value");
  return DIS_OK;
}

int dis_flow_batch_host(const void* host_frame1, const void* host_frame2, int32_t dtype,
                        int32_t B, int32_t H, int32_t W, const dis_params_t* p,
                        double* host_flow_out, void* workspace, size_t workspace_bytes,
                        void* stream) {
  return host_batch_impl(host_frame1, host_frame2, dtype, B, H, W, p, host_flow_out, workspace,
                         workspace_bytes, stream, false);
}

int dis_stereo_batch_host(const void* host_left, const void* host_right, int32_t dtype,
                          int32_t B, int32_t H, int32_t W, const dis_params_t* p,
                          double* host_flow_out, void* workspace, size_t workspace_bytes,
                          void* stream) {
  return host_batch_impl(host_left, host_right, dtype, B, H, W, p, host_flow_out, workspace,
                         workspace_bytes, stream, true);
}


int dis_flow_batch_host_async(const void* host_frame1, const void* host_frame2, int32_t dtype,
                              int32_t B, int32_t H, int32_t W, const dis_params_t* p,
                              double* host_flow_out, void* workspace, size_t workspace_bytes,
                              void* stream) {
  return host_batch_impl(host_frame1, host_frame2, dtype, B, H, W, p, host_flow_out, workspace,
                         workspace_bytes, stream, false, false);
}

int dis_stereo_batch_host_async(const void* host_left, const void* host_right, int32_t dtype,
                                int32_t B, int32_t H, int32_t W, const dis_params_t* p,
                                double* host_flow_out, void* workspace, size_t workspace_bytes,
                                void* stream) {
  return host_batch_impl(host_left, host_right, dtype, B, H, W, p, host_flow_out, workspace,
                         workspace_bytes, stream, true, false);
}

int dis_host_batch_finish(const void* workspace, int32_t B, int32_t H, int32_t W, int32_t dtype,
                          const dis_params_t* p, void* stream) {
  return host_batch_finish(workspace, B, H, W, dtype, p, stream);
}

int dis_flow_batch_host_ex(const void* host_frame1, const void* host_frame2, int32_t dtype,
                           int32_t B, int32_t H, int32_t W, const dis_params_t* p,
                           void* host_flow_out, void* workspace, size_t workspace_bytes,
                           void* stream, uint32_t flags) {
  if (flags & ~(uint32_t)(DIS_HOST_ASYNC | DIS_HOST_FLOW_F32 | DIS_HOST_STEREO))
    return fail(DIS_ERR_VALUE, "dis_flow_batch_host_ex: unknown flags 0x%x", flags);
  return host_batch_impl(host_frame1, host_frame2, dtype, B, H, W, p,
                         static_cast<double*>(host_flow_out), workspace, workspace_bytes, stream,
                         (flags & DIS_HOST_STEREO) != 0, !(flags & DIS_HOST_ASYNC),
                         (flags & DIS_HOST_FLOW_F32) != 0);
}

}  // extern "C"

namespace {
// The host path's whole enqueue (copies in, every chunk's kernels, copies
// out on the chunk streams) is replayed as one CUDA graph when the call
// repeats with the same pinned host buffers, workspace, stream and problem
// (captured on the second such call; the first runs eagerly and performs
// the kernels' one-time set-up).  Saves the per-launch gaps of the
// latency-bound per-chunk pipelines.
struct HostGraph {
  const void* f1 = nullptr;
  const void* f2 = nullptr;
  const void* out = nullptr;
  const void* ws = nullptr;
  void* stream = nullptr;
  int32_t dtype = -1, B = 0, H = 0, W = 0;
  bool stereo = false;
  bool f32 = false;
  int dev = -1;
  dis_params_t p{};
  int seen = 0;
  cudaGraphExec_t exec = nullptr;
  long long launches = 0;
};
constexpr int kHostGraphs = 8;  // (blocking, two in flight, float32 variants of two problems)
HostGraph g_hgraph[kHostGraphs];
int g_hgraph_next = 0;

bool host_graphs_on() {
  static const bool on = [] {
    const char* e = getenv("DIS_HOST_GRAPH");  // experiments only
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}

bool is_pinned(const void* ptr) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

int host_batch_enqueue(const void* host_frame1, const void* host_frame2, int32_t dtype,
                       int32_t B, int32_t H, int32_t W, const dis_params_t* p,
                       double* host_flow_out, void* workspace, cudaStream_t st, bool stereo,
                       const ChunkPlan& cp, size_t per, int* used_out, bool f32);

// experiments only (DIS_HOST_TRACE=1 with DIS_HOST_GRAPH=0): per-chunk event
// times (frames landed, kernels done, flow copied) printed after each call
bool host_trace_on() {
  static const bool on = [] {
    const char* e = getenv("DIS_HOST_TRACE");
    return e && atoi(e) != 0;
  }();
  return on;
}
cudaEvent_t g_tr[kHostChunksMax][3];
cudaEvent_t g_tr0;
int g_tr_n = 0;
void host_trace_mark(int c, cudaStream_t in, cudaStream_t cs, cudaStream_t out) {
  if (!g_tr0) {
    cudaEventCreate(&g_tr0);
    for (int i = 0; i < kHostChunksMax; ++i)
      for (int j = 0; j < 3; ++j) cudaEventCreate(&g_tr[i][j]);
  }
  if (c == 0) cudaEventRecord(g_tr0, in);  // (recorded after chunk 0's copies were enqueued)
  cudaEventRecord(g_tr[c][0], in);
  cudaEventRecord(g_tr[c][1], cs);
  cudaEventRecord(g_tr[c][2], out);
  g_tr_n = c + 1;
}
void host_trace_print() {
  cudaDeviceSynchronize();
  for (int c = 0; c < g_tr_n; ++c) {
    float t[3];
    for (int j = 0; j < 3; ++j) cudaEventElapsedTime(&t[j], g_tr0, g_tr[c][j]);
    fprintf(stderr, "chunk %2d: landed %7.3f  computed %7.3f  copied out %7.3f ms\n", c, t[0],
            t[1], t[2]);
  }
}

int host_batch_impl(const void* host_frame1, const void* host_frame2, int32_t dtype, int32_t B,
                    int32_t H, int32_t W, const dis_params_t* p, double* host_flow_out,
                    void* workspace, size_t workspace_bytes, void* stream, bool stereo,
                    bool wait, bool f32) {
  int rc = dis_params_validate(p);
  if (rc) return rc;
  if (!stereo && p->mode == 1)
    return fail(DIS_ERR_VALUE, "use dis_stereo for stereo-mode parameters");
  if (dtype < 0 || dtype > 2) return fail(DIS_ERR_VALUE, "unsupported frame dtype %d", dtype);
  rc = check_dims(p, B, H, W);
  if (rc) return rc;
  const size_t need = dis_host_workspace_bytes(B, H, W, dtype, p);
  if (workspace_bytes < need)
    return fail(DIS_ERR_WORKSPACE, "workspace holds %zu bytes, need %zu", workspace_bytes, need);
  const ChunkPlan cp = host_chunks(B);
  const size_t per = host_chunk_bytes(cp.bmax, H, W, dtype, p);
  int dev = 0;
  cudaGetDevice(&dev);
  std::unique_lock<std::mutex> guard(g_host_mu);
  HostStreams& hs = g_host[dev & 15];
  if (hs.dev != dev) {
    // the first (small) chunks get the highest stream priority: the flow's
    // device->host copy, the pipeline's bottleneck, starts once chunk 0 is done
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    for (int i = 0; i < kHostChunksMax; ++i) {
      const int pr = prio_hi + i < prio_lo ? prio_hi + i : prio_lo;
      cudaStreamCreateWithPriority(&hs.s[i], cudaStreamNonBlocking, pr);
      cudaEventCreateWithFlags(&hs.done[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&hs.landed[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&hs.computed[i], cudaEventDisableTiming);
    }
    cudaStreamCreateWithFlags(&hs.in, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&hs.out, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&hs.start, cudaEventDisableTiming);
    cudaStreamCreateWithFlags(&hs.cap, cudaStreamNonBlocking);
    hs.dev = dev;
  }
  cudaStream_t st = as_stream(stream);
  // graph cache lookup (pinned host buffers only: pageable copies cannot be
  // captured)
  HostGraph* hg = nullptr;
  if (host_graphs_on()) {
    for (int i = 0; i < kHostGraphs; ++i) {
      HostGraph& g = g_hgraph[i];
      if (g.f1 == host_frame1 && g.f2 == host_frame2 && g.out == host_flow_out &&
          g.ws == workspace && g.stream == stream && g.dtype == dtype && g.B == B && g.H == H &&
          g.W == W && g.stereo == stereo && g.f32 == f32 && g.dev == dev &&
          std::memcmp(&g.p, p, sizeof(dis_params_t)) == 0) {
        hg = &g;
        break;
      }
    }
    if (!hg && is_pinned(host_frame1) && is_pinned(host_frame2) && is_pinned(host_flow_out)) {
      hg = &g_hgraph[g_hgraph_next];
      g_hgraph_next = (g_hgraph_next + 1) % kHostGraphs;
      if (hg->exec) cudaGraphExecDestroy(hg->exec);
      *hg = HostGraph{};
      hg->f1 = host_frame1;
      hg->f2 = host_frame2;
      hg->out = host_flow_out;
      hg->ws = workspace;
      hg->stream = stream;
      hg->dtype = dtype;
      hg->B = B;
      hg->H = H;
      hg->W = W;
      hg->stereo = stereo;
      hg->f32 = f32;
      hg->dev = dev;
      hg->p = *p;
    }
  }
  int used = 0;
  if (hg && hg->exec) {  // replay
    if (cudaGraphLaunch(hg->exec, st) != cudaSuccess)
      return fail(DIS_ERR_CUDA, "dis_flow_batch_host: graph launch failed");
    used = cp.n;
    g_launches = hg->launches;
  } else if (hg && hg->seen >= 1) {  // capture this call, then replay it
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(hs.cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
      return fail(DIS_ERR_CUDA, "dis_flow_batch_host: stream capture failed");
    rc = host_batch_enqueue(host_frame1, host_frame2, dtype, B, H, W, p, host_flow_out,
                            workspace, hs.cap, stereo, cp, per, &used, f32);
    const cudaError_t ce = cudaStreamEndCapture(hs.cap, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (ce != cudaSuccess || cudaGraphInstantiate(&hg->exec, graph, 0) != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      hg->exec = nullptr;
      return fail(DIS_ERR_CUDA, "dis_flow_batch_host: graph capture failed");
    }
    cudaGraphDestroy(graph);
    hg->launches = g_launches.load();
    if (cudaGraphLaunch(hg->exec, st) != cudaSuccess)
      return fail(DIS_ERR_CUDA, "dis_flow_batch_host: graph launch failed");
  } else {
    if (hg) ++hg->seen;
    rc = host_batch_enqueue(host_frame1, host_frame2, dtype, B, H, W, p, host_flow_out,
                            workspace, st, stereo, cp, per, &used, f32);
    if (rc) return rc;
  }
  (void)used;
  if (!wait) return DIS_OK;  // the caller finishes the call with dis_host_batch_finish
  guard.unlock();
  return host_batch_finish(workspace, B, H, W, dtype, p, stream);
}

// The blocking half of a host-buffer call: wait for the stream the call was
// enqueued on (its flow copies have then landed in the host buffer) and turn
// the chunks' status words into a return code.
int host_batch_finish(const void* workspace, int32_t B, int32_t H, int32_t W, int32_t dtype,
                      const dis_params_t* p, void* stream) {
  int rc = dis_params_validate(p);
  if (rc) return rc;
  if (!workspace) return fail(DIS_ERR_VALUE, "workspace is NULL");
  rc = check_dims(p, B, H, W);
  if (rc) return rc;
  const ChunkPlan cp = host_chunks(B);
  const size_t per = host_chunk_bytes(cp.bmax, H, W, dtype, p);
  int used = 0;
  for (int c = 0; c < cp.n; ++c)
    if (cp.first[c + 1] - cp.first[c] > 0) ++used;
  cudaError_t e = cudaStreamSynchronize(as_stream(stream));
  if (e != cudaSuccess) return fail(DIS_ERR_CUDA, "dis_flow_batch_host: %s", cudaGetErrorString(e));
  if (host_trace_on()) host_trace_print();
  uint32_t any = 0;
  const uint32_t* hst = nullptr;
  {
    std::lock_guard<std::mutex> guard(g_host_mu);
    hst = host_status_for(workspace, false);
  }
  for (int c = 0; c < used; ++c) {
    uint32_t status = 0;
    if (hst) {
      status = hst[c];
    } else {
      e = cudaMemcpy(&status, static_cast<const char*>(workspace) + (size_t)c * per,
                     sizeof(uint32_t), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess)
        return fail(DIS_ERR_CUDA, "dis_flow_batch_host: %s", cudaGetErrorString(e));
    }
    any |= status;
  }
  return dis_status_to_error(any);
}
int host_batch_enqueue(const void* host_frame1, const void* host_frame2, int32_t dtype,
                       int32_t B, int32_t H, int32_t W, const dis_params_t* p,
                       double* host_flow_out, void* workspace, cudaStream_t st, bool stereo,
                       const ChunkPlan& cp, size_t per, int* used_out, bool f32) {
  int dev = 0;
  cudaGetDevice(&dev);
  HostStreams& hs = g_host[dev & 15];
  int rc = DIS_OK;
  cudaEventRecord(hs.start, st);  // chunks start after the caller's prior work
  const size_t esz = dtype_size(dtype);
  const size_t px = (size_t)H * W;
  long long launches = 0;
  int used = 0;
  // copies in chunk order on one stream per direction (each chunk's frames
  // land as early as possible, the flow leaves in order without the copy
  // engine interleaving the chunks); each chunk's kernels on its own stream
  // so that they overlap each other and the copies
  const int Bc = cp.bmax;
  uint32_t* hst = host_status_for(workspace, true);  // (the caller holds g_host_mu)
  cudaStreamWaitEvent(hs.in, hs.start, 0);
  cudaStreamWaitEvent(hs.out, hs.start, 0);
  for (int c = 0; c < cp.n; ++c) {
    const int b0 = cp.first[c];
    const int bn = cp.first[c + 1] - b0;
    if (bn <= 0) break;
    ++used;
    cudaStream_t cs = hs.s[c];
    char* wsc = static_cast<char*>(workspace) + (size_t)c * per;
    Plan pl;
    make_plan(p, bn, H, W, &pl);
    size_t cur = dis_workspace_bytes(Bc, H, W, p);
    const size_t fbytes = (size_t)bn * px * esz;
    const size_t obytes = (size_t)bn * px * 2 * sizeof(double);
    void* d1 = wsc + take(cur, (size_t)Bc * px * esz);
    void* d2 = wsc + take(cur, (size_t)Bc * px * esz);
    double* dout = reinterpret_cast<double*>(wsc + take(cur, (size_t)Bc * px * 2 * sizeof(double)));
    cudaMemcpyAsync(d1, static_cast<const char*>(host_frame1) + (size_t)b0 * px * esz, fbytes,
                    cudaMemcpyHostToDevice, hs.in);
    cudaMemcpyAsync(d2, static_cast<const char*>(host_frame2) + (size_t)b0 * px * esz, fbytes,
                    cudaMemcpyHostToDevice, hs.in);
    cudaEventRecord(hs.landed[c], hs.in);
    cudaStreamWaitEvent(cs, hs.landed[c], 0);
    rc = flow_batch_impl(d1, d2, dtype, bn, H, W, p, dout, wsc, pl.total, cs, stereo);
    if (rc) return rc;
    launches += g_launches.load();
    cudaEventRecord(hs.computed[c], cs);
    cudaStreamWaitEvent(hs.out, hs.computed[c], 0);
    if (f32) {
      // the flow rounded to float32 on the device (round to nearest, like
      // numpy's astype): half the copy-out.  The staging area is the head of
      // the chunk's pipeline workspace, free once its kernels are done.
      float* d32 = reinterpret_cast<float*>(wsc + 256);
      launch_flow_to_f32(dout, d32, (size_t)bn * px * 2, cs);
      ++launches;
      cudaEventRecord(hs.computed[c], cs);
      cudaStreamWaitEvent(hs.out, hs.computed[c], 0);
      cudaMemcpyAsync(reinterpret_cast<float*>(host_flow_out) + (size_t)b0 * px * 2, d32,
                      obytes / 2, cudaMemcpyDeviceToHost, hs.out);
    } else {
      cudaMemcpyAsync(host_flow_out + (size_t)b0 * px * 2, dout, obytes, cudaMemcpyDeviceToHost,
                      hs.out);
    }
    if (hst)
      cudaMemcpyAsync(hst + c, wsc, sizeof(uint32_t), cudaMemcpyDeviceToHost, hs.out);
    if (host_trace_on()) host_trace_mark(c, hs.in, cs, hs.out);
  }
  cudaEventRecord(hs.done[0], hs.out);
  cudaStreamWaitEvent(st, hs.done[0], 0);
  for (int c = 0; c < used; ++c) {  // every chunk stream joins (graph capture)
    cudaEventRecord(hs.done[c], hs.s[c]);
    cudaStreamWaitEvent(st, hs.done[c], 0);
  }
  g_launches = launches;
  *used_out = used;
  return DIS_OK;
}
}  // namespace

extern "C" {

// ---- stage entry points -----------------------------------------------------

int dis_build_pyramid(const void* frames, int32_t dtype, int32_t B, int32_t H, int32_t W,
                      int32_t coarsest, int32_t downscale, double* const* levels_img,
                      double* const* levels_gx, double* const* levels_gy,
                      double* const* levels_dd, uint32_t* status, void* stream) {
  if (coarsest < 0) return fail(DIS_ERR_PARAMETER, "coarsest_scale must be >= 0");
  if (downscale < 2) return fail(DIS_ERR_PARAMETER, "downscale must be an integer >= 2");
  if (downscale > 128)
    return fail(DIS_ERR_PARAMETER, "this path implements downscale factors up to 128");
  if (coarsest > 30) return fail(DIS_ERR_PARAMETER, "coarsest_scale too large");
  if (H < 2 || W < 2) return fail(DIS_ERR_VALUE, "image must be at least 2x2");
  {
    int h = H, w = W;
    for (int s = 1; s <= coarsest; ++s) {
      h /= downscale;
      w /= downscale;
      if (h < 2 || w < 2)
        return fail(DIS_ERR_VALUE,
                    "downsampled level would be %dx%d; levels below 2 pixels per axis are not "
                    "representable",
                    w, h);
    }
  }
  if (!levels_img) return fail(DIS_ERR_VALUE, "levels_img is NULL");
  for (int s = 1; s <= coarsest; ++s)
    if (!levels_img[s]) return fail(DIS_ERR_VALUE, "levels_img[%d] is NULL", s);
  std::vector<double*> gx(coarsest + 1, nullptr), gy(coarsest + 1, nullptr);
  for (int s = 0; s <= coarsest; ++s) {
    if (levels_gx) gx[s] = levels_gx[s];
    if (levels_gy) gy[s] = levels_gy[s];
    if ((gx[s] || gy[s] || (levels_dd && levels_dd[s])) && !levels_img[s])
      return fail(DIS_ERR_VALUE, "gradients of level %d need its image", s);
  }
  launch_pyramid(frames, dtype, B, H, W, coarsest, downscale, levels_img, gx.data(), gy.data(),
                 levels_dd, status, as_stream(stream));
  return check_cuda("dis_build_pyramid");
}

int32_t dis_grid_axis(int32_t dim, int32_t patch_size, double overlap, int32_t* origins_out,
                      int32_t max_out) {
  if (!(overlap >= 0.0 && overlap < 1.0)) return fail(DIS_ERR_VALUE, "overlap must lie in [0, 1)");
  if (dim < patch_size)
    return fail(DIS_ERR_VALUE, "level %d is smaller than the patch size %d", dim, patch_size);
  GridAxis a = make_axis(dim, patch_size, grid_spacing(patch_size, overlap));
  if (origins_out)
    for (int j = 0; j < a.n && j < max_out; ++j) origins_out[j] = a.origin(j);
  return a.n;
}

size_t dis_patch_search_workspace_bytes(int32_t B, int32_t W, int32_t H,
                                        const dis_params_t* p) {
  if (dis_params_validate(p) || W < p->patch_size || H < p->patch_size) return 0;
  const int sp = grid_spacing(p->patch_size, p->overlap);
  return patch_search_scratch_bytes(
      B, make_axis(W, p->patch_size, sp).n * make_axis(H, p->patch_size, sp).n, W, H);
}

int dis_patch_search(const double* ref_img, const double* ref_gx, const double* ref_gy,
                     const double* qry_img, int32_t B, int32_t W, int32_t H,
                     const double* coarse_flow_u, const double* coarse_flow_v, int32_t Wc,
                     int32_t Hc, const dis_params_t* p, double* out_u, double* out_v,
                     double* out_off, double* out_mar, double* out_init_u, double* out_init_v,
                     uint8_t* out_valid, void* workspace, size_t workspace_bytes,
                     void* stream) {
  if (dis_params_validate(p)) return DIS_ERR_PARAMETER;
  if (workspace_bytes < dis_patch_search_workspace_bytes(B, W, H, p))
    return fail(DIS_ERR_WORKSPACE, "patch search workspace too small");
  if (W < p->patch_size || H < p->patch_size)
    return fail(DIS_ERR_VALUE, "level %dx%d is smaller than the patch size %d", W, H,
                p->patch_size);
  const int sp = grid_spacing(p->patch_size, p->overlap);
  SearchArgs a{};
  a.ref = ref_img;
  a.rgx = ref_gx;
  a.rgy = ref_gy;
  a.qry = qry_img;
  a.B = B;
  a.W = W;
  a.H = H;
  a.cu = coarse_flow_u;
  a.cv = coarse_flow_v;
  a.Wc = Wc;
  a.Hc = Hc;
  a.ax = make_axis(W, p->patch_size, sp);
  a.ay = make_axis(H, p->patch_size, sp);
  a.ps = p->patch_size;
  a.iters = p->iterations;
  a.mean_norm = p->use_mean_normalization;
  a.code = p->residual_norm;
  a.hb = p->huber_b;
  a.ds = p->downscale;
  a.out_u = out_u;
  a.out_v = out_v;
  a.out_off = out_off;
  a.out_mar = out_mar;
  a.out_iu = out_init_u;
  a.out_iv = out_init_v;
  a.out_valid = out_valid;
  a.horizontal = p->mode == 1;  // horizontal_only (inverse_search.py:259-264)
  launch_patch_search(a, workspace, as_stream(stream));
  return check_cuda("dis_patch_search");
}

// ---- the reference's inverse-search stage functions (inverse_search.py:306-387)
// and init / reset (densification.py:82-107) on materialised arrays ----------

int dis_precompute_patch_set(const double* img, const double* gx, const double* gy, int32_t W,
                             int32_t H, const double* x_starts, const double* y_starts,
                             int32_t n, int32_t patch_size, int32_t horizontal_only,
                             double* templates, double* steep_x, double* steep_y,
                             double* template_mean, double* hessian, double* hessian_inv,
                             uint8_t* valid, void* stream) {
  if (patch_size < 1) return fail(DIS_ERR_PARAMETER, "patch_size must be >= 1");
  if (W < 1 || H < 1 || n < 0) return fail(DIS_ERR_VALUE, "bad level or patch count");
  g_launches = 0;
  if (n == 0) return DIS_OK;
  launch_precompute_set(img, gx, gy, W, H, x_starts, y_starts, n, patch_size, horizontal_only,
                        templates, steep_x, steep_y, template_mean, hessian, hessian_inv, valid,
                        as_stream(stream));
  return check_cuda("dis_precompute_patch_set");
}

int dis_optimize_patch_set(const double* qry, int32_t W, int32_t H, const double* x_starts,
                           const double* y_starts, int32_t n, int32_t patch_size,
                           const double* templates, const double* steep_x, const double* steep_y,
                           const double* hessian_inv, const double* template_mean,
                           const uint8_t* valid, const double* init_displacement,
                           int32_t iterations, int32_t mean_normalization, int32_t residual_norm,
                           double huber_b, double* displacement, double* offset,
                           double* mean_abs_residual, void* stream) {
  if (residual_norm < 0 || residual_norm > 2)
    return fail(DIS_ERR_VALUE, "unknown residual norm code %d", residual_norm);
  if (W < 1 || H < 1 || n < 0 || patch_size < 1)
    return fail(DIS_ERR_VALUE, "bad level, patch size or patch count");
  g_launches = 0;
  if (n == 0) return DIS_OK;
  launch_optimize_set(qry, W, H, x_starts, y_starts, n, patch_size, templates, steep_x, steep_y,
                      hessian_inv, template_mean, valid, init_displacement, iterations,
                      mean_normalization, residual_norm, huber_b, displacement, offset,
                      mean_abs_residual, as_stream(stream));
  return check_cuda("dis_optimize_patch_set");
}

int dis_refresh_patch_stats(const double* qry, int32_t W, int32_t H, const double* x_starts,
                            const double* y_starts, int32_t n, int32_t patch_size,
                            const double* templates, const double* template_mean,
                            const uint8_t* select, const double* displacement,
                            int32_t mean_normalization, double* offset,
                            double* mean_abs_residual, void* stream) {
  if (W < 1 || H < 1 || n < 0 || patch_size < 1)
    return fail(DIS_ERR_VALUE, "bad level, patch size or patch count");
  g_launches = 0;
  if (n == 0) return DIS_OK;
  launch_window_stats(qry, W, H, x_starts, y_starts, n, patch_size, templates, template_mean,
                      select, displacement, mean_normalization, offset, mean_abs_residual,
                      as_stream(stream));
  return check_cuda("dis_refresh_patch_stats");
}

int dis_init_patches(const double* coarser_flow, int32_t Wc, int32_t Hc, const double* centers,
                     int32_t n, int32_t downscale, double* init_out, void* stream) {
  if (downscale < 1) return fail(DIS_ERR_PARAMETER, "downscale must be >= 1");
  if (coarser_flow && (Wc < 1 || Hc < 1)) return fail(DIS_ERR_VALUE, "empty coarser field");
  g_launches = 0;
  if (n <= 0) return DIS_OK;
  launch_init_patches(coarser_flow, Wc, Hc, centers, n, downscale, init_out, as_stream(stream));
  return check_cuda("dis_init_patches");
}

int dis_reset_outliers(const double* displacement, const double* init_displacement, int32_t n,
                       int32_t patch_size, double* out, uint8_t* was_reset, void* stream) {
  g_launches = 0;
  if (n <= 0) return DIS_OK;
  launch_reset_outliers(displacement, init_displacement, n, patch_size, out, was_reset,
                        as_stream(stream));
  return check_cuda("dis_reset_outliers");
}

int dis_densify(const double* ref_img, const double* qry_img, int32_t B, int32_t W, int32_t H,
                const dis_params_t* p, const double* patch_u, const double* patch_v,
                const double* patch_off, double* flow_u, double* flow_v, uint32_t* status,
                void* stream) {
  if (dis_params_validate(p)) return DIS_ERR_PARAMETER;
  if (W < p->patch_size || H < p->patch_size)
    return fail(DIS_ERR_VALUE, "level %dx%d is smaller than the patch size %d", W, H,
                p->patch_size);
  const int sp = grid_spacing(p->patch_size, p->overlap);
  launch_densify(ref_img, qry_img, B, W, H, make_axis(W, p->patch_size, sp),
                 make_axis(H, p->patch_size, sp), p->patch_size, patch_u, patch_v, patch_off,
                 flow_u, flow_v, status, as_stream(stream));
  return check_cuda("dis_densify");
}

// ---- sparse correspondences (pipeline.py:202-287) --------------------------
}  // extern "C"
namespace {
struct SparsePlan {
  dis_params_t q;  // params with refinement off (refine=False, pipeline.py:266-268)
  Plan pl;
  size_t off_seeds, off_valid, off_out, off_scratch, total;
};
void make_sparse_plan(const dis_params_t* p, int H, int W, int n, SparsePlan* sp) {
  sp->q = *p;
  sp->q.variational = 0;
  make_plan(&sp->q, 1, H, W, &sp->pl);
  size_t cur = sp->pl.total;
  const size_t nn = (size_t)(n > 0 ? n : 1);
  sp->off_seeds = take(cur, nn * 2 * sizeof(double));
  sp->off_valid = take(cur, nn);
  sp->off_out = take(cur, nn * 2 * sizeof(double));
  sp->off_scratch =
      take(cur, nn * 3 * (size_t)p->patch_size * p->patch_size * sizeof(double));
  sp->total = (cur + 255) & ~size_t(255);
}
}  // namespace
extern "C" {

size_t dis_sparse_workspace_bytes(int32_t H, int32_t W, int32_t n_seeds, const dis_params_t* p) {
  if (dis_params_validate(p) || n_seeds < 0) return 0;
  dis_params_t q = *p;
  q.variational = 0;
  if (check_dims(&q, 1, H, W)) return 0;
  SparsePlan sp;
  make_sparse_plan(p, H, W, n_seeds, &sp);
  return sp.total;
}

int dis_sparse_correspondences(const void* frame1, const void* frame2, int32_t dtype,
                               int32_t H, int32_t W, const dis_params_t* p,
                               const double* host_seeds, int32_t n_seeds,
                               double* host_disp_out, uint8_t* host_valid_out, void* workspace,
                               size_t workspace_bytes, void* stream) {
  int rc = dis_params_validate(p);
  if (rc) return rc;
  if (dtype < 0 || dtype > 2) return fail(DIS_ERR_VALUE, "unsupported frame dtype %d", dtype);
  if (n_seeds < 0) return fail(DIS_ERR_VALUE, "negative seed count");
  dis_params_t q = *p;
  q.variational = 0;
  rc = check_dims(&q, 1, H, W);  // as_image / _check_pair / _check_levels
  if (rc) return rc;
  SparsePlan sp;
  make_sparse_plan(p, H, W, n_seeds, &sp);
  if (workspace_bytes < sp.total)
    return fail(DIS_ERR_WORKSPACE, "workspace holds %zu bytes, need %zu", workspace_bytes,
                sp.total);
  // in-bounds test (pipeline.py:257-261); out-of-bounds seeds are (0, 0), invalid
  std::vector<uint8_t> valid((size_t)n_seeds);
  int ngood = 0;
  for (int i = 0; i < n_seeds; ++i) {
    const double x = host_seeds[2 * i], y = host_seeds[2 * i + 1];
    valid[i] = (x >= 0) && (x <= W - 1) && (y >= 0) && (y <= H - 1);
    ngood += valid[i];
    host_disp_out[2 * i] = host_disp_out[2 * i + 1] = 0.0;
    host_valid_out[i] = valid[i];
  }
  g_launches = 0;
  if (!ngood) return DIS_OK;  // the reference skips the pyramid descent
  cudaStream_t st = as_stream(stream);
  const Plan& pl = sp.pl;
  double* d_seeds = at<double>(workspace, sp.off_seeds);
  uint8_t* d_valid = at<uint8_t>(workspace, sp.off_valid);
  double* d_out = at<double>(workspace, sp.off_out);
  cudaMemsetAsync(at<char>(workspace, pl.off_status), 0, 256, st);
  cudaMemcpyAsync(d_seeds, host_seeds, (size_t)n_seeds * 2 * sizeof(double),
                  cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_valid, valid.data(), (size_t)n_seeds, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(d_out, 0, (size_t)n_seeds * 2 * sizeof(double), st);
  build_pyramids(pl, frame1, frame2, dtype, workspace, st);
  rc = check_cuda("pyramid");
  if (rc) return rc;
  if (p->use_densification) {
    rc = run_pipeline(pl, &sp.q, nullptr, workspace, st, false, false);
    if (rc) return rc;
    const int sf = pl.sf;
    double scale = 1.0;  // params.downscale ** finest_scale (pipeline.py:266)
    for (int s = 0; s < sf; ++s) scale *= (double)pl.ds;
    launch_sparse_sample(at<double>(workspace, pl.off_fu[sf]), at<double>(workspace, pl.off_fv[sf]),
                         pl.ws[sf], pl.hs[sf], scale, d_seeds, d_valid, n_seeds, d_out, st);
  } else {
    SparseChainArgs a{};
    for (int s = 0; s <= pl.ss; ++s) {
      a.img[s] = at<double>(workspace, pl.off_img[0][s]);
      a.gx[s] = at<double>(workspace, pl.off_gx[0][s]);
      a.gy[s] = at<double>(workspace, pl.off_gy[0][s]);
      a.qry[s] = at<double>(workspace, pl.off_img[1][s]);
      a.W[s] = pl.ws[s];
      a.H[s] = pl.hs[s];
    }
    a.coarsest = pl.ss;
    a.finest = pl.sf;
    a.ps = p->patch_size;
    a.iters = p->iterations;
    a.mean_norm = p->use_mean_normalization;
    a.code = p->residual_norm;
    a.hb = p->huber_b;
    a.ds = p->downscale;
    a.seeds = d_seeds;
    a.valid = d_valid;
    a.n = n_seeds;
    a.scratch = at<double>(workspace, sp.off_scratch);
    a.out = d_out;
    launch_sparse_chain(a, st);
  }
  rc = check_cuda("dis_sparse_correspondences");
  if (rc) return rc;
  cudaMemcpyAsync(host_disp_out, d_out, (size_t)n_seeds * 2 * sizeof(double),
                  cudaMemcpyDeviceToHost, st);
  uint32_t status = 0;
  cudaMemcpyAsync(&status, at<char>(workspace, pl.off_status), sizeof status,
                  cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess)
    return fail(DIS_ERR_CUDA, "dis_sparse_correspondences: %s", cudaGetErrorString(e));
  rc = dis_status_to_error(status);
  if (rc) {
    for (int i = 0; i < 2 * n_seeds; ++i) host_disp_out[i] = 0.0;
  }
  return rc;
}

size_t dis_densify_bidirectional_workspace_bytes(int32_t B, int32_t W, int32_t H,
                                                 const dis_params_t* p) {
  if (dis_params_validate(p) || W < p->patch_size || H < p->patch_size) return 0;
  const int sp = grid_spacing(p->patch_size, p->overlap);
  const int P = make_axis(W, p->patch_size, sp).n * make_axis(H, p->patch_size, sp).n;
  return bidir_scratch_bytes(B, W, H, P, p->patch_size);
}

int dis_densify_bidirectional(const double* ref_img, const double* qry_img, int32_t B,
                              int32_t W, int32_t H, const dis_params_t* p,
                              const double* fwd_u, const double* fwd_v, const double* fwd_off,
                              const double* bwd_u, const double* bwd_v, const double* bwd_off,
                              double* flow_u, double* flow_v, void* workspace,
                              size_t workspace_bytes, uint32_t* status, void* stream) {
  if (dis_params_validate(p)) return DIS_ERR_PARAMETER;
  if (W < p->patch_size || H < p->patch_size)
    return fail(DIS_ERR_VALUE, "level %dx%d is smaller than the patch size %d", W, H,
                p->patch_size);
  if (workspace_bytes < dis_densify_bidirectional_workspace_bytes(B, W, H, p))
    return fail(DIS_ERR_WORKSPACE, "bidirectional densify workspace too small");
  const int sp = grid_spacing(p->patch_size, p->overlap);
  launch_densify_bidir(ref_img, qry_img, B, W, H, make_axis(W, p->patch_size, sp),
                       make_axis(H, p->patch_size, sp), p->patch_size, fwd_u, fwd_v, fwd_off,
                       bwd_u, bwd_v, bwd_off, flow_u, flow_v, workspace, status,
                       as_stream(stream));
  return check_cuda("dis_densify_bidirectional");
}

size_t dis_refine_workspace_bytes(int32_t B, int32_t W, int32_t H) {
  return refine_scratch_doubles(B, W, H) * sizeof(double);
}

int dis_refine(const double* ref_img, const double* ref_gx, const double* ref_gy,
               const double* ref_dd, const double* qry_img, const double* qry_gx,
               const double* qry_gy, const double* qry_dd, int32_t B, int32_t W, int32_t H,
               const dis_params_t* p, int32_t outer_iters, double* flow_u, double* flow_v,
               void* workspace, size_t workspace_bytes, uint32_t* status, void* stream) {
  if (dis_params_validate(p)) return DIS_ERR_PARAMETER;
  if (workspace_bytes < dis_refine_workspace_bytes(B, W, H))
    return fail(DIS_ERR_WORKSPACE, "refine workspace too small");
  if (H > 2048)
    return fail(DIS_ERR_VALUE, "variational refinement of a level taller than 2048 rows is not "
                               "supported by this build");
  RefineArgs r{};
  r.ref = ref_img;
  r.rgx = ref_gx;
  r.rgy = ref_gy;
  (void)ref_dd;  // second derivatives are formed on the fly
  r.qry = qry_img;
  r.qgx = qry_gx;
  r.qgy = qry_gy;
  (void)qry_dd;
  r.B = B;
  r.W = W;
  r.H = H;
  r.delta = p->var_intensity_weight;
  r.gamma = p->var_gradient_weight;
  r.alpha = p->var_smoothness_weight;
  r.eps = p->var_penalizer_eps;
  r.omega = p->var_sor_omega;
  r.sweeps = p->var_inner_sor_iters;
  r.outer = outer_iters;
  r.horizontal = p->mode == 1;  // horizontal_only (variational.py:161)
  r.fu = flow_u;
  r.fv = flow_v;
  r.rec = static_cast<double*>(workspace);
  r.status = status;
  int rc = launch_refine(r, as_stream(stream));
  if (rc) return fail(rc, "refine launch failed");
  return check_cuda("dis_refine");
}

int dis_upsample_flow(const double* in_u, const double* in_v, int32_t B, int32_t W, int32_t H,
                      double* out_u, double* out_v, int32_t Wn, int32_t Hn, int32_t scale_factor,
                      void* stream) {
  if (scale_factor < 1) return fail(DIS_ERR_PARAMETER, "scale_factor must be >= 1");
  launch_upsample(in_u, in_v, B, W, H, out_u, out_v, nullptr, Wn, Hn, scale_factor,
                  as_stream(stream));
  return check_cuda("dis_upsample_flow");
}

int dis_compose_flows(const double* flow_ab, const double* flow_bc, int32_t B, int32_t H,
                      int32_t W, double* flow_out, void* stream) {
  if (B < 1 || H < 1 || W < 1)
    return fail(DIS_ERR_VALUE, "flow fields must be non-empty, got (%d, %d, %d)", B, H, W);
  if (!flow_ab || !flow_bc || !flow_out)
    return fail(DIS_ERR_VALUE, "compose_flows: null field pointer");
  const size_t bytes = (size_t)B * H * W * 2 * sizeof(double);
  auto overlap = [&](const double* a) {
    return (const char*)a < (const char*)flow_out + bytes &&
           (const char*)flow_out < (const char*)a + bytes;
  };
  if (overlap(flow_ab) || overlap(flow_bc))
    return fail(DIS_ERR_VALUE, "compose_flows: the output must not alias an input field");
  g_launches = 0;
  launch_compose(flow_ab, flow_bc, B, H, W, flow_out, as_stream(stream));
  return check_cuda("dis_compose_flows");
}

}  // extern "C"
