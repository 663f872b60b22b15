// kernels.cuh — host-side launchers of the DIS kernels (one per stage).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace disb200 {

// ---- instrumentation (api.cu) ----
// Kernel classes timed by the optional per-stage CUDA-event profiler and
// counted by the launch counter (dis_profile_*, dis_last_launch_count).
enum KernelClass {
  KC_PYRAMID = 0,
  KC_SEARCH = 1,
  KC_DENSIFY = 2,
  KC_TENSOR = 3,
  KC_SOR = 4,
  KC_UPSAMPLE = 5,
  KC_COUNT = 6
};
void prof_begin(int cls, cudaStream_t st);
void prof_end(int cls, cudaStream_t st);
void prof_level(int level);  // tags the following launches with their pyramid level
void note_launch(int n = 1);
// evaluation census (bench roofline): device counters or null when off
unsigned long long* census_counters();
// the current CUDA device and its SM count; per-device launch settings
// (kernel attributes, occupancy-derived grid caps) are cached per device
// index, so one process may drive several GPUs
constexpr int kMaxDevices = 64;
int current_device();
int device_sm_count();

// pyramid.cu
// downscale: the pyramid factor k (core.py:88-128); level s is floor(dim / k^s)
void launch_pyramid(const void* frames, int dtype, int B, int H, int W, int coarsest,
                    int downscale, double* const* img, double* const* gx, double* const* gy,
                    double* const* dd, uint32_t* status, cudaStream_t st);

// both frames of a batch at once (the flow path): img[f][s] / gx / gy per
// frame f and level s (null = not needed); no second derivatives
void launch_pyramid_pair(const void* f1, const void* f2, int dtype, int B, int H, int W,
                         int coarsest, int downscale, double* const (*img)[32],
                         double* const (*gx)[32], double* const (*gy)[32], uint32_t* status,
                         cudaStream_t st);

// patch_search.cu — init + precompute + condition + GN + reset + refresh
struct SearchArgs {
  const double* ref;
  const double* rgx;
  const double* rgy;
  const double* qry;
  int B, W, H;
  const double* cu;  // coarse flow (level s+1), row-major planar, or null
  const double* cv;
  int Wc, Hc;
  GridAxis ax, ay;
  int ps, iters, mean_norm, code;
  double hb;
  int ds;            // pyramid factor (init_patches: centre / ds, times ds)
  double* out_u;
  double* out_v;
  double* out_off;
  double* out_mar;    // optional
  double* out_iu;     // optional
  double* out_iv;     // optional
  uint8_t* out_valid; // optional
  int32_t* out_evals; // optional
  unsigned long long* census;  // optional: [0] += evaluations, [1] += patches
  int horizontal;     // stereo: _condition_hessians horizontal_only (259-264)
  // set by launch_patch_search: the query level with a replicated border
  // (patch_search.cu, kQPad), read by the lane kernel
  const double* qpad;
  int qp_pitch;
  // lane kernel: once the work queue is empty, a warp with at most this many
  // patches still running hands them to the lane-group kernel (0: never)
  int stragglers;
};
// scratch of one level's search: per-patch prep + parked state + counters +
// the padded query level (W x H level, P patches per pair)
size_t patch_search_scratch_bytes(int B, int P, int W, int H);
void launch_patch_search(const SearchArgs& a, void* scratch, cudaStream_t st);

// stage_search.cu — the reference's inverse-search / init / reset stage
// functions on materialised per-patch arrays (one thread per patch)
void launch_precompute_set(const double* img, const double* gx, const double* gy, int W, int H,
                           const double* xs, const double* ys, int n, int ps, int horizontal,
                           double* tmpl, double* sdx, double* sdy, double* mean_t, double* hess,
                           double* hinv, uint8_t* valid, cudaStream_t st);
void launch_optimize_set(const double* qry, int W, int H, const double* xs, const double* ys,
                         int n, int ps, const double* tmpl, const double* sdx, const double* sdy,
                         const double* hinv, const double* mean_t, const uint8_t* valid,
                         const double* init, int iters, int mean_norm, int code, double hb,
                         double* disp, double* offset, double* mar, cudaStream_t st);
void launch_window_stats(const double* qry, int W, int H, const double* xs, const double* ys,
                         int n, int ps, const double* tmpl, const double* mean_t,
                         const uint8_t* sel, const double* disp, int mean_norm, double* offset,
                         double* mar, cudaStream_t st);
void launch_init_patches(const double* coarse, int Wc, int Hc, const double* centers, int n,
                         int ds, double* init, cudaStream_t st);
void launch_reset_outliers(const double* disp, const double* init, int n, int ps, double* out,
                           uint8_t* was_reset, cudaStream_t st);

// densify.cu
void launch_densify(const double* ref, const double* qry, int B, int W, int H, GridAxis ax,
                    GridAxis ay, int ps, const double* pu, const double* pv,
                    const double* poff, double* fu, double* fv, uint32_t* status,
                    cudaStream_t st);

// densify.cu — bidirectional merge (densify_bidirectional): forward set
// gathered per pixel, backward set binned by window tile
size_t bidir_scratch_bytes(int B, int W, int H, int P, int ps);
void launch_densify_bidir(const double* ref, const double* qry, int B, int W, int H,
                          GridAxis ax, GridAxis ay, int ps, const double* fu_p,
                          const double* fv_p, const double* foff_p, const double* bu_p,
                          const double* bv_p, const double* boff_p, double* fu, double* fv,
                          void* scratch, uint32_t* status, cudaStream_t st);

// variational.cu
struct RefineArgs {
  const double* ref;
  const double* rgx;
  const double* rgy;
  const double* qry;
  const double* qgx;
  const double* qgy;
  int B, W, H;
  double delta, gamma, alpha, eps, omega;
  int sweeps, outer;
  int horizontal;  // stereo: _sor_sweeps horizontal_only (variational.py:161)
  double* fu;  // flow, row-major planar, refined in place
  double* fv;
  double* rec;  // 8 * B * (W + H - 1) * H doubles of scratch
  uint32_t* status;
};
size_t refine_scratch_doubles(int B, int W, int H);
int launch_refine(const RefineArgs& a, cudaStream_t st);

// upsample.cu — upsample_flow by the pyramid factor (planar in, planar or
// interleaved out)
void launch_upsample(const double* iu, const double* iv, int B, int W, int H, double* ou,
                     double* ov, double* out_interleaved, int Wn, int Hn, int factor,
                     cudaStream_t st);
void launch_interleave(const double* u, const double* v, int B, int W, int H, double* out,
                       cudaStream_t st);
void launch_flow_to_f32(const double* in, float* out, size_t n, cudaStream_t st);

// sparse.cu — sparse_correspondences (pipeline.py:202-287)
struct SparseChainArgs {
  const double* img[32];
  const double* gx[32];
  const double* gy[32];
  const double* qry[32];
  int W[32], H[32];
  int coarsest, finest, ps, iters, mean_norm, code;
  double hb;
  int ds;                // pyramid factor
  const double* seeds;   // (n, 2) device
  const uint8_t* valid;  // (n) device
  int n;
  double* scratch;       // n * 3 * ps^2 doubles
  double* out;           // (n, 2)
};
void launch_sparse_chain(const SparseChainArgs& a, cudaStream_t st);
void launch_sparse_sample(const double* fu, const double* fv, int W, int H, double scale,
                          const double* seeds, const uint8_t* valid, int n, double* out,
                          cudaStream_t st);

// compose.cu — compose_flows (interleaved (B, H, W, 2) fields)
void launch_compose(const double* ab, const double* bc, int B, int H, int W, double* out,
                    cudaStream_t st);

}  // namespace disb200
