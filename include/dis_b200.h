/*
 * dis_b200.h — C ABI of the B200-native Dense Inverse Search (DIS) flow path.
 *
 * This is the drop-in boundary for the reference's `dis_flow` hot path
 * (reference: pkg/src/disflow/pipeline.py:150-163 `dis_flow`,
 *  pipeline.py:136-147 `dis_flow_on_pyramids`) and for the numba operator
 * layer underneath it (the `@njit` kernels in inverse_search.py,
 * densification.py and variational.py, plus the numpy stages in core.py).
 *
 * Conventions (all entry points):
 *  - plain pointers and sizes only; device pointers are CUDA global-memory
 *    addresses (e.g. torch.Tensor.data_ptr()), `stream` is a cudaStream_t
 *    passed as void* (NULL = legacy default stream).
 *  - every call is stream-ordered and asynchronous; nothing allocates;
 *    scratch comes from a caller-owned workspace sized by
 *    dis_workspace_bytes().
 *  - return value: DIS_OK or a negative status (below); a human readable
 *    message for the last failing call on this host thread is available from
 *    dis_last_error().  The status values mirror the reference's exception
 *    types: ParameterError (core.py:25-26), ValueError for shapes
 *    (core.py:68-71, 92-96, 113-119; pipeline.py:30-41), AssertionError for
 *    densification coverage (densification.py:189-190) and RuntimeError for
 *    non-finite refinement output (variational.py:268-274).
 *  - numerics: IEEE float64 in the reference's exact operation order
 *    (no FMA contraction, sequential sums), so results are bit-identical to
 *    the reference on the same inputs.
 *
 * Raster layout on the device: every per-level raster of a pair (image,
 * gradients, second derivatives, dense flow components u and v) is float64
 * row-major (H_s, W_s) exactly like the reference (core.py:1-14); a batch of
 * B pairs stores B such rasters back to back.  Frames passed in are (B, H, W)
 * row-major; the flow returned is (B, H, W, 2) float64 row-major (u, v).
 */
#ifndef DIS_B200_H
#define DIS_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DIS_API __attribute__((visibility("default")))
#else
#define DIS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define DIS_B200_ABI_VERSION 2

/* status codes */
#define DIS_OK 0
#define DIS_ERR_PARAMETER (-1)   /* ParameterError(ValueError)  core.py:25-26      */
#define DIS_ERR_VALUE (-2)       /* ValueError (shapes, non-finite input frames)    */
#define DIS_ERR_COVERAGE (-3)    /* AssertionError densification.py:189-190        */
#define DIS_ERR_NONFINITE (-4)   /* RuntimeError variational.py:268-274            */
#define DIS_ERR_CUDA (-5)        /* CUDA launch / runtime failure                   */
#define DIS_ERR_WORKSPACE (-6)   /* workspace too small                             */

/* residual norms: inverse_search.py:20 NORM_CODES */
#define DIS_NORM_L2 0
#define DIS_NORM_L1 1
#define DIS_NORM_HUBER 2

/* frame element types accepted by the entry points (as_image core.py:65-72
 * converts any real raster to float64; these are the ones we take) */
#define DIS_DTYPE_F32 0
#define DIS_DTYPE_F64 1
#define DIS_DTYPE_U8 2

/* device-status bits written into the workspace status word */
#define DIS_STATUS_NONFINITE_INPUT 1u
#define DIS_STATUS_COVERAGE 2u
#define DIS_STATUS_NONFINITE_FLOW 4u

/*
 * Parameter set: field-for-field the reference's DisParams (core.py:237-257)
 * and VarParams (core.py:197-210).  Two documented extensions:
 *  - outer_iters_fixed: > 0 overrides VarParams.outer_iters(s) = s + 1
 *    (core.py:212-213) with a constant (BASELINE configs use 1);
 *    <= 0 keeps the reference rule.
 *  - mode: 0 "flow", 1 "stereo".  dis_flow_batch rejects stereo-mode
 *    parameters like dis_flow_on_pyramids (pipeline.py:141-142);
 *    dis_stereo_batch runs horizontal-only search and refinement with either
 *    mode (pipeline.py:166-183).
 *  - bidirectional: forward and backward searches merged by
 *    densify_bidirectional at every scale (pipeline.py:97-124).
 */
typedef struct dis_params_t {
  int32_t patch_size;            /* theta_ps                          */
  int32_t iterations;            /* theta_it                          */
  int32_t finest_scale;          /* theta_sf                          */
  int32_t coarsest_scale;        /* theta_ss                          */
  int32_t downscale;             /* pyramid factor k, 2..128          */
  int32_t use_mean_normalization;
  int32_t use_densification;     /* carried; dense path always densifies */
  int32_t residual_norm;         /* DIS_NORM_*                        */
  double overlap;                /* theta_ov                          */
  double huber_b;
  int32_t variational;           /* 0: DisParams.variational is None  */
  int32_t var_inner_sor_iters;   /* theta_vi                          */
  double var_intensity_weight;   /* delta                             */
  double var_gradient_weight;    /* gamma                             */
  double var_smoothness_weight;  /* alpha                             */
  double var_penalizer_eps;
  double var_sor_omega;
  int32_t outer_iters_fixed;     /* extension, see above              */
  int32_t mode;                  /* 0 flow, 1 stereo                  */
  int32_t bidirectional;         /* densify_bidirectional per scale   */
  int32_t reserved;
} dis_params_t;

/* Fill `p` with DisParams() defaults (core.py:246-257, operating point 2). */
DIS_API void dis_params_default(dis_params_t* p);

/* DisParams.validate + VarParams.validate (core.py:296-316, 215-223) plus
 * this path's own limit downscale <= 128. */
DIS_API int dis_params_validate(const dis_params_t* p);

/* Workspace bytes for dis_flow_batch on B pairs of H x W frames. */
DIS_API size_t dis_workspace_bytes(int32_t B, int32_t H, int32_t W, const dis_params_t* p);

/*
 * Fused coarse-to-fine flow for a batch of B independent pairs
 * (dis_flow, pipeline.py:150-163, applied pair by pair).
 *   frame1, frame2 : device, B x H x W row-major, element type `dtype`
 *   flow_out       : device, B x H x W x 2 float64 row-major (u, v)
 *   workspace      : device, >= dis_workspace_bytes(B, H, W, p) bytes
 * Enqueues all work on `stream` and returns without synchronizing.  The
 * device-side status word (non-finite input, coverage, non-finite flow) is
 * at offset 0 of the workspace; read it with dis_read_status() after the
 * stream completes and convert with dis_status_to_error().
 */
DIS_API int dis_flow_batch(const void* frame1, const void* frame2, int32_t dtype,
                   int32_t B, int32_t H, int32_t W, const dis_params_t* p,
                   double* flow_out, void* workspace, size_t workspace_bytes,
                   void* stream);

/* dis_flow_on_pyramids (pipeline.py:136-147) for a batch: the pyramids are
 * given (device arrays of level pointers, index 0..coarsest; each level
 * B x (H>>s) x (W>>s) float64 row-major: image and build_pyramid's
 * image_gradients).  Only the levels the parameters read are used (images of
 * levels >= 1 or of the finest level, gradients of levels >= finest_scale);
 * they are copied into the workspace (dis_workspace_bytes) and the
 * coarse-to-fine loop runs as in dis_flow_batch.  Stereo-mode parameters
 * raise ValueError (pipeline.py:141-142). */
DIS_API int dis_flow_batch_levels(const double* const* img1, const double* const* gx1,
                                  const double* const* gy1, const double* const* img2,
                                  const double* const* gx2, const double* const* gy2,
                                  int32_t B, int32_t H, int32_t W, const dis_params_t* p,
                                  double* flow_out, void* workspace, size_t workspace_bytes,
                                  void* stream);

/* dis_stereo (pipeline.py:166-183) for a batch of rectified pairs: the
 * same pipeline with horizontal-only conditioning (inverse_search.py:
 * 259-264) and SOR (variational.py:161); v comes out identically 0.  Same
 * arguments and workspace as dis_flow_batch. */
DIS_API int dis_stereo_batch(const void* left, const void* right, int32_t dtype,
                             int32_t B, int32_t H, int32_t W, const dis_params_t* p,
                             double* flow_out, void* workspace, size_t workspace_bytes,
                             void* stream);

/* Workspace bytes for dis_flow_batch_host (adds device staging for the
 * frames and the flow). */
DIS_API size_t dis_host_workspace_bytes(int32_t B, int32_t H, int32_t W, int32_t dtype,
                                const dis_params_t* p);

/* Synchronous host-buffer variant (the e2e boundary): host frames in, host
 * flow out; the batch runs as up to 16 chunks on internal streams (copies
 * in, kernels, copies out overlapping across chunks), ordered after prior
 * work on `stream`, and the call returns once they have drained, with the
 * status word already converted to a return code.  Host buffers should be
 * pinned: a call repeating the same pinned buffers, workspace, stream and
 * problem is captured once (its second occurrence) and then replayed as one
 * CUDA graph (same kernels and arguments, so the same results). */
DIS_API int dis_flow_batch_host(const void* host_frame1, const void* host_frame2,
                        int32_t dtype, int32_t B, int32_t H, int32_t W,
                        const dis_params_t* p, double* host_flow_out,
                        void* workspace, size_t workspace_bytes, void* stream);

/* Host-buffer dis_stereo_batch (same contract as dis_flow_batch_host). */
DIS_API int dis_stereo_batch_host(const void* host_left, const void* host_right,
                                  int32_t dtype, int32_t B, int32_t H, int32_t W,
                                  const dis_params_t* p, double* host_flow_out,
                                  void* workspace, size_t workspace_bytes, void* stream);

/* The same calls split in two, for callers that keep several batches in
 * flight (the reference's dis_flow, pipeline.py:150-163, is one blocking call
 * per pair; a streaming caller double-buffers): *_async enqueues the whole
 * call (copies in, kernels, copies out, ordered after prior work on
 * `stream`) and returns without waiting; dis_host_batch_finish waits for
 * `stream` and converts the call's status words (copied to pinned host
 * memory behind the flow) into the return code dis_flow_batch_host would
 * have given.  Between the two the host buffers and the workspace belong to
 * the call.  Calls in flight at the same time need their own workspace, host
 * buffers and stream each; their copies share the PCIe link in call order
 * and their kernels overlap, so one call's copy-out hides the next call's
 * copy-in and compute.  dis_flow_batch_host == *_async + finish. */
DIS_API int dis_flow_batch_host_async(const void* host_frame1, const void* host_frame2,
                                      int32_t dtype, int32_t B, int32_t H, int32_t W,
                                      const dis_params_t* p, double* host_flow_out,
                                      void* workspace, size_t workspace_bytes, void* stream);
DIS_API int dis_stereo_batch_host_async(const void* host_left, const void* host_right,
                                        int32_t dtype, int32_t B, int32_t H, int32_t W,
                                        const dis_params_t* p, double* host_flow_out,
                                        void* workspace, size_t workspace_bytes, void* stream);
DIS_API int dis_host_batch_finish(const void* workspace, int32_t B, int32_t H, int32_t W,
                                  int32_t dtype, const dis_params_t* p, void* stream);

/* The general host-buffer entry point: dis_flow_batch_host with flags.
 *   DIS_HOST_ASYNC     enqueue only (finish with dis_host_batch_finish)
 *   DIS_HOST_STEREO    dis_stereo (pipeline.py:166-183) instead of dis_flow
 *   DIS_HOST_FLOW_F32  host_flow_out is float32 (B, H, W, 2): the float64 flow
 *                      of the same computation, rounded to nearest on the
 *                      device before the copy-out (== numpy's
 *                      flow.astype(float32); rounding error <= 2^-18 px for
 *                      |flow| < 64 px).  Halves the device->host bytes, which
 *                      bound the host path; not the reference's return type,
 *                      so opt-in.
 * flags = 0 is dis_flow_batch_host. */
#define DIS_HOST_ASYNC 1u
#define DIS_HOST_FLOW_F32 2u
#define DIS_HOST_STEREO 4u
DIS_API int dis_flow_batch_host_ex(const void* host_frame1, const void* host_frame2,
                                   int32_t dtype, int32_t B, int32_t H, int32_t W,
                                   const dis_params_t* p, void* host_flow_out,
                                   void* workspace, size_t workspace_bytes, void* stream,
                                   uint32_t flags);

/* sparse_correspondences (pipeline.py:230-287) for one pair: displacements
 * at `n_seeds` seed locations (host (n, 2) x, y in full-resolution pixels)
 * -> host (n, 2) displacements and (n) validity flags.  Seeds outside the
 * image are invalid with (0, 0).  use_densification: the unrefined dense
 * field of the finest scale sampled at the seeds; otherwise one patch chain
 * per seed down the scales (_sparse_chain 202-227).  Frames on the device;
 * synchronous (returns after the results reached the host). */
DIS_API size_t dis_sparse_workspace_bytes(int32_t H, int32_t W, int32_t n_seeds,
                                          const dis_params_t* p);
DIS_API int dis_sparse_correspondences(const void* frame1, const void* frame2,
                                       int32_t dtype, int32_t H, int32_t W,
                                       const dis_params_t* p, const double* host_seeds,
                                       int32_t n_seeds, double* host_disp_out,
                                       uint8_t* host_valid_out, void* workspace,
                                       size_t workspace_bytes, void* stream);

/* Copy the status word out of the workspace (blocking on `stream`). */
DIS_API int dis_read_status(const void* workspace, uint32_t* status_out, void* stream);
/* Map a device status word to DIS_OK / DIS_ERR_* and set dis_last_error(). */
DIS_API int dis_status_to_error(uint32_t status);

/* ------------------------------------------------------------------------
 * Stage entry points (the operator layer), each parity-testable against the
 * reference function named beside it.  Level rasters are row-major float64
 * as described at the top; `B` pairs are processed per call.
 * ---------------------------------------------------------------------- */

/* build_pyramid (core.py:106-128): levels 0..coarsest of B frames, factor
 * `downscale` (k >= 2; level s is floor(dim / k^s), _box_downsample
 * core.py:88-98 in numpy's summation order).
 *   levels_img[s]  : device B x H_s x W_s float64 for every s in
 *                    0..coarsest (levels_img[0] may be NULL: level 1 is then
 *                    computed from the frames directly)
 *   levels_gx/gy[s]: gradients (image_gradients core.py:75-85), NULL = skip
 *   levels_dd[s]   : 4 consecutive rasters gxx, gxy, gyx, gyy
 *                    (_second_derivatives variational.py:168-171), NULL = skip
 *   status         : device uint32, OR-ed with DIS_STATUS_NONFINITE_INPUT */
DIS_API int dis_build_pyramid(const void* frames, int32_t dtype, int32_t B, int32_t H,
                      int32_t W, int32_t coarsest, int32_t downscale,
                      double* const* levels_img, double* const* levels_gx,
                      double* const* levels_gy, double* const* levels_dd, uint32_t* status,
                      void* stream);

/* init_patches + precompute_patch_set + optimize_patch_set + reset_outliers
 * + refresh_patch_stats for one scale (pipeline.py:54-82).  p->mode == 1
 * selects the horizontal_only conditioning (stereo).
 *   ref_img/ref_gx/ref_gy/qry_img : level s, B x H x W
 *   coarse_flow_u/v : level s+1 flow (B x Hc x Wc) or NULL (zeros)
 *   out_u/out_v/out_off/out_mar : B x P_s, P_s in grid row-major order
 *   out_init_u/v (optional, may be NULL): B x P_s initial displacements
 *   out_valid (optional): B x P_s uint8 */
DIS_API int dis_patch_search(const double* ref_img, const double* ref_gx,
                     const double* ref_gy, const double* qry_img, int32_t B,
                     int32_t W, int32_t H, const double* coarse_flow_u,
                     const double* coarse_flow_v, int32_t Wc, int32_t Hc,
                     const dis_params_t* p, double* out_u, double* out_v,
                     double* out_off, double* out_mar, double* out_init_u,
                     double* out_init_v, uint8_t* out_valid, void* workspace,
                     size_t workspace_bytes, void* stream);
/* Scratch for dis_patch_search (per-patch prep records + work counter). */
DIS_API size_t dis_patch_search_workspace_bytes(int32_t B, int32_t W, int32_t H,
                                                const dis_params_t* p);

/* densify (densification.py:173-191): dense flow of level s. */
DIS_API int dis_densify(const double* ref_img, const double* qry_img, int32_t B,
                int32_t W, int32_t H, const dis_params_t* p,
                const double* patch_u, const double* patch_v,
                const double* patch_off, double* flow_u, double* flow_v,
                uint32_t* status, void* stream);

/* densify_bidirectional (densification.py:194-234): forward patches (on
 * ref_img, grid of the level) merged with the negated backward patches (on
 * qry_img, same grid) whose displaced windows cover each pixel
 * (_accumulate_backward 131-153); per-pixel sums in ascending patch index.
 * The workspace holds the backward windows' tile bins. */
DIS_API size_t dis_densify_bidirectional_workspace_bytes(int32_t B, int32_t W, int32_t H,
                                                         const dis_params_t* p);
DIS_API int dis_densify_bidirectional(const double* ref_img, const double* qry_img,
                                      int32_t B, int32_t W, int32_t H,
                                      const dis_params_t* p, const double* fwd_u,
                                      const double* fwd_v, const double* fwd_off,
                                      const double* bwd_u, const double* bwd_v,
                                      const double* bwd_off, double* flow_u,
                                      double* flow_v, void* workspace,
                                      size_t workspace_bytes, uint32_t* status,
                                      void* stream);

/* Workspace for dis_refine on one level. */
DIS_API size_t dis_refine_workspace_bytes(int32_t B, int32_t W, int32_t H);

/* refine (variational.py:220-275) in place on flow_u/flow_v (p->mode == 1:
 * horizontal_only), running `outer_iters` fixed-point iterations (pass
 * params->outer_iters_fixed or scale_index + 1).  ref_dd/qry_dd (the 4
 * second-derivative rasters gxx, gxy, gyx, gyy of each level) are accepted
 * for interface compatibility and may be NULL: the kernel forms them from
 * the gradient rasters on the fly (_second_derivatives, variational.py:
 * 168-171). */
DIS_API int dis_refine(const double* ref_img, const double* ref_gx, const double* ref_gy,
               const double* ref_dd, const double* qry_img, const double* qry_gx,
               const double* qry_gy, const double* qry_dd, int32_t B, int32_t W,
               int32_t H, const dis_params_t* p, int32_t outer_iters,
               double* flow_u, double* flow_v, void* workspace,
               size_t workspace_bytes, uint32_t* status, void* stream);

/* upsample_flow (core.py:178-190) by `scale_factor` from a W x H level to
 * a Wn x Hn level (planar u, v in and out):
 * out(x) = scale_factor * bilinear_map(flow, x / scale_factor). */
DIS_API int dis_upsample_flow(const double* in_u, const double* in_v, int32_t B,
                      int32_t W, int32_t H, double* out_u, double* out_v,
                      int32_t Wn, int32_t Hn, int32_t scale_factor, void* stream);

/* ---- the reference's inverse-search stage functions on materialised
 * per-patch arrays (device memory; one level, n patches; the flow path fuses
 * these inside dis_patch_search) -------------------------------------------
 * precompute_patch_set (inverse_search.py:306-341): window origins x_starts,
 * y_starts (n, real coordinates) -> templates, steep_x, steep_y (n, ps*ps),
 * template_mean (n), hessian / hessian_inv (n, 3 packed [00, 01, 11]) and
 * valid (n, uint8) from _patch_precompute (75-98) and _condition_hessians
 * (255-276; horizontal_only = the stereo form 259-264). */
DIS_API int dis_precompute_patch_set(const double* img, const double* gx, const double* gy,
                                     int32_t W, int32_t H, const double* x_starts,
                                     const double* y_starts, int32_t n, int32_t patch_size,
                                     int32_t horizontal_only, double* templates,
                                     double* steep_x, double* steep_y, double* template_mean,
                                     double* hessian, double* hessian_inv, uint8_t* valid,
                                     void* stream);

/* optimize_patch_set (inverse_search.py:344-371): _patch_optimize (113-189)
 * for every patch from init_displacement (n, 2) -> displacement (n, 2),
 * offset (n), mean_abs_residual (n).  residual_norm: DIS_NORM_*. */
DIS_API int dis_optimize_patch_set(const double* qry, int32_t W, int32_t H,
                                   const double* x_starts, const double* y_starts, int32_t n,
                                   int32_t patch_size, const double* templates,
                                   const double* steep_x, const double* steep_y,
                                   const double* hessian_inv, const double* template_mean,
                                   const uint8_t* valid, const double* init_displacement,
                                   int32_t iterations, int32_t mean_normalization,
                                   int32_t residual_norm, double huber_b, double* displacement,
                                   double* offset, double* mean_abs_residual, void* stream);

/* refresh_patch_stats (inverse_search.py:374-387, _window_stats 227-248):
 * offset and mean_abs_residual of the selected patches (select, n uint8) at
 * their displacement (n, 2); the others are left untouched. */
DIS_API int dis_refresh_patch_stats(const double* qry, int32_t W, int32_t H,
                                    const double* x_starts, const double* y_starts, int32_t n,
                                    int32_t patch_size, const double* templates,
                                    const double* template_mean, const uint8_t* select,
                                    const double* displacement, int32_t mean_normalization,
                                    double* offset, double* mean_abs_residual, void* stream);

/* init_patches (densification.py:82-95): the coarser field (Hc x Wc x 2
 * interleaved, or NULL = zeros) sampled with bilinear_map at centers (n, 2)
 * / downscale, times downscale -> init_out (n, 2). */
DIS_API int dis_init_patches(const double* coarser_flow, int32_t Wc, int32_t Hc,
                             const double* centers, int32_t n, int32_t downscale,
                             double* init_out, void* stream);

/* reset_outliers (densification.py:98-107): out = init where
 * hypot(displacement - init) > patch_size (correctly rounded), else
 * displacement; was_reset (optional, n uint8) marks the reset patches. */
DIS_API int dis_reset_outliers(const double* displacement, const double* init_displacement,
                               int32_t n, int32_t patch_size, double* out, uint8_t* was_reset,
                               void* stream);

/* compose_flows (pipeline.py:186-199): out(x) = ab(x) + bc(x + ab(x)) with
 * bc sampled by bilinear_map (core.py:154-170).  B fields, each H x W x 2
 * float64 interleaved (u, v), device memory; `out` must not alias the
 * inputs.  Frame chaining (cli.py chain) composes consecutive fields. */
DIS_API int dis_compose_flows(const double* flow_ab, const double* flow_bc, int32_t B,
                              int32_t H, int32_t W, double* flow_out, void* stream);

/* Patch grid (create_grid densification.py:58-79): number of window
 * origins per axis and the origins themselves (host memory).  Returns the
 * count, or a negative status. */
DIS_API int32_t dis_grid_axis(int32_t dim, int32_t patch_size, double overlap,
                      int32_t* origins_out, int32_t max_out);

/* ------------------------------------------------------------------------
 * Instrumentation (not part of the reference interface; used by bench.py).
 * ---------------------------------------------------------------------- */
/* Kernels this library launched since the last dis_flow_batch() began. */
DIS_API long long dis_last_launch_count(void);
/* Per-stage CUDA-event timing: classes 0 pyramid, 1 patch search,
 * 2 densify, 3 tensor+assemble, 4 SOR, 5 upsample. */
DIS_API void dis_profile_enable(int32_t on);
DIS_API void dis_profile_reset(void);
/* Blocks on the recorded events; writes total ms and launch counts. */
DIS_API int dis_profile_read(double* ms_out, int64_t* count_out, int32_t n_classes);
/* Every timed launch since dis_profile_reset, in enqueue order: its class,
 * its pyramid level (-1 outside the coarse-to-fine loop) and its ms (up to
 * `max` entries).  Blocks like dis_profile_read; returns the entry count or
 * a negative status. */
DIS_API int32_t dis_profile_log(int32_t* cls_out, int32_t* level_out, double* ms_out,
                                int32_t max);

/* Evaluation census (bench roofline): while on, the patch-search kernels
 * count window evaluations and finished patches on the device; read with
 * dis_census_read (blocking).  Turning it on resets the counters. */
DIS_API int dis_census_enable(int32_t on);
DIS_API int dis_census_read(long long* evals_out, long long* patches_out);

/* Measured FP64 peak of this device for the roofline denominator:
 * independent DADD and DMUL chains (no FMA, as in the exact-parity
 * kernels) over all SMs; writes Gop/s of each. */
DIS_API int dis_selftest_fp64_peak(double* dadd_gops, double* dmul_gops, void* stream);

/* Test hook: exact_div_pos (the SOR's division) and IEEE `/` on device
 * arrays n, d -> fast, ieee (count elements). */
DIS_API int dis_selftest_div(const double* n, const double* d, double* fast,
                             double* ieee, size_t count, void* stream);

/* Human-readable message of the last failing call on this host thread. */
DIS_API const char* dis_last_error(void);
/* DIS_B200_ABI_VERSION of the loaded library. */
DIS_API int32_t dis_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DIS_B200_H */
