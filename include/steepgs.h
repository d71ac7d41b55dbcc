/* steepgs.h — C ABI of the SteepGS hot path on B200 (sm_100a only).
 *
 * Paper: arXiv 2505.05587 (SteepGS, "Steepest Density Control").  Citations P:L<n> are lines of
 * /root/reference/PAPER.md; canonical definitions C1..C24 and readings Z1..Z27 are DESIGN.md §3.
 * Hot path: project, bin_sort, render_fwd, l1_grad, render_bwd_split, densify.
 * Widened rows (§8(f)): Algorithm-1 optimiser (adam_step, reset_moments), budget / gate variants of
 * densify, SH colour (project_sh, sh_bwd, adam_step_planes, copy_offspring), the SSIM loss
 * (l1_ssim_grad), the ADC baseline (densify_adc).
 *
 * Conventions for every call
 *  - Pointers are CUDA DEVICE pointers owned by the caller unless tagged [host].  The library never
 *    allocates, frees or reallocates device memory and keeps no global state except a
 *    thread-local error string, a launch counter and the binning generation counter.
 *  - `stream` is a cudaStream_t passed as void*.  Calls are asynchronous on `stream` and never
 *    synchronise it, except steepgs_densify_host_count (documented below).  Nothing is
 *    read back to the host, so every call can be captured in a CUDA graph.  Most kernels are
 *    launched with programmatic dependent launch (they may be scheduled while the preceding kernel
 *    of the stream drains, and wait for it to complete before reading anything), so stream order
 *    holds exactly as for plain launches.
 *  - Reentrant; concurrent calls must not share output or workspace buffers.
 *  - Errors are returned as steepgs_status; no exception crosses the ABI.  Asynchronous device
 *    faults surface as STEEPGS_ERR_CUDA at a later call.  steepgs_last_error() gives detail.
 *  - No CPU fallback: without a compute-capability 10.x device every call returns
 *    STEEPGS_ERR_UNSUPPORTED_DEVICE.
 *
 * Data layouts
 *  - params  [14][ld] fp32 planar (ld >= capacity >= n): 0-2 mean p, 3-5 log-scale, 6-9 quaternion
 *            (w,x,y,z; normalised on use), 10 opacity logit, 11-13 rgb.          (C1)
 *  - grad_S  [20][ldg] fp32 planar: 0-13 dL/d(param plane k), 14-19 splitting matrix S
 *            (xx,xy,xz,yy,yz,zz).  Summed over views (and, by the caller, over steps/ranks).
 *  - splats  [V][n] steepgs_splat (64 B): the per-(view, Gaussian) projected record.
 *  - images  [V][3][H][W] fp32; per-pixel planes [V][H][W].  All views of a call share W, H.
 */
#ifndef STEEPGS_H
#define STEEPGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  STEEPGS_OK = 0,
  STEEPGS_ERR_INVALID_ARGUMENT = 1,    /* null/misaligned pointer, n < 0, V outside [1, 64],
                                          width/height <= 0 or differing across views, ld < n,
                                          tile != 16, denom <= 0, gate not 0/1/2 */
  STEEPGS_ERR_WORKSPACE_TOO_SMALL = 2, /* ws_bytes < steepgs_bin_sort_workspace_size(...) */
  STEEPGS_ERR_CAPACITY = 3,            /* densify: n + n_split > capacity (host-count variant) */
  STEEPGS_ERR_STALE_STATE = 4,         /* render_bwd: the binning was not rendered forward with these
                                          splats / cameras / raster params since its bin_sort (§8(b)) */
  STEEPGS_ERR_UNSUPPORTED_DEVICE = 5,  /* no CUDA device of compute capability 10.x */
  STEEPGS_ERR_CUDA = 6                 /* launch / runtime error, see steepgs_last_error() */
} steepgs_status;

/* One camera (view), [host].  World -> camera: t_c = R p + t, R row-major.  Camera looks down +z,
 * image y down, pixel (j, k) samples (j + 0.5, k + 0.5) (Z5).
 * model 0: pinhole, EWA local affine P = J(t_c) R ("approx"); model 1: affine
 * Pi(p) = diag(fx, fy)[R p + t]_xy + (cx, cy), the paper's exact Eq. eqn:sigma_2D footnote.
 * Pinhole culls: z <= znear, |x/z| > guard (W/2)/fx, |y/z| > guard (H/2)/fy (C3). */
typedef struct {
  float R[9], t[3];
  float fx, fy, cx, cy;
  int32_t width, height, model;
  float znear, guard;
} steepgs_camera;

/* Compositing parameters (C8, Z3).  Defaults 1/255, 0.99, 1e-4, 0.3, {0,0,0}, 16.
 * Smooth mode (used by the theorem pins): 0, 1, 0, 0.  tile must be 16. */
typedef struct {
  float alpha_min, alpha_max, t_min, dilation;
  float bg[3];
  int32_t tile;
} steepgs_raster_params;

/* Densify parameters (Thm 2, Alg. 1).  eps_split default -1e-6; eta >= 0:
 * eps = eta sqrt(v^T Sigma v) (default 0.5, Z13), eta < 0: eps = eps_abs; denom = number of
 * accumulated views/steps (S_bar = S / denom), must be > 0.
 * gate = 1: the "compactest" variant (App. A.2): a Gaussian is split only if also
 *   ||G_p / denom||_2 <= eps_grad, G_p = the accumulated position-gradient planes 0-2 (Z12, Z21).
 * gate = 2: Alg. 1's "condition on G" read as 3DGS's densification condition (C24): split
 *   only if grad_S[0][i] / grad_S[1][i] >= eps_grad, planes 0, 1 holding the view_grad_stats of
 *   steepgs_gauss_bwd_split (sum of ||dL/dPi(p)|| over visible views, their count).
 * budget >= 0: "densification with increment budget" (App. A.2): of the Gaussians
 *   that pass the rule, split at most `budget`, those with the least lambda_min (ties: lower
 *   index first); budget < 0: unlimited. */
typedef struct {
  float eps_split, eta, eps_abs, eps_grad, denom;
  int32_t gate;
  int64_t budget;
} steepgs_densify_params;

/* Projected splat (a1 output), 64 B.  mean Pi(p) in pixels kept in fp64 so that per-pair offsets
 * are exact to ~1e-7 px after tile-relative rounding; conic Q = Pi(Sigma)^-1 (with dilation)
 * stored pre-scaled for exp2 as (Qxx, 2 Qxy, Qyy) * log2(e)/2, so sigma = 2^(log2_opacity - m'),
 * m' = conic[0] dx^2 + conic[1] dx dy + conic[2] dy^2; opacity o = sigmoid(logit); rgb;
 * extent = padded half-extents (pixels) of the alpha support {d^T Q d <= tau} along x and y;
 * tau = 2 ln(o / alpha_min).  Conic, mean and extents are formed in fp64 and rounded once. */
typedef struct {
  double mean[2];
  float conic[3];
  float log2_opacity;
  float rgb[3];
  float opacity;
  float extent[2];
  float tau;
  float reserved;
} steepgs_splat;

/* Binning result: device pointers into the caller's workspace.  [host] struct. */
typedef struct {
  const uint32_t* ids;          /* [max_instances] Gaussian index per tile instance, ordered by
                                   (view, tile, depth key, index); valid prefix = *n_instances */
  const uint32_t* ranges;       /* [V * tiles_x * tiles_y][2] (start, end) into ids */
  const int64_t* n_instances;   /* device scalar I */
  const int64_t* n_visible;     /* device scalar: visible (view, Gaussian) pairs */
  const int32_t* overflow;      /* device flag: 1 if I > max_instances (results then invalid) */
  uint32_t* tile_last;          /* [V * tiles_x * tiles_y]: zeroed by bin_sort; render_fwd stores the
                                   tile's composited list prefix (max over its pixels of n_contrib),
                                   which render_bwd reads: the backward needs the forward's binning */
  uint8_t* inst_mask;           /* [max_instances]: render_fwd stores, per tile instance it stages
                                   and its consumers finish, the 8-bit mask of the tile's 8x4
                                   sub-blocks in which at least one pixel composited the splat (bit
                                   2 strip + column); render_bwd reads it to visit only contributing
                                   (block, splat) pairs.  Instances after the forward's early exit
                                   (all pixels of the tile terminated) are not written; the backward
                                   never reaches them (it stops at tile_last) */
  int64_t max_instances;
  int32_t tiles_x, tiles_y, V;
  uint64_t generation;          /* set by bin_sort: a process-wide counter, distinct per bin_sort call */
  uint64_t fwd_token;           /* set by render_fwd(_l1): a hash of (generation, splats, n, cameras,
                                   raster params) of the forward that filled tile_last / inst_mask;
                                   render_bwd recomputes it from its own arguments and returns
                                   STEEPGS_ERR_STALE_STATE on a mismatch (0: no forward yet) */
  const uint32_t* tile_order;   /* [V * tiles_x * tiles_y]: set by bin_sort, the (view, tile) indices
                                   by descending tile-list length (half-octave buckets); the raster kernels
                                   take their tiles in this order (a scheduling permutation only) */
} steepgs_binning;

/* ---- a1: projection (Eq. eqn:sigma_2D + footnote P:L135-139).  Per (view, Gaussian):
 * activations, camera transform, culls, P = J R, Pi(Sigma) = P Sigma P^T + dil I, conic, opacity,
 * alpha-support tile rect and tiles_touched, depth key (DESIGN.md §3.2 decision chain, bit-exact
 * with the oracle).  Culled Gaussians get tiles_touched = 0.
 * Outputs: splats [V][n]; depth_key [V][n] (orderable uint32 of fp32 z); tile_rect [V][n] packed
 * uint32x2 (x0 | x1 << 16, y0 | y1 << 16, inclusive tile coords); tiles_touched [V][n] int32. */
steepgs_status steepgs_project(const float* params, int64_t ld, int64_t n, const steepgs_camera* cams,
                               int32_t V, const steepgs_raster_params* rp, steepgs_splat* splats,
                               uint32_t* depth_key, uint32_t* tile_rect, int32_t* tiles_touched,
                               void* stream);

/* ---- NEXT f3: view-dependent colour from real spherical harmonics (3DGS ordering and
 * constants, degree 0..3, K = (degree + 1)^2).  colour = max(0, sum_k Y_k(dir) f_k + 1/2) per
 * (view, Gaussian), dir = (p - o)/|p - o| with o = -R^T t (pinhole) or R^T e_z (affine).  The DC
 * coefficients f_0 are parameter planes 11-13; sh_rest [3 (K - 1)][ld_sh] holds f_k, plane
 * 3 (k - 1) + ch.  Same outputs as steepgs_project; the splat record carries the view's colour. */
steepgs_status steepgs_project_sh(const float* params, int64_t ld, int64_t n, const float* sh_rest, int64_t ld_sh,
                                  int32_t sh_degree, const steepgs_camera* cams, int32_t V,
                                  const steepgs_raster_params* rp, steepgs_splat* splats, uint32_t* depth_key,
                                  uint32_t* tile_rect, int32_t* tiles_touched, void* stream);

/* ---- a2: bin & sort ("sorts points according to view-dependent depth"; C7).
 * Stable depth sort of visible (view, Gaussian) pairs, duplication per touched tile, stable sort
 * by (view, tile), tile ranges.  Result order within a tile: ascending (depth key, index) —
 * bit-exact.  No host synchronisation: sizes live on the device; max_instances bounds I. */
steepgs_status steepgs_bin_sort_workspace_size(int64_t n, int32_t V, int32_t width, int32_t height,
                                               int64_t max_instances, size_t* bytes /*[host]*/);
steepgs_status steepgs_bin_sort(const uint32_t* depth_key, const uint32_t* tile_rect,
                                const int32_t* tiles_touched, int64_t n, const steepgs_camera* cams,
                                int32_t V, const steepgs_raster_params* rp, void* workspace,
                                size_t ws_bytes, int64_t max_instances,
                                steepgs_binning* out /*[host]*/, void* stream);

/* ---- a3: forward compositing, Eq. eqn:alpha_blend, C8.
 * image [V][3][H][W]; final_T [V][H][W]; n_contrib [V][H][W] = length of the tile-list prefix
 * up to the last composited Gaussian (consumed by the backward).
 * pair_counts: NULL, or a device int64[2] that receives += (composited pairs, evaluated pairs)
 * (the units of the roofline model). */
steepgs_status steepgs_render_fwd(const steepgs_splat* splats, int64_t n, steepgs_binning* b /*[host], fwd_token set*/,
                                  const steepgs_camera* cams, int32_t V, const steepgs_raster_params* rp,
                                  float* image, float* final_T, int32_t* n_contrib, int64_t* pair_counts,
                                  void* stream);

/* a3 + a4 fused: the forward above, and in its epilogue the l1 gradient of steepgs_l1_grad
 * (dL_dimage = scale * sign(image - target), loss[v] = scale * sum |image - target| if loss != NULL,
 * the same expressions), so the image is not read back by a separate pass.  target / dL_dimage
 * [V][3][H][W]. */
steepgs_status steepgs_render_fwd_l1(const steepgs_splat* splats, int64_t n, steepgs_binning* b /*[host]*/,
                                     const steepgs_camera* cams, int32_t V, const steepgs_raster_params* rp,
                                     float* image, float* final_T, int32_t* n_contrib, const float* target,
                                     float scale, float* dL_dimage, float* loss, int64_t* pair_counts, void* stream);

/* The same with 8-bit targets (the photographs' own format: a quarter of the bytes to upload per step):
 * target [V][3][H][W] uint8, decoded as C_hat = (float)target * (1.0f / 255.0f) (fp32, one rounding), then the
 * expressions above; results bit-identical to steepgs_render_fwd_l1 on the decoded float targets. */
steepgs_status steepgs_render_fwd_l1_u8(const steepgs_splat* splats, int64_t n, steepgs_binning* b /*[host]*/,
                                        const steepgs_camera* cams, int32_t V, const steepgs_raster_params* rp,
                                        float* image, float* final_T, int32_t* n_contrib, const uint8_t* target,
                                        float scale, float* dL_dimage, float* loss, int64_t* pair_counts,
                                        void* stream);

/* ---- a4: l1 loss gradient helper (Eq. eqn:loss; C9, Z8):
 * dL_dimage = scale * sign(image - target) (sign(0) = 0) over V*count elements; if loss != NULL,
 * loss[v] (device, [V]) = scale * sum |image - target| over view v. */
steepgs_status steepgs_l1_grad(const float* image, const float* target, int32_t V, int64_t count,
                               float scale, float* dL_dimage, float* loss, void* stream);

/* NEXT f3: the 3DGS photometric loss with the SSIM term (P:L150 footnote), per view
 *   loss[v] = (1 - lambda) mean |C - C_hat| + lambda (1 - SSIM(C, C_hat))   (3DGS: lambda = 0.2),
 * SSIM = mean over [3][H][W] of the SSIM map (11x11 Gaussian window, sigma 1.5, zero padding,
 * C1 = 0.01^2, C2 = 0.03^2); dL_dimage = scale * d loss[v] / d image (scale = 1/V for a batch
 * mean).  image, target, dL_dimage [V][3][H][W]; loss [V] device or NULL; workspace >=
 * steepgs_loss_workspace_size(V, H, W) bytes (SSIM partial maps + per-view sums). */
steepgs_status steepgs_loss_workspace_size(int32_t V, int32_t height, int32_t width, size_t* bytes /*[host]*/);
steepgs_status steepgs_l1_ssim_grad(const float* image, const float* target, int32_t V, int32_t height, int32_t width,
                                    float lambda_ssim, float scale, float* dL_dimage, float* loss, void* workspace,
                                    size_t ws_bytes, void* stream);

/* ---- a5 + a6: backward with the splitting matrix (Thm 1; S per P:L356-358; Alg. 1
 * P:L537-538).  Replays each pixel back to front, accumulates per (view, Gaussian) 9 moments of
 * w = dL/dsigma * sigma (sum w, sum w d, sum w d d^T, sum alpha T dL/dC) into moments_ws, then per
 * Gaussian chains them to dL/dparams and S_view = P^T (Q M Q - m0 Q) P, summed over the V views.
 * grad_S (columns [0, n)): accumulate = 0: grad_S = result; 1: grad_S += result; 2: gradient planes
 * 0-13 = result, S planes 14-19 += result (Alg. 1: per-step gradients, S summed over T_split steps).
 * accumulate | 4 (SH colour, after steepgs_sh_bwd): planes 0-2 are added to, planes 11-13 untouched.
 * moments_ws [V][n][12] fp32 must be all-zero on first use; the call leaves it all-zero.
 * view_grad_stats [2][ldg] fp32 or NULL (NEXT f4, the ADC statistic of P:L154): plane 0 gets the sum
 * over this call's views v with tiles_touched[v][i] > 0 of ||dL/dPi(p_i)||_2 (pixel units), plane 1
 * the number of such views; written (accumulate = 0) or added (1, 2) like the S planes.
 * tiles_touched ([V][n], from steepgs_project) is read only then.
 * Precondition: splats, b, cams and rp are those of the steepgs_render_fwd call that produced
 * final_T and n_contrib (the replay also reads b->tile_last and b->inst_mask, which that forward
 * wrote).  Checked on the host through b->fwd_token: a binning re-sorted since, or a forward run
 * with other splats / n / cameras / raster params, returns STEEPGS_ERR_STALE_STATE (nothing is
 * launched).  (final_T / n_contrib / dL_dimage are not covered: the caller owns those buffers.) */
steepgs_status steepgs_render_bwd_split(const float* params, int64_t ld, int64_t n,
                                        const steepgs_splat* splats, const steepgs_binning* b,
                                        const steepgs_camera* cams, int32_t V,
                                        const steepgs_raster_params* rp, const float* final_T,
                                        const int32_t* n_contrib, const float* dL_dimage,
                                        float* moments_ws, float* grad_S, int64_t ldg, int32_t accumulate,
                                        const int32_t* tiles_touched, float* view_grad_stats, void* stream);

/* The two halves of steepgs_render_bwd_split, exported separately so each kernel can be timed:
 * a5 (per-pixel replay -> moments_ws) and a6 (moments -> grad_S, S; clears moments_ws). */
steepgs_status steepgs_render_bwd_moments(const steepgs_splat* splats, int64_t n, const steepgs_binning* b,
                                          const steepgs_camera* cams, int32_t V, const steepgs_raster_params* rp,
                                          const float* final_T, const int32_t* n_contrib, const float* dL_dimage,
                                          float* moments_ws, void* stream);
steepgs_status steepgs_gauss_bwd_split(const float* params, int64_t ld, int64_t n, const steepgs_camera* cams,
                                       int32_t V, const steepgs_raster_params* rp,
                                       float* moments_ws, float* grad_S, int64_t ldg, int32_t accumulate,
                                       const int32_t* tiles_touched, float* view_grad_stats, void* stream);

/* NEXT f3 backward: call after steepgs_render_bwd_moments and before steepgs_gauss_bwd_split (which
 * then takes accumulate | 4).  From the per-(view, Gaussian) colour gradient in moments_ws (left in
 * place) through the clamp and the SH expansion: grad_S planes 11-13 = dL/d(DC coefficients), planes
 * 0-2 = the view-direction part of dL/dp (pinhole), grad_sh [3 (K - 1)][ldg_sh] = dL/d(rest);
 * written (accumulate 0, 2) or added (1) like the gradient planes of steepgs_gauss_bwd_split. */
steepgs_status steepgs_sh_bwd(const float* params, int64_t ld, int64_t n, const float* sh_rest, int64_t ld_sh,
                              int32_t sh_degree, const steepgs_camera* cams, int32_t V, const float* moments_ws,
                              float* grad_S, int64_t ldg, float* grad_sh, int64_t ldg_sh, int32_t accumulate,
                              void* stream);

/* ---- a8: steepest density control (Thm 2; Alg. 1; eigen App. A.3
 * P:L584-604).  Per Gaussian: S_bar = S / denom; lambda_min by the trigonometric roots (fp32,
 * recomputed in fp64 within a guard band of eps_split); v_min (unit, canonical sign); split iff
 * lambda_min < eps_split; rank by exclusive scan; offspring A in slot i at p + eps v, B in slot
 * n + rank at p - eps v, both logit(o/2), other planes copied (C15).  S planes zeroed on
 * [0, n + n_split); all 20 accumulator planes of new slots zeroed.
 * Outputs: split_mask [n] u8, dest_index [n] i32 (n + rank or -1), lambda_min [n] f32 or NULL,
 * n_split [1] int64 device scalar, status [1] int32 device scalar (0 ok, 3 = capacity exceeded:
 * then params/grad_S are untouched).  workspace: >= steepgs_densify_workspace_size(n) bytes. */
steepgs_status steepgs_densify_workspace_size(int64_t n, size_t* bytes /*[host]*/);
steepgs_status steepgs_densify(float* params, int64_t ld, int64_t n, int64_t capacity, float* grad_S,
                               int64_t ldg, const steepgs_densify_params* dp, uint8_t* split_mask,
                               int32_t* dest_index, float* lambda_min, int64_t* n_split,
                               int32_t* status, void* workspace, size_t ws_bytes, void* stream);
/* Convenience: same as steepgs_densify, then synchronises `stream` and returns the count in
 * *n_split_host; STEEPGS_ERR_CAPACITY if n + n_split > capacity. */
steepgs_status steepgs_densify_host_count(float* params, int64_t ld, int64_t n, int64_t capacity,
                                          float* grad_S, int64_t ldg, const steepgs_densify_params* dp,
                                          uint8_t* split_mask, int32_t* dest_index, float* lambda_min,
                                          int64_t* n_split, int32_t* status, void* workspace,
                                          size_t ws_bytes, int64_t* n_split_host, void* stream);

/* ---- NEXT f4: 3DGS Adaptive Density Control baseline.  Per Gaussian:
 * g = view_grad_stats[0][i] / view_grad_stats[1][i] (0 if never visible); selected iff g >= eps_adc;
 * clone iff ||Sigma||_2 = max_k s_k^2 <= tau_adc, else split.  Rank by exclusive scan, dest = n + rank.
 * Clone: parent unchanged, copy appended at p - clone_step * G / denom (G = grad_S planes 0-2, the
 * accumulated position gradient).  Split: both offspring at p + R(q) diag(s) z_j (z_0 = normals
 * planes 0-2, z_1 = planes 3-5, column i; caller-drawn N(0, I)), log-scale + ln(scale_factor)
 * (0.8: Sigma_j = 0.64 Sigma); A in slot i, B appended; opacity, quaternion, colour copied.
 * view_grad_stats and all 20 grad_S planes are zeroed on [0, n + n_new).  Outputs: kind [n] u8
 * (0 keep, 1 clone, 2 split), dest_index [n] i32, n_new [1] int64 and status [1] int32 device
 * scalars (3 = capacity exceeded: params untouched). */
typedef struct {
  float eps_adc;       /* mean view-space gradient-norm threshold */
  float tau_adc;       /* clone / split boundary on ||Sigma||_2 */
  float clone_step;    /* clone displacement along -G / denom */
  float scale_factor;  /* split offspring scale factor (> 0) */
  float denom;         /* accumulated steps for G (> 0) */
  int32_t reserved;
} steepgs_adc_params;
steepgs_status steepgs_adc_workspace_size(int64_t n, size_t* bytes /*[host]*/);
steepgs_status steepgs_densify_adc(float* params, int64_t ld, int64_t n, int64_t capacity, float* grad_S,
                                   int64_t ldg, float* view_grad_stats, const float* normals, int64_t ldz,
                                   const steepgs_adc_params* ap, uint8_t* kind, int32_t* dest_index,
                                   int64_t* n_new, int32_t* status, void* workspace, size_t ws_bytes,
                                   void* stream);

/* ---- Algorithm 1 optimiser step (NEXT f1; "update each Gaussian's parameters via standard
 * gradient descent", 3DGS default Adam).  One fused pass over the 14 parameter planes:
 * m = b1 m + (1-b1) g, v = b2 v + (1-b2) g^2, p -= lr_group * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps),
 * g = grad_S planes 0-13 (columns [0, n)); lr groups: mean, log-scale, quaternion, opacity logit, rgb.
 * step t >= 1 (number of optimiser steps taken, including this one; bias corrections 1 - beta^t).
 * gacc [3][ldm] or NULL: the position-gradient accumulator G of Alg. 1 (read by the compactest
 * gate): gacc = g (gacc_accumulate = 0, first step of a densification window) or gacc += g (1). */
typedef struct {              /* hyper-parameters in fp64; the kernel rounds lr, beta, 1 - beta, eps to fp32 */
  double lr[5];
  double beta1, beta2, eps;
} steepgs_adam_params;
steepgs_status steepgs_adam_step(float* params, int64_t ld, int64_t n, const float* grad_S, int64_t ldg,
                                 float* adam_m, float* adam_v, int64_t ldm, const steepgs_adam_params* ap,
                                 int64_t step, float* gacc, int32_t gacc_accumulate, void* stream);
/* After a densify: zero the Adam moments (`planes` planes of m and v: 14 for the parameter planes,
 * 3 (K - 1) for SH rest coefficients) of the replaced parents
 * (split_mask[i] == mask_value: 1 for steepgs_densify's mask, 2 for ADC splits in steepgs_densify_adc's
 * kind) and of the appended offspring [n, n + *n_split) — new Gaussians (Alg. 1, C20). */
steepgs_status steepgs_reset_moments(float* adam_m, float* adam_v, int64_t ldm, int64_t n,
                                     const uint8_t* split_mask, const int64_t* n_split, int32_t mask_value,
                                     int32_t planes, void* stream);

/* Adam over `planes` dense planes with the single learning rate ap->lr[0] (SH rest coefficients,
 * f3; 3DGS uses feature_lr / 20), same update and bias corrections as steepgs_adam_step. */
steepgs_status steepgs_adam_step_planes(float* params, int64_t ld, int32_t planes, int64_t n, const float* grad,
                                        int64_t ldg, float* adam_m, float* adam_v, int64_t ldm,
                                        const steepgs_adam_params* ap, int64_t step, void* stream);
/* After a densify: arr[:, dest_index[i]] = arr[:, i] for every parent with dest_index[i] >= 0 (extra
 * per-Gaussian planes such as SH rest coefficients follow their parent into the appended slot). */
steepgs_status steepgs_copy_offspring(float* arr, int64_t ld, int32_t planes, int64_t n, const int32_t* dest_index,
                                      void* stream);

/* Opacity pruning kept from 3DGS's density control ("prunes invisible points"; 3DGS removes
 * Gaussians with opacity < 0.005 at each densification).  keep iff params[10][i] (the opacity logit)
 * >= logit_min (compared in logit space: an exact decision); new_index [n] i32 = rank among the kept
 * (index order) or -1; n_keep [1] int64 device scalar.  workspace >= steepgs_prune_workspace_size(n). */
steepgs_status steepgs_prune_workspace_size(int64_t n, size_t* bytes /*[host]*/);
steepgs_status steepgs_prune_decide(const float* params, int64_t ld, int64_t n, float logit_min, int32_t* new_index,
                                    int64_t* n_keep, void* workspace, size_t ws_bytes, void* stream);
/* dst[k][new_index[i]] = src[k][i] for k < planes and every kept i (new_index >= 0); out of place
 * (src != dst), so the kept columns keep their order. */
steepgs_status steepgs_compact_planes(const float* src, int64_t ld_src, float* dst, int64_t ld_dst, int32_t planes,
                                      int64_t n, const int32_t* new_index, void* stream);

/* Copy planes [first, first + count) of a planar [*][ld] fp32 array, columns [0, n), device to
 * device (one vectorised copy kernel).  Used to checkpoint / restore Gaussian sets. */
steepgs_status steepgs_copy_planes(float* dst, int64_t ld_dst, const float* src, int64_t ld_src, int64_t n,
                                   int32_t first, int32_t count, void* stream);

const char* steepgs_status_string(steepgs_status s);
const char* steepgs_last_error(void);
/* Number of kernels this library has launched in this process (all threads). */
uint64_t steepgs_launch_count(void);
/* Library version / build string. */
const char* steepgs_version(void);

/* ---- a7 fused with a6 (SURVEY §8(e) B200-native variant of the allreduce of grads + S): the
 * columns [0, n) are split into R owner ranges of `chunk` columns (rank q owns [q chunk, q chunk +
 * chunk) ∩ [0, n); chunk = steepgs_scatter_chunk(n, R), a multiple of 32).
 * steepgs_gauss_bwd_scatter is steepgs_gauss_bwd_split whose per-Gaussian result (20 planes, as
 * accumulate = 0 would write them) goes straight to the owner: rank `rank` stores the columns of
 * range q into peer_partials[q] + (rank * 20 + plane) * chunk (each peer buffer [R][20][chunk] fp32;
 * device pointers valid on this device — peer / P2P-mapped memory of the other ranks, e.g. torch
 * symmetric memory; [host] array of R pointers).  No SH colour, no view_grad_stats on this path.
 * Then, after a cross-rank barrier (the caller's), steepgs_reduce_bcast on rank q sums the R partials
 * of its range in rank order, applies `accumulate` (0, 1 or 2 as in steepgs_gauss_bwd_split, against
 * its own grad_S, which equals every rank's) and stores the result into every rank's grad_S
 * (peer_grad_S [host][R] device pointers, planar [20][ldg]); a second barrier ends the exchange.
 * Together they replace the allreduce: the reduce-scatter is fused into the compute kernel and the
 * all-gather into the reduction.  R <= 8. */
steepgs_status steepgs_scatter_chunk(int64_t n, int32_t R, int64_t* chunk /*[host]*/);
steepgs_status steepgs_gauss_bwd_scatter(const float* params, int64_t ld, int64_t n, const steepgs_camera* cams,
                                         int32_t V, const steepgs_raster_params* rp, float* moments_ws,
                                         const uint64_t* peer_partials /*[host][R]*/, int32_t R, int32_t rank,
                                         int64_t chunk, void* stream);
steepgs_status steepgs_reduce_bcast(const float* partials, int32_t R, int32_t rank, int64_t n, int64_t chunk,
                                    const uint64_t* peer_grad_S /*[host][R]*/, int64_t ldg, int32_t accumulate,
                                    void* stream);

/* Debugging: the device-side invariant checks of the checked build (libsteepgs_checked.so, built with
 * -DSTEEPGS_CHECKS): ring-stage identity under the mbarrier protocol of the raster kernels, list / row
 * / instance-id bounds, radix scatter bounds, densify offspring slots.  *compiled = 0 in the release
 * build (nothing is checked there); otherwise *failures = failed checks since the last reset and
 * *first_line = the source line of the first (0 if none).  reset != 0 zeroes the counters after reading. */
steepgs_status steepgs_debug_checks(int32_t* compiled /*[host]*/, uint64_t* failures /*[host]*/,
                                    uint32_t* first_line /*[host]*/, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* STEEPGS_H */
