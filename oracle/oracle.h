/* oracle.h — SteepGS CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load liboracle.so.  The product (paper_2505_05587_b200/, include/steepgs.h) never includes,
 * links or calls anything here, and this file includes nothing from the product.
 *
 * A plain, slow, fp64 implementation of what the hot path computes, written from the paper
 * (/root/reference/PAPER.md, cited "P:L<line>") and the readings in DESIGN.md §3:
 *   - projection  Eq. eqn:sigma_2D + footnote fn:Pi, quaternion+scale
 *   - compositing Eq. eqn:alpha_blend, per pixel, all candidates, depth order
 *   - backward    Lemma lem:derivatives_orig first line: explicit per-pair chain rule
 *   - splitting matrix per pair: S += dl/dsigma * Hessian (Thm 1; Alg. 1) with the
 *                 closed-form Hessian sigma*(U U^T - P^T Pi(Sigma)^-1 P) (App. C.4)
 *   - eigen       cyclic Jacobi (textbook; deliberately NOT the trigonometric formula of P:L588-604)
 *   - densify     Thm 2, Alg. 1 densify branch
 *
 * Integer decisions that floating point takes (visibility/cull, depth order key, tile rect) are
 * taken in fp32 with the canonical operation order of DESIGN.md §3.2 ("same precision as the
 * kernel"), implemented here independently of the CUDA code.  All values are fp64.
 *
 * Parameter planes [14][ld]: 0-2 mean, 3-5 log-scale, 6-9 quat (w,x,y,z), 10 opacity logit,
 * 11-13 rgb.  Accumulator planes [20][ld]: 0-13 dL/dparam (same order), 14-19 S (xx,xy,xz,yy,yz,zz).
 */
#ifndef STEEPGS_ORACLE_H
#define STEEPGS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double R[9], t[3];          /* world -> camera, row-major; values are exact fp32 numbers */
  double fx, fy, cx, cy;
  int32_t width, height, model; /* model 0 = pinhole (EWA local affine), 1 = affine (exact Eq. 3) */
  double znear, guard;
} orc_camera;

typedef struct {
  double alpha_min, alpha_max, t_min, dilation;
  double bg[3];
  int32_t tile;
} orc_raster;

typedef struct {               /* merged-slot split of one Gaussian, for theorem pins */
  int64_t index;
  int32_t m;
  double w[4];
  double delta[4][3];          /* position offsets of the offspring */
} orc_split;

/* View-dependent SH colour (NEXT f3): the DC coefficients are parameter planes 11-13, the
 * rest [3 ((degree + 1)^2 - 1)][ld] planes, plane 3 (k - 1) + ch = coefficient k of channel ch. */
typedef struct {
  const double* rest;
  int64_t ld;
  int32_t degree;              /* 0..3 */
} orc_sh;
/* Real SH basis (3DGS ordering / constants) at unit direction dir: Y[16] (zero above the degree),
 * dY[16][3] (optional) = partial derivatives of the basis polynomials. */
void orc_sh_basis(const double* dir, int32_t degree, double* Y, double* dY);

/* fp32 decision chain: visibility, depth key, pixel rect [n][4] = jmin,jmax,
 * kmin,kmax (inclusive, -1 if culled), tiles_touched.  Returns number visible. */
int64_t orc_decide_f32(const double* params, int64_t ld, int64_t n, const orc_camera* cam,
                       const orc_raster* rp, uint8_t* visible, uint32_t* depth_key,
                       int32_t* rect_px, int32_t* tiles_touched);

/* fp64 projected quantities (all Gaussians, whether visible or not):
 * mu [n][2], cov2d [n][3] (xx,xy,yy incl. dilation), conic [n][3], opacity [n], depth [n]. */
void orc_project_f64(const double* params, int64_t ld, int64_t n, const orc_camera* cam,
                     const orc_raster* rp, double* mu, double* cov2d, double* conic,
                     double* opacity, double* depth);

/* sigma_Pi(x; theta_i) of Eq. eqn:sigma_2D at pixel-plane point (x, y), fp64. */
double orc_eval_sigma(const double* params, int64_t ld, int64_t i, const orc_camera* cam,
                      const orc_raster* rp, double x, double y);
/* Closed-form position Hessian of sigma (App. C.4, P is frozen), H row-major [9]. */
void orc_position_hessian(const double* params, int64_t ld, int64_t i, const orc_camera* cam,
                          const orc_raster* rp, double x, double y, double* H);

/* Render one view over the pixel window [x0,x0+w) x [y0,y0+h) (Eq. eqn:alpha_blend), and when
 * dL_dimage != NULL the backward pass: grad[20][ld] += dL/dparam and S, absg[20][ld] += |per-pair
 * contributions|, amb_g[n] |= 1 for Gaussians in an ambiguous pixel's candidate list.
 * brute_force = 1: candidates = every visible Gaussian; 0: per-Gaussian fp64 AABB scatter.
 * amb_px[h][w] = 1 where some candidate sits within a rounding band of a threshold
 * (DESIGN.md §3.4).  split != NULL renders the merged-slot model (fwd only).  grad_mu (optional,
 * [2][ld]) += dL/dPi(p) of this view, the 2D-mean gradient ADC thresholds.  sh != NULL:
 * colours from spherical harmonics (f3); grad_sh [3 (K - 1)][ld] += the rest-coefficient gradients,
 * grad planes 11-13 get the DC-coefficient gradients and planes 0-2 include the view-direction term.
 * Returns the number of composited pairs, or -1 on allocation failure. */
int64_t orc_render_view(const double* params, int64_t ld, int64_t n, const orc_camera* cam,
                        const orc_raster* rp, const uint8_t* visible, const uint32_t* depth_key,
                        int32_t x0, int32_t y0, int32_t w, int32_t h, int32_t brute_force,
                        const orc_split* split, const double* dL_dimage,
                        double* image, double* final_T, int32_t* n_comp, uint8_t* amb_px,
                        double* grad, double* absg, uint8_t* amb_g, double* grad_mu,
                        const orc_sh* sh, double* grad_sh);

/* Symmetric 3x3 eigen-decomposition by cyclic Jacobi.  A = (xx,xy,xz,yy,yz,zz).
 * lam ascending; V columns are unit eigenvectors (V[3*r + c] = component r of vector c), each
 * with canonical sign (largest-|.| component positive, ties -> lowest index).  Degenerate
 * (p < 1e-12 (1+|q|)): lam = q, V = I.  Returns the number of sweeps. */
int orc_eig_sym3(const double* A, double* lam, double* V);

/* SDC densify (Thm 2, Alg. 1) on fp64 planes, in place.  Variants of App. A.2:
 * gate = 1 also requires ||acc[0..2] / denom||_2 <= eps_grad (compactest); gate = 2
 * requires acc[0] / acc[1] >= eps_grad (Alg. 1's "condition on G" read as 3DGS's mean view-space
 * gradient-norm threshold, acc[0] = sum of norms, acc[1] = visible views; C24); budget >= 0
 * keeps at most `budget` splits, those with the least lambda_min, ties by index.
 * S planes are read from
 * acc[14..19][ld].  Offspring A in slot i (p + eps v), B in slot n + rank (p - eps v), both with
 * opacity o/2 (stored as logit), eps = eta sqrt(v^T Sigma v) (eta >= 0) or eps_abs.  S planes are
 * zeroed for [0, n').  mask[n], dest[n] (-1 if kept), lambda[n] (may be NULL).
 * Returns n_split, or -1 if n + n_split > capacity (then nothing but mask/dest/lambda written). */
int64_t orc_densify(double* params, int64_t ld, int64_t n, int64_t capacity, double* acc,
                    int64_t ldg, double denom, double eps_split, double eta, double eps_abs,
                    int32_t gate, double eps_grad, int64_t budget,
                    uint8_t* mask, int32_t* dest, double* lambda);

int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
