/* oracle.c — SteepGS CPU ORACLE.  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain, slow, fp64.  Each function cites the PAPER.md passage (P:L<line>) it follows; readings
 * of silent/ambiguous points are DESIGN.md §3 ("Z<k>").  Compile with -ffp-contract=off so the
 * fp32 decision chain (orc_decide_f32) evaluates exactly the operations written.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define AMB_BAND 1e-4 /* relative rounding band for threshold ambiguity */

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

static inline double sigmoid(double l) { return 1.0 / (1.0 + exp(-l)); }

/* ------------------------------------------------------------------------------------------
 * 1. fp32 decision chain — DESIGN.md §3.2.  Visibility (cull set, Z4), depth-order key (Z6),
 *    pixel rect of the opacity-aware alpha support (Z4).  Every line is one IEEE fp32 operation
 *    in the order written; exp/log are evaluated in double and rounded once to fp32.
 * ------------------------------------------------------------------------------------------ */
static uint32_t orderable_key(float z) {
  uint32_t u;
  memcpy(&u, &z, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

int64_t orc_decide_f32(const double* params, int64_t ld, int64_t n, const orc_camera* cam,
                       const orc_raster* rp, uint8_t* visible, uint32_t* depth_key,
                       int32_t* rect_px, int32_t* tiles_touched) {
  float Rc[9], tc[3];
  for (int k = 0; k < 9; ++k) Rc[k] = (float)cam->R[k];
  for (int k = 0; k < 3; ++k) tc[k] = (float)cam->t[k];
  const float fx = (float)cam->fx, fy = (float)cam->fy, cx = (float)cam->cx, cy = (float)cam->cy;
  const float znear = (float)cam->znear, guard = (float)cam->guard;
  const float dil = (float)rp->dilation, amin = (float)rp->alpha_min;
  const int W = cam->width, H = cam->height, T = rp->tile;
  int64_t nvis = 0;
  for (int64_t i = 0; i < n; ++i) {
    visible[i] = 0;
    depth_key[i] = 0;
    rect_px[4 * i + 0] = rect_px[4 * i + 1] = rect_px[4 * i + 2] = rect_px[4 * i + 3] = -1;
    tiles_touched[i] = 0;
    const float p0 = (float)params[0 * ld + i], p1 = (float)params[1 * ld + i], p2 = (float)params[2 * ld + i];
    /* camera-space mean t = R p + t (P:L135-139 footnote: Pi(x) = P x + b) */
    float tx = Rc[0] * p0; tx = tx + Rc[1] * p1; tx = tx + Rc[2] * p2; tx = tx + tc[0];
    float ty = Rc[3] * p0; ty = ty + Rc[4] * p1; ty = ty + Rc[5] * p2; ty = ty + tc[1];
    float tz = Rc[6] * p0; tz = tz + Rc[7] * p1; tz = tz + Rc[8] * p2; tz = tz + tc[2];
    float mux, muy, J00, J02, J11, J12;
    if (cam->model == 0) {
      if (!(tz > znear)) continue;
      const float xz = tx / tz, yz = ty / tz;
      const float limx = guard * ((0.5f * (float)W) / fx);
      const float limy = guard * ((0.5f * (float)H) / fy);
      if (!(fabsf(xz) <= limx) || !(fabsf(yz) <= limy)) continue;
      mux = fx * xz; mux = mux + cx;
      muy = fy * yz; muy = muy + cy;
      J00 = fx / tz; J02 = -((fx * xz) / tz);
      J11 = fy / tz; J12 = -((fy * yz) / tz);
    } else {
      mux = fx * tx; mux = mux + cx;
      muy = fy * ty; muy = muy + cy;
      J00 = fx; J02 = 0.0f; J11 = fy; J12 = 0.0f;
    }
    float P[6];
    for (int b = 0; b < 3; ++b) {
      float a0 = J00 * Rc[0 + b]; a0 = a0 + J02 * Rc[6 + b]; P[b] = a0;
      float a1 = J11 * Rc[3 + b]; a1 = a1 + J12 * Rc[6 + b]; P[3 + b] = a1;
    }
    /* covariance from quaternion + scale */
    const float qw = (float)params[6 * ld + i], qx = (float)params[7 * ld + i];
    const float qy = (float)params[8 * ld + i], qz = (float)params[9 * ld + i];
    float nq2 = qw * qw; nq2 = nq2 + qx * qx; nq2 = nq2 + qy * qy; nq2 = nq2 + qz * qz;
    if (!(nq2 > 0.0f)) continue;
    const float nq = sqrtf(nq2);
    const float w = qw / nq, x = qx / nq, y = qy / nq, z = qz / nq;
    float r[9];
    r[0] = 1.0f - 2.0f * (y * y + z * z);
    r[1] = 2.0f * (x * y - w * z);
    r[2] = 2.0f * (x * z + w * y);
    r[3] = 2.0f * (x * y + w * z);
    r[4] = 1.0f - 2.0f * (x * x + z * z);
    r[5] = 2.0f * (y * z - w * x);
    r[6] = 2.0f * (x * z - w * y);
    r[7] = 2.0f * (y * z + w * x);
    r[8] = 1.0f - 2.0f * (x * x + y * y);
    float s[3];
    for (int k = 0; k < 3; ++k) s[k] = (float)exp((double)(float)params[(3 + k) * ld + i]);
    float M[9];
    for (int a = 0; a < 3; ++a)
      for (int k = 0; k < 3; ++k) M[3 * a + k] = r[3 * a + k] * s[k];
    float Sg[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        float acc = M[3 * a + 0] * M[3 * b + 0];
        acc = acc + M[3 * a + 1] * M[3 * b + 1];
        acc = acc + M[3 * a + 2] * M[3 * b + 2];
        Sg[3 * a + b] = acc;
      }
    float Tm[6];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) {
        float acc = P[3 * a + 0] * Sg[0 + b];
        acc = acc + P[3 * a + 1] * Sg[3 + b];
        acc = acc + P[3 * a + 2] * Sg[6 + b];
        Tm[3 * a + b] = acc;
      }
    float A = Tm[0] * P[0]; A = A + Tm[1] * P[1]; A = A + Tm[2] * P[2]; A = A + dil;
    float B = Tm[0] * P[3]; B = B + Tm[1] * P[4]; B = B + Tm[2] * P[5];
    float C = Tm[3] * P[3]; C = C + Tm[4] * P[4]; C = C + Tm[5] * P[5]; C = C + dil;
    const float det = A * C - B * B;
    if (!(det > 0.0f)) continue;
    const float o = (float)(1.0 / (1.0 + exp(-(double)(float)params[10 * ld + i])));
    if (!(o > amin)) continue;
    const float tau = (float)(2.0 * log((double)o / (double)amin));
    const float ex = sqrtf(tau * A), ey = sqrtf(tau * C);
    float lox = mux - ex; lox = lox - 0.5f; lox = lox - 1e-3f;
    float hix = mux + ex; hix = hix - 0.5f; hix = hix + 1e-3f;
    float loy = muy - ey; loy = loy - 0.5f; loy = loy - 1e-3f;
    float hiy = muy + ey; hiy = hiy - 0.5f; hiy = hiy + 1e-3f;
    if (lox != lox || hix != hix || loy != loy || hiy != hiy) continue;
    const float jmin = fmaxf(ceilf(lox), 0.0f), jmax = fminf(floorf(hix), (float)(W - 1));
    const float kmin = fmaxf(ceilf(loy), 0.0f), kmax = fminf(floorf(hiy), (float)(H - 1));
    if (!(jmin <= jmax) || !(kmin <= kmax)) continue;
    const int j0 = (int)jmin, j1 = (int)jmax, k0 = (int)kmin, k1 = (int)kmax;
    visible[i] = 1;
    depth_key[i] = orderable_key(tz);
    rect_px[4 * i + 0] = j0; rect_px[4 * i + 1] = j1;
    rect_px[4 * i + 2] = k0; rect_px[4 * i + 3] = k1;
    tiles_touched[i] = (j1 / T - j0 / T + 1) * (k1 / T - k0 / T + 1);
    ++nvis;
  }
  return nvis;
}

/* ------------------------------------------------------------------------------------------
 * 2. fp64 projection with explicit forward-mode Jacobians (for the per-pair chain rule).
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  double mu[2], cov[3], conic[3], o, z, tau;
  double P[6];              /* 2x3, P = J W (P:L139 footnote) */
  double col[3];
  int sh_k;                 /* 0: colour = rgb planes; else (degree + 1)^2 SH coefficients per channel */
  double Y[16];             /* SH basis at the view direction */
  double cmask[3];          /* 1 where the colour is not clamped at 0 */
  double dcol_dp[3][3];     /* d colour_ch / d p_k through the view direction */
  double dcov[10][3];       /* d(cov xx, xy, yy)/d theta_k; k = p0..2, ls0..2, q0..3 */
  double dmu[2][3];         /* d mu / d p */
} gproj;

static void mat3_mul(const double* A, const double* B, double* C) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += A[3 * i + k] * B[3 * k + j];
      C[3 * i + j] = s;
    }
}

static void rot_from_quat(const double* q, double* R) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}

/* dR/dq_hat_c for the unit-quaternion rotation above. */
static void drot_dquat(const double* q, int c, double* D) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  switch (c) {
    case 0: { double d[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0}; memcpy(D, d, sizeof d); } break;
    case 1: { double d[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x}; memcpy(D, d, sizeof d); } break;
    case 2: { double d[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y}; memcpy(D, d, sizeof d); } break;
    default: { double d[9] = {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0}; memcpy(D, d, sizeof d); } break;
  }
}

/* cov2 = P A P^T restricted to (xx, xy, yy) */
static void sandwich2(const double* P, const double* A, double* out) {
  double T[6];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += P[3 * a + k] * A[3 * k + b];
      T[3 * a + b] = s;
    }
  double c[4];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += T[3 * a + k] * P[3 * b + k];
      c[2 * a + b] = s;
    }
  out[0] = c[0]; out[1] = 0.5 * (c[1] + c[2]); out[2] = c[3];
}

/* View-dependent colour (NEXT f3): real spherical harmonics of degree <= 3 in the 3DGS
 * ordering and constants, colour = max(0, sum_k Y_k(dir) f_k + 1/2).  Y[k] and the partial
 * derivatives dY[k][j] = dY_k / d dir_j of the polynomials (x, y, z = dir). */
static const double SH_C0 = 0.28209479177387814, SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

static void sh_basis(const double* v, int deg, double* Y, double (*dY)[3]) {
  const double x = v[0], y = v[1], z = v[2];
  for (int k = 0; k < 16; ++k) { Y[k] = 0; dY[k][0] = dY[k][1] = dY[k][2] = 0; }
  Y[0] = SH_C0;
  if (deg < 1) return;
  Y[1] = -SH_C1 * y; dY[1][1] = -SH_C1;
  Y[2] = SH_C1 * z;  dY[2][2] = SH_C1;
  Y[3] = -SH_C1 * x; dY[3][0] = -SH_C1;
  if (deg < 2) return;
  Y[4] = SH_C2[0] * x * y;                   dY[4][0] = SH_C2[0] * y; dY[4][1] = SH_C2[0] * x;
  Y[5] = SH_C2[1] * y * z;                   dY[5][1] = SH_C2[1] * z; dY[5][2] = SH_C2[1] * y;
  Y[6] = SH_C2[2] * (2 * z * z - x * x - y * y);
  dY[6][0] = -2 * SH_C2[2] * x; dY[6][1] = -2 * SH_C2[2] * y; dY[6][2] = 4 * SH_C2[2] * z;
  Y[7] = SH_C2[3] * x * z;                   dY[7][0] = SH_C2[3] * z; dY[7][2] = SH_C2[3] * x;
  Y[8] = SH_C2[4] * (x * x - y * y);         dY[8][0] = 2 * SH_C2[4] * x; dY[8][1] = -2 * SH_C2[4] * y;
  if (deg < 3) return;
  Y[9] = SH_C3[0] * y * (3 * x * x - y * y);
  dY[9][0] = 6 * SH_C3[0] * x * y; dY[9][1] = SH_C3[0] * (3 * x * x - 3 * y * y);
  Y[10] = SH_C3[1] * x * y * z;
  dY[10][0] = SH_C3[1] * y * z; dY[10][1] = SH_C3[1] * x * z; dY[10][2] = SH_C3[1] * x * y;
  Y[11] = SH_C3[2] * y * (4 * z * z - x * x - y * y);
  dY[11][0] = -2 * SH_C3[2] * x * y; dY[11][1] = SH_C3[2] * (4 * z * z - x * x - 3 * y * y);
  dY[11][2] = 8 * SH_C3[2] * y * z;
  Y[12] = SH_C3[3] * z * (2 * z * z - 3 * x * x - 3 * y * y);
  dY[12][0] = -6 * SH_C3[3] * x * z; dY[12][1] = -6 * SH_C3[3] * y * z;
  dY[12][2] = SH_C3[3] * (6 * z * z - 3 * x * x - 3 * y * y);
  Y[13] = SH_C3[4] * x * (4 * z * z - x * x - y * y);
  dY[13][0] = SH_C3[4] * (4 * z * z - 3 * x * x - y * y); dY[13][1] = -2 * SH_C3[4] * x * y;
  dY[13][2] = 8 * SH_C3[4] * x * z;
  Y[14] = SH_C3[5] * z * (x * x - y * y);
  dY[14][0] = 2 * SH_C3[5] * x * z; dY[14][1] = -2 * SH_C3[5] * y * z; dY[14][2] = SH_C3[5] * (x * x - y * y);
  Y[15] = SH_C3[6] * x * (x * x - 3 * y * y);
  dY[15][0] = SH_C3[6] * (3 * x * x - 3 * y * y); dY[15][1] = -6 * SH_C3[6] * x * y;
}

void orc_sh_basis(const double* dir, int32_t degree, double* Y, double* dY) {
  double d[16][3];
  sh_basis(dir, degree, Y, d);
  if (dY) for (int k = 0; k < 16; ++k) for (int j = 0; j < 3; ++j) dY[3 * k + j] = d[k][j];
}

/* colour of Gaussian i seen from `cam` (C1 / f3): view direction dir = (p - o)/|p - o| with the
 * camera centre o = -R^T t (pinhole) or the camera axis R^T e_z (affine, no dependence on p). */
static void sh_colour(const double* params, int64_t ld, int64_t i, const orc_sh* sh, const orc_camera* cam,
                      const double* p, gproj* g, int want_jac) {
  const double* W = cam->R;
  double dir[3], r = 1.0;
  if (cam->model == 0) {
    double v[3];
    for (int k = 0; k < 3; ++k) {
      const double o = -(W[k] * cam->t[0] + W[3 + k] * cam->t[1] + W[6 + k] * cam->t[2]);
      v[k] = p[k] - o;
    }
    r = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int k = 0; k < 3; ++k) dir[k] = v[k] / r;
  } else {
    for (int k = 0; k < 3; ++k) dir[k] = W[6 + k];
  }
  double dY[16][3];
  sh_basis(dir, sh->degree, g->Y, dY);
  g->sh_k = (sh->degree + 1) * (sh->degree + 1);
  double f[16][3];
  for (int ch = 0; ch < 3; ++ch) f[0][ch] = params[(11 + ch) * ld + i];
  for (int k = 1; k < g->sh_k; ++k)
    for (int ch = 0; ch < 3; ++ch) f[k][ch] = sh->rest[(int64_t)(3 * (k - 1) + ch) * sh->ld + i];
  for (int ch = 0; ch < 3; ++ch) {
    double raw = 0.5;
    for (int k = 0; k < g->sh_k; ++k) raw += g->Y[k] * f[k][ch];
    g->col[ch] = raw > 0 ? raw : 0.0;
    g->cmask[ch] = raw > 0 ? 1.0 : 0.0;
  }
  for (int ch = 0; ch < 3; ++ch)
    for (int m = 0; m < 3; ++m) g->dcol_dp[ch][m] = 0.0;
  if (!want_jac || cam->model != 0) return;
  /* d dir / d p = (I - dir dir^T) / r */
  for (int ch = 0; ch < 3; ++ch) {
    double gd[3] = {0, 0, 0};   /* d raw_ch / d dir */
    for (int k = 1; k < g->sh_k; ++k)
      for (int j = 0; j < 3; ++j) gd[j] += f[k][ch] * dY[k][j];
    const double dot = gd[0] * dir[0] + gd[1] * dir[1] + gd[2] * dir[2];
    for (int m = 0; m < 3; ++m) g->dcol_dp[ch][m] = g->cmask[ch] * (gd[m] - dot * dir[m]) / r;
  }
}

/* Projection of Gaussian i with mean overridden by `pm` (NULL = own mean). */
static void project_one(const double* params, int64_t ld, int64_t i, const orc_camera* cam,
                        const orc_raster* rp, const double* pm, gproj* g, int want_jac, const orc_sh* sh) {
  const double* W = cam->R;
  double p[3];
  for (int k = 0; k < 3; ++k) p[k] = pm ? pm[k] : params[k * ld + i];
  double t[3];
  for (int a = 0; a < 3; ++a) t[a] = W[3 * a] * p[0] + W[3 * a + 1] * p[1] + W[3 * a + 2] * p[2] + cam->t[a];
  const double fx = cam->fx, fy = cam->fy;
  double J[6] = {0, 0, 0, 0, 0, 0};
  if (cam->model == 0) {
    const double z = t[2];
    g->mu[0] = fx * t[0] / z + cam->cx;
    g->mu[1] = fy * t[1] / z + cam->cy;
    J[0] = fx / z; J[2] = -fx * t[0] / (z * z);
    J[4] = fy / z; J[5] = -fy * t[1] / (z * z);
  } else {
    g->mu[0] = fx * t[0] + cam->cx;
    g->mu[1] = fy * t[1] + cam->cy;
    J[0] = fx; J[4] = fy;
  }
  g->z = t[2];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += J[3 * a + k] * W[3 * k + b];
      g->P[3 * a + b] = s;
    }
  double q[4];
  for (int k = 0; k < 4; ++k) q[k] = params[(6 + k) * ld + i];
  const double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  double qh[4];
  for (int k = 0; k < 4; ++k) qh[k] = q[k] / qn;
  double R[9];
  rot_from_quat(qh, R);
  double s2[3];
  for (int k = 0; k < 3; ++k) { const double s = exp(params[(3 + k) * ld + i]); s2[k] = s * s; }
  double Sig[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0;
      for (int k = 0; k < 3; ++k) acc += R[3 * a + k] * s2[k] * R[3 * b + k];
      Sig[3 * a + b] = acc;
    }
  sandwich2(g->P, Sig, g->cov);
  g->cov[0] += rp->dilation;
  g->cov[2] += rp->dilation;
  const double det = g->cov[0] * g->cov[2] - g->cov[1] * g->cov[1];
  g->conic[0] = g->cov[2] / det; g->conic[1] = -g->cov[1] / det; g->conic[2] = g->cov[0] / det;
  g->o = sigmoid(params[10 * ld + i]);
  g->tau = (rp->alpha_min > 0) ? 2.0 * log(g->o / rp->alpha_min) : INFINITY;
  g->sh_k = 0;
  if (sh) {
    sh_colour(params, ld, i, sh, cam, p, g, want_jac);
  } else {
    for (int k = 0; k < 3; ++k) g->col[k] = params[(11 + k) * ld + i];
  }
  if (!want_jac) return;

  /* d mu / d p = J W = P (mean path) */
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b) g->dmu[a][b] = g->P[3 * a + b];
  /* d cov / d p through J(t) (pinhole; zero for affine).  cov = J Sc J^T, Sc = W Sig W^T. */
  double Sc[9], tmp[9], Wt[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) Wt[3 * a + b] = W[3 * b + a];
  mat3_mul(W, Sig, tmp);
  mat3_mul(tmp, Wt, Sc);
  double dcov_dt[3][3];
  memset(dcov_dt, 0, sizeof dcov_dt);
  if (cam->model == 0) {
    const double z = t[2];
    for (int m = 0; m < 3; ++m) {
      double dJ[6] = {0, 0, 0, 0, 0, 0};
      if (m == 0) dJ[2] = -fx / (z * z);
      if (m == 1) dJ[5] = -fy / (z * z);
      if (m == 2) {
        dJ[0] = -fx / (z * z); dJ[2] = 2 * fx * t[0] / (z * z * z);
        dJ[4] = -fy / (z * z); dJ[5] = 2 * fy * t[1] / (z * z * z);
      }
      /* d(J Sc J^T) = dJ Sc J^T + J Sc dJ^T */
      double A1[6], c[4];
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) {
          double s = 0;
          for (int k = 0; k < 3; ++k) s += dJ[3 * a + k] * Sc[3 * k + b];
          A1[3 * a + b] = s;
        }
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
          double s = 0;
          for (int k = 0; k < 3; ++k) s += A1[3 * a + k] * J[3 * b + k];
          c[2 * a + b] = s;
        }
      dcov_dt[m][0] = 2 * c[0];
      dcov_dt[m][1] = c[1] + c[2];
      dcov_dt[m][2] = 2 * c[3];
    }
  }
  for (int k = 0; k < 3; ++k)
    for (int e = 0; e < 3; ++e)
      g->dcov[k][e] = dcov_dt[0][e] * W[0 * 3 + k] + dcov_dt[1][e] * W[1 * 3 + k] + dcov_dt[2][e] * W[2 * 3 + k];
  /* d cov / d log s_k = P (2 s_k^2 r_k r_k^T) P^T */
  for (int k = 0; k < 3; ++k) {
    double dS[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) dS[3 * a + b] = 2 * s2[k] * R[3 * a + k] * R[3 * b + k];
    sandwich2(g->P, dS, g->dcov[3 + k]);
  }
  /* d cov / d q_c:  dSig = dR S2 R^T + R S2 dR^T,  dR/dq_c = sum_d dR/dqh_d (delta_dc - qh_d qh_c)/|q| */
  for (int c = 0; c < 4; ++c) {
    double dR[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int d = 0; d < 4; ++d) {
      const double f = ((d == c ? 1.0 : 0.0) - qh[d] * qh[c]) / qn;
      double D[9];
      drot_dquat(qh, d, D);
      for (int k = 0; k < 9; ++k) dR[k] += f * D[k];
    }
    double dS[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0;
        for (int k = 0; k < 3; ++k) acc += dR[3 * a + k] * s2[k] * R[3 * b + k] + R[3 * a + k] * s2[k] * dR[3 * b + k];
        dS[3 * a + b] = acc;
      }
    sandwich2(g->P, dS, g->dcov[6 + c]);
  }
}

void orc_project_f64(const double* params, int64_t ld, int64_t n, const orc_camera* cam,
                     const orc_raster* rp, double* mu, double* cov2d, double* conic,
                     double* opacity, double* depth) {
  for (int64_t i = 0; i < n; ++i) {
    gproj g;
    project_one(params, ld, i, cam, rp, NULL, &g, 0, NULL);
    if (mu) { mu[2 * i] = g.mu[0]; mu[2 * i + 1] = g.mu[1]; }
    if (cov2d) for (int k = 0; k < 3; ++k) cov2d[3 * i + k] = g.cov[k];
    if (conic) for (int k = 0; k < 3; ++k) conic[3 * i + k] = g.conic[k];
    if (opacity) opacity[i] = g.o;
    if (depth) depth[i] = g.z;
  }
}

/* sigma_Pi(x) = o exp(-1/2 d^T Pi(Sigma)^-1 d), d = x - Pi(p)  (Eq. eqn:sigma_2D) */
static double sigma_at(const gproj* g, double x, double y, double* d) {
  d[0] = x - g->mu[0];
  d[1] = y - g->mu[1];
  const double m = g->conic[0] * d[0] * d[0] + 2 * g->conic[1] * d[0] * d[1] + g->conic[2] * d[1] * d[1];
  return g->o * exp(-0.5 * m);
}

double orc_eval_sigma(const double* params, int64_t ld, int64_t i, const orc_camera* cam,
                      const orc_raster* rp, double x, double y) {
  gproj g;
  double d[2];
  project_one(params, ld, i, cam, rp, NULL, &g, 0, NULL);
  return sigma_at(&g, x, y, d);
}

/* Hessian of sigma w.r.t. the mean, P frozen (App. C.4):
 *   H = sigma (U U^T - P^T Q P),  U = P^T Q (x - Pi(p)). */
static void hessian_pair(const gproj* g, double sigma, const double* d, double* H) {
  const double u0 = g->conic[0] * d[0] + g->conic[1] * d[1];
  const double u1 = g->conic[1] * d[0] + g->conic[2] * d[1];
  double U[3];
  for (int a = 0; a < 3; ++a) U[a] = g->P[a] * u0 + g->P[3 + a] * u1;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      /* (P^T Q P)_ab = sum_{c,e} P_ca Q_ce P_eb */
      const double PQP = g->P[a] * (g->conic[0] * g->P[b] + g->conic[1] * g->P[3 + b]) +
                         g->P[3 + a] * (g->conic[1] * g->P[b] + g->conic[2] * g->P[3 + b]);
      H[3 * a + b] = sigma * (U[a] * U[b] - PQP);
    }
}

/* Magnitudes of the two terms of each Hessian entry: sigma (|U_a U_b| + |(P^T Q P)_ab|).  Test
 * infrastructure: the GPU forms S from per-Gaussian moments, P^T (Q M Q - m0 Q) P (C12), so its fp32
 * error scales with these magnitudes summed over the pairs, not with |H_ab|. */
static void hessian_terms_abs(const gproj* g, double sigma, const double* d, double* Hm) {
  const double u0 = g->conic[0] * d[0] + g->conic[1] * d[1];
  const double u1 = g->conic[1] * d[0] + g->conic[2] * d[1];
  double U[3];
  for (int a = 0; a < 3; ++a) U[a] = g->P[a] * u0 + g->P[3 + a] * u1;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      const double PQP = g->P[a] * (g->conic[0] * g->P[b] + g->conic[1] * g->P[3 + b]) +
                         g->P[3 + a] * (g->conic[1] * g->P[b] + g->conic[2] * g->P[3 + b]);
      Hm[3 * a + b] = sigma * (fabs(U[a] * U[b]) + fabs(PQP));
    }
}

void orc_position_hessian(const double* params, int64_t ld, int64_t i, const orc_camera* cam,
                          const orc_raster* rp, double x, double y, double* H) {
  gproj g;
  double d[2];
  project_one(params, ld, i, cam, rp, NULL, &g, 0, NULL);
  const double sigma = sigma_at(&g, x, y, d);
  hessian_pair(&g, sigma, d, H);
}

/* ------------------------------------------------------------------------------------------
 * 3. Per-pixel compositing (Eq. eqn:alpha_blend) and its backward,
 *    with S accumulated per pair (Thm 1, Alg. 1, Hessian P:L356).
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  int64_t gid;       /* global Gaussian index */
  uint32_t key;
  gproj g;
  double bb[4];      /* fp64 AABB of the alpha support in pixel-centre coordinates */
} cand_t;

static int cmp_cand(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->gid < y->gid ? -1 : (x->gid > y->gid ? 1 : 0);
}

typedef struct {
  int32_t c;        /* candidate (local) index */
  double sigma, alpha, T, d[2];
} rec_t;

static double slot_sigma(const cand_t* cd, const orc_split* split, const double* params, int64_t ld,
                         const orc_camera* cam, const orc_raster* rp, gproj* off, double x, double y,
                         double* d) {
  if (split && cd->gid == split->index) {
    double s = 0, dd[2];
    for (int j = 0; j < split->m; ++j) s += split->w[j] * sigma_at(&off[j], x, y, dd);
    d[0] = x - cd->g.mu[0];
    d[1] = y - cd->g.mu[1];
    return s;
  }
  (void)params; (void)ld; (void)cam; (void)rp;
  return sigma_at(&cd->g, x, y, d);
}

#define ACCW 48

int64_t orc_render_view(const double* params, int64_t ld, int64_t n, const orc_camera* cam,
                        const orc_raster* rp, const uint8_t* visible, const uint32_t* depth_key,
                        int32_t x0, int32_t y0, int32_t w, int32_t h, int32_t brute_force,
                        const orc_split* split, const double* dL_dimage,
                        double* image, double* final_T, int32_t* n_comp, uint8_t* amb_px,
                        double* grad, double* absg, uint8_t* amb_g, double* grad_mu,
                        const orc_sh* sh, double* grad_sh) {
  const int want_bwd = dL_dimage != NULL;
  /* Candidates: visible Gaussians (fp32 decision) whose alpha support can reach the window. */
  int64_t ncand = 0, cap = 1024;
  cand_t* cand = (cand_t*)malloc(sizeof(cand_t) * (size_t)cap);
  if (!cand) return -1;
  gproj off[4];
  if (split) {
    for (int j = 0; j < split->m; ++j) {
      double pm[3];
      for (int k = 0; k < 3; ++k) pm[k] = params[k * ld + split->index] + split->delta[j][k];
      project_one(params, ld, split->index, cam, rp, pm, &off[j], 0, sh);
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    if (!visible[i]) continue;
    if (ncand == cap) {
      cap *= 2;
      cand_t* nc = (cand_t*)realloc(cand, sizeof(cand_t) * (size_t)cap);
      if (!nc) { free(cand); return -1; }
      cand = nc;
    }
    cand_t* c = &cand[ncand];
    c->gid = i;
    c->key = depth_key[i];
    project_one(params, ld, i, cam, rp, NULL, &c->g, want_bwd, sh);
    /* exact AABB of {d : d^T Q d <= tau} is |d_x| <= sqrt(tau cov_xx) (plus 1e-6 px) */
    const double ex = sqrt(c->g.tau * c->g.cov[0]) + 1e-6, ey = sqrt(c->g.tau * c->g.cov[2]) + 1e-6;
    c->bb[0] = c->g.mu[0] - ex; c->bb[1] = c->g.mu[0] + ex;
    c->bb[2] = c->g.mu[1] - ey; c->bb[3] = c->g.mu[1] + ey;
    if (split && i == split->index) { /* merged slot: union of the offspring supports */
      c->bb[0] = -INFINITY; c->bb[1] = INFINITY; c->bb[2] = -INFINITY; c->bb[3] = INFINITY;
    }
    if (!brute_force && (c->bb[1] < x0 + 0.5 || c->bb[0] > x0 + w - 0.5 || c->bb[3] < y0 + 0.5 ||
                         c->bb[2] > y0 + h - 0.5))
      continue;
    ++ncand;
  }
  /* depth order: ascending (fp32 depth key, index) — P:L129, Z6 */
  qsort(cand, (size_t)ncand, sizeof(cand_t), cmp_cand);

  /* per-pixel candidate lists (in depth order) */
  const int64_t npx = (int64_t)w * h;
  int64_t* start = (int64_t*)calloc((size_t)npx + 1, sizeof(int64_t));
  int32_t* list = NULL;
  if (!start) { free(cand); return -1; }
  if (!brute_force) {
    for (int64_t c = 0; c < ncand; ++c) {
      const cand_t* cd = &cand[c];
      int ja = (int)ceil(cd->bb[0] - 0.5), jb = (int)floor(cd->bb[1] - 0.5);
      int ka = (int)ceil(cd->bb[2] - 0.5), kb = (int)floor(cd->bb[3] - 0.5);
      if (!isfinite(cd->bb[0])) ja = x0;
      if (!isfinite(cd->bb[1])) jb = x0 + w - 1;
      if (!isfinite(cd->bb[2])) ka = y0;
      if (!isfinite(cd->bb[3])) kb = y0 + h - 1;
      if (ja < x0) ja = x0;
      if (jb > x0 + w - 1) jb = x0 + w - 1;
      if (ka < y0) ka = y0;
      if (kb > y0 + h - 1) kb = y0 + h - 1;
      for (int k = ka; k <= kb; ++k)
        for (int j = ja; j <= jb; ++j) start[(int64_t)(k - y0) * w + (j - x0) + 1]++;
    }
    for (int64_t p = 0; p < npx; ++p) start[p + 1] += start[p];
    list = (int32_t*)malloc(sizeof(int32_t) * (size_t)(start[npx] > 0 ? start[npx] : 1));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(npx > 0 ? npx : 1));
    if (!list || !fill) { free(cand); free(start); free(list); free(fill); return -1; }
    memcpy(fill, start, sizeof(int64_t) * (size_t)npx);
    for (int64_t c = 0; c < ncand; ++c) {
      const cand_t* cd = &cand[c];
      int ja = (int)ceil(cd->bb[0] - 0.5), jb = (int)floor(cd->bb[1] - 0.5);
      int ka = (int)ceil(cd->bb[2] - 0.5), kb = (int)floor(cd->bb[3] - 0.5);
      if (!isfinite(cd->bb[0])) ja = x0;
      if (!isfinite(cd->bb[1])) jb = x0 + w - 1;
      if (!isfinite(cd->bb[2])) ka = y0;
      if (!isfinite(cd->bb[3])) kb = y0 + h - 1;
      if (ja < x0) ja = x0;
      if (jb > x0 + w - 1) jb = x0 + w - 1;
      if (ka < y0) ka = y0;
      if (kb > y0 + h - 1) kb = y0 + h - 1;
      for (int k = ka; k <= kb; ++k)
        for (int j = ja; j <= jb; ++j) list[fill[(int64_t)(k - y0) * w + (j - x0)]++] = (int32_t)c;
    }
    free(fill);
  }

  const int nthr = orc_num_threads();
  double* tacc = NULL;   /* per-thread [ncand][ACCW] accumulators (grad 20 + abs 20 + dL/dmu 2 + S term magnitudes 6) */
  double* tsh = NULL;    /* per-thread [ncand][45] SH rest-coefficient accumulators (f3) */
  uint8_t* tamb = NULL;
  const int nrest = sh ? 3 * ((sh->degree + 1) * (sh->degree + 1) - 1) : 0;
  if (want_bwd) {
    tacc = (double*)calloc((size_t)nthr * (size_t)(ncand > 0 ? ncand : 1) * ACCW, sizeof(double));
    tamb = (uint8_t*)calloc((size_t)(ncand > 0 ? ncand : 1), 1);
    if (nrest > 0) tsh = (double*)calloc((size_t)nthr * (size_t)(ncand > 0 ? ncand : 1) * 45, sizeof(double));
    if (!tacc || !tamb || (nrest > 0 && !tsh)) {
      free(cand); free(start); free(list); free(tacc); free(tamb); free(tsh); return -1;
    }
  }
  int64_t total_comp = 0;
  const double amin = rp->alpha_min, amax = rp->alpha_max, tmin = rp->t_min;

#pragma omp parallel reduction(+ : total_comp)
  {
#ifdef _OPENMP
    const int tid = omp_get_thread_num();
#else
    const int tid = 0;
#endif
    double* acc = want_bwd ? tacc + (size_t)tid * (size_t)ncand * ACCW : NULL;
    double* ash = tsh ? tsh + (size_t)tid * (size_t)ncand * 45 : NULL;
    rec_t* recs = (rec_t*)malloc(sizeof(rec_t) * (size_t)(ncand > 0 ? ncand : 1));
#pragma omp for schedule(static)
    for (int32_t ky = 0; ky < h; ++ky) {
      for (int32_t jx = 0; jx < w; ++jx) {
        const int64_t pix = (int64_t)ky * w + jx;
        const double x = x0 + jx + 0.5, y = y0 + ky + 0.5;   /* pixel centre (Z5) */
        int64_t lb, le;
        if (brute_force) { lb = 0; le = ncand; } else { lb = start[pix]; le = start[pix + 1]; }
        double T = 1.0, C[3] = {0, 0, 0};
        int nr = 0, amb = 0;
        for (int64_t li = lb; li < le; ++li) {
          const int32_t c = brute_force ? (int32_t)li : list[li];
          const cand_t* cd = &cand[c];
          double d[2];
          const double sigma = slot_sigma(cd, split, params, ld, cam, rp, off, x, y, d);
          const double alpha = sigma < amax ? sigma : amax;
          if (amin > 0 && fabs(alpha - amin) <= AMB_BAND * amin) amb = 1;
          if (fabs(sigma - amax) <= AMB_BAND * amax) amb = 1;
          if (alpha < amin) continue;                       /* C8: skip */
          const double Tn = T * (1.0 - alpha);
          if (tmin > 0 && fabs(Tn - tmin) <= AMB_BAND * tmin) amb = 1;
          if (Tn < tmin) break;                             /* C8: terminate */
          for (int ch = 0; ch < 3; ++ch) C[ch] += alpha * T * cd->g.col[ch];
          recs[nr].c = c; recs[nr].sigma = sigma; recs[nr].alpha = alpha; recs[nr].T = T;
          recs[nr].d[0] = d[0]; recs[nr].d[1] = d[1];
          ++nr;
          T = Tn;
        }
        for (int ch = 0; ch < 3; ++ch) C[ch] += T * rp->bg[ch];
        if (image) for (int ch = 0; ch < 3; ++ch) image[(int64_t)ch * npx + pix] = C[ch];
        if (final_T) final_T[pix] = T;
        if (n_comp) n_comp[pix] = nr;
        if (amb_px) amb_px[pix] = (uint8_t)amb;
        total_comp += nr;
        if (!want_bwd) continue;
        if (amb) {
          for (int64_t li = lb; li < le; ++li) tamb[brute_force ? (int32_t)li : list[li]] = 1;
        }
        /* backward by reverse replay (C10):  g_i = T_i sum_ch dL/dC_ch (c_i,ch - B_ch) */
        double dLdC[3];
        for (int ch = 0; ch < 3; ++ch) dLdC[ch] = dL_dimage[(int64_t)ch * npx + pix];
        double Bc[3] = {rp->bg[0], rp->bg[1], rp->bg[2]};
        for (int r = nr - 1; r >= 0; --r) {
          const rec_t* rc = &recs[r];
          const cand_t* cd = &cand[rc->c];
          const gproj* g = &cd->g;
          double gsum = 0;
          for (int ch = 0; ch < 3; ++ch) gsum += dLdC[ch] * (g->col[ch] - Bc[ch]);
          const double ga = rc->T * gsum;  /* dL/dalpha = dL/dsigma (straight-through, Z3) */
          for (int ch = 0; ch < 3; ++ch) Bc[ch] = rc->alpha * g->col[ch] + (1 - rc->alpha) * Bc[ch];
          const double sg = rc->sigma;
          const double* d = rc->d;
          const double u0 = g->conic[0] * d[0] + g->conic[1] * d[1];
          const double u1 = g->conic[1] * d[0] + g->conic[2] * d[1];
          /* dsigma/dmu = sigma Q d ; dsigma/dcov(xx,xy,yy) = sigma (u0^2/2, u0 u1, u1^2/2) */
          const double dsdmu[2] = {sg * u0, sg * u1};
          const double dsdcov[3] = {0.5 * sg * u0 * u0, sg * u0 * u1, 0.5 * sg * u1 * u1};
          double contrib[20];
          for (int k = 0; k < 10; ++k) {
            double v = dsdcov[0] * g->dcov[k][0] + dsdcov[1] * g->dcov[k][1] + dsdcov[2] * g->dcov[k][2];
            if (k < 3) v += dsdmu[0] * g->dmu[0][k] + dsdmu[1] * g->dmu[1][k];
            contrib[k] = ga * v;
          }
          contrib[10] = ga * sg * (1.0 - g->o);                 /* d sigma / d logit */
          for (int ch = 0; ch < 3; ++ch) contrib[11 + ch] = rc->alpha * rc->T * dLdC[ch];
          if (g->sh_k) {   /* f3: dL/dcolour -> SH coefficients (masked by the clamp) and the mean */
            for (int ch = 0; ch < 3; ++ch) {
              const double gc = contrib[11 + ch] * g->cmask[ch];
              for (int k = 0; k < 3; ++k) contrib[k] += contrib[11 + ch] * g->dcol_dp[ch][k];
              for (int k = 1; k < g->sh_k; ++k) ash[(size_t)rc->c * 45 + 3 * (k - 1) + ch] += gc * g->Y[k];
              contrib[11 + ch] = gc * g->Y[0];
            }
          }
          double H[9];
          hessian_pair(g, sg, d, H);
          contrib[14] = ga * H[0]; contrib[15] = ga * H[1]; contrib[16] = ga * H[2];
          contrib[17] = ga * H[4]; contrib[18] = ga * H[5]; contrib[19] = ga * H[8];
          double* a = acc + (size_t)rc->c * ACCW;
          for (int k = 0; k < 20; ++k) { a[k] += contrib[k]; a[20 + k] += fabs(contrib[k]); }
          a[40] += ga * dsdmu[0];                               /* dL/dPi(p) (ADC statistic) */
          a[41] += ga * dsdmu[1];
          {   /* test infrastructure: the S entries' term magnitudes (absg rows 20-25) */
            double Hm[9];
            hessian_terms_abs(g, sg, d, Hm);
            const int e6[6] = {0, 1, 2, 4, 5, 8};
            for (int k = 0; k < 6; ++k) a[42 + k] += fabs(ga) * Hm[e6[k]];
          }
        }
      }
    }
    free(recs);
  }
  if (want_bwd) {
    for (int64_t c = 0; c < ncand; ++c) {
      const int64_t gi = cand[c].gid;
      for (int t = 0; t < nthr; ++t) {
        const double* a = tacc + ((size_t)t * (size_t)ncand + (size_t)c) * ACCW;
        for (int k = 0; k < 20; ++k) {
          if (grad) grad[k * ld + gi] += a[k];
          if (absg) absg[k * ld + gi] += a[20 + k];
        }
        for (int k = 0; k < 6; ++k)
          if (absg) absg[(20 + k) * ld + gi] += a[42 + k];
        if (grad_mu) { grad_mu[gi] += a[40]; grad_mu[ld + gi] += a[41]; }
        if (grad_sh && tsh) {
          const double* b = tsh + ((size_t)t * (size_t)ncand + (size_t)c) * 45;
          for (int k = 0; k < nrest; ++k) grad_sh[(int64_t)k * ld + gi] += b[k];
        }
      }
      if (amb_g && tamb[c]) amb_g[gi] = 1;
    }
  }
  free(tacc); free(tsh); free(tamb); free(cand); free(start); free(list);
  return total_comp;
}

/* ------------------------------------------------------------------------------------------
 * 4. Symmetric 3x3 eigen-decomposition by cyclic Jacobi (textbook; independent of the trig
 *    root formula of P:L588-604 that the kernels use).
 * ------------------------------------------------------------------------------------------ */
int orc_eig_sym3(const double* A6, double* lam, double* V) {
  double a[3][3] = {{A6[0], A6[1], A6[2]}, {A6[1], A6[3], A6[4]}, {A6[2], A6[4], A6[5]}};
  double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  const double q = (a[0][0] + a[1][1] + a[2][2]) / 3.0;
  double pp = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double b = a[i][j] - (i == j ? q : 0.0);
      pp += b * b;
    }
  const double p = sqrt(pp / 6.0);
  if (p < 1e-12 * (1.0 + fabs(q))) {           /* degenerate branch (Z17) */
    lam[0] = lam[1] = lam[2] = q;
    for (int k = 0; k < 9; ++k) V[k] = (k % 4 == 0) ? 1.0 : 0.0;
    return 0;
  }
  int sweep;
  for (sweep = 0; sweep < 100; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    const double diag = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2];
    if (off <= 1e-34 * diag || off == 0.0) break;
    for (int pi = 0; pi < 2; ++pi)
      for (int qi = pi + 1; qi < 3; ++qi) {
        if (a[pi][qi] == 0.0) continue;
        const double theta = (a[qi][qi] - a[pi][pi]) / (2.0 * a[pi][qi]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {           /* A <- A J (columns p,q) */
          const double akp = a[k][pi], akq = a[k][qi];
          a[k][pi] = c * akp - s * akq;
          a[k][qi] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {           /* A <- J^T A (rows p,q) */
          const double apk = a[pi][k], aqk = a[qi][k];
          a[pi][k] = c * apk - s * aqk;
          a[qi][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {           /* V <- V J */
          const double vkp = v[k][pi], vkq = v[k][qi];
          v[k][pi] = c * vkp - s * vkq;
          v[k][qi] = s * vkp + c * vkq;
        }
      }
  }
  int order[3] = {0, 1, 2};
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (a[order[j]][order[j]] < a[order[i]][order[i]]) { const int t = order[i]; order[i] = order[j]; order[j] = t; }
  for (int c = 0; c < 3; ++c) {
    const int o = order[c];
    lam[c] = a[o][o];
    double col[3] = {v[0][o], v[1][o], v[2][o]};
    const double nrm = sqrt(col[0] * col[0] + col[1] * col[1] + col[2] * col[2]);
    int big = 0;
    for (int k = 0; k < 3; ++k) col[k] /= nrm;
    for (int k = 1; k < 3; ++k)
      if (fabs(col[k]) > fabs(col[big])) big = k;
    const double sg = col[big] < 0 ? -1.0 : 1.0;   /* canonical sign (C13) */
    for (int k = 0; k < 3; ++k) V[3 * k + c] = sg * col[k];
  }
  return sweep;
}

/* ------------------------------------------------------------------------------------------
 * 5. Steepest density control (Thm 2; Alg. 1).
 * ------------------------------------------------------------------------------------------ */
int64_t orc_densify(double* params, int64_t ld, int64_t n, int64_t capacity, double* acc,
                    int64_t ldg, double denom, double eps_split, double eta, double eps_abs,
                    int32_t gate, double eps_grad, int64_t budget,
                    uint8_t* mask, int32_t* dest, double* lambda) {
  int64_t nsplit = 0;
  double* vmin = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  double* lam0 = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (!vmin || !lam0) { free(vmin); free(lam0); return -2; }
  int64_t ncand = 0;
  for (int64_t i = 0; i < n; ++i) {
    double Sbar[6];
    for (int k = 0; k < 6; ++k) Sbar[k] = acc[(14 + k) * ldg + i] / denom;
    double lam[3], V[9];
    orc_eig_sym3(Sbar, lam, V);
    if (lambda) lambda[i] = lam[0];
    lam0[i] = lam[0];
    for (int k = 0; k < 3; ++k) vmin[3 * i + k] = V[3 * k + 0];
    int split = lam[0] < eps_split;                                            /* P:L545, Z11 */
    if (split && gate == 1) {
      double g2 = 0;
      for (int k = 0; k < 3; ++k) { const double g = acc[k * ldg + i] / denom; g2 += g * g; }
      split = sqrt(g2) <= eps_grad;
    } else if (split && gate == 2) {          /* Alg. 1 "condition on G" as 3DGS's (C24) */
      const double cnt = acc[1 * ldg + i];
      split = cnt > 0 && acc[0 * ldg + i] / cnt >= eps_grad;
    }
    mask[i] = (uint8_t)split;
    ncand += split;
  }
  if (budget >= 0 && ncand > budget) {
    /* keep the `budget` least lambda_min (ties: lower index) — selection by repeated minimum */
    uint8_t* keep = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
    for (int64_t r = 0; r < budget; ++r) {
      int64_t best = -1;
      for (int64_t i = 0; i < n; ++i)
        if (mask[i] && !keep[i] && (best < 0 || lam0[i] < lam0[best])) best = i;
      keep[best] = 1;
    }
    for (int64_t i = 0; i < n; ++i) mask[i] = keep[i];
    free(keep);
  }
  for (int64_t i = 0; i < n; ++i) {
    dest[i] = mask[i] ? (int32_t)(n + nsplit) : -1;                            /* Z24 */
    nsplit += mask[i];
  }
  free(lam0);
  if (n + nsplit > capacity) { free(vmin); return -1; }                        /* C16 */
  for (int64_t i = 0; i < n; ++i) {
    if (!mask[i]) continue;
    const int64_t b = dest[i];
    const double* v = &vmin[3 * i];
    double eps = eps_abs;
    if (eta >= 0) {                                                            /* Z13 */
      double q[4];
      for (int k = 0; k < 4; ++k) q[k] = params[(6 + k) * ld + i];
      const double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
      for (int k = 0; k < 4; ++k) q[k] /= qn;
      double R[9];
      rot_from_quat(q, R);
      double vSv = 0;
      for (int k = 0; k < 3; ++k) {
        const double s = exp(params[(3 + k) * ld + i]);
        const double rv = R[0 * 3 + k] * v[0] + R[1 * 3 + k] * v[1] + R[2 * 3 + k] * v[2];
        vSv += s * s * rv * rv;
      }
      eps = eta * sqrt(vSv);
    }
    const double o = sigmoid(params[10 * ld + i]);
    const double half = 0.5 * o;                                               /* Z15 */
    const double lg = log(half) - log1p(-half);
    for (int k = 0; k < 14; ++k) params[k * ld + b] = params[k * ld + i];     /* Z14: copy */
    for (int k = 0; k < 3; ++k) {
      const double p = params[k * ld + i];
      params[k * ld + i] = p + eps * v[k];
      params[k * ld + b] = p - eps * v[k];
    }
    params[10 * ld + i] = lg;
    params[10 * ld + b] = lg;
  }
  for (int64_t i = 0; i < n + nsplit; ++i)
    for (int k = 14; k < 20; ++k) acc[k * ldg + i] = 0.0;                      /* Z23 */
  free(vmin);
  return nsplit;
}
