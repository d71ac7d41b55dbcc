// project.cu — a1: per-(view, Gaussian) projection (Eq. eqn:sigma_2D + footnote fn:Pi,
// P:L135-139; quaternion + scale re-parameterisation P:L114).
//
// Decision chain (visibility, depth key, tile rect): the exact fp32 operation sequence of DESIGN.md
// §3.2, written with explicit round-to-nearest intrinsics (__fmul_rn / __fadd_rn / __fsub_rn /
// __fdiv_rn / __fsqrt_rn are never contracted into FMAs), exp/log evaluated in double and rounded
// once, so the integer results match the oracle's independent evaluation bit for bit.
// Render values: the pixel mean (kept in fp64), the conic (formed as M M^T + dil I with
// M = P R diag(s), det from |m0 x m1|^2, rounded once), log2 o and the padded alpha-support
// extents, written as one 64-B exp2-ready record per visible (view, Gaussian).
//
// One thread per Gaussian; the 14 parameter planes are read once (coalesced SoA) and the V views
// of the call are produced from registers.  Bound: HBM (56 B read + 64 B + 16 B written per
// visible (view, Gaussian)).
#include <math.h>

#include "common.cuh"

namespace sgs {

#define MUL(a, b) __fmul_rn((a), (b))
#define ADD(a, b) __fadd_rn((a), (b))
#define SUB(a, b) __fsub_rn((a), (b))
#define DIV(a, b) __fdiv_rn((a), (b))

__device__ __forceinline__ uint32_t orderable_key(float z) {
  const uint32_t u = __float_as_uint(z);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// 1/x in fp64 from the fp32 reciprocal and two Newton steps (|rel err| < 1e-15 for normal x).
__device__ __forceinline__ double drcp(double x) {
  double r = (double)__frcp_rn((float)x);
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}

// kSH = -1: colour = rgb planes 11-13; kSH = 0..3: view-dependent colour from real spherical harmonics
// (NEXT f3): colour = max(0, sum_k Y_k(dir) f_k + 1/2), DC f_0 = planes 11-13, the rest from
// sh_rest (plane 3 (k - 1) + ch), dir = (p - o)/|p - o| with o = -R^T t (pinhole) or R^T e_z (affine).
template <int kSH>
__global__ void __launch_bounds__(256, kSH < 0 ? 4 : 1) k_project(const float* __restrict__ params, int64_t ld, int64_t n,
                                                 const float* __restrict__ sh_rest, int64_t ld_sh,
                                                 const CamPack cams, int V, const RasterK rk,
                                                 steepgs_splat* __restrict__ splats,
                                                 uint32_t* __restrict__ depth_key, uint2* __restrict__ tile_rect,
                                                 int32_t* __restrict__ tiles_touched) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float p0 = params[0 * ld + i], p1 = params[1 * ld + i], p2 = params[2 * ld + i];
  const float ls0 = params[3 * ld + i], ls1 = params[4 * ld + i], ls2 = params[5 * ld + i];
  const float qw = params[6 * ld + i], qx = params[7 * ld + i], qy = params[8 * ld + i], qz = params[9 * ld + i];
  const float logit = params[10 * ld + i];
  const float cr = params[11 * ld + i], cg = params[12 * ld + i], cb = params[13 * ld + i];

  // ---- view-independent part of the decision chain: R(q), s, Sigma, opacity ----
  const float nq2 = ADD(ADD(ADD(MUL(qw, qw), MUL(qx, qx)), MUL(qy, qy)), MUL(qz, qz));
  const bool qok = nq2 > 0.0f;
  const float nq = __fsqrt_rn(nq2);
  const float w = DIV(qw, nq), x = DIV(qx, nq), y = DIV(qy, nq), z = DIV(qz, nq);
  float r[9];
  r[0] = SUB(1.0f, MUL(2.0f, ADD(MUL(y, y), MUL(z, z))));
  r[1] = MUL(2.0f, SUB(MUL(x, y), MUL(w, z)));
  r[2] = MUL(2.0f, ADD(MUL(x, z), MUL(w, y)));
  r[3] = MUL(2.0f, ADD(MUL(x, y), MUL(w, z)));
  r[4] = SUB(1.0f, MUL(2.0f, ADD(MUL(x, x), MUL(z, z))));
  r[5] = MUL(2.0f, SUB(MUL(y, z), MUL(w, x)));
  r[6] = MUL(2.0f, SUB(MUL(x, z), MUL(w, y)));
  r[7] = MUL(2.0f, ADD(MUL(y, z), MUL(w, x)));
  r[8] = SUB(1.0f, MUL(2.0f, ADD(MUL(x, x), MUL(y, y))));
  const double ds0 = exp((double)ls0), ds1 = exp((double)ls1), ds2 = exp((double)ls2);
  const float s[3] = {(float)ds0, (float)ds1, (float)ds2};
  float M[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) M[3 * a + k] = MUL(r[3 * a + k], s[k]);
  float Sg[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      Sg[3 * a + b] = ADD(ADD(MUL(M[3 * a + 0], M[3 * b + 0]), MUL(M[3 * a + 1], M[3 * b + 1])),
                          MUL(M[3 * a + 2], M[3 * b + 2]));
  const double dopac = 1.0 / (1.0 + exp(-(double)logit));
  const float o = (float)dopac;
  const bool ook = o > rk.alpha_min;
  const float tau = (float)(2.0 * log((double)o / (double)rk.alpha_min));
  const float log2o = (float)log2((double)o);
  // fp64 R(q_hat) diag(s) for the render values (columns scaled by s_k)
  double dr[9];
  {
    const double dq = sqrt((double)qw * qw + (double)qx * qx + (double)qy * qy + (double)qz * qz);
    const double iq = 1.0 / dq;
    const double W_ = qw * iq, X = qx * iq, Y = qy * iq, Z = qz * iq;
    dr[0] = (1.0 - 2.0 * (Y * Y + Z * Z)) * ds0; dr[1] = 2.0 * (X * Y - W_ * Z) * ds1; dr[2] = 2.0 * (X * Z + W_ * Y) * ds2;
    dr[3] = 2.0 * (X * Y + W_ * Z) * ds0; dr[4] = (1.0 - 2.0 * (X * X + Z * Z)) * ds1; dr[5] = 2.0 * (Y * Z - W_ * X) * ds2;
    dr[6] = 2.0 * (X * Z - W_ * Y) * ds0; dr[7] = 2.0 * (Y * Z + W_ * X) * ds1; dr[8] = (1.0 - 2.0 * (X * X + Y * Y)) * ds2;
  }

  const double dp0 = p0, dp1 = p1, dp2 = p2;
  // SH rest coefficients: read once, used by every view (kSH >= 1)
  constexpr int kRest = kSH >= 1 ? 3 * ((kSH + 1) * (kSH + 1) - 1) : 1;
  float shc[kRest];
#pragma unroll
  for (int k = 0; k < kRest; ++k) shc[k] = kSH >= 1 ? __ldg(sh_rest + (int64_t)k * ld_sh + i) : 0.0f;
  for (int v = 0; v < V; ++v) {
    const steepgs_camera& c = cams.cam[v];
    const int64_t vi = (int64_t)v * n + i;
    const float* R = c.R;
    // ---- decision chain, view part ----
    const float tx = ADD(ADD(ADD(MUL(R[0], p0), MUL(R[1], p1)), MUL(R[2], p2)), c.t[0]);
    const float ty = ADD(ADD(ADD(MUL(R[3], p0), MUL(R[4], p1)), MUL(R[5], p2)), c.t[1]);
    const float tz = ADD(ADD(ADD(MUL(R[6], p0), MUL(R[7], p1)), MUL(R[8], p2)), c.t[2]);
    bool vis = qok && ook;
    float mux, muy, J00, J02, J11, J12;
    if (c.model == 0) {
      vis = vis && (tz > c.znear);
      const float xz = DIV(tx, tz), yz = DIV(ty, tz);
      const float limx = cams.lim[v][0], limy = cams.lim[v][1];   // MUL(guard, DIV(MUL(0.5, W), fx)), host
      vis = vis && (fabsf(xz) <= limx) && (fabsf(yz) <= limy);
      mux = ADD(MUL(c.fx, xz), c.cx);
      muy = ADD(MUL(c.fy, yz), c.cy);
      J00 = DIV(c.fx, tz); J02 = -DIV(MUL(c.fx, xz), tz);
      J11 = DIV(c.fy, tz); J12 = -DIV(MUL(c.fy, yz), tz);
    } else {
      mux = ADD(MUL(c.fx, tx), c.cx);
      muy = ADD(MUL(c.fy, ty), c.cy);
      J00 = c.fx; J02 = 0.0f; J11 = c.fy; J12 = 0.0f;
    }
    float P[6];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      P[b] = ADD(MUL(J00, R[0 + b]), MUL(J02, R[6 + b]));
      P[3 + b] = ADD(MUL(J11, R[3 + b]), MUL(J12, R[6 + b]));
    }
    float Tm[6];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b)
        Tm[3 * a + b] = ADD(ADD(MUL(P[3 * a + 0], Sg[0 + b]), MUL(P[3 * a + 1], Sg[3 + b])), MUL(P[3 * a + 2], Sg[6 + b]));
    const float A = ADD(ADD(ADD(MUL(Tm[0], P[0]), MUL(Tm[1], P[1])), MUL(Tm[2], P[2])), rk.dilation);
    const float B = ADD(ADD(MUL(Tm[0], P[3]), MUL(Tm[1], P[4])), MUL(Tm[2], P[5]));
    const float C = ADD(ADD(ADD(MUL(Tm[3], P[3]), MUL(Tm[4], P[4])), MUL(Tm[5], P[5])), rk.dilation);
    const float det = SUB(MUL(A, C), MUL(B, B));
    vis = vis && (det > 0.0f);
    const float ex = __fsqrt_rn(MUL(tau, A)), ey = __fsqrt_rn(MUL(tau, C));
    const float lox = SUB(SUB(SUB(mux, ex), 0.5f), 1e-3f);
    const float hix = ADD(SUB(ADD(mux, ex), 0.5f), 1e-3f);
    const float loy = SUB(SUB(SUB(muy, ey), 0.5f), 1e-3f);
    const float hiy = ADD(SUB(ADD(muy, ey), 0.5f), 1e-3f);
    vis = vis && !(lox != lox || hix != hix || loy != loy || hiy != hiy);
    const float jmin = fmaxf(ceilf(lox), 0.0f), jmax = fminf(floorf(hix), (float)(c.width - 1));
    const float kmin = fmaxf(ceilf(loy), 0.0f), kmax = fminf(floorf(hiy), (float)(c.height - 1));
    vis = vis && (jmin <= jmax) && (kmin <= kmax);
    if (!vis) {
      tiles_touched[vi] = 0;
      depth_key[vi] = 0xFFFFFFFFu;
      tile_rect[vi] = make_uint2(0u, 0u);
      continue;
    }
    const int tx0 = (int)jmin / kTile, tx1 = (int)jmax / kTile;
    const int ty0 = (int)kmin / kTile, ty1 = (int)kmax / kTile;
    tiles_touched[vi] = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
    depth_key[vi] = orderable_key(tz);
    tile_rect[vi] = make_uint2((uint32_t)tx0 | ((uint32_t)tx1 << 16), (uint32_t)ty0 | ((uint32_t)ty1 << 16));

    // ---- render values in fp64, rounded once.  fp32 rounding of P alone would perturb thin,
    // large footprints by ~1e-7 lambda_max / lambda_min, so Sigma2D = M M^T + dil I with
    // M = P R diag(s) and det = |m0 x m1|^2 + dil (|m0|^2 + |m1|^2) + dil^2 (no cancellation).
    const double* Dc = cams.dc[v];   // R (0-8), t (9-11), fx, fy, cx, cy in fp64
    const double dtx = fma(Dc[0], dp0, fma(Dc[1], dp1, fma(Dc[2], dp2, Dc[9])));
    const double dty = fma(Dc[3], dp0, fma(Dc[4], dp1, fma(Dc[5], dp2, Dc[10])));
    const double dtz = fma(Dc[6], dp0, fma(Dc[7], dp1, fma(Dc[8], dp2, Dc[11])));
    double mx, my, j00, j02, j11, j12;
    if (c.model == 0) {
      const double iz = drcp(dtz);
      const double xz = dtx * iz, yz = dty * iz;
      mx = fma(Dc[12], xz, Dc[14]);
      my = fma(Dc[13], yz, Dc[15]);
      j00 = Dc[12] * iz; j02 = -Dc[12] * xz * iz;
      j11 = Dc[13] * iz; j12 = -Dc[13] * yz * iz;
    } else {
      mx = fma(Dc[12], dtx, Dc[14]);
      my = fma(Dc[13], dty, Dc[15]);
      j00 = Dc[12]; j02 = 0.0; j11 = Dc[13]; j12 = 0.0;
    }
    double m0[3], m1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      // column k of R(q) diag(s) taken to camera space, then through J
      const double wx = dr[k], wy = dr[3 + k], wz = dr[6 + k];
      const double cx_ = fma(Dc[0], wx, fma(Dc[1], wy, Dc[2] * wz));
      const double cy_ = fma(Dc[3], wx, fma(Dc[4], wy, Dc[5] * wz));
      const double cz_ = fma(Dc[6], wx, fma(Dc[7], wy, Dc[8] * wz));
      m0[k] = fma(j00, cx_, j02 * cz_);
      m1[k] = fma(j11, cy_, j12 * cz_);
    }
    const double dil = (double)rk.dilation;
    const double a00 = fma(m0[0], m0[0], fma(m0[1], m0[1], m0[2] * m0[2]));
    const double a11 = fma(m1[0], m1[0], fma(m1[1], m1[1], m1[2] * m1[2]));
    const double a01 = fma(m0[0], m1[0], fma(m0[1], m1[1], m0[2] * m1[2]));
    const double x0 = fma(m0[1], m1[2], -m0[2] * m1[1]), x1 = fma(m0[2], m1[0], -m0[0] * m1[2]);
    const double x2 = fma(m0[0], m1[1], -m0[1] * m1[0]);
    const double ddet = fma(x0, x0, fma(x1, x1, x2 * x2)) + dil * (a00 + a11 + dil);
    const double hl2e = 0.72134752044448170;  // log2(e) / 2: exp2-ready conic
    const double sc = drcp(ddet) * hl2e;
    const float hx = sqrtf(tau * (float)(a00 + dil)) * 1.001f + 0.01f;   // padded half-extents of {m <= tau}
    const float hy = sqrtf(tau * (float)(a11 + dil)) * 1.001f + 0.01f;
    steepgs_splat* sp = splats + vi;
    double2* s0 = reinterpret_cast<double2*>(sp);
    float4* s1 = reinterpret_cast<float4*>(sp) + 1;
    *s0 = make_double2(mx, my);
    s1[0] = make_float4((float)((a11 + dil) * sc), (float)(-2.0 * a01 * sc), (float)((a00 + dil) * sc), log2o);
    float col[3] = {cr, cg, cb};
    if (kSH >= 0) {
      float d[3];
      if (c.model == 0) {
        float v3[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) v3[k] = (k == 0 ? p0 : (k == 1 ? p1 : p2)) +
                                             (R[k] * c.t[0] + R[3 + k] * c.t[1] + R[6 + k] * c.t[2]);
        const float rn = rsqrtf(v3[0] * v3[0] + v3[1] * v3[1] + v3[2] * v3[2]);
        d[0] = v3[0] * rn; d[1] = v3[1] * rn; d[2] = v3[2] * rn;
      } else {
        d[0] = R[6]; d[1] = R[7]; d[2] = R[8];
      }
      float Y[16];
      sh_basis<kSH>(d, Y);
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        float raw = 0.5f + Y[0] * col[ch];
#pragma unroll
        for (int k = 1; k < (kSH + 1) * (kSH + 1); ++k) raw += Y[k] * shc[3 * (k - 1) + ch];
        col[ch] = fmaxf(raw, 0.0f);
      }
    }
    s1[1] = make_float4(col[0], col[1], col[2], o);
    s1[2] = make_float4(hx, hy, tau, 0.0f);
  }
}

#undef MUL
#undef ADD
#undef SUB
#undef DIV

cudaError_t launch_project(const float* params, int64_t ld, int64_t n, const float* sh_rest, int64_t ld_sh,
                           int sh_degree, const CamPack& cams, int V, const RasterK& rk, steepgs_splat* splats,
                           uint32_t* depth_key, uint32_t* tile_rect, int32_t* tiles_touched, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  const unsigned blocks = (unsigned)((n + threads - 1) / threads);
#define SGS_PROJECT(D)                                                                                     \
  launch_pdl(k_project<D>, dim3(blocks), dim3(threads), 0, st, params, ld, n, sh_rest, ld_sh, cams, V, rk, splats, \
             depth_key, reinterpret_cast<uint2*>(tile_rect), tiles_touched)
  switch (sh_degree) {
    case 0: SGS_PROJECT(0); break;
    case 1: SGS_PROJECT(1); break;
    case 2: SGS_PROJECT(2); break;
    case 3: SGS_PROJECT(3); break;
    default: SGS_PROJECT(-1); break;
  }
#undef SGS_PROJECT
  note_launch();
  return check_launch("k_project");
}

}  // namespace sgs
