// project.cu — a1: per-(view, Gaussian) projection (Eq. eqn:sigma_2D + footnote fn:Pi,
// P:L135-139; quaternion + scale re-parameterisation P:L114).
//
// Compiled with -fmad=false: the decision chain (visibility, depth key, tile rect) is the exact
// fp32 operation sequence of DESIGN.md §3.2, each line one IEEE round-to-nearest operation, with
// exp/log evaluated in double and rounded once.  The render values (pixel mean) are computed in
// fp64 and kept in fp64 in the splat record.
//
// One thread per Gaussian; the 14 parameter planes are read once (coalesced SoA) and the V views
// of the call are produced from registers.  Bound: HBM (56 B read + 64 B + 16 B written per
// visible (view, Gaussian)).
#include <math.h>

#include "common.cuh"

namespace sgs {

__device__ __forceinline__ uint32_t orderable_key(float z) {
  const uint32_t u = __float_as_uint(z);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void __launch_bounds__(256) k_project(const float* __restrict__ params, int64_t ld, int64_t n,
                                                 const CamPack cams, int V, const RasterK rk,
                                                 steepgs_splat* __restrict__ splats,
                                                 uint32_t* __restrict__ depth_key, uint2* __restrict__ tile_rect,
                                                 int32_t* __restrict__ tiles_touched) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float p0 = params[0 * ld + i], p1 = params[1 * ld + i], p2 = params[2 * ld + i];
  const float ls0 = params[3 * ld + i], ls1 = params[4 * ld + i], ls2 = params[5 * ld + i];
  const float qw = params[6 * ld + i], qx = params[7 * ld + i], qy = params[8 * ld + i], qz = params[9 * ld + i];
  const float logit = params[10 * ld + i];
  const float cr = params[11 * ld + i], cg = params[12 * ld + i], cb = params[13 * ld + i];

  // ---- view-independent part of the chain: R(q), s, Sigma, opacity ----
  float nq2 = qw * qw; nq2 = nq2 + qx * qx; nq2 = nq2 + qy * qy; nq2 = nq2 + qz * qz;
  const bool qok = nq2 > 0.0f;
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
  const float s[3] = {(float)exp((double)ls0), (float)exp((double)ls1), (float)exp((double)ls2)};
  float M[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) M[3 * a + k] = r[3 * a + k] * s[k];
  float Sg[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      float acc = M[3 * a + 0] * M[3 * b + 0];
      acc = acc + M[3 * a + 1] * M[3 * b + 1];
      acc = acc + M[3 * a + 2] * M[3 * b + 2];
      Sg[3 * a + b] = acc;
    }
  // fp64 R(q_hat) diag(s) for the render values (columns scaled by s_k)
  double dr[9];
  {
    const double dq = sqrt((double)qw * qw + (double)qx * qx + (double)qy * qy + (double)qz * qz);
    const double W_ = qw / dq, X = qx / dq, Y = qy / dq, Z = qz / dq;
    const double ds0 = exp((double)ls0), ds1 = exp((double)ls1), ds2 = exp((double)ls2);
    dr[0] = (1.0 - 2.0 * (Y * Y + Z * Z)) * ds0; dr[1] = 2.0 * (X * Y - W_ * Z) * ds1; dr[2] = 2.0 * (X * Z + W_ * Y) * ds2;
    dr[3] = 2.0 * (X * Y + W_ * Z) * ds0; dr[4] = (1.0 - 2.0 * (X * X + Z * Z)) * ds1; dr[5] = 2.0 * (Y * Z - W_ * X) * ds2;
    dr[6] = 2.0 * (X * Z - W_ * Y) * ds0; dr[7] = 2.0 * (Y * Z + W_ * X) * ds1; dr[8] = (1.0 - 2.0 * (X * X + Y * Y)) * ds2;
  }
  const float o = (float)(1.0 / (1.0 + exp(-(double)logit)));
  const bool ook = o > rk.alpha_min;
  const float tau = (float)(2.0 * log((double)o / (double)rk.alpha_min));

  for (int v = 0; v < V; ++v) {
    const steepgs_camera& c = cams.cam[v];
    const int64_t vi = (int64_t)v * n + i;
    const float* R = c.R;
    float tx = R[0] * p0; tx = tx + R[1] * p1; tx = tx + R[2] * p2; tx = tx + c.t[0];
    float ty = R[3] * p0; ty = ty + R[4] * p1; ty = ty + R[5] * p2; ty = ty + c.t[1];
    float tz = R[6] * p0; tz = tz + R[7] * p1; tz = tz + R[8] * p2; tz = tz + c.t[2];
    bool vis = qok && ook;
    float mux, muy, J00, J02, J11, J12;
    if (c.model == 0) {
      vis = vis && (tz > c.znear);
      const float xz = tx / tz, yz = ty / tz;
      const float limx = c.guard * ((0.5f * (float)c.width) / c.fx);
      const float limy = c.guard * ((0.5f * (float)c.height) / c.fy);
      vis = vis && (fabsf(xz) <= limx) && (fabsf(yz) <= limy);
      mux = c.fx * xz; mux = mux + c.cx;
      muy = c.fy * yz; muy = muy + c.cy;
      J00 = c.fx / tz; J02 = -((c.fx * xz) / tz);
      J11 = c.fy / tz; J12 = -((c.fy * yz) / tz);
    } else {
      mux = c.fx * tx; mux = mux + c.cx;
      muy = c.fy * ty; muy = muy + c.cy;
      J00 = c.fx; J02 = 0.0f; J11 = c.fy; J12 = 0.0f;
    }
    float P[6];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      float a0 = J00 * R[0 + b]; a0 = a0 + J02 * R[6 + b]; P[b] = a0;
      float a1 = J11 * R[3 + b]; a1 = a1 + J12 * R[6 + b]; P[3 + b] = a1;
    }
    float Tm[6];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        float acc = P[3 * a + 0] * Sg[0 + b];
        acc = acc + P[3 * a + 1] * Sg[3 + b];
        acc = acc + P[3 * a + 2] * Sg[6 + b];
        Tm[3 * a + b] = acc;
      }
    float A = Tm[0] * P[0]; A = A + Tm[1] * P[1]; A = A + Tm[2] * P[2]; A = A + rk.dilation;
    float B = Tm[0] * P[3]; B = B + Tm[1] * P[4]; B = B + Tm[2] * P[5];
    float C = Tm[3] * P[3]; C = C + Tm[4] * P[4]; C = C + Tm[5] * P[5]; C = C + rk.dilation;
    const float det = A * C - B * B;
    vis = vis && (det > 0.0f);
    const float ex = sqrtf(tau * A), ey = sqrtf(tau * C);
    float lox = mux - ex; lox = lox - 0.5f; lox = lox - 1e-3f;
    float hix = mux + ex; hix = hix - 0.5f; hix = hix + 1e-3f;
    float loy = muy - ey; loy = loy - 0.5f; loy = loy - 1e-3f;
    float hiy = muy + ey; hiy = hiy - 0.5f; hiy = hiy + 1e-3f;
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

    // ---- render values in fp64, rounded once: the pixel mean (kept in fp64) and the conic.  fp32
    // rounding of P alone perturbs thin, large footprints by ~1e-7 lambda_max / lambda_min, so the
    // projected covariance is formed as Sigma2D = M M^T + dil I with M = P R diag(s) and
    // det = |m0 x m1|^2 + dil (|m0|^2 + |m1|^2) + dil^2 (no cancellation).
    const double dtx = ((double)R[0] * p0 + (double)R[1] * p1) + ((double)R[2] * p2 + (double)c.t[0]);
    const double dty = ((double)R[3] * p0 + (double)R[4] * p1) + ((double)R[5] * p2 + (double)c.t[1]);
    const double dtz = ((double)R[6] * p0 + (double)R[7] * p1) + ((double)R[8] * p2 + (double)c.t[2]);
    double mx, my, j00, j02, j11, j12;
    if (c.model == 0) {
      const double iz = 1.0 / dtz;
      mx = (double)c.fx * (dtx * iz) + (double)c.cx;
      my = (double)c.fy * (dty * iz) + (double)c.cy;
      j00 = (double)c.fx * iz; j02 = -(double)c.fx * dtx * iz * iz;
      j11 = (double)c.fy * iz; j12 = -(double)c.fy * dty * iz * iz;
    } else {
      mx = (double)c.fx * dtx + (double)c.cx;
      my = (double)c.fy * dty + (double)c.cy;
      j00 = c.fx; j02 = 0.0; j11 = c.fy; j12 = 0.0;
    }
    double m0[3], m1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      // column k of R(q) diag(s) in world space, then through P = J W
      const double wx = dr[k], wy = dr[3 + k], wz = dr[6 + k];
      const double cx_ = (double)R[0] * wx + (double)R[1] * wy + (double)R[2] * wz;
      const double cy_ = (double)R[3] * wx + (double)R[4] * wy + (double)R[5] * wz;
      const double cz_ = (double)R[6] * wx + (double)R[7] * wy + (double)R[8] * wz;
      m0[k] = j00 * cx_ + j02 * cz_;
      m1[k] = j11 * cy_ + j12 * cz_;
    }
    const double dil = (double)rk.dilation;
    const double a00 = m0[0] * m0[0] + m0[1] * m0[1] + m0[2] * m0[2];
    const double a11 = m1[0] * m1[0] + m1[1] * m1[1] + m1[2] * m1[2];
    const double a01 = m0[0] * m1[0] + m0[1] * m1[1] + m0[2] * m1[2];
    const double x0 = m0[1] * m1[2] - m0[2] * m1[1], x1 = m0[2] * m1[0] - m0[0] * m1[2], x2 = m0[0] * m1[1] - m0[1] * m1[0];
    const double ddet = (x0 * x0 + x1 * x1 + x2 * x2) + dil * (a00 + a11) + dil * dil;
    const double idet = 1.0 / ddet;
    // exp2-ready record: conic * log2(e)/2, log2(o), and the padded half-extents of {m <= tau}
    const double hl2e = 0.72134752044448170;  // log2(e) / 2
    const double dtau = (double)tau;
    const float hx = (float)(sqrt(dtau * (a00 + dil)) * 1.001 + 0.01);
    const float hy = (float)(sqrt(dtau * (a11 + dil)) * 1.001 + 0.01);
    steepgs_splat* sp = splats + vi;
    double2* s0 = reinterpret_cast<double2*>(sp);
    float4* s1 = reinterpret_cast<float4*>(sp) + 1;
    *s0 = make_double2(mx, my);
    s1[0] = make_float4((float)((a11 + dil) * idet * hl2e), (float)(-2.0 * a01 * idet * hl2e),
                        (float)((a00 + dil) * idet * hl2e), (float)log2((double)o));
    s1[1] = make_float4(cr, cg, cb, o);
    s1[2] = make_float4(hx, hy, tau, 0.0f);
  }
}

cudaError_t launch_project(const float* params, int64_t ld, int64_t n, const CamPack& cams, int V,
                           const RasterK& rk, steepgs_splat* splats, uint32_t* depth_key, uint32_t* tile_rect,
                           int32_t* tiles_touched, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  const unsigned blocks = (unsigned)((n + threads - 1) / threads);
  k_project<<<blocks, threads, 0, st>>>(params, ld, n, cams, V, rk, splats, depth_key,
                                        reinterpret_cast<uint2*>(tile_rect), tiles_touched);
  note_launch();
  return check_launch("k_project");
}

}  // namespace sgs
