// gauss_bwd.cu — a6: per-Gaussian backward and the splitting matrix (App. C.4
// P:L1133-1157; Alg. 1).
//
// From the 9 per-(view, Gaussian) moments of w = dL/dsigma * sigma accumulated by k_render_bwd2
//   m0 = sum w,  m1 = sum w d,  M = sum w d d^T,  cg = sum alpha T dL/dC     (d = x - Pi(p))
// and sigma = o exp(-1/2 d^T Q d):
//   dL/dmu = Q m1,  dL/dPi(Sigma) = 1/2 Q M Q,  dL/do = m0 / o,  dL/dc = cg,
//   S_view = sum_x g sigma P^T (Q d d^T Q - Q) P = P^T (Q M Q - m0 Q) P          (C12)
// because P and Q are constant per (view, Gaussian).  dL/dSigma_3D = P^T (1/2 Q M Q) P is summed
// over the views and chained to log-scale and quaternion once.  Pinhole: J(t) depends on p, so
// dL/dt gets the J-derivative terms (C11); S keeps P frozen.
//
// One thread per Gaussian, views looped inside (no atomics); the moments are read and cleared
// (read-and-zero keeps the workspace zero for the next call), with the next view's moments in
// flight while the current view is chained.  Bound: HBM.
#include "common.cuh"

namespace sgs {

namespace {

__global__ void __launch_bounds__(128, 5) k_gauss_bwd(const float* __restrict__ params, int64_t ld, int64_t n,
                                                   const CamPack cams, int V, const RasterK rk,
                                                   float* __restrict__ moments, float* __restrict__ grad_S,
                                                   int64_t ldg, int accumulate,
                                                   const int32_t* __restrict__ tiles_touched,
                                                   float* __restrict__ vstats, const ScatterOut sc) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float p0 = params[0 * ld + i], p1 = params[1 * ld + i], p2 = params[2 * ld + i];
  const float ls[3] = {params[3 * ld + i], params[4 * ld + i], params[5 * ld + i]};
  const float qw = params[6 * ld + i], qx = params[7 * ld + i], qy = params[8 * ld + i], qz = params[9 * ld + i];
  const float logit = params[10 * ld + i];
  const float qn = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
  const float w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
  float r[9];
  r[0] = 1.f - 2.f * (y * y + z * z); r[1] = 2.f * (x * y - w * z); r[2] = 2.f * (x * z + w * y);
  r[3] = 2.f * (x * y + w * z); r[4] = 1.f - 2.f * (x * x + z * z); r[5] = 2.f * (y * z - w * x);
  r[6] = 2.f * (x * z - w * y); r[7] = 2.f * (y * z + w * x); r[8] = 1.f - 2.f * (x * x + y * y);
  const float s[3] = {expf(ls[0]), expf(ls[1]), expf(ls[2])};
  float Mm[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) Mm[3 * a + k] = r[3 * a + k] * s[k];
  const float o = 1.0f / (1.0f + expf(-logit));

  float gp[3] = {0.f, 0.f, 0.f};
  float G3[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // dL/dSigma_3D (symmetric, full)
  float glogit = 0.f, gc[3] = {0.f, 0.f, 0.f};
  float S6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float vsum = 0.f, vcnt = 0.f;   // ADC statistics (f4): sum of ||dL/dPi(p)|| over visible views, count

  // Moments of view v + 1 are loaded (unconditionally: never-touched entries are zero) while view
  // v is processed, so each thread keeps one 48-B load in flight behind the arithmetic.
  const float4* mbase = reinterpret_cast<const float4*>(moments) + i * 3;
  const int64_t vstride = n * 3;  // float4 per view
  float4 na = __ldcg(mbase), nb = __ldcg(mbase + 1), nc = __ldcg(mbase + 2);
  for (int v = 0; v < V; ++v) {
    const float4 ma = na, mb = nb, mc = nc;
    if (v + 1 < V) {
      const float4* q = mbase + (int64_t)(v + 1) * vstride;
      na = __ldcg(q); nb = __ldcg(q + 1); nc = __ldcg(q + 2);
    }
    const float m0 = ma.x, m1x = ma.y, m1y = ma.z, Mxx = ma.w, Mxy = mb.x, Myy = mb.y;
    const float cg0 = mb.z, cg1 = mb.w, cg2 = mc.x;
    const bool vis = vstats != nullptr && __ldg(tiles_touched + (int64_t)v * n + i) > 0;
    if (vis) vcnt += 1.f;
    if (m0 == 0.f && m1x == 0.f && m1y == 0.f && Mxx == 0.f && Mxy == 0.f && Myy == 0.f && cg0 == 0.f &&
        cg1 == 0.f && cg2 == 0.f)
      continue;
    {
      float4* mp = reinterpret_cast<float4*>(moments) + ((int64_t)v * n + i) * 3;  // read-and-clear
      const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
      __stcg(mp, zero); __stcg(mp + 1, zero); __stcg(mp + 2, zero);
    }
    const steepgs_camera& c = cams.cam[v];
    const float* W = c.R;
    const float tx = W[0] * p0 + W[1] * p1 + W[2] * p2 + c.t[0];
    const float ty = W[3] * p0 + W[4] * p1 + W[5] * p2 + c.t[1];
    const float tz = W[6] * p0 + W[7] * p1 + W[8] * p2 + c.t[2];
    float J00, J02, J11, J12;
    const bool pin = c.model == 0;
    if (pin) {
      const float iz = 1.0f / tz;
      J00 = c.fx * iz; J02 = -c.fx * tx * iz * iz;
      J11 = c.fy * iz; J12 = -c.fy * ty * iz * iz;
    } else {
      J00 = c.fx; J02 = 0.f; J11 = c.fy; J12 = 0.f;
    }
    float P[6];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      P[b] = J00 * W[b] + J02 * W[6 + b];
      P[3 + b] = J11 * W[3 + b] + J12 * W[6 + b];
    }
    // Pi(Sigma) = (P M)(P M)^T + dil I with M = R diag(s); det from |m0 x m1|^2 (no cancellation)
    float m0v[3], m1v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      m0v[k] = P[0] * Mm[k] + P[1] * Mm[3 + k] + P[2] * Mm[6 + k];
      m1v[k] = P[3] * Mm[k] + P[4] * Mm[3 + k] + P[5] * Mm[6 + k];
    }
    float U[6];  // U = P Sigma = (P M) M^T
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      U[b] = m0v[0] * Mm[3 * b] + m0v[1] * Mm[3 * b + 1] + m0v[2] * Mm[3 * b + 2];
      U[3 + b] = m1v[0] * Mm[3 * b] + m1v[1] * Mm[3 * b + 1] + m1v[2] * Mm[3 * b + 2];
    }
    const float a00 = m0v[0] * m0v[0] + m0v[1] * m0v[1] + m0v[2] * m0v[2];
    const float a11 = m1v[0] * m1v[0] + m1v[1] * m1v[1] + m1v[2] * m1v[2];
    const float B = m0v[0] * m1v[0] + m0v[1] * m1v[1] + m0v[2] * m1v[2];
    const float cx0 = m0v[1] * m1v[2] - m0v[2] * m1v[1], cx1 = m0v[2] * m1v[0] - m0v[0] * m1v[2];
    const float cx2 = m0v[0] * m1v[1] - m0v[1] * m1v[0];
    const float dil = rk.dilation;
    const float A = a00 + dil, C = a11 + dil;
    const float idet = 1.0f / ((cx0 * cx0 + cx1 * cx1 + cx2 * cx2) + dil * (a00 + a11) + dil * dil);
    const float Qa = C * idet, Qb = -B * idet, Qc = A * idet;
    // dL/dmu = Q m1
    const float gmx = Qa * m1x + Qb * m1y, gmy = Qb * m1x + Qc * m1y;
    if (vis) vsum += sqrtf(gmx * gmx + gmy * gmy);
    // K = Q M Q (2x2 sym)
    const float QM00 = Qa * Mxx + Qb * Mxy, QM01 = Qa * Mxy + Qb * Myy;
    const float QM10 = Qb * Mxx + Qc * Mxy, QM11 = Qb * Mxy + Qc * Myy;
    const float K00 = QM00 * Qa + QM01 * Qb, K01 = QM00 * Qb + QM01 * Qc, K11 = QM10 * Qb + QM11 * Qc;
    // G2 = 1/2 K  -> dL/dSigma_3D += P^T G2 P ;  S += P^T (K - m0 Q) P
    const float H00 = K00 - m0 * Qa, H01 = K01 - m0 * Qb, H11 = K11 - m0 * Qc;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const float pa0 = P[a], pa1 = P[3 + a], pb0 = P[b], pb1 = P[3 + b];
        G3[3 * a + b] += 0.5f * (pa0 * (K00 * pb0 + K01 * pb1) + pa1 * (K01 * pb0 + K11 * pb1));
      }
    {
      int k = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b) {
          const float pa0 = P[a], pa1 = P[3 + a], pb0 = P[b], pb1 = P[3 + b];
          S6[k++] += pa0 * (H00 * pb0 + H01 * pb1) + pa1 * (H01 * pb0 + H11 * pb1);
        }
    }
    // mean path: dL/dt = J^T dL/dmu (+ J(t) terms for pinhole)
    float gtx = J00 * gmx, gty = J11 * gmy, gtz = J02 * gmx + J12 * gmy;
    if (pin) {
      // dL/dJ = 2 G2 (P Sigma W^T) = K X,  X = U W^T (2x3)
      float X[6];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) X[3 * a + b] = U[3 * a] * W[3 * b] + U[3 * a + 1] * W[3 * b + 1] + U[3 * a + 2] * W[3 * b + 2];
      const float dJ00 = K00 * X[0] + K01 * X[3];
      const float dJ02 = K00 * X[2] + K01 * X[5];
      const float dJ11 = K01 * X[1] + K11 * X[4];
      const float dJ12 = K01 * X[2] + K11 * X[5];
      const float iz = 1.0f / tz, iz2 = iz * iz, iz3 = iz2 * iz;
      gtx += -c.fx * iz2 * dJ02;
      gty += -c.fy * iz2 * dJ12;
      gtz += -c.fx * iz2 * dJ00 - c.fy * iz2 * dJ11 + 2.f * c.fx * tx * iz3 * dJ02 + 2.f * c.fy * ty * iz3 * dJ12;
    }
    gp[0] += W[0] * gtx + W[3] * gty + W[6] * gtz;
    gp[1] += W[1] * gtx + W[4] * gty + W[7] * gtz;
    gp[2] += W[2] * gtx + W[5] * gty + W[8] * gtz;
    glogit += m0 * (1.0f - o);
    gc[0] += cg0; gc[1] += cg1; gc[2] += cg2;
  }

  // Sigma = M M^T, M = R diag(s):  dL/dM = 2 G3 M ; dL/ds_k = sum_j R_jk dLdM_jk ; dL/dR_jk = dLdM_jk s_k
  float dM[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) dM[3 * a + k] = 2.f * (G3[3 * a] * Mm[k] + G3[3 * a + 1] * Mm[3 + k] + G3[3 * a + 2] * Mm[6 + k]);
  float gls[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) gls[k] = s[k] * (r[k] * dM[k] + r[3 + k] * dM[3 + k] + r[6 + k] * dM[6 + k]);
  float G[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) G[3 * a + k] = dM[3 * a + k] * s[k];
  // dL/dq_hat from R(q_hat) (C1)
  const float gw = 2.f * (-z * G[1] + y * G[2] + z * G[3] - x * G[5] - y * G[6] + x * G[7]);
  const float gx = 2.f * (y * G[1] + z * G[2] + y * G[3] - 2.f * x * G[4] - w * G[5] + z * G[6] + w * G[7] - 2.f * x * G[8]);
  const float gy = 2.f * (-2.f * y * G[0] + x * G[1] + w * G[2] + x * G[3] + z * G[5] - w * G[6] + z * G[7] - 2.f * y * G[8]);
  const float gz = 2.f * (-2.f * z * G[0] - w * G[1] + x * G[2] + w * G[3] - 2.f * z * G[4] + y * G[5] + x * G[6] + y * G[7]);
  const float dot = w * gw + x * gx + y * gy + z * gz;
  const float iq = 1.0f / qn;
  const float gq[4] = {(gw - w * dot) * iq, (gx - x * dot) * iq, (gy - y * dot) * iq, (gz - z * dot) * iq};

  float out[20];
  out[0] = gp[0]; out[1] = gp[1]; out[2] = gp[2];
  out[3] = gls[0]; out[4] = gls[1]; out[5] = gls[2];
  out[6] = gq[0]; out[7] = gq[1]; out[8] = gq[2]; out[9] = gq[3];
  out[10] = glogit;
  out[11] = gc[0]; out[12] = gc[1]; out[13] = gc[2];
#pragma unroll
  for (int k = 0; k < 6; ++k) out[14 + k] = S6[k];
  // accumulate & 3: 0 = overwrite all 20 planes, 1 = += all, 2 = overwrite the 14 gradient planes and
  // += the 6 S planes (Alg. 1: per-step gradients for the optimizer, S summed over T_split steps).
  // accumulate & 4 (SH colour, f3): k_sh_bwd has written planes 0-2 (view-direction term) and 11-13
  // (DC coefficients) for this call, so planes 0-2 are added to and 11-13 left alone.
  if (sc.R > 0) {   // fused reduce-scatter: this rank's partial goes straight to the owner of column i
    const int q = (int)(i / sc.chunk);
    const int64_t j = i - (int64_t)q * sc.chunk;
    float* dst = sc.peers[q] + (int64_t)sc.rank * 20 * sc.chunk + j;
#pragma unroll
    for (int k = 0; k < 20; ++k) dst[(int64_t)k * sc.chunk] = out[k];   // coalesced over i (P2P over NVLink)
    return;
  }
  const int mode = accumulate & 3;
  const bool shm = (accumulate & 4) != 0;
  const bool acc_g = mode == 1, acc_s = mode != 0;
#pragma unroll
  for (int k = 0; k < 14; ++k) {
    if (shm && k >= 11) continue;
    grad_S[k * ldg + i] = (acc_g || (shm && k < 3)) ? grad_S[k * ldg + i] + out[k] : out[k];
  }
#pragma unroll
  for (int k = 14; k < 20; ++k) grad_S[k * ldg + i] = acc_s ? grad_S[k * ldg + i] + out[k] : out[k];
  if (vstats) {   // same window semantics as S: mode 0 opens a new window
    vstats[i] = mode ? vstats[i] + vsum : vsum;
    vstats[ldg + i] = mode ? vstats[ldg + i] + vcnt : vcnt;
  }
}

// The owner's half of the fused reduce (rank q owns columns [q chunk, q chunk + len)): sums the R
// partials the ranks' k_gauss_bwd stored into its buffer, applies the accumulate mode of the 20
// planes (the owner's grad_S equals every rank's: they are replicated), and stores the result into
// every rank's grad_S (P2P stores over NVLink: the all-gather, fused into the reduction).
__global__ void __launch_bounds__(256) k_reduce_bcast(const float* __restrict__ partials, int R, int rank,
                                                      int64_t n, int64_t chunk, const PeerPtrs gs, int64_t ldg,
                                                      int accumulate) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = (int64_t)rank * chunk + j;
  if (j >= chunk || i >= n) return;
  const int mode = accumulate & 3;
  const float* own = gs.p[rank];
#pragma unroll 4
  for (int k = 0; k < 20; ++k) {
    float v = 0.0f;
    for (int r = 0; r < R; ++r) v += partials[((int64_t)r * 20 + k) * chunk + j];   // rank order
    const bool acc = k < 14 ? mode == 1 : mode != 0;
    if (acc) v = own[(int64_t)k * ldg + i] + v;
    for (int t = 0; t < R; ++t) gs.p[t][(int64_t)k * ldg + i] = v;
  }
}

}  // namespace

cudaError_t launch_gauss_bwd(const float* params, int64_t ld, int64_t n, const CamPack& cams, int V,
                             const RasterK& rk, float* moments, float* grad_S, int64_t ldg, int accumulate,
                             const int32_t* tiles_touched, float* view_grad_stats, cudaStream_t st,
                             const ScatterOut& sc) {
  if (n == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((n + 127) / 128);
  // launched without the programmatic-dependent attribute: with it, the whole-step graph measured
  // 60-70 us slower per C2 step (its blocks parked on griddepcontrol.wait during render_bwd's tail)
  launch_k<false>(k_gauss_bwd, dim3(blocks), dim3(128), 0, st, params, ld, n, cams, V, rk, moments, grad_S, ldg, accumulate,
             tiles_touched, view_grad_stats, sc);
  note_launch();
  return check_launch("k_gauss_bwd");
}

cudaError_t launch_reduce_bcast(const float* partials, int R, int rank, int64_t n, int64_t chunk, const PeerPtrs& gs,
                                int64_t ldg, int accumulate, cudaStream_t st) {
  const int64_t len = chunk;
  if (len <= 0 || (int64_t)rank * chunk >= n) return cudaSuccess;
  k_reduce_bcast<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(partials, R, rank, n, chunk, gs, ldg, accumulate);
  note_launch();
  return check_launch("k_reduce_bcast");
}

}  // namespace sgs
