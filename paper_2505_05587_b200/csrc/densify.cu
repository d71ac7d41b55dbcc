// densify.cu — a8: steepest density control (Thm 2; Alg. 1 densify branch,
// P:L541-548; closed-form 3x3 eigen, App. A.3).
//
//   k_densify_decide  per Gaussian: S_bar = S / denom; lambda_min by the trigonometric
//                     roots (k = 1 root, Z19) in fp32, re-evaluated in fp64 when it falls within a
//                     guard band of eps_split; split iff lambda_min < eps_split (strict, Z11);
//                     single-pass exclusive scan of the mask (decoupled look-back) -> dest_index.
//   k_densify_apply   capacity check on the device (C16); S planes zeroed on [0, n + n_split) (Z23);
//                     for split parents: unit v_min (robust cross-product / 2x2-complement method,
//                     canonical sign, C13), eps = eta sqrt(v^T Sigma v) (Z13), offspring
//                     A = (p + eps v, o/2) in place, B = (p - eps v, o/2) appended at n + rank (Z24),
//                     log-scale / quaternion / colour copied (Z14).
// With capacity >= 2n (a densify can at most double n) both steps run as one fused kernel.
// Bound: HBM (~53 B per Gaussian + 192 B per split).
#include <math.h>

#include "common.cuh"
#include "scan.cuh"

namespace sgs {

SGS_CHECKS_TU(densify)

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTileItems = kThreads * kItems;

__device__ __forceinline__ double eig_min_f64(const float* S6) {
  const double a = S6[0], b = S6[1], c = S6[2], d = S6[3], g = S6[4], f = S6[5];
  const double q = (a + d + f) / 3.0;
  const double A = a - q, D = d - q, F = f - q;
  const double p = sqrt((A * A + D * D + F * F + 2.0 * (b * b + c * c + g * g)) / 6.0);
  if (p <= 1e-12 * (1.0 + fabs(q))) return q;
  const double Ba = A / p, Bb = b / p, Bc = c / p, Bd = D / p, Be = g / p, Bf = F / p;
  const double det = Ba * (Bd * Bf - Be * Be) - Bb * (Bb * Bf - Be * Bc) + Bc * (Bb * Be - Bd * Bc);
  const double r = fmin(1.0, fmax(-1.0, 0.5 * det));
  return q + 2.0 * p * cos(acos(r) / 3.0 + 2.0943951023931957);
}

__device__ __forceinline__ void load_sbar(const float* __restrict__ grad_S, int64_t ldg, int64_t i, float inv_denom,
                                          float* S6) {
#pragma unroll
  for (int k = 0; k < 6; ++k) S6[k] = grad_S[(14 + k) * ldg + i] * inv_denom;
}

// largest cross product of two rows of (S - lam I) -> unit vector (or false if all vanish)
__device__ __forceinline__ bool null_vector(const float* S6, float lam, float* v) {
  const float r0[3] = {S6[0] - lam, S6[1], S6[2]};
  const float r1[3] = {S6[1], S6[3] - lam, S6[4]};
  const float r2[3] = {S6[2], S6[4], S6[5] - lam};
  const float c01[3] = {r0[1] * r1[2] - r0[2] * r1[1], r0[2] * r1[0] - r0[0] * r1[2], r0[0] * r1[1] - r0[1] * r1[0]};
  const float c02[3] = {r0[1] * r2[2] - r0[2] * r2[1], r0[2] * r2[0] - r0[0] * r2[2], r0[0] * r2[1] - r0[1] * r2[0]};
  const float c12[3] = {r1[1] * r2[2] - r1[2] * r2[1], r1[2] * r2[0] - r1[0] * r2[2], r1[0] * r2[1] - r1[1] * r2[0]};
  const float n01 = c01[0] * c01[0] + c01[1] * c01[1] + c01[2] * c01[2];
  const float n02 = c02[0] * c02[0] + c02[1] * c02[1] + c02[2] * c02[2];
  const float n12 = c12[0] * c12[0] + c12[1] * c12[1] + c12[2] * c12[2];
  float nb = n01;
  v[0] = c01[0]; v[1] = c01[1]; v[2] = c01[2];
  if (n02 > nb) { nb = n02; v[0] = c02[0]; v[1] = c02[1]; v[2] = c02[2]; }
  if (n12 > nb) { nb = n12; v[0] = c12[0]; v[1] = c12[1]; v[2] = c12[2]; }
  if (!(nb > 0.f)) return false;
  const float in = rsqrtf(nb);
  v[0] *= in; v[1] *= in; v[2] *= in;
  return true;
}

// Fallback when every cross product of the rows of (S - lambda I) vanishes in fp32: inverse iteration
// in fp64 on (S - mu I), mu just below lambda (three steps from (1, 1, 1); the solve by the adjugate,
// which stays finite when the shifted matrix is nearly singular — that is what makes it converge).
__device__ void inverse_iteration(const float* S6, float lam, float* v) {
  const double a = S6[0], b = S6[1], c = S6[2], d = S6[3], e = S6[4], f = S6[5];
  const double sc = fmax(fmax(fabs(a), fabs(d)), fmax(fabs(f), fmax(fabs(b), fmax(fabs(c), fabs(e)))));
  const double mu = (double)lam - 1e-6 * sc;
  const double A = a - mu, D = d - mu, F = f - mu;
  // adjugate of the symmetric [[A, b, c], [b, D, e], [c, e, F]]
  const double j00 = D * F - e * e, j01 = c * e - b * F, j02 = b * e - c * D;
  const double j11 = A * F - c * c, j12 = b * c - A * e, j22 = A * D - b * b;
  double x0 = 1.0, x1 = 1.0, x2 = 1.0;
  for (int it = 0; it < 3; ++it) {
    const double y0 = j00 * x0 + j01 * x1 + j02 * x2;
    const double y1 = j01 * x0 + j11 * x1 + j12 * x2;
    const double y2 = j02 * x0 + j12 * x1 + j22 * x2;
    const double nn = sqrt(y0 * y0 + y1 * y1 + y2 * y2);
    if (!(nn > 0.0)) break;
    x0 = y0 / nn; x1 = y1 / nn; x2 = y2 / nn;
  }
  v[0] = (float)x0; v[1] = (float)x1; v[2] = (float)x2;
}

// lambda_min and (optionally) unit v_min of the symmetric S6 = (xx,xy,xz,yy,yz,zz), fp32.
// Eigenvalues by Smith's trigonometric roots (App. A.3: q = tr/3, p, B = (A - qI)/p,
// beta = 2 cos(acos(det B / 2)/3 + 2k pi/3)), organised so both outputs stay accurate when two
// roots nearly coincide: with r = det(B)/2 >= 0 the maximum root (k = 0) is the isolated one, so
// v_max comes from a cross product and (lambda_min, v_min) from the 2x2 problem in its orthogonal
// complement; with r < 0 the minimum root (k = 1, Z19) is isolated and is used directly.
__device__ void eig_min_robust(const float* S6in, bool want_vec, float& lam, float* v) {
  v[0] = 1.f; v[1] = 0.f; v[2] = 0.f;
  float sc = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) sc = fmaxf(sc, fabsf(S6in[k]));
  if (!(sc > 0.f)) { lam = 0.f; return; }                      // zero matrix
  const float is = 1.0f / sc;
  float S6[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) S6[k] = S6in[k] * is;
  const float q = (S6[0] + S6[3] + S6[5]) * (1.0f / 3.0f);
  const float A = S6[0] - q, D = S6[3] - q, F = S6[5] - q;
  const float p = sqrtf((A * A + D * D + F * F + 2.0f * (S6[1] * S6[1] + S6[2] * S6[2] + S6[4] * S6[4])) * (1.0f / 6.0f));
  if (p * sc <= 1e-12f * (1.0f + fabsf(q * sc))) { lam = q * sc; return; }   // S ~ qI: v = e_x (Z17)
  const float ip = 1.0f / p;
  const float Ba = A * ip, Bb = S6[1] * ip, Bc = S6[2] * ip, Bd = D * ip, Be = S6[4] * ip, Bf = F * ip;
  const float det = Ba * (Bd * Bf - Be * Be) - Bb * (Bb * Bf - Be * Bc) + Bc * (Bb * Be - Bd * Bc);
  const float r = fminf(1.0f, fmaxf(-1.0f, 0.5f * det));        // Z18
  const float phi = acosf(r) * (1.0f / 3.0f);
  bool have_vec = false;
  if (r >= 0.f) {
    const float lmax = q + 2.0f * p * cosf(phi);
    float u3[3];
    if (null_vector(S6, lmax, u3)) {
      float a[3];
      if (fabsf(u3[0]) > fabsf(u3[1])) {
        const float il = rsqrtf(u3[0] * u3[0] + u3[2] * u3[2]);
        a[0] = -u3[2] * il; a[1] = 0.f; a[2] = u3[0] * il;
      } else {
        const float il = rsqrtf(u3[1] * u3[1] + u3[2] * u3[2]);
        a[0] = 0.f; a[1] = u3[2] * il; a[2] = -u3[1] * il;
      }
      const float b[3] = {u3[1] * a[2] - u3[2] * a[1], u3[2] * a[0] - u3[0] * a[2], u3[0] * a[1] - u3[1] * a[0]};
      const float Sa[3] = {S6[0] * a[0] + S6[1] * a[1] + S6[2] * a[2], S6[1] * a[0] + S6[3] * a[1] + S6[4] * a[2],
                           S6[2] * a[0] + S6[4] * a[1] + S6[5] * a[2]};
      const float Sb[3] = {S6[0] * b[0] + S6[1] * b[1] + S6[2] * b[2], S6[1] * b[0] + S6[3] * b[1] + S6[4] * b[2],
                           S6[2] * b[0] + S6[4] * b[1] + S6[5] * b[2]};
      const float m00 = a[0] * Sa[0] + a[1] * Sa[1] + a[2] * Sa[2];
      const float m01 = a[0] * Sb[0] + a[1] * Sb[1] + a[2] * Sb[2];
      const float m11 = b[0] * Sb[0] + b[1] * Sb[1] + b[2] * Sb[2];
      const float hd = 0.5f * (m00 - m11);
      const float rad = sqrtf(hd * hd + m01 * m01);
      lam = (0.5f * (m00 + m11) - rad) * sc;
      if (want_vec) {
        // min eigenvector of [[m00, m01], [m01, m11]]: orthogonal to the larger row of (M - lam2 I)
        const float e0 = hd + rad, e1 = rad - hd;               // m00 - lam2, m11 - lam2 (>= 0)
        float c0, c1;
        if (e0 >= e1) { c0 = -m01; c1 = e0; } else { c0 = e1; c1 = -m01; }
        const float nn = c0 * c0 + c1 * c1;
        if (nn > 0.f) { const float in = rsqrtf(nn); c0 *= in; c1 *= in; } else { c0 = 1.f; c1 = 0.f; }
        v[0] = c0 * a[0] + c1 * b[0];
        v[1] = c0 * a[1] + c1 * b[1];
        v[2] = c0 * a[2] + c1 * b[2];
        have_vec = true;
      }
    } else {
      lam = (q + 2.0f * p * cosf(phi + 2.0943951023931957f)) * sc;
    }
  } else {
    const float l = q + 2.0f * p * cosf(phi + 2.0943951023931957f);  // k = 1 root is the minimum (Z19)
    lam = l * sc;
    if (want_vec) have_vec = null_vector(S6, l, v);
  }
  if (!want_vec) return;
  if (!have_vec) inverse_iteration(S6, lam / sc, v);   // (scaled S6; no arbitrary e_x)
  const float nn = rsqrtf(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  v[0] *= nn; v[1] *= nn; v[2] *= nn;
  int big = 0;  // canonical sign: largest |component| positive, ties -> lowest index (C13)
  if (fabsf(v[1]) > fabsf(v[big])) big = 1;
  if (fabsf(v[2]) > fabsf(v[big])) big = 2;
  if (v[big] < 0.f) { v[0] = -v[0]; v[1] = -v[1]; v[2] = -v[2]; }
}

// lambda_min for the split decision; with v != nullptr also the unit v_min of the same fp32 solve (the
// fused kernel keeps it for the offspring instead of solving again: bit-identical to spawn_prepare's).
__device__ __forceinline__ float decide_lambda(const float* S6, float eps_split, float* v = nullptr) {
  float lam, vv[3];
  eig_min_robust(S6, v != nullptr, lam, v != nullptr ? v : vv);
  float fro = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) fro += (k == 1 || k == 2 || k == 4 ? 2.f : 1.f) * S6[k] * S6[k];
  fro = sqrtf(fro);
  // guard band: within 1e-5 ||S||_F of eps_split the decision is taken on the fp64 eigenvalue.  The
  // fp32 lambda_min is accurate to O(10 eps) ||S||_F ~ 1e-6 ||S||_F: the r < 0 root is first-order
  // insensitive to r near -1, and for r >= 0 it comes from the 2x2 complement of the isolated
  // lambda_max; tests/test_gpu_parity.py::test_densify_decisions_near_the_threshold checks 120k
  // matrices at 1e-7 .. 1e-3 ||S||_F from the threshold (no band: mismatches; 1e-3 (round 1): densify
  // 0.080 vs 0.075 ms per C2 step, warps entering the fp64 path)
  if (fabsf(lam - eps_split) <= 1e-5f * fro + 1e-30f) lam = (float)eig_min_f64(S6);
  return lam;
}

// Offspring of split parent i (Thm 2 / Alg. 1): A in slot i at p + eps v, B in slot b at
// p - eps v, both with opacity logit(o/2) (Z15), other planes copied (Z14); B's accumulators zeroed.
// Split in two so the fused kernel can do the arithmetic and the parent loads before its look-back
// completes and only the stores after it.
struct Spawn {
  float v[3], eps, p[3], lg;
  float rest[10];   // planes 3-9 (log-scale, quaternion) and 11-13 (colour)
};

// v_min: given (the decide step already solved), else solved here from S6.
__device__ __forceinline__ void spawn_prepare(const float* __restrict__ params, int64_t ld, int64_t i,
                                              const float* S6, const float* vmin, float eta, float eps_abs,
                                              Spawn& sp) {
  if (vmin != nullptr) {
    sp.v[0] = vmin[0]; sp.v[1] = vmin[1]; sp.v[2] = vmin[2];
  } else {
    float lam_unused;
    eig_min_robust(S6, true, lam_unused, sp.v);
  }
  // parent: p, Sigma = R diag(s^2) R^T, o
  sp.p[0] = params[0 * ld + i]; sp.p[1] = params[1 * ld + i]; sp.p[2] = params[2 * ld + i];
#pragma unroll
  for (int k = 0; k < 7; ++k) sp.rest[k] = params[(3 + k) * ld + i];
#pragma unroll
  for (int k = 0; k < 3; ++k) sp.rest[7 + k] = params[(11 + k) * ld + i];
  float eps = eps_abs;
  if (eta >= 0.f) {
    const float qw = sp.rest[3], qx = sp.rest[4], qy = sp.rest[5], qz = sp.rest[6];
    const float qn = rsqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
    const float w = qw * qn, x = qx * qn, y = qy * qn, z = qz * qn;
    const float r[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                        2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                        2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
    float vsv = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float s = expf(sp.rest[k]);
      const float rv = r[k] * sp.v[0] + r[3 + k] * sp.v[1] + r[6 + k] * sp.v[2];
      vsv += s * s * rv * rv;
    }
    eps = eta * sqrtf(vsv);
  }
  sp.eps = eps;
  // Z15: w = 1/2 absorbed in opacity, logit(sigmoid(x) / 2) = -log(1 + 2 e^-x) (fp64, then rounded)
  sp.lg = (float)(-log1p(2.0 * exp(-(double)params[10 * ld + i])));
}

__device__ __forceinline__ void spawn_commit(float* __restrict__ params, int64_t ld, float* __restrict__ grad_S,
                                             int64_t ldg, int64_t i, int64_t b, const Spawn& sp) {
#pragma unroll
  for (int k = 0; k < 7; ++k) params[(3 + k) * ld + b] = sp.rest[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) params[(11 + k) * ld + b] = sp.rest[7 + k];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    params[a * ld + b] = sp.p[a] - sp.eps * sp.v[a];
    params[a * ld + i] = sp.p[a] + sp.eps * sp.v[a];
  }
  params[10 * ld + b] = sp.lg;
  params[10 * ld + i] = sp.lg;
#pragma unroll
  for (int k = 0; k < 20; ++k) grad_S[k * ldg + b] = 0.f;
}

__device__ __forceinline__ void spawn(float* __restrict__ params, int64_t ld, float* __restrict__ grad_S,
                                      int64_t ldg, int64_t i, int64_t b, const float* S6, float eta, float eps_abs) {
  Spawn sp;
  spawn_prepare(params, ld, i, S6, nullptr, eta, eps_abs, sp);
  spawn_commit(params, ld, grad_S, ldg, i, b, sp);
}

// gate 1 — compactest (App. A.2): ||G_p / denom||_2 <= eps_grad on the position gradient;
// gate 2 — Alg. 1's "condition on G" read as 3DGS's densification condition (C24): the mean view-space
// gradient norm (planes 0, 1 = sum of ||dL/dPi(p)||, visible views) >= eps_grad.
__device__ __forceinline__ bool gate_ok(const float* __restrict__ grad_S, int64_t ldg, int64_t i, float inv_denom,
                                        int gate, float eps_grad) {
  if (gate == 2) {
    const float cnt = grad_S[1 * ldg + i];
    return cnt > 0.0f && __fdiv_rn(grad_S[0 * ldg + i], cnt) >= eps_grad;
  }
  const float g0 = grad_S[0 * ldg + i] * inv_denom, g1 = grad_S[1 * ldg + i] * inv_denom;
  const float g2 = grad_S[2 * ldg + i] * inv_denom;
  return sqrtf(g0 * g0 + g1 * g1 + g2 * g2) <= eps_grad;
}

__device__ __forceinline__ uint32_t orderable(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// ---- increment budget (App. A.2): keep the `budget` least lambda_min among the
// candidates, ties by index.  Radix select of the threshold key over 4 byte-passes on the device. --
struct SelState {
  uint32_t hist[256];
  uint32_t prefix, pmask, remaining, count;
};

__global__ void __launch_bounds__(kThreads) k_budget_keys(const float* __restrict__ grad_S, int64_t ldg, int64_t n,
                                                          float inv_denom, float eps_split, int gate, float eps_grad,
                                                          uint32_t* __restrict__ keys, float* __restrict__ lambda,
                                                          SelState* st) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool cand = false;
  if (i < n) {
    float S6[6];
    load_sbar(grad_S, ldg, i, inv_denom, S6);
    const float lam = decide_lambda(S6, eps_split);
    if (lambda) lambda[i] = lam;
    cand = lam < eps_split && (!gate || gate_ok(grad_S, ldg, i, inv_denom, gate, eps_grad));
    keys[i] = cand ? orderable(lam) : 0xFFFFFFFFu;
  }
  const uint32_t b = __ballot_sync(0xffffffffu, cand);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(&st->count, (uint32_t)__popc(b));
}

__global__ void __launch_bounds__(kThreads) k_select_hist(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                          int64_t budget, SelState* st) {
  if ((int64_t)st->count <= budget) return;  // every candidate is kept: nothing to select
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0u;
  __syncthreads();
  const uint32_t prefix = st->prefix, pmask = st->pmask;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    if (k != 0xFFFFFFFFu && (k & pmask) == prefix) atomicAdd(&h[(k >> shift) & 255u], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_select_pick(int shift, int64_t budget, SelState* st) {
  if ((int64_t)st->count <= budget) return;
  __shared__ uint32_t s_warp[8];
  const int d = threadIdx.x, lane = d & 31, warp = d >> 5;
  const uint32_t c = st->hist[d];
  uint32_t inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  uint32_t wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += s_warp[w];
  const uint32_t excl = wpre + inc - c;
  const uint32_t rem = shift == 24 ? (uint32_t)budget : st->remaining;
  __syncthreads();
  if (rem == 0u) {                       // budget 0: select nothing
    if (d == 0) { st->prefix = 0u; st->pmask = 0xFFFFFFFFu; st->remaining = 0u; }
  } else if (excl < rem && rem <= excl + c) {
    st->prefix |= (uint32_t)d << shift;
    st->pmask |= 0xFFu << shift;
    st->remaining = rem - excl;
  }
  st->hist[d] = 0u;
}

// kFused (capacity >= 2n, so n + n_split <= capacity holds for any mask): the same kernel also
// writes the offspring and clears S, one pass over the data and no second launch.
// kSel: the split set was already chosen (budget path): split = candidate key < threshold, or
// == threshold within the first `remaining` ties in index order (tie ranks by this kernel's scan of
// the ties would need a second look-back; ties are resolved by k_budget_ties first).
template <bool kFused, int kIt, bool kSel>
__global__ void __launch_bounds__(kThreads) k_densify_decide(float* __restrict__ params, int64_t ld,
                                                             float* __restrict__ grad_S, int64_t ldg, int64_t n,
                                                             float inv_denom, float eps_split, float eta, float eps_abs,
                                                             int gate, float eps_grad,
                                                             const uint8_t* __restrict__ sel,
                                                             uint8_t* __restrict__ mask, int32_t* __restrict__ dest,
                                                             float* __restrict__ lambda, uint64_t* status,
                                                             int* tile_counter, int64_t* n_split,
                                                             int32_t* __restrict__ dstatus) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_tile;
  __shared__ uint32_t s_cnt[kIt][kThreads / 32];
  __shared__ uint64_t s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * (kThreads * kIt);
  bool split[kIt];
  uint32_t pos[kIt];
  // fused: v_min kept for the offspring (decide path), or S_bar to solve it (budget path)
  float S6k[kFused && kSel ? kIt : 1][6];
  float vk[kFused && !kSel ? kIt : 1][3];
#pragma unroll
  for (int j = 0; j < kIt; ++j) {
    const int64_t i = base + (int64_t)j * kThreads + tid;
    split[j] = false;
    if (i < n) {
      float S6[6];
      if (kSel) {
        split[j] = sel[i] != 0;
        if (kFused && split[j]) load_sbar(grad_S, ldg, i, inv_denom, S6);
      } else {
        load_sbar(grad_S, ldg, i, inv_denom, S6);
        const float lam = decide_lambda(S6, eps_split, kFused ? vk[kFused && !kSel ? j : 0] : nullptr);
        split[j] = lam < eps_split;                   // Thm 2 / Alg. 1 P:L545 (strict, Z11)
        if (gate && split[j]) split[j] = gate_ok(grad_S, ldg, i, inv_denom, gate, eps_grad);
        if (lambda) lambda[i] = lam;
      }
      if (kFused && kSel) {
#pragma unroll
        for (int k = 0; k < 6; ++k) S6k[kFused && kSel ? j : 0][k] = S6[k];
      }
    }
    const uint32_t b = __ballot_sync(0xffffffffu, split[j]);
    pos[j] = __popc(b & lanemask_lt());
    if (lane == 0) s_cnt[j][warp] = __popc(b);
  }
  __syncthreads();
  __shared__ uint32_t s_agg;
  if (warp == 0) {
    constexpr int nw = kThreads / 32, nv = kIt * nw;   // <= 64 counts, two per lane, (j, warp) order
    uint32_t* cnt = &s_cnt[0][0];
    const uint32_t a = 2 * lane < nv ? cnt[2 * lane] : 0u, bb = 2 * lane + 1 < nv ? cnt[2 * lane + 1] : 0u;
    uint32_t sum = a + bb, inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t ex = inc - sum;
    if (2 * lane < nv) cnt[2 * lane] = ex;
    if (2 * lane + 1 < nv) cnt[2 * lane + 1] = ex + a;
    const uint32_t agg = __shfl_sync(0xffffffffu, inc, 31);
    if (lane == 0) {
      publish_aggregate(status, tile, agg);        // early: successors can look past this tile
      s_agg = agg;
    }
  }
  // fused: the offspring arithmetic and parent loads overlap the look-back
  Spawn sp[kFused ? kIt : 1];
  if (kFused) {
#pragma unroll
    for (int j = 0; j < kIt; ++j) {
      const int64_t i = base + (int64_t)j * kThreads + tid;
      if (i < n && split[j])
        spawn_prepare(params, ld, i, S6k[kFused && kSel ? j : 0], kSel ? nullptr : vk[kFused && !kSel ? j : 0], eta,
                      eps_abs, sp[kFused ? j : 0]);
    }
  }
  if (warp == 0) {
    const uint32_t agg = __shfl_sync(0xffffffffu, s_agg, 0);
    const uint64_t excl = lookback_published(status, tile, agg);
    if (lane == 0) {
      s_excl = excl;
      if (base + kThreads * kIt >= n) *n_split = (int64_t)(excl + agg);
    }
  }
  __syncthreads();
  if (kFused && tile == 0 && tid == 0) *dstatus = 0;
#pragma unroll
  for (int j = 0; j < kIt; ++j) {
    const int64_t i = base + (int64_t)j * kThreads + tid;
    if (i >= n) continue;
    const int64_t b = n + (int64_t)(s_excl + s_cnt[j][warp] + pos[j]);
    mask[i] = split[j] ? 1 : 0;
    dest[i] = split[j] ? (int32_t)b : -1;  // Z24
    SGS_CHECK(!split[j] || (b >= n && b < 2 * n));            // (the fused path needs capacity >= 2n)
    if (kFused) {
#pragma unroll
      for (int k = 14; k < 20; ++k) grad_S[k * ldg + i] = 0.f;   // Z23
      if (split[j]) spawn_commit(params, ld, grad_S, ldg, i, b, sp[kFused ? j : 0]);
    }
  }
}

// Budget path, final selection: sel = key < t, or key == t and among the first `remaining` ties of t in
// index order (decoupled look-back scan of the tie flags).  With count <= budget every candidate is kept.
__global__ void __launch_bounds__(kThreads) k_budget_ties(const uint32_t* __restrict__ keys, int64_t n, int64_t budget,
                                                          const SelState* st, uint8_t* __restrict__ sel,
                                                          uint64_t* status, int* tile_counter) {
  __shared__ int s_tile;
  __shared__ uint32_t s_cnt[kItems][kThreads / 32];
  __shared__ uint64_t s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * kTileItems;
  const bool all = (int64_t)st->count <= budget;
  const uint32_t t = st->prefix, rem = st->remaining;
  bool tie[kItems];
  uint32_t key[kItems], pos[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int64_t i = base + (int64_t)j * kThreads + tid;
    key[j] = i < n ? keys[i] : 0xFFFFFFFFu;
    tie[j] = !all && key[j] != 0xFFFFFFFFu && key[j] == t;
    const uint32_t b = __ballot_sync(0xffffffffu, tie[j]);
    pos[j] = __popc(b & lanemask_lt());
    if (lane == 0) s_cnt[j][warp] = __popc(b);
  }
  __syncthreads();
  if (warp == 0) {
    constexpr int nw = kThreads / 32;
    uint32_t* cnt = &s_cnt[0][0];
    const uint32_t a = cnt[2 * lane], bb = cnt[2 * lane + 1];
    uint32_t sum = a + bb, inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    const uint32_t ex = inc - sum;
    cnt[2 * lane] = ex;
    cnt[2 * lane + 1] = ex + a;
    const uint32_t agg = __shfl_sync(0xffffffffu, inc, 31);
    const uint64_t excl = lookback_warp(status, tile, agg);
    if (lane == 0) s_excl = excl;
    (void)nw;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int64_t i = base + (int64_t)j * kThreads + tid;
    if (i >= n) continue;
    bool s = false;
    if (key[j] != 0xFFFFFFFFu) {
      if (all) s = true;
      else if (key[j] < t) s = true;
      else if (tie[j]) s = (s_excl + s_cnt[j][warp] + pos[j]) < rem;
    }
    sel[i] = s ? 1 : 0;
  }
}

__global__ void __launch_bounds__(kThreads) k_densify_apply(float* __restrict__ params, int64_t ld, int64_t n,
                                                            int64_t capacity, float* __restrict__ grad_S, int64_t ldg,
                                                            float inv_denom, float eta, float eps_abs,
                                                            const uint8_t* __restrict__ mask,
                                                            const int32_t* __restrict__ dest,
                                                            const int64_t* __restrict__ n_split,
                                                            int32_t* __restrict__ status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ns = *n_split;
  const bool ok = n + ns <= capacity;
  if (i == 0) *status = ok ? 0 : (int32_t)STEEPGS_ERR_CAPACITY;
  if (!ok || i >= n) return;
  float S6[6];
  load_sbar(grad_S, ldg, i, inv_denom, S6);
#pragma unroll
  for (int k = 14; k < 20; ++k) grad_S[k * ldg + i] = 0.f;
  if (!mask[i]) return;
  SGS_CHECK(dest[i] >= n && dest[i] < n + ns);
  spawn(params, ld, grad_S, ldg, i, dest[i], S6, eta, eps_abs);
}


inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

constexpr int kItemsFused = 1;   // one Gaussian per thread when the offspring are written too

namespace {
struct DensWs {
  size_t st_decide, st_ties, counters, sel_state, keys, sel, end;
};
DensWs dens_layout(int64_t n) {
  DensWs L;
  const int64_t tiles1 = (n + kThreads * kItemsFused - 1) / (kThreads * kItemsFused);
  const int64_t tiles8 = (n + kTileItems - 1) / kTileItems;
  size_t o = 0;
  auto take = [&](size_t b) { const size_t at = o; o = align_up(o + b); return at; };
  L.st_decide = take(8 * (size_t)(tiles1 > 0 ? tiles1 : 1));
  L.st_ties = take(8 * (size_t)(tiles8 > 0 ? tiles8 : 1));
  L.counters = take(16 * sizeof(int));
  L.sel_state = take(sizeof(SelState));
  L.keys = take(4 * (size_t)(n > 0 ? n : 1));
  L.sel = take((size_t)(n > 0 ? n : 1));
  L.end = o;
  return L;
}
}  // namespace

size_t densify_ws_bytes(int64_t n) { return dens_layout(n).end; }

cudaError_t launch_densify(float* params, int64_t ld, int64_t n, int64_t capacity, float* grad_S, int64_t ldg,
                           const steepgs_densify_params& dp, uint8_t* mask, int32_t* dest, float* lambda,
                           int64_t* n_split, int32_t* status, void* ws, size_t ws_bytes, cudaStream_t st) {
  const DensWs L = dens_layout(n);
  if (ws_bytes < L.end) return cudaErrorInvalidValue;
  const bool fused = capacity >= 2 * n;
  const bool budget = dp.budget >= 0;
  char* w = static_cast<char*>(ws);
  uint64_t* st_decide = reinterpret_cast<uint64_t*>(w + L.st_decide);
  uint64_t* st_ties = reinterpret_cast<uint64_t*>(w + L.st_ties);
  int* counter = reinterpret_cast<int*>(w + L.counters);
  SelState* sst = reinterpret_cast<SelState*>(w + L.sel_state);
  uint32_t* keys = reinterpret_cast<uint32_t*>(w + L.keys);
  uint8_t* sel = reinterpret_cast<uint8_t*>(w + L.sel);
  cudaError_t e = cudaMemsetAsync(ws, 0, L.keys, st);   // scan states, counters, selection state
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(n_split, 0, sizeof(int64_t), st);
  if (e != cudaSuccess) return e;
  const float inv_denom = 1.0f / dp.denom;
  const unsigned b1 = (unsigned)((n + kThreads - 1) / kThreads);
  if (n > 0 && budget) {
    k_budget_keys<<<b1, kThreads, 0, st>>>(grad_S, ldg, n, inv_denom, dp.eps_split, dp.gate, dp.eps_grad, keys, lambda,
                                           sst);
    note_launch();
    if ((e = check_launch("k_budget_keys")) != cudaSuccess) return e;
    unsigned hb = b1 < 148 * 8 ? b1 : 148 * 8;
    for (int shift = 24; shift >= 0; shift -= 8) {
      k_select_hist<<<hb, kThreads, 0, st>>>(keys, n, shift, dp.budget, sst);
      k_select_pick<<<1, 256, 0, st>>>(shift, dp.budget, sst);
      note_launch(2);
      if ((e = check_launch("k_select")) != cudaSuccess) return e;
    }
    const unsigned bt = (unsigned)((n + kTileItems - 1) / kTileItems);
    k_budget_ties<<<bt, kThreads, 0, st>>>(keys, n, dp.budget, sst, sel, st_ties, counter + 1);
    note_launch();
    if ((e = check_launch("k_budget_ties")) != cudaSuccess) return e;
  }
  const int64_t tiles = fused ? (n + kThreads * kItemsFused - 1) / (kThreads * kItemsFused)
                              : (n + kTileItems - 1) / kTileItems;
  if (n > 0) {
#define SGS_DECIDE(F, IT, SEL)                                                                              \
  launch_pdl(k_densify_decide<F, IT, SEL>, dim3((unsigned)tiles), dim3(kThreads), 0, st, params, ld, grad_S, ldg, n,  \
             inv_denom, dp.eps_split, dp.eta, dp.eps_abs, dp.gate, dp.eps_grad, (const uint8_t*)sel, mask, dest,   \
             budget ? nullptr : lambda, st_decide, counter, n_split, status)
    if (fused && budget) SGS_DECIDE(true, kItemsFused, true);
    else if (fused) SGS_DECIDE(true, kItemsFused, false);
    else if (budget) SGS_DECIDE(false, kItems, true);
    else SGS_DECIDE(false, kItems, false);
#undef SGS_DECIDE
    note_launch();
    if ((e = check_launch("k_densify_decide")) != cudaSuccess) return e;
    if (fused) return cudaSuccess;
  }
  k_densify_apply<<<b1 > 0 ? b1 : 1, kThreads, 0, st>>>(params, ld, n, capacity, grad_S, ldg, inv_denom, dp.eta,
                                                        dp.eps_abs, mask, dest, n_split, status);
  note_launch();
  return check_launch("k_densify_apply");
}

}  // namespace sgs
