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
  if (!have_vec) { v[0] = 1.f; v[1] = 0.f; v[2] = 0.f; return; }
  const float nn = rsqrtf(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  v[0] *= nn; v[1] *= nn; v[2] *= nn;
  int big = 0;  // canonical sign: largest |component| positive, ties -> lowest index (C13)
  if (fabsf(v[1]) > fabsf(v[big])) big = 1;
  if (fabsf(v[2]) > fabsf(v[big])) big = 2;
  if (v[big] < 0.f) { v[0] = -v[0]; v[1] = -v[1]; v[2] = -v[2]; }
}

__device__ __forceinline__ float decide_lambda(const float* S6, float eps_split) {
  float lam, v[3];
  eig_min_robust(S6, false, lam, v);
  float fro = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) fro += (k == 1 || k == 2 || k == 4 ? 2.f : 1.f) * S6[k] * S6[k];
  fro = sqrtf(fro);
  if (fabsf(lam - eps_split) <= 1e-3f * fro + 1e-30f) lam = (float)eig_min_f64(S6);  // guard band: fp64
  return lam;
}

// Offspring of split parent i (Thm 2 / Alg. 1): A in slot i at p + eps v, B in slot b at
// p - eps v, both with opacity logit(o/2) (Z15), other planes copied (Z14); B's accumulators zeroed.
__device__ __forceinline__ void spawn(float* __restrict__ params, int64_t ld, float* __restrict__ grad_S,
                                      int64_t ldg, int64_t i, int64_t b, const float* S6, float eta, float eps_abs) {
  float v[3], lam_unused;
  eig_min_robust(S6, true, lam_unused, v);
  // parent: p, Sigma = R diag(s^2) R^T, o
  const float p0 = params[0 * ld + i], p1 = params[1 * ld + i], p2 = params[2 * ld + i];
  float eps = eps_abs;
  if (eta >= 0.f) {
    const float qw = params[6 * ld + i], qx = params[7 * ld + i], qy = params[8 * ld + i], qz = params[9 * ld + i];
    const float qn = rsqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
    const float w = qw * qn, x = qx * qn, y = qy * qn, z = qz * qn;
    const float r[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                        2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                        2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
    float vsv = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float s = expf(params[(3 + k) * ld + i]);
      const float rv = r[k] * v[0] + r[3 + k] * v[1] + r[6 + k] * v[2];
      vsv += s * s * rv * rv;
    }
    eps = eta * sqrtf(vsv);
  }
  const double o = 1.0 / (1.0 + exp(-(double)params[10 * ld + i]));
  const double h = 0.5 * o;                                   // Z15: w = 1/2 absorbed in opacity
  const float lg = (float)(log(h) - log1p(-h));
#pragma unroll
  for (int k = 3; k < 14; ++k) params[k * ld + b] = params[k * ld + i];
  params[0 * ld + b] = p0 - eps * v[0];
  params[1 * ld + b] = p1 - eps * v[1];
  params[2 * ld + b] = p2 - eps * v[2];
  params[10 * ld + b] = lg;
  params[0 * ld + i] = p0 + eps * v[0];
  params[1 * ld + i] = p1 + eps * v[1];
  params[2 * ld + i] = p2 + eps * v[2];
  params[10 * ld + i] = lg;
#pragma unroll
  for (int k = 0; k < 20; ++k) grad_S[k * ldg + b] = 0.f;
}

// kFused (capacity >= 2n, so n + n_split <= capacity holds for any mask): the same kernel also
// writes the offspring and clears S, one pass over the data and no second launch.
template <bool kFused, int kIt>
__global__ void __launch_bounds__(kThreads) k_densify_decide(float* __restrict__ params, int64_t ld,
                                                             float* __restrict__ grad_S, int64_t ldg, int64_t n,
                                                             float inv_denom, float eps_split, float eta, float eps_abs,
                                                             uint8_t* __restrict__ mask, int32_t* __restrict__ dest,
                                                             float* __restrict__ lambda, uint64_t* status,
                                                             int* tile_counter, int64_t* n_split,
                                                             int32_t* __restrict__ dstatus) {
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
#pragma unroll
  for (int j = 0; j < kIt; ++j) {
    const int64_t i = base + (int64_t)j * kThreads + tid;
    split[j] = false;
    if (i < n) {
      float S6[6];
      load_sbar(grad_S, ldg, i, inv_denom, S6);
      const float lam = decide_lambda(S6, eps_split);
      split[j] = lam < eps_split;                     // Thm 2 / Alg. 1 P:L545 (strict, Z11)
      if (lambda) lambda[i] = lam;
    }
    const uint32_t b = __ballot_sync(0xffffffffu, split[j]);
    pos[j] = __popc(b & lanemask_lt());
    if (lane == 0) s_cnt[j][warp] = __popc(b);
  }
  __syncthreads();
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
    const uint64_t excl = lookback_warp(status, tile, agg);
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
    if (kFused) {
      float S6[6];
      if (split[j]) load_sbar(grad_S, ldg, i, inv_denom, S6);
#pragma unroll
      for (int k = 14; k < 20; ++k) grad_S[k * ldg + i] = 0.f;   // Z23
      if (split[j]) spawn(params, ld, grad_S, ldg, i, b, S6, eta, eps_abs);
    }
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
  spawn(params, ld, grad_S, ldg, i, dest[i], S6, eta, eps_abs);
}


inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

constexpr int kItemsFused = 1;   // one Gaussian per thread when the offspring are written too

size_t densify_ws_bytes(int64_t n) {
  const int64_t tiles = (n + kThreads * kItemsFused - 1) / (kThreads * kItemsFused);
  return align_up(8 * (size_t)(tiles > 0 ? tiles : 1)) + 256;
}

cudaError_t launch_densify(float* params, int64_t ld, int64_t n, int64_t capacity, float* grad_S, int64_t ldg,
                           const steepgs_densify_params& dp, uint8_t* mask, int32_t* dest, float* lambda,
                           int64_t* n_split, int32_t* status, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (ws_bytes < densify_ws_bytes(n)) return cudaErrorInvalidValue;
  const bool fused = capacity >= 2 * n;
  const int64_t tiles = fused ? (n + kThreads * kItemsFused - 1) / (kThreads * kItemsFused)
                              : (n + kTileItems - 1) / kTileItems;
  char* w = static_cast<char*>(ws);
  uint64_t* sstatus = reinterpret_cast<uint64_t*>(w);
  int* counter = reinterpret_cast<int*>(w + align_up(8 * (size_t)(tiles > 0 ? tiles : 1)));
  cudaError_t e = cudaMemsetAsync(ws, 0, densify_ws_bytes(n), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(n_split, 0, sizeof(int64_t), st);
  if (e != cudaSuccess) return e;
  const float inv_denom = 1.0f / dp.denom;
  if (n > 0 && fused) {
    k_densify_decide<true, kItemsFused><<<(unsigned)tiles, kThreads, 0, st>>>(params, ld, grad_S, ldg, n, inv_denom, dp.eps_split,
                                                                 dp.eta, dp.eps_abs, mask, dest, lambda, sstatus,
                                                                 counter, n_split, status);
    note_launch();
    return check_launch("k_densify_decide<fused>");
  }
  if (n > 0) {
    k_densify_decide<false, kItems><<<(unsigned)tiles, kThreads, 0, st>>>(params, ld, grad_S, ldg, n, inv_denom, dp.eps_split,
                                                                  dp.eta, dp.eps_abs, mask, dest, lambda, sstatus,
                                                                  counter, n_split, status);
    note_launch();
    if ((e = check_launch("k_densify_decide")) != cudaSuccess) return e;
  }
  const unsigned blocks = (unsigned)((n + kThreads - 1) / kThreads);
  k_densify_apply<<<blocks > 0 ? blocks : 1, kThreads, 0, st>>>(params, ld, n, capacity, grad_S, ldg, inv_denom, dp.eta,
                                                                dp.eps_abs, mask, dest, n_split, status);
  note_launch();
  return check_launch("k_densify_apply");
}

}  // namespace sgs
