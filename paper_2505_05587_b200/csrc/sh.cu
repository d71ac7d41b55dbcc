// sh.cu — NEXT f3: view-dependent colour from real spherical harmonics on the backward side,
// and the plane-generic helpers the extra coefficient planes need (Adam, offspring copies).
//
//   k_sh_bwd         per Gaussian, over the views of the call: the per-(view, Gaussian) colour gradient
//                    cg = sum alpha T dL/dC (moments 6-8, left in place for k_gauss_bwd) is taken through
//                    the clamp max(0, .) and the SH expansion: dL/df_k = Y_k(dir) cg (DC -> grad_S planes
//                    11-13, the rest -> grad_sh), and, for a pinhole camera, through dir = (p - o)/|p - o|
//                    into dL/dp (-> grad_S planes 0-2; k_gauss_bwd then adds the splat terms).
//   k_adam_planes    Adam over `planes` dense planes with one learning rate (the SH rest coefficients).
//   k_copy_offspring arr[:, dest[i]] = arr[:, i] for densified parents (extra planes follow the parent).
//   k_copy_planes    plane-range copies (checkpoint / restore of Gaussian sets, steepgs_copy_planes).
// Bound: HBM.
#include <math.h>

#include "common.cuh"

namespace sgs {

namespace {

// sum_k w_k grad Y_k(d) for the basis of sh_basis<D> (partial derivatives of the polynomials).
template <int D>
__device__ __forceinline__ void sh_grad(const float* d, const float* w, float* g) {
  const float x = d[0], y = d[1], z = d[2];
  g[0] = g[1] = g[2] = 0.0f;
  if (D < 1) return;
  const float c1 = 0.4886025119029199f;
  g[1] += -c1 * w[1];
  g[2] += c1 * w[2];
  g[0] += -c1 * w[3];
  if (D < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z;
  const float a0 = 1.0925484305920792f, a1 = -1.0925484305920792f, a2 = 0.31539156525252005f,
              a3 = -1.0925484305920792f, a4 = 0.5462742152960396f;
  g[0] += a0 * y * w[4];                 g[1] += a0 * x * w[4];
  g[1] += a1 * z * w[5];                 g[2] += a1 * y * w[5];
  g[0] += -2.0f * a2 * x * w[6];         g[1] += -2.0f * a2 * y * w[6];  g[2] += 4.0f * a2 * z * w[6];
  g[0] += a3 * z * w[7];                 g[2] += a3 * x * w[7];
  g[0] += 2.0f * a4 * x * w[8];          g[1] += -2.0f * a4 * y * w[8];
  if (D < 3) return;
  const float b0 = -0.5900435899266435f, b1 = 2.890611442640554f, b2 = -0.4570457994644658f,
              b3 = 0.3731763325901154f, b4 = -0.4570457994644658f, b5 = 1.445305721320277f,
              b6 = -0.5900435899266435f;
  g[0] += 6.0f * b0 * x * y * w[9];                     g[1] += b0 * (3.0f * xx - 3.0f * yy) * w[9];
  g[0] += b1 * y * z * w[10];  g[1] += b1 * x * z * w[10];  g[2] += b1 * x * y * w[10];
  g[0] += -2.0f * b2 * x * y * w[11];  g[1] += b2 * (4.0f * zz - xx - 3.0f * yy) * w[11];
  g[2] += 8.0f * b2 * y * z * w[11];
  g[0] += -6.0f * b3 * x * z * w[12];  g[1] += -6.0f * b3 * y * z * w[12];
  g[2] += b3 * (6.0f * zz - 3.0f * xx - 3.0f * yy) * w[12];
  g[0] += b4 * (4.0f * zz - 3.0f * xx - yy) * w[13];  g[1] += -2.0f * b4 * x * y * w[13];
  g[2] += 8.0f * b4 * x * z * w[13];
  g[0] += 2.0f * b5 * x * z * w[14];  g[1] += -2.0f * b5 * y * z * w[14];  g[2] += b5 * (xx - yy) * w[14];
  g[0] += b6 * (3.0f * xx - 3.0f * yy) * w[15];  g[1] += -6.0f * b6 * x * y * w[15];
}

template <int D>
__global__ void __launch_bounds__(128) k_sh_bwd(const float* __restrict__ params, int64_t ld, int64_t n,
                                                const float* __restrict__ sh_rest, int64_t ld_sh,
                                                const CamPack cams, int V, const float* __restrict__ moments,
                                                float* __restrict__ grad_S, int64_t ldg, float* __restrict__ grad_sh,
                                                int64_t ldg_sh, int accumulate) {
  constexpr int K = (D + 1) * (D + 1);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float p[3] = {params[0 * ld + i], params[1 * ld + i], params[2 * ld + i]};
  float f[K][3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) f[0][ch] = params[(11 + ch) * ld + i];
#pragma unroll
  for (int k = 1; k < K; ++k)
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) f[k][ch] = sh_rest[(int64_t)(3 * (k - 1) + ch) * ld_sh + i];
  float gf[K][3];
#pragma unroll
  for (int k = 0; k < K; ++k) gf[k][0] = gf[k][1] = gf[k][2] = 0.0f;
  float gp[3] = {0.0f, 0.0f, 0.0f};
  for (int v = 0; v < V; ++v) {
    const float* mp = moments + ((int64_t)v * n + i) * 12;
    const float4 mb = __ldcg(reinterpret_cast<const float4*>(mp) + 1);
    const float cg[3] = {mb.z, mb.w, __ldcg(mp + 8)};
    if (cg[0] == 0.0f && cg[1] == 0.0f && cg[2] == 0.0f) continue;
    const steepgs_camera& c = cams.cam[v];
    const float* R = c.R;
    float d[3], rinv = 0.0f;
    if (c.model == 0) {
      float v3[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) v3[k] = p[k] + (R[k] * c.t[0] + R[3 + k] * c.t[1] + R[6 + k] * c.t[2]);
      rinv = rsqrtf(v3[0] * v3[0] + v3[1] * v3[1] + v3[2] * v3[2]);
      d[0] = v3[0] * rinv; d[1] = v3[1] * rinv; d[2] = v3[2] * rinv;
    } else {
      d[0] = R[6]; d[1] = R[7]; d[2] = R[8];
    }
    float Y[16];
    sh_basis<D>(d, Y);
    float g[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float raw = 0.5f;
#pragma unroll
      for (int k = 0; k < K; ++k) raw += Y[k] * f[k][ch];
      g[ch] = raw > 0.0f ? cg[ch] : 0.0f;                       // clamp max(0, .)
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) gf[k][ch] += Y[k] * g[ch];
    if (D >= 1 && c.model == 0) {
      float w[16];
#pragma unroll
      for (int k = 0; k < K; ++k) w[k] = f[k][0] * g[0] + f[k][1] * g[1] + f[k][2] * g[2];
      float gd[3];
      sh_grad<D>(d, w, gd);
      const float dot = gd[0] * d[0] + gd[1] * d[1] + gd[2] * d[2];
#pragma unroll
      for (int k = 0; k < 3; ++k) gp[k] += (gd[k] - dot * d[k]) * rinv;   // (I - d d^T) / r
    }
  }
  const bool acc = (accumulate & 3) == 1;
#pragma unroll
  for (int k = 0; k < 3; ++k) grad_S[k * ldg + i] = acc ? grad_S[k * ldg + i] + gp[k] : gp[k];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) grad_S[(11 + ch) * ldg + i] = acc ? grad_S[(11 + ch) * ldg + i] + gf[0][ch] : gf[0][ch];
#pragma unroll
  for (int k = 1; k < K; ++k)
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float* q = grad_sh + (int64_t)(3 * (k - 1) + ch) * ldg_sh + i;
      *q = acc ? *q + gf[k][ch] : gf[k][ch];
    }
}

__global__ void __launch_bounds__(256) k_adam_planes(float* __restrict__ params, int64_t ld, int planes, int64_t n,
                                                     const float* __restrict__ grad, int64_t ldg,
                                                     float* __restrict__ m, float* __restrict__ v, int64_t ldm,
                                                     float lr, float b1, float omb1, float b2, float omb2, float eps,
                                                     float bc1, float bc2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < planes; ++k) {
    const float g = grad[k * ldg + i];
    const float mk = b1 * m[k * ldm + i] + omb1 * g;
    const float vk = b2 * v[k * ldm + i] + omb2 * (g * g);
    m[k * ldm + i] = mk;
    v[k * ldm + i] = vk;
    params[k * ld + i] -= lr * (mk / bc1) / (sqrtf(vk / bc2) + eps);
  }
}

__global__ void __launch_bounds__(256) k_copy_offspring(float* __restrict__ arr, int64_t ld, int planes, int64_t n,
                                                        const int32_t* __restrict__ dest) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t b = dest[i];
  if (b < 0) return;
  for (int k = 0; k < planes; ++k) arr[k * ld + b] = arr[k * ld + i];
}

// dst[first + k][i] = src[first + k][i] for k < count, i < n: 16-B vector copies when both row
// pitches and bases allow it (the planar arrays here are 256-B aligned with ld % 4 == 0)
__global__ void __launch_bounds__(256) k_copy_planes(float* __restrict__ dst, int64_t ld_dst,
                                                     const float* __restrict__ src, int64_t ld_src, int64_t n,
                                                     int count, bool vec) {
  pdl_wait();
  pdl_trigger();
  const int k = blockIdx.y;
  float* d = dst + k * ld_dst;
  const float* s = src + k * ld_src;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    const int64_t n4 = n / 4;
    for (int64_t q = i; q < n4; q += stride)
      reinterpret_cast<float4*>(d)[q] = __ldg(reinterpret_cast<const float4*>(s) + q);
    for (int64_t q = 4 * n4 + i; q < n; q += stride) d[q] = s[q];
  } else {
    for (; i < n; i += stride) d[i] = s[i];
  }
}

}  // namespace

cudaError_t launch_copy_planes(float* dst, int64_t ld_dst, const float* src, int64_t ld_src, int64_t n, int first,
                               int count, cudaStream_t st) {
  if (n == 0 || count == 0) return cudaSuccess;
  float* d = dst + first * ld_dst;
  const float* s = src + first * ld_src;
  const bool vec = (ld_dst % 4 == 0) && (ld_src % 4 == 0) && ((uintptr_t)d % 16 == 0) && ((uintptr_t)s % 16 == 0);
  int64_t blocks = (n / (vec ? 4 : 1) + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch_pdl(k_copy_planes, dim3((unsigned)(blocks > 0 ? blocks : 1), (unsigned)count), dim3(256), 0, st, d, ld_dst,
             s, ld_src, n, count, vec);
  note_launch();
  return check_launch("k_copy_planes");
}

cudaError_t launch_sh_bwd(const float* params, int64_t ld, int64_t n, const float* sh_rest, int64_t ld_sh,
                          int sh_degree, const CamPack& cams, int V, const float* moments, float* grad_S,
                          int64_t ldg, float* grad_sh, int64_t ldg_sh, int accumulate, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((n + 127) / 128);
#define SGS_SHB(D)                                                                                             \
  k_sh_bwd<D><<<blocks, 128, 0, st>>>(params, ld, n, sh_rest, ld_sh, cams, V, moments, grad_S, ldg, grad_sh, \
                                      ldg_sh, accumulate)
  switch (sh_degree) {
    case 0: SGS_SHB(0); break;
    case 1: SGS_SHB(1); break;
    case 2: SGS_SHB(2); break;
    default: SGS_SHB(3); break;
  }
#undef SGS_SHB
  note_launch();
  return check_launch("k_sh_bwd");
}

cudaError_t launch_adam_planes(float* params, int64_t ld, int planes, int64_t n, const float* grad, int64_t ldg,
                               float* m, float* v, int64_t ldm, const steepgs_adam_params& ap, int64_t step,
                               cudaStream_t st) {
  if (n == 0 || planes == 0) return cudaSuccess;
  const float bc1 = (float)(1.0 - pow(ap.beta1, (double)step));
  const float bc2 = (float)(1.0 - pow(ap.beta2, (double)step));
  k_adam_planes<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      params, ld, planes, n, grad, ldg, m, v, ldm, (float)ap.lr[0], (float)ap.beta1, (float)(1.0 - ap.beta1),
      (float)ap.beta2, (float)(1.0 - ap.beta2), (float)ap.eps, bc1, bc2);
  note_launch();
  return check_launch("k_adam_planes");
}

cudaError_t launch_copy_offspring(float* arr, int64_t ld, int planes, int64_t n, const int32_t* dest,
                                  cudaStream_t st) {
  if (n == 0 || planes == 0) return cudaSuccess;
  k_copy_offspring<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(arr, ld, planes, n, dest);
  note_launch();
  return check_launch("k_copy_offspring");
}

}  // namespace sgs
