// ssim.cu — NEXT f3: the 3DGS photometric loss with the SSIM term (P:L150 footnote; 3DGS trains
// with L = (1 - lam) L1 + lam (1 - SSIM), lam = 0.2) and its gradient, fused with the l1 part.
//
//   k_ssim_fwd   per (view, channel) plane and 32x16 output tile: the 11x11 Gaussian window (sigma 1.5,
//                zero padding) as two separable passes in shared memory over the 5 moments
//                x, y, x^2, y^2, x y; per pixel the SSIM value S and its partials
//                G1 = dS/dmu_x, G11 = dS/d(w * x^2), G12 = dS/d(w * x y) (written to the workspace);
//                per-view sum of S.
//   k_ssim_bwd   the same window over (G1, G11, G12) (the window is symmetric: its adjoint is itself),
//                dSSIM/dx = [w * G1 + 2 x (w * G11) + y (w * G12)] / N, fused with the l1 term:
//                dL/dx = scale ((1 - lam) sign(x - y) / N - lam dSSIM/dx); per-view sum of |x - y|.
//   k_loss_final loss[v] = (1 - lam) L1 + lam (1 - SSIM).
// Bound: HBM (each pass reads its inputs once, the halo re-reads hit L2).
#include <math.h>

#include "common.cuh"

namespace sgs {

namespace {

constexpr int kTW = 32, kTH = 16, kR = 5, kWin = 2 * kR + 1;
constexpr int kIW = kTW + 2 * kR, kIH = kTH + 2 * kR;
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

// the normalised Gaussian window (sigma 1.5), computed once on the host in fp64 and rounded to fp32,
// passed by value (kernel parameter space)
struct Win {
  float w[kWin];
};

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float s = 0.0f;
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return s;
}

// Register-blocked separable window.  The input tile (kIH x kIW, zero outside the image) is stored
// with a 16-B aligned row stride; the horizontal pass gives each thread 4 consecutive outputs of a
// row (14 inputs loaded with 4 vector loads, each input's products formed once and added to the
// up-to-4 outputs its taps reach), the vertical pass 2 consecutive rows of a column.
constexpr int kIWP = 44;                 // padded input row (16-B multiple)

// h[q][r][c0 .. c0 + 3] = sum_t w[t] v_q[r][c0 + o + t] for the NQ planes v of `in` (fwd: x, y and the
// products x^2, y^2, x y formed here from the two input planes)
template <bool kProducts, int NIN, int NQ>
__device__ __forceinline__ void hpass(const Win& win, const float (*in)[kIH][kIWP], float (*h)[kIH][kTW]) {
  for (int e = threadIdx.x; e < kIH * (kTW / 4); e += blockDim.x) {
    const int r = e / (kTW / 4), c0 = (e % (kTW / 4)) * 4;
    float v[NIN][16];
#pragma unroll
    for (int q = 0; q < NIN; ++q)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 t = *reinterpret_cast<const float4*>(&in[q][r][c0 + 4 * k]);
        v[q][4 * k] = t.x; v[q][4 * k + 1] = t.y; v[q][4 * k + 2] = t.z; v[q][4 * k + 3] = t.w;
      }
    float acc[NQ][4];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int o = 0; o < 4; ++o) acc[q][o] = 0.0f;
#pragma unroll
    for (int k = 0; k < kWin + 3; ++k) {
      float val[NQ];
      if (kProducts) {
        const float a = v[0][k], b = v[1][k];
        val[0] = a; val[1] = b; val[2] = a * a; val[3] = b * b; val[4] = a * b;
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q) val[q] = v[q][k];
      }
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const int t = k - o;
        if (t < 0 || t >= kWin) continue;
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q][o] = fmaf(win.w[t], val[q], acc[q][o]);
      }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      *reinterpret_cast<float4*>(&h[q][r][c0]) = make_float4(acc[q][0], acc[q][1], acc[q][2], acc[q][3]);
  }
  __syncthreads();
}

// m[q][o] = sum_t w[t] h[q][r0 + o + t][c] for o = 0, 1
template <int NQ>
__device__ __forceinline__ void vpass(const Win& win, const float (*h)[kIH][kTW], int r0, int c, float (*m)[2]) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
    for (int k = 0; k < kWin + 1; ++k) {
      const float x = h[q][r0 + k][c];
      if (k < kWin) a0 = fmaf(win.w[k], x, a0);
      if (k >= 1) a1 = fmaf(win.w[k - 1], x, a1);
    }
    m[q][0] = a0;
    m[q][1] = a1;
  }
}

__global__ void __launch_bounds__(256) k_ssim_fwd(const float* __restrict__ image, const float* __restrict__ target,
                                                  int H, int W, float* __restrict__ maps, float* __restrict__ ssim_sum,
                                                  const Win win) {
  __shared__ __align__(16) float in[2][kIH][kIWP];
  __shared__ __align__(16) float h[5][kIH][kTW];
  __shared__ float red[8];
  const int plane = blockIdx.z;                 // view * 3 + channel
  const int view = plane / 3;
  const int64_t HW = (int64_t)H * W;
  const float* x = image + plane * HW;
  const float* y = target + plane * HW;
  const int ox = blockIdx.x * kTW - kR, oy = blockIdx.y * kTH - kR;
  for (int e = threadIdx.x; e < kIH * kIW; e += blockDim.x) {
    const int r = e / kIW, c = e % kIW;
    const int gy = oy + r, gx = ox + c;
    const bool ok = gy >= 0 && gy < H && gx >= 0 && gx < W;
    in[0][r][c] = ok ? x[(int64_t)gy * W + gx] : 0.0f;
    in[1][r][c] = ok ? y[(int64_t)gy * W + gx] : 0.0f;
  }
  __syncthreads();
  hpass<true, 2, 5>(win, in, h);
  const int c = threadIdx.x % kTW, r0 = 2 * (threadIdx.x / kTW);   // 2 rows x 32 columns per 256 threads
  float m[5][2];
  vpass<5>(win, h, r0, c, m);
  float acc = 0.0f;
  float* mp = maps + plane * 3 * HW;
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    const int gy = blockIdx.y * kTH + r0 + o, gx = blockIdx.x * kTW + c;
    if (gy >= H || gx >= W) continue;
    const float mx = m[0][o], my = m[1][o];
    const float sxx = m[2][o] - mx * mx, syy = m[3][o] - my * my, sxy = m[4][o] - mx * my;
    const float an = 2.f * mx * my + kC1, bn = 2.f * sxy + kC2;
    const float ad = mx * mx + my * my + kC1, bd = sxx + syy + kC2;
    const float D = ad * bd;
    const float S = an * bn / D;
    const float G1 = (2.f * my * bn - 2.f * my * an) / D - S * (2.f * mx / ad - 2.f * mx / bd);
    const float G11 = -S / bd;
    const float G12 = 2.f * an / D;
    const int64_t pix = (int64_t)gy * W + gx;
    mp[pix] = G1; mp[HW + pix] = G11; mp[2 * HW + pix] = G12;
    acc += S;
  }
  const float s = block_sum(acc, red);
  if (threadIdx.x == 0) atomicAdd(ssim_sum + view, s);
}

__global__ void __launch_bounds__(256) k_ssim_bwd(const float* __restrict__ image, const float* __restrict__ target,
                                                  int H, int W, const float* __restrict__ maps, float lam,
                                                  float scale, float* __restrict__ dL, float* __restrict__ l1_sum,
                                                  const Win win) {
  __shared__ __align__(16) float in[3][kIH][kIWP];
  __shared__ __align__(16) float h[3][kIH][kTW];
  __shared__ float red[8];
  const int plane = blockIdx.z;
  const int view = plane / 3;
  const int64_t HW = (int64_t)H * W;
  const float* mp = maps + plane * 3 * HW;
  const int ox = blockIdx.x * kTW - kR, oy = blockIdx.y * kTH - kR;
  for (int e = threadIdx.x; e < kIH * kIW; e += blockDim.x) {
    const int r = e / kIW, c = e % kIW;
    const int gy = oy + r, gx = ox + c;
    const bool ok = gy >= 0 && gy < H && gx >= 0 && gx < W;
    const int64_t pix = (int64_t)gy * W + gx;
#pragma unroll
    for (int q = 0; q < 3; ++q) in[q][r][c] = ok ? mp[q * HW + pix] : 0.0f;
  }
  __syncthreads();
  hpass<false, 3, 3>(win, in, h);
  const int c = threadIdx.x % kTW, r0 = 2 * (threadIdx.x / kTW);
  float f[3][2];
  vpass<3>(win, h, r0, c, f);
  const float invN = 1.0f / (float)(3 * HW);
  float acc = 0.0f;
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    const int gy = blockIdx.y * kTH + r0 + o, gx = blockIdx.x * kTW + c;
    if (gy >= H || gx >= W) continue;
    const int64_t pix = plane * HW + (int64_t)gy * W + gx;
    const float xv = image[pix], yv = target[pix];
    const float gs = (f[0][o] + 2.f * xv * f[1][o] + yv * f[2][o]) * invN;
    const float d = xv - yv;
    const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
    dL[pix] = scale * ((1.f - lam) * sg * invN - lam * gs);
    acc += fabsf(d);
  }
  const float s = block_sum(acc, red);
  if (threadIdx.x == 0) atomicAdd(l1_sum + view, s);
}

__global__ void k_loss_final(const float* __restrict__ sums, int V, float invN, float lam, float* __restrict__ loss) {
  const int v = threadIdx.x;
  if (v < V) loss[v] = (1.f - lam) * sums[V + v] * invN + lam * (1.f - sums[v] * invN);
}

}  // namespace

size_t loss_ws_bytes(int V, int H, int W) { return (size_t)V * 3 * 3 * H * W * sizeof(float) + 2 * 64 * sizeof(float); }

cudaError_t launch_ssim_loss(const float* image, const float* target, int V, int H, int W, float lam, float scale,
                             float* dL, float* loss, void* ws, cudaStream_t st) {
  cudaError_t e;
  float* maps = static_cast<float*>(ws);
  float* sums = maps + (size_t)V * 9 * H * W;       // [2][V]: SSIM sums, L1 sums
  if ((e = cudaMemsetAsync(sums, 0, 2 * 64 * sizeof(float), st)) != cudaSuccess) return e;
  Win win;
  {
    double g[kWin], s = 0.0;
    for (int t = 0; t < kWin; ++t) {
      g[t] = exp(-(double)((t - kR) * (t - kR)) / (2.0 * 1.5 * 1.5));
      s += g[t];
    }
    for (int t = 0; t < kWin; ++t) win.w[t] = (float)(g[t] / s);
  }
  dim3 grid((W + kTW - 1) / kTW, (H + kTH - 1) / kTH, 3 * V);
  k_ssim_fwd<<<grid, 256, 0, st>>>(image, target, H, W, maps, sums, win);
  k_ssim_bwd<<<grid, 256, 0, st>>>(image, target, H, W, maps, lam, scale, dL, sums + V, win);
  note_launch(2);
  if ((e = check_launch("k_ssim")) != cudaSuccess) return e;
  if (loss) {
    k_loss_final<<<1, 64, 0, st>>>(sums, V, 1.0f / (float)(3 * (int64_t)H * W), lam, loss);
    note_launch();
    return check_launch("k_loss_final");
  }
  return cudaSuccess;
}

}  // namespace sgs
