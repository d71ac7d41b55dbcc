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

// the normalised Gaussian window (sigma 1.5), computed in fp64 and rounded once, per block
__device__ __forceinline__ void load_window(float* win) {
  if (threadIdx.x < kWin) {
    double s = 0.0, g = 0.0;
    for (int t = 0; t < kWin; ++t) {
      const double e = exp(-(double)((t - kR) * (t - kR)) / (2.0 * 1.5 * 1.5));
      s += e;
      if (t == (int)threadIdx.x) g = e;
    }
    win[threadIdx.x] = (float)(g / s);
  }
}

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

// Separable window over NQ planes staged in `in` ([NQ][kIH][kIW], zero outside the image):
// horizontal pass into `h` ([NQ][kIH][kTW]), then the vertical pass for output (r, c) -> out[q].
template <int NQ>
__device__ __forceinline__ void window_pass(const float* c_win, const float (*in)[kIH][kIW], float (*h)[kIH][kTW]) {
  for (int e = threadIdx.x; e < kIH * kTW; e += blockDim.x) {
    const int r = e / kTW, c = e % kTW;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float s = 0.0f;
#pragma unroll
      for (int t = 0; t < kWin; ++t) s = fmaf(c_win[t], in[q][r][c + t], s);
      h[q][r][c] = s;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_ssim_fwd(const float* __restrict__ image, const float* __restrict__ target,
                                                  int H, int W, float* __restrict__ maps, float* __restrict__ ssim_sum) {
  __shared__ float in[2][kIH][kIW];
  __shared__ float h[5][kIH][kTW];
  __shared__ float red[8];
  __shared__ float c_win[kWin];
  load_window(c_win);
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
  for (int e = threadIdx.x; e < kIH * kTW; e += blockDim.x) {
    const int r = e / kTW, c = e % kTW;
    float sx = 0.f, sy = 0.f, sxx = 0.f, syy = 0.f, sxy = 0.f;
#pragma unroll
    for (int t = 0; t < kWin; ++t) {
      const float a = in[0][r][c + t], b = in[1][r][c + t], w = c_win[t];
      sx = fmaf(w, a, sx); sy = fmaf(w, b, sy);
      sxx = fmaf(w, a * a, sxx); syy = fmaf(w, b * b, syy); sxy = fmaf(w, a * b, sxy);
    }
    h[0][r][c] = sx; h[1][r][c] = sy; h[2][r][c] = sxx; h[3][r][c] = syy; h[4][r][c] = sxy;
  }
  __syncthreads();
  float acc = 0.0f;
  for (int e = threadIdx.x; e < kTH * kTW; e += blockDim.x) {
    const int r = e / kTW, c = e % kTW;
    const int gy = blockIdx.y * kTH + r, gx = blockIdx.x * kTW + c;
    if (gy >= H || gx >= W) continue;
    float m[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      float s = 0.0f;
#pragma unroll
      for (int t = 0; t < kWin; ++t) s = fmaf(c_win[t], h[q][r + t][c], s);
      m[q] = s;
    }
    const float mx = m[0], my = m[1];
    const float sxx = m[2] - mx * mx, syy = m[3] - my * my, sxy = m[4] - mx * my;
    const float an = 2.f * mx * my + kC1, bn = 2.f * sxy + kC2;
    const float ad = mx * mx + my * my + kC1, bd = sxx + syy + kC2;
    const float D = ad * bd;
    const float S = an * bn / D;
    const float G1 = (2.f * my * bn - 2.f * my * an) / D - S * (2.f * mx / ad - 2.f * mx / bd);
    const float G11 = -S / bd;
    const float G12 = 2.f * an / D;
    const int64_t pix = (int64_t)gy * W + gx;
    float* mp = maps + plane * 3 * HW;
    mp[pix] = G1; mp[HW + pix] = G11; mp[2 * HW + pix] = G12;
    acc += S;
  }
  const float s = block_sum(acc, red);
  if (threadIdx.x == 0) atomicAdd(ssim_sum + view, s);
}

__global__ void __launch_bounds__(256) k_ssim_bwd(const float* __restrict__ image, const float* __restrict__ target,
                                                  int H, int W, const float* __restrict__ maps, float lam,
                                                  float scale, float* __restrict__ dL, float* __restrict__ l1_sum) {
  __shared__ float in[3][kIH][kIW];
  __shared__ float h[3][kIH][kTW];
  __shared__ float red[8];
  __shared__ float c_win[kWin];
  load_window(c_win);
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
  window_pass<3>(c_win, in, h);
  const float invN = 1.0f / (float)(3 * HW);
  float acc = 0.0f;
  for (int e = threadIdx.x; e < kTH * kTW; e += blockDim.x) {
    const int r = e / kTW, c = e % kTW;
    const int gy = blockIdx.y * kTH + r, gx = blockIdx.x * kTW + c;
    if (gy >= H || gx >= W) continue;
    float f[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float s = 0.0f;
#pragma unroll
      for (int t = 0; t < kWin; ++t) s = fmaf(c_win[t], h[q][r + t][c], s);
      f[q] = s;
    }
    const int64_t pix = plane * HW + (int64_t)gy * W + gx;
    const float xv = image[pix], yv = target[pix];
    const float gs = (f[0] + 2.f * xv * f[1] + yv * f[2]) * invN;
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
  dim3 grid((W + kTW - 1) / kTW, (H + kTH - 1) / kTH, 3 * V);
  k_ssim_fwd<<<grid, 256, 0, st>>>(image, target, H, W, maps, sums);
  k_ssim_bwd<<<grid, 256, 0, st>>>(image, target, H, W, maps, lam, scale, dL, sums + V);
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
