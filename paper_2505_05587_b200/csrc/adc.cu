// adc.cu — NEXT f4: the 3DGS Adaptive Density Control baseline (as a splitting rule
// P:L185-188), on the same planar buffers and the same in-place + append layout as SDC.
//
//   k_adc_decide  per Gaussian: mean view-space gradient norm g = stats[0] / stats[1] (0 if never
//                 visible); selected iff g >= eps_adc (ADC (i)); clone iff ||Sigma||_2 =
//                 max_k s_k^2 <= tau_adc (ADC (ii)), else split (ADC (iii)); single-pass exclusive
//                 scan of the selection (decoupled look-back) -> dest = n + rank.
//   k_adc_apply   capacity check on the device; clone: the parent stays, the copy appended at
//                 p - clone_step * G / denom ("p_j - p proportional to grad_p L", C22);
//                 split: both offspring at p + R diag(s) z_j with caller-drawn z_j ~ N(0, I) and
//                 log-scale + ln(scale_factor) (Sigma_j = 0.64 Sigma), A in place, B
//                 appended; opacity unchanged (w = 1).  The gradient statistics and the
//                 accumulator planes of [0, n + n_new) restart at zero.
// Bound: HBM.
#include <math.h>

#include "common.cuh"
#include "scan.cuh"

namespace sgs {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTileItems = kThreads * kItems;
static_assert(kItems * (kThreads / 32) == 64, "the block scan gives each of 32 lanes two (item, warp) counts");

__global__ void __launch_bounds__(kThreads) k_adc_decide(const float* __restrict__ params, int64_t ld, int64_t n,
                                                         const float* __restrict__ stats, int64_t lds,
                                                         float eps_adc, float tau_adc, uint8_t* __restrict__ kind,
                                                         int32_t* __restrict__ dest, uint64_t* status,
                                                         int* tile_counter, int64_t* n_new) {
  __shared__ int s_tile;
  __shared__ uint32_t s_cnt[kItems][kThreads / 32];
  __shared__ uint64_t s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * kTileItems;
  uint8_t kd[kItems];
  uint32_t pos[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int64_t i = base + (int64_t)j * kThreads + tid;
    kd[j] = 0;
    if (i < n) {
      const float cnt = stats[lds + i];
      const float g = cnt > 0.f ? __fdiv_rn(stats[i], cnt) : 0.f;
      if (g >= eps_adc) {
        float smax = params[3 * ld + i];
        smax = fmaxf(smax, params[4 * ld + i]);
        smax = fmaxf(smax, params[5 * ld + i]);
        const float s = expf(smax);
        kd[j] = (s * s <= tau_adc) ? 1 : 2;
      }
    }
    const uint32_t b = __ballot_sync(0xffffffffu, kd[j] != 0);
    pos[j] = __popc(b & lanemask_lt());
    if (lane == 0) s_cnt[j][warp] = __popc(b);
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t* cnt = &s_cnt[0][0];
    const uint32_t a = cnt[2 * lane], bb = cnt[2 * lane + 1];   // 64 counts in (j, warp) order
    uint32_t sum = a + bb, inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t ex = inc - sum;
    cnt[2 * lane] = ex;
    cnt[2 * lane + 1] = ex + a;
    const uint32_t agg = __shfl_sync(0xffffffffu, inc, 31);
    const uint64_t excl = lookback_warp(status, tile, agg);
    if (lane == 0) {
      s_excl = excl;
      if (base + kTileItems >= n) *n_new = (int64_t)(excl + agg);
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int64_t i = base + (int64_t)j * kThreads + tid;
    if (i >= n) continue;
    kind[i] = kd[j];
    dest[i] = kd[j] ? (int32_t)(n + (int64_t)(s_excl + s_cnt[j][warp] + pos[j])) : -1;
  }
}

__global__ void __launch_bounds__(kThreads) k_adc_apply(float* __restrict__ params, int64_t ld, int64_t n,
                                                        int64_t capacity, float* __restrict__ grad_S, int64_t ldg,
                                                        float* __restrict__ stats, int64_t lds,
                                                        const float* __restrict__ normals, int64_t ldz,
                                                        float clone_step, float inv_denom, float log_scale_factor,
                                                        const uint8_t* __restrict__ kind,
                                                        const int32_t* __restrict__ dest,
                                                        const int64_t* __restrict__ n_new,
                                                        int32_t* __restrict__ status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nn = *n_new;
  const bool ok = n + nn <= capacity;
  if (i == 0) *status = ok ? 0 : (int32_t)STEEPGS_ERR_CAPACITY;
  if (!ok || i >= n) return;
  const int k = kind[i];
  float g[3] = {0.f, 0.f, 0.f};
  if (k == 1) {
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = grad_S[a * ldg + i] * inv_denom;
  }
  stats[i] = 0.f;
  stats[lds + i] = 0.f;
#pragma unroll
  for (int q = 0; q < 20; ++q) grad_S[q * ldg + i] = 0.f;
  if (k == 0) return;
  const int64_t b = dest[i];
#pragma unroll
  for (int q = 0; q < 14; ++q) params[q * ld + b] = params[q * ld + i];
#pragma unroll
  for (int q = 0; q < 20; ++q) grad_S[q * ldg + b] = 0.f;
  stats[b] = 0.f;
  stats[lds + b] = 0.f;
  if (k == 1) {                                        // clone (ADC (ii)): copy displaced along -G
#pragma unroll
    for (int a = 0; a < 3; ++a) params[a * ld + b] = params[a * ld + i] - clone_step * g[a];
    return;
  }
  // split (ADC (iii)): p_j = p + R diag(s) z_j, s_j = scale_factor * s
  const float qw = params[6 * ld + i], qx = params[7 * ld + i], qy = params[8 * ld + i], qz = params[9 * ld + i];
  const float qn = 1.0f / sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
  const float w = qw * qn, x = qx * qn, y = qy * qn, z = qz * qn;
  const float r[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                      2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                      2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
  const float ls[3] = {params[3 * ld + i], params[4 * ld + i], params[5 * ld + i]};
  const float s[3] = {expf(ls[0]), expf(ls[1]), expf(ls[2])};
  const float p[3] = {params[0 * ld + i], params[1 * ld + i], params[2 * ld + i]};
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int64_t slot = j == 0 ? i : b;
    const float u[3] = {s[0] * normals[(3 * j + 0) * ldz + i], s[1] * normals[(3 * j + 1) * ldz + i],
                        s[2] * normals[(3 * j + 2) * ldz + i]};
#pragma unroll
    for (int a = 0; a < 3; ++a) params[a * ld + slot] = p[a] + (r[3 * a] * u[0] + r[3 * a + 1] * u[1] + r[3 * a + 2] * u[2]);
#pragma unroll
    for (int a = 0; a < 3; ++a) params[(3 + a) * ld + slot] = ls[a] + log_scale_factor;
  }
}

inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

size_t adc_ws_bytes(int64_t n) {
  const int64_t tiles = (n + kTileItems - 1) / kTileItems;
  return align_up(8 * (size_t)(tiles > 0 ? tiles : 1)) + 256;
}

cudaError_t launch_adc(float* params, int64_t ld, int64_t n, int64_t capacity, float* grad_S, int64_t ldg,
                       float* stats, int64_t lds, const float* normals, int64_t ldz, const steepgs_adc_params& ap,
                       uint8_t* kind, int32_t* dest, int64_t* n_new, int32_t* status, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
  const size_t need = adc_ws_bytes(n);
  if (ws_bytes < need) return cudaErrorInvalidValue;
  char* w = static_cast<char*>(ws);
  uint64_t* lb = reinterpret_cast<uint64_t*>(w);
  int* counter = reinterpret_cast<int*>(w + need - 256);
  cudaError_t e = cudaMemsetAsync(ws, 0, need, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(n_new, 0, sizeof(int64_t), st);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    const unsigned tiles = (unsigned)((n + kTileItems - 1) / kTileItems);
    k_adc_decide<<<tiles, kThreads, 0, st>>>(params, ld, n, stats, lds, ap.eps_adc, ap.tau_adc, kind, dest, lb,
                                            counter, n_new);
    note_launch();
    if ((e = check_launch("k_adc_decide")) != cudaSuccess) return e;
  }
  const unsigned b1 = (unsigned)((n + kThreads - 1) / kThreads);
  k_adc_apply<<<b1 > 0 ? b1 : 1, kThreads, 0, st>>>(params, ld, n, capacity, grad_S, ldg, stats, lds, normals, ldz,
                                                    ap.clone_step, 1.0f / ap.denom, logf(ap.scale_factor), kind, dest,
                                                    n_new, status);
  note_launch();
  return check_launch("k_adc_apply");
}

}  // namespace sgs
