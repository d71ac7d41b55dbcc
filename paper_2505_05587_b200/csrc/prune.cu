// prune.cu — the opacity pruning of the 3DGS density control that SteepGS keeps ("ADC ...
// prunes invisible points"; 3DGS removes Gaussians with opacity < 0.005 at every densification).
//
//   k_prune_decide   keep iff logit >= logit_min (the threshold compared in logit space, so the
//                    decision is exact: no sigmoid rounding); single-pass exclusive scan of the keep
//                    flags (decoupled look-back) -> new_index (-1 for pruned), n_keep.
//   k_compact_planes dst[:, new_index[i]] = src[:, i] for every plane (out of place: stable order).
// Bound: HBM.
#include "common.cuh"
#include "scan.cuh"

namespace sgs {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kPTile = kThreads * kItems;
static_assert(kItems * (kThreads / 32) == 64, "the block scan gives each of 32 lanes two (item, warp) counts");

__global__ void __launch_bounds__(kThreads) k_prune_decide(const float* __restrict__ logit, int64_t n, float logit_min,
                                                           int32_t* __restrict__ new_index, uint64_t* status,
                                                           int* tile_counter, int64_t* n_keep) {
  __shared__ int s_tile;
  __shared__ uint32_t s_cnt[kItems][kThreads / 32];
  __shared__ uint64_t s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * kPTile;
  bool keep[kItems];
  uint32_t pos[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int64_t i = base + (int64_t)j * kThreads + tid;
    keep[j] = i < n && logit[i] >= logit_min;
    const uint32_t b = __ballot_sync(0xffffffffu, keep[j]);
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
      if (base + kPTile >= n) *n_keep = (int64_t)(excl + agg);
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int64_t i = base + (int64_t)j * kThreads + tid;
    if (i < n) new_index[i] = keep[j] ? (int32_t)(s_excl + s_cnt[j][warp] + pos[j]) : -1;
  }
}

__global__ void __launch_bounds__(256) k_compact_planes(const float* __restrict__ src, int64_t ld_src,
                                                        float* __restrict__ dst, int64_t ld_dst, int planes, int64_t n,
                                                        const int32_t* __restrict__ new_index) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t d = new_index[i];
  if (d < 0) return;
  for (int k = 0; k < planes; ++k) dst[k * ld_dst + d] = src[k * ld_src + i];
}

}  // namespace

size_t prune_ws_bytes(int64_t n) {
  const int64_t tiles = (n + kPTile - 1) / kPTile;
  return (size_t)(8 * (tiles > 0 ? tiles : 1) + 255) / 256 * 256 + 256;
}

cudaError_t launch_prune_decide(const float* logit, int64_t n, float logit_min, int32_t* new_index, int64_t* n_keep,
                                void* ws, size_t ws_bytes, cudaStream_t st) {
  const size_t need = prune_ws_bytes(n);
  if (ws_bytes < need) return cudaErrorInvalidValue;
  char* w = static_cast<char*>(ws);
  cudaError_t e = cudaMemsetAsync(ws, 0, need, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(n_keep, 0, sizeof(int64_t), st);
  if (e != cudaSuccess) return e;
  if (n == 0) return cudaSuccess;
  const unsigned tiles = (unsigned)((n + kPTile - 1) / kPTile);
  k_prune_decide<<<tiles, kThreads, 0, st>>>(logit, n, logit_min, new_index, reinterpret_cast<uint64_t*>(w),
                                            reinterpret_cast<int*>(w + need - 256), n_keep);
  note_launch();
  return check_launch("k_prune_decide");
}

cudaError_t launch_compact_planes(const float* src, int64_t ld_src, float* dst, int64_t ld_dst, int planes, int64_t n,
                                  const int32_t* new_index, cudaStream_t st) {
  if (n == 0 || planes == 0) return cudaSuccess;
  k_compact_planes<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, ld_src, dst, ld_dst, planes, n, new_index);
  note_launch();
  return check_launch("k_compact_planes");
}

}  // namespace sgs
