// sort.cu — a2: bin & sort ("3DGS first sorts points according to view-dependent depth", P:L129;
// order C7 = ascending (depth key, index) within each (view, tile)).
//
// B200 design (no host synchronisation, graph-capturable):
//   1. k_count_visible + k_scan_tile_counts + k_compact: visible (view, Gaussian) pairs -> (depth
//                       key, slot) + 16-B record at offsets from a reduce-then-scan of per-tile
//                       counts; builds the 4 depth-digit histograms on the fly.
//   2. 4 x k_radix_pass  stable LSD radix sort of the 32-bit depth keys (8-bit digits, onesweep-style:
//                       warp match-based ranking, per-digit decoupled look-back, smem-staged coalesced
//                       scatter).  Ties keep (view, index) order because the input is in that order.
//   3. k_duplicate      exclusive scan of tiles_touched in depth order (look-back) and emission of one
//                       (view*tiles + tile, index) instance per touched tile; builds the tile-digit
//                       histograms on the fly.
//   4. 1-2 x k_radix_pass stable sort by tile key -> (view, tile, depth, index) order.
//   5. k_ranges         [start, end) per (view, tile).
// Sizes that are only known on the device (visible count, instance count) are read by the kernels;
// grids are sized by the host-known upper bounds and surplus blocks exit at once.
#include "common.cuh"
#include "scan.cuh"

namespace sgs {

SGS_CHECKS_TU(sort)

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;                      // items per thread per scan tile
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048
static_assert(kScanItems * (kScanThreads / 32) == 64, "the block scan gives each of 32 lanes two (item, warp) counts");
constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 12;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 3072
constexpr int kRadixItemsSmall = 4;                      // small sorts (one view): 1024-item tiles
constexpr int kRadixTileSmall = kRadixThreads * kRadixItemsSmall;
constexpr int64_t kRadixSmallBelow = 1 << 21;  // sorts of fewer items use the small tile
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixLook = 4;  // predecessors per look-back round trip (16 / 32: measured slower)

// Items per radix tile for a sort of up to `count` keys: 3072 fills 148 SMs x 3 blocks from ~1.4M
// keys up; below 2M keys (a one-view step: ~0.55M visible pairs) 1024-key tiles give 3x the blocks.
inline int radix_tile_for(int64_t count) { return count < kRadixSmallBelow ? kRadixTileSmall : kRadixTile; }

constexpr uint32_t kRadFlagAgg = 1u << 30;
constexpr uint32_t kRadFlagPre = 2u << 30;
constexpr uint32_t kRadValMask = (1u << 30) - 1;

// ------------------------------------------------------------------------------------------------
// 1. compaction of visible pairs + depth-digit histograms
// ------------------------------------------------------------------------------------------------
// Visible items per compaction tile (tiles_touched > 0), then one exclusive scan of the tile counts:
// k_compact then knows its output offset at once (a decoupled look-back here walks back over most of
// the first wave's tiles, whose aggregates appear together but whose prefixes resolve one by one).
__global__ void __launch_bounds__(kScanThreads) k_count_visible(const int32_t* __restrict__ tiles_touched,
                                                                int64_t total, uint64_t* __restrict__ tile_count) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_w[kScanThreads / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t idx = base + (int64_t)j * kScanThreads + tid;
    c += (idx < total && __ldg(tiles_touched + idx) > 0) ? 1u : 0u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) s_w[warp] = c;
  __syncthreads();
  if (tid == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) t += s_w[w];
    tile_count[blockIdx.x] = t;
  }
}

// In-place exclusive scan of the tile counts (one block of 1024 threads, contiguous chunks).
__global__ void __launch_bounds__(1024) k_scan_tile_counts(uint64_t* __restrict__ v, int m, int64_t* total_out) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint64_t s_w[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int per = (m + 1023) / 1024;
  const int a = min(m, tid * per), b = min(m, a + per);
  uint64_t sum = 0;
  for (int i = a; i < b; ++i) sum += v[i];
  uint64_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint64_t x = s_w[lane];
    uint64_t y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += t;
    }
    s_w[lane] = y - x;
    if (lane == 31) *total_out = (int64_t)y;
  }
  __syncthreads();
  uint64_t run = s_w[warp] + inc - sum;
  for (int i = a; i < b; ++i) {
    const uint64_t c = v[i];
    v[i] = run;
    run += c;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_compact(const uint32_t* __restrict__ depth_key,
                                                          const uint2* __restrict__ tile_rect,
                                                          const int32_t* __restrict__ tiles_touched, int64_t n,
                                                          int64_t total, uint32_t* __restrict__ keys_out,
                                                          uint32_t* __restrict__ vals_out, uint4* __restrict__ recs,
                                                          const uint64_t* __restrict__ tile_offset, uint32_t* hist4) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_cnt[kScanItems][kScanThreads / 32];
  __shared__ uint32_t s_hist[4][256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int k = tid; k < 4 * 256; k += kScanThreads) (&s_hist[0][0])[k] = 0;
  const int tile = blockIdx.x;
  const int64_t base = (int64_t)tile * kScanTile;
  bool flag[kScanItems];
  uint32_t pos_in_warp[kScanItems];
  uint32_t key[kScanItems];
  uint2 rect[kScanItems];
  int32_t tt[kScanItems];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t idx = base + (int64_t)j * kScanThreads + tid;
    tt[j] = idx < total ? tiles_touched[idx] : 0;
  }
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t idx = base + (int64_t)j * kScanThreads + tid;
    flag[j] = tt[j] > 0;
    // the visible items' key and rect are loaded here, so their latency overlaps the block scan
    if (flag[j]) { key[j] = depth_key[idx]; rect[j] = tile_rect[idx]; }
    const uint32_t b = __ballot_sync(0xffffffffu, flag[j]);
    pos_in_warp[j] = __popc(b & lanemask_lt());
    if (lane == 0) s_cnt[j][warp] = __popc(b);
  }
  __syncthreads();
  // exclusive scan of the 64 warp counts in (j, warp) order by warp 0
  if (warp == 0) {
    const int nw = kScanThreads / 32;
    uint32_t a = s_cnt[(2 * lane) / nw][(2 * lane) % nw], b = s_cnt[(2 * lane + 1) / nw][(2 * lane + 1) % nw];
    uint32_t sum = a + b, inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t ex = inc - sum;
    s_cnt[(2 * lane) / nw][(2 * lane) % nw] = ex;
    s_cnt[(2 * lane + 1) / nw][(2 * lane + 1) % nw] = ex + a;
  }
  __syncthreads();
  const uint64_t bex = tile_offset[tile];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    if (!flag[j]) continue;
    const int64_t idx = base + (int64_t)j * kScanThreads + tid;
    const uint64_t pos = bex + s_cnt[j][warp] + pos_in_warp[j];
    keys_out[pos] = key[j];
    vals_out[pos] = (uint32_t)pos;
    const uint32_t v = (uint32_t)(idx / n), i = (uint32_t)(idx - (int64_t)v * n);
    recs[pos] = make_uint4(rect[j].x, rect[j].y, i, (v << 24) | (uint32_t)tt[j]);
#pragma unroll
    for (int p = 0; p < 4; ++p) atomicAdd(&s_hist[p][(key[j] >> (8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int k = tid; k < 4 * 256; k += kScanThreads) {
    const uint32_t c = (&s_hist[0][0])[k];
    if (c) atomicAdd(&hist4[k], c);
  }
}

// ------------------------------------------------------------------------------------------------
// 2/4. one stable LSD radix pass (8-bit digit at `shift`), onesweep-style.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t v, uint32_t* s_warp /*[8]*/) {
  // 256 threads, one value each -> exclusive scan (all threads participate)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  uint32_t wpre = 0;
#pragma unroll
  for (int w = 0; w < kRadixWarps; ++w) wpre += (w < warp) ? s_warp[w] : 0u;
  __syncthreads();
  return wpre + inc - v;
}

template <int kItems, int kMinBlocks, int kLook>
__global__ void __launch_bounds__(kRadixThreads, kMinBlocks) k_radix_pass(const uint32_t* __restrict__ keys_in,
                                                              const uint32_t* __restrict__ vals_in,
                                                              uint32_t* __restrict__ keys_out,
                                                              uint32_t* __restrict__ vals_out, const int64_t* n_dev,
                                                              int64_t n_max, int shift,
                                                              const uint32_t* __restrict__ ghist /*[256]*/,
                                                              uint32_t* status /*[tiles][256]*/, int* tile_counter) {
  pdl_wait();
  pdl_trigger();
  constexpr int kTile = kRadixThreads * kItems;
  __shared__ uint32_t s_keys[kTile];
  __shared__ uint32_t s_vals[kTile];
  __shared__ uint32_t s_whist[kRadixWarps][256];
  __shared__ uint32_t s_local[256];
  __shared__ uint32_t s_dbase[256];
  __shared__ uint32_t s_tmp[kRadixWarps];
  __shared__ int s_tile;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1);
  for (int k = tid; k < kRadixWarps * 256; k += kRadixThreads) (&s_whist[0][0])[k] = 0;
  __syncthreads();
  const int tile = s_tile;
  int64_t n = *n_dev;
  if (n > n_max) n = n_max;
  const int64_t base = (int64_t)tile * kTile;
  if (base >= n) return;
  const int64_t wbase = base + (int64_t)warp * (32 * kItems);
  uint32_t k[kItems], v[kItems];
  uint32_t d[kItems], rank[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int64_t idx = wbase + j * 32 + lane;
    const bool ok = idx < n;
    k[j] = ok ? keys_in[idx] : 0u;
    v[j] = ok ? vals_in[idx] : 0u;
    d[j] = ok ? ((k[j] >> shift) & 255u) : 256u;
  }
  const uint32_t lt = lanemask_lt();
  // warp-level ranking: peers by match.any; the lowest peer adds the group's size to the warp's
  // digit counter with a returning shared atomic.  The kItems atomics are independent instructions
  // issued in item order (one warp, in-order issue), so their latencies overlap instead of
  // forming a load -> store chain through shared memory, and equal digits keep item order.
  uint32_t peers[kItems], old[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) peers[j] = __match_any_sync(0xffffffffu, d[j]);
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    old[j] = 0u;
    if (d[j] < 256u && (peers[j] & lt) == 0u) old[j] = atomicAdd(&s_whist[warp][d[j]], (uint32_t)__popc(peers[j]));
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t before = __shfl_sync(0xffffffffu, old[j], __ffs(peers[j]) - 1);
    rank[j] = before + __popc(peers[j] & lt);
  }
  __syncthreads();
  // per digit (thread = digit): exclusive over warps, block total, look-back, bases
  const uint32_t dig = (uint32_t)tid;
  uint32_t tot = 0;
#pragma unroll
  for (int w = 0; w < kRadixWarps; ++w) {
    const uint32_t c = s_whist[w][dig];
    s_whist[w][dig] = tot;
    tot += c;
  }
  uint32_t excl = 0;
  if (tile == 0) {
    st_volatile(&status[dig], kRadFlagPre | tot);
  } else {
    st_volatile(&status[(int64_t)tile * 256 + dig], kRadFlagAgg | tot);
    // look back kLook predecessors per round trip (independent loads in flight), in order
    int p = tile - 1;
    bool found = false;
    while (!found) {
      uint32_t sv[kLook];
#pragma unroll
      for (int q = 0; q < kLook; ++q)
        sv[q] = p - q >= 0 ? ld_volatile(&status[(int64_t)(p - q) * 256 + dig]) : kRadFlagPre;
#pragma unroll
      for (int q = 0; q < kLook; ++q) {
        if (found) break;
        while ((sv[q] >> 30) == 0) sv[q] = ld_volatile(&status[(int64_t)(p - q) * 256 + dig]);
        excl += sv[q] & kRadValMask;
        found = (sv[q] >> 30) == 2;
      }
      p -= kLook;
    }
    st_volatile(&status[(int64_t)tile * 256 + dig], kRadFlagPre | (excl + tot));
  }
  const uint32_t gstart = block_excl_scan_256(ghist[dig], s_tmp);
  const uint32_t lstart = block_excl_scan_256(tot, s_tmp);
  s_local[dig] = lstart;
  s_dbase[dig] = gstart + excl;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (d[j] < 256u) {
      const uint32_t lp = s_local[d[j]] + s_whist[warp][d[j]] + rank[j];
      SGS_CHECK(lp < (uint32_t)kTile);
      s_keys[lp] = k[j];
      s_vals[lp] = v[j];
    }
  }
  __syncthreads();
  const int cnt = (int)((n - base) < kTile ? (n - base) : kTile);
  for (int idx = tid; idx < cnt; idx += kRadixThreads) {
    const uint32_t kk = s_keys[idx];
    const uint32_t dd = (kk >> shift) & 255u;
    const uint32_t g = s_dbase[dd] + (uint32_t)idx - s_local[dd];
    SGS_CHECK((int64_t)g < n);
    keys_out[g] = kk;
    vals_out[g] = s_vals[idx];
  }
}

// ------------------------------------------------------------------------------------------------
// 3. duplication: scan of tiles_touched in depth order, one instance per touched tile
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kScanThreads, 4) k_duplicate(const uint32_t* __restrict__ sorted_slots,
                                                            const uint4* __restrict__ recs, const int64_t* n_vis_dev,
                                                            int tiles_x, int tiles_per_view, int64_t max_instances,
                                                            uint32_t* __restrict__ inst_keys,
                                                            uint32_t* __restrict__ inst_ids, uint64_t* status,
                                                            int* tile_counter, uint32_t* hist2, int64_t* n_inst,
                                                            int32_t* overflow, int tile_passes) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_tile;
  __shared__ uint32_t s_cnt[kScanItems][kScanThreads / 32];
  __shared__ uint32_t s_hist[3][256];
  __shared__ uint64_t s_excl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1);
  for (int k = tid; k < 3 * 256; k += kScanThreads) (&s_hist[0][0])[k] = 0;
  __syncthreads();
  const int tile = s_tile;
  const int64_t nvis = *n_vis_dev;
  const int64_t base = (int64_t)tile * kScanTile;
  if (base >= nvis) return;
  uint4 rec[kScanItems];
  uint32_t pre[kScanItems];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t idx = base + (int64_t)j * kScanThreads + tid;
    rec[j] = idx < nvis ? recs[sorted_slots[idx]] : make_uint4(0, 0, 0, 0);
    const uint32_t tt = rec[j].w & 0xFFFFFFu;
    uint32_t inc = tt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    pre[j] = inc - tt;
    if (lane == 31) s_cnt[j][warp] = inc;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = kScanThreads / 32;
    uint32_t a = s_cnt[(2 * lane) / nw][(2 * lane) % nw], b = s_cnt[(2 * lane + 1) / nw][(2 * lane + 1) % nw];
    uint32_t sum = a + b, inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t ex = inc - sum;
    s_cnt[(2 * lane) / nw][(2 * lane) % nw] = ex;
    s_cnt[(2 * lane + 1) / nw][(2 * lane + 1) % nw] = ex + a;
    const uint32_t agg = __shfl_sync(0xffffffffu, inc, 31);
    const uint64_t excl = lookback_warp(status, tile, agg);
    if (lane == 0) {
      s_excl = excl;
      if (base + kScanTile >= nvis) {
        const int64_t I = (int64_t)(excl + agg);
        *n_inst = I;
        *overflow = I > max_instances ? 1 : 0;
      }
    }
  }
  __syncthreads();
  const uint64_t bex = s_excl;
  // Load-balanced emission: the warp emits the instances of its 32 items of group j together,
  // lane e handling instance e, e + 32, ... of the group; the source item is the last lane whose
  // exclusive prefix is <= e (5-step shuffle search), so a Gaussian covering many tiles is spread
  // over the warp and each store instruction writes 32 consecutive instances.
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const uint32_t tt = rec[j].w & 0xFFFFFFu;
    const uint32_t total = __shfl_sync(0xffffffffu, pre[j] + tt, 31);
    if (total == 0) continue;
    const uint64_t gbase = bex + s_cnt[j][warp];
    const uint32_t w = (rec[j].x >> 16) - (rec[j].x & 0xFFFFu) + 1u;
    for (uint32_t e0 = 0; e0 < total; e0 += 32) {
      const uint32_t e = e0 + (uint32_t)lane;
      int src = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint32_t p = __shfl_sync(0xffffffffu, pre[j], src + step);
        if (p <= e) src += step;
      }
      const uint32_t local = e - __shfl_sync(0xffffffffu, pre[j], src);
      const uint32_t sw = __shfl_sync(0xffffffffu, w, src);
      const uint32_t sx = __shfl_sync(0xffffffffu, rec[j].x, src);
      const uint32_t sy = __shfl_sync(0xffffffffu, rec[j].y, src);
      const uint32_t sid = __shfl_sync(0xffffffffu, rec[j].z, src);
      const uint32_t sview = __shfl_sync(0xffffffffu, rec[j].w, src) >> 24;
      if (e >= total) continue;
      const uint32_t dy = local / sw, dx = local - dy * sw;
      const uint32_t key = sview * (uint32_t)tiles_per_view + ((sy & 0xFFFFu) + dy) * (uint32_t)tiles_x +
                           (sx & 0xFFFFu) + dx;
      const uint64_t pos = gbase + e;
      if ((int64_t)pos >= max_instances) continue;
      inst_keys[pos] = key;
      inst_ids[pos] = sid;
      atomicAdd(&s_hist[0][key & 255u], 1u);
      if (tile_passes > 1) atomicAdd(&s_hist[1][(key >> 8) & 255u], 1u);
      if (tile_passes > 2) atomicAdd(&s_hist[2][(key >> 16) & 255u], 1u);
    }
  }
  __syncthreads();
  for (int k = tid; k < 3 * 256; k += kScanThreads) {
    const uint32_t c = (&s_hist[0][0])[k];
    if (c) atomicAdd(&hist2[k], c);
  }
}

// ------------------------------------------------------------------------------------------------
// 5. tile ranges
// ------------------------------------------------------------------------------------------------
// Four consecutive keys per thread (one 16-B load; the neighbours across the group boundary come
// from the adjacent lanes or one extra load).
__global__ void k_ranges(const uint32_t* __restrict__ keys, const int64_t* n_inst, int64_t max_instances,
                         uint2* __restrict__ ranges) {
  pdl_wait();
  pdl_trigger();
  int64_t I = *n_inst;
  if (I > max_instances) I = max_instances;
  const int64_t groups = (I + 3) / 4;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = 4 * g;
    uint32_t k[6];   // keys i0 - 1 .. i0 + 4
    if (i0 + 4 <= I) {
      const uint4 q = *reinterpret_cast<const uint4*>(keys + i0);   // keys buffer is 256-B aligned
      k[1] = q.x; k[2] = q.y; k[3] = q.z; k[4] = q.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) k[1 + j] = i0 + j < I ? keys[i0 + j] : 0u;
    }
    k[0] = i0 > 0 ? __ldg(keys + i0 - 1) : ~0u;
    k[5] = i0 + 4 < I ? __ldg(keys + i0 + 4) : ~0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t i = i0 + j;
      if (i >= I) break;
      const uint32_t kk = k[1 + j];
      if (i == 0 || k[j] != kk) ranges[kk].x = (uint32_t)i;
      if (i == I - 1 || k[2 + j] != kk) ranges[kk].y = (uint32_t)(i + 1);
    }
  }
}

cudaError_t launch_radix(int tile, int grid, cudaStream_t st, const uint32_t* ki, const uint32_t* vi, uint32_t* ko,
                  uint32_t* vo, const int64_t* n_dev, int64_t n_max, int shift, const uint32_t* ghist, uint32_t* status,
                  int* counter) {
  if (tile == kRadixTileSmall)
    return launch_pdl(k_radix_pass<kRadixItemsSmall, 5, kRadixLook>, dim3(grid), dim3(kRadixThreads), 0, st, ki, vi, ko,
                      vo, n_dev, n_max, shift, ghist, status, counter);
  else
    return launch_pdl(k_radix_pass<kRadixItems, 3, kRadixLook>, dim3(grid), dim3(kRadixThreads), 0, st, ki, vi, ko, vo,
                      n_dev, n_max, shift, ghist, status, counter);
}

// 6. tile order for the raster kernels: (view, tile) indices by descending list length, in half-octave
// buckets (one block; the order inside a bucket is whatever the shared atomics give — it only decides
// which block runs which tile, never a result).  Long tiles start first, so the last wave is short.
__global__ void __launch_bounds__(1024) k_tile_order(const uint2* __restrict__ ranges, int m, int tiles_per_view,
                                                     int by_length, uint32_t* __restrict__ order) {
  pdl_wait();
  pdl_trigger();
    constexpr uint32_t kB = 65;
  __shared__ uint32_t s_cnt[kB];
  const int tid = threadIdx.x;
  if (!by_length) {
    for (int i = tid; i < m; i += 1024) {
      const uint32_t v = (uint32_t)(i / tiles_per_view), t = (uint32_t)(i - (int)v * tiles_per_view);
      order[i] = (v << 20) | t;
    }
    return;
  }
  if (tid < (int)kB) s_cnt[tid] = 0u;
  __syncthreads();
  auto key = [&](int i) {
    const uint2 r = ranges[i];
    const uint32_t len = r.y - r.x;
    if (len == 0u) return 64u;   // half-octave buckets, 0 for the longest lists
    const uint32_t c = (uint32_t)__clz(len), p = 31u - c;
    const uint32_t nb = p > 0u ? (len >> (p - 1u)) & 1u : 0u;
    return 2u * c + 1u - nb;
  };
  auto pack = [&](int i) {
    const uint32_t v = (uint32_t)(i / tiles_per_view), t = (uint32_t)(i - (int)v * tiles_per_view);
    return (v << 20) | t;   // (view, tile) packed: no division in the kernels
  };
  constexpr int kPer = 24;   // keys per thread kept in registers (all loads issued together)
  if (m <= 1024 * kPer) {
    uint32_t kk[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) kk[j] = j * 1024 + tid < m ? key(j * 1024 + tid) : kB;
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (kk[j] < kB) atomicAdd(&s_cnt[kk[j]], 1u);
    __syncthreads();
    if (tid == 0) {
      uint32_t run = 0;
      for (uint32_t k = 0; k < kB; ++k) {
        const uint32_t c = s_cnt[k];
        s_cnt[k] = run;
        run += c;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (kk[j] < kB) order[atomicAdd(&s_cnt[kk[j]], 1u)] = pack(j * 1024 + tid);
    return;
  }
  for (int i = tid; i < m; i += 1024) atomicAdd(&s_cnt[key(i)], 1u);
  __syncthreads();
  if (tid == 0) {
    uint32_t run = 0;
    for (uint32_t k = 0; k < kB; ++k) {
      const uint32_t c = s_cnt[k];
      s_cnt[k] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int i = tid; i < m; i += 1024) order[atomicAdd(&s_cnt[key(i)], 1u)] = pack(i);
}

cudaError_t launch_tile_order(const uint2* ranges, int tiles_total, int tiles_per_view, uint32_t* order,
                              cudaStream_t st) {
#ifdef SGS_NO_TILE_ORDER
  const bool identity = true;
#else
  const bool identity = false;
#endif
  const cudaError_t e = launch_pdl(k_tile_order, dim3(1), dim3(1024), 0, st, ranges, tiles_total, tiles_per_view,
                                   identity ? 0 : 1, order);
  note_launch();
  if (e != cudaSuccess) return e;
  return check_launch("k_tile_order");
}

inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
  size_t keysA, valsA, keysB, valsB, recs, keysC, valsC, keysD, valsD, ranges, tile_last, inst_mask, order;
  size_t st_compact, st_dup, st_depth, st_tile, counters, hist, scalars, end;
  size_t zero_begin, zero_end;
  int64_t items;
  int depth_tiles, inst_tiles, compact_tiles, depth_tile, inst_tile;
};

Layout layout(int64_t n, int V, int tiles_total, int64_t max_instances) {
  Layout L;
  const int64_t items = (int64_t)V * n;
  L.items = items;
  L.compact_tiles = (int)((items + kScanTile - 1) / kScanTile);
  L.depth_tile = radix_tile_for(items);
  L.inst_tile = radix_tile_for(max_instances);
  L.depth_tiles = (int)((items + L.depth_tile - 1) / L.depth_tile);
  L.inst_tiles = (int)((max_instances + L.inst_tile - 1) / L.inst_tile);
  size_t o = 0;
  auto take = [&](size_t bytes) { const size_t at = o; o = align_up(o + bytes); return at; };
  L.keysA = take(4 * (size_t)items);
  L.valsA = take(4 * (size_t)items);
  L.keysB = take(4 * (size_t)items);
  L.valsB = take(4 * (size_t)items);
  L.recs = take(16 * (size_t)items);
  L.keysC = take(4 * (size_t)max_instances);
  L.valsC = take(4 * (size_t)max_instances);
  L.keysD = take(4 * (size_t)max_instances);
  L.valsD = take(4 * (size_t)max_instances);
  L.ranges = take(8 * (size_t)tiles_total);
  L.inst_mask = take((size_t)max_instances);
  L.order = take(4 * (size_t)tiles_total);
  L.zero_begin = o;
  L.tile_last = take(4 * (size_t)tiles_total);
  L.st_compact = take(8 * (size_t)L.compact_tiles);
  L.st_dup = take(8 * (size_t)L.compact_tiles);
  L.st_depth = take(4 * 256 * 4 * (size_t)L.depth_tiles);
  L.st_tile = take(3 * 256 * 4 * (size_t)L.inst_tiles);
  L.counters = take(16 * sizeof(int));
  L.hist = take(7 * 256 * 4);
  L.scalars = take(4 * 8);
  L.zero_end = o;
  L.end = o;
  return L;
}

}  // namespace

size_t bin_sort_ws_bytes(int64_t n, int V, int tiles, int64_t max_instances) {
  return layout(n, V, tiles * V, max_instances).end;
}

cudaError_t launch_bin_sort(const uint32_t* depth_key, const uint32_t* tile_rect, const int32_t* tiles_touched,
                            int64_t n, int V, int tiles_x, int tiles_y, void* ws, size_t ws_bytes,
                            int64_t max_instances, steepgs_binning* out, cudaStream_t st) {
  const int tiles_per_view = tiles_x * tiles_y;
  const int tiles_total = tiles_per_view * V;
  const Layout L = layout(n, V, tiles_total, max_instances);
  if (ws_bytes < L.end) return cudaErrorInvalidValue;
  if (tiles_per_view >= (1 << 20) || V >= (1 << 12)) return cudaErrorInvalidValue;   // tile_order packing
  char* w = static_cast<char*>(ws);
  auto U32 = [&](size_t off) { return reinterpret_cast<uint32_t*>(w + off); };
  uint32_t* keysA = U32(L.keysA);
  uint32_t* valsA = U32(L.valsA);
  uint32_t* keysB = U32(L.keysB);
  uint32_t* valsB = U32(L.valsB);
  uint4* recs = reinterpret_cast<uint4*>(w + L.recs);
  uint32_t* keysC = U32(L.keysC);
  uint32_t* valsC = U32(L.valsC);
  uint32_t* keysD = U32(L.keysD);
  uint32_t* valsD = U32(L.valsD);
  uint2* ranges = reinterpret_cast<uint2*>(w + L.ranges);
  uint64_t* st_compact = reinterpret_cast<uint64_t*>(w + L.st_compact);
  uint64_t* st_dup = reinterpret_cast<uint64_t*>(w + L.st_dup);
  uint32_t* st_depth = U32(L.st_depth);
  uint32_t* st_tile = U32(L.st_tile);
  int* counters = reinterpret_cast<int*>(w + L.counters);
  uint32_t* hist = U32(L.hist);
  int64_t* scalars = reinterpret_cast<int64_t*>(w + L.scalars);
  int64_t* n_visible = scalars + 0;
  int64_t* n_inst = scalars + 1;
  int32_t* overflow = reinterpret_cast<int32_t*>(scalars + 2);

  cudaError_t e = cudaMemsetAsync(w + L.zero_begin, 0, L.zero_end - L.zero_begin, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(ranges, 0, 8 * (size_t)tiles_total, st);
  if (e != cudaSuccess) return e;
  out->ids = valsC;
  out->ranges = reinterpret_cast<const uint32_t*>(ranges);
  out->n_instances = n_inst;
  out->n_visible = n_visible;
  out->overflow = overflow;
  out->tile_last = U32(L.tile_last);
  out->inst_mask = reinterpret_cast<uint8_t*>(w + L.inst_mask);
  out->tile_order = reinterpret_cast<const uint32_t*>(w + L.order);
  out->max_instances = max_instances;
  out->tiles_x = tiles_x;
  out->tiles_y = tiles_y;
  out->V = V;
  if (L.items == 0) return launch_tile_order(reinterpret_cast<const uint2*>(ranges), tiles_total, tiles_per_view,
                                             U32(L.order), st);

  e = launch_pdl(k_count_visible, dim3(L.compact_tiles), dim3(kScanThreads), 0, st, tiles_touched, L.items, st_compact);
  note_launch();
  if (e != cudaSuccess) return e;
  if ((e = check_launch("k_count_visible")) != cudaSuccess) return e;
  e = launch_pdl(k_scan_tile_counts, dim3(1), dim3(1024), 0, st, st_compact, L.compact_tiles, n_visible);
  note_launch();
  if (e != cudaSuccess) return e;
  if ((e = check_launch("k_scan_tile_counts")) != cudaSuccess) return e;
  e = launch_pdl(k_compact, dim3(L.compact_tiles), dim3(kScanThreads), 0, st, depth_key,
                 reinterpret_cast<const uint2*>(tile_rect), tiles_touched, n, L.items, keysA, valsA, recs,
                 (const uint64_t*)st_compact, hist);
  note_launch();
  if (e != cudaSuccess) return e;
  if ((e = check_launch("k_compact")) != cudaSuccess) return e;
  // depth sort: A -> B -> A -> B -> A
  uint32_t *ki = keysA, *vi = valsA, *ko = keysB, *vo = valsB;
  for (int p = 0; p < 4; ++p) {
    e = launch_radix(L.depth_tile, L.depth_tiles, st, ki, vi, ko, vo, n_visible, L.items, 8 * p, hist + 256 * p,
                     st_depth + (size_t)p * 256 * L.depth_tiles, counters + 1 + p);
    note_launch();
    if (e != cudaSuccess) return e;
    if ((e = check_launch("k_radix_pass(depth)")) != cudaSuccess) return e;
    uint32_t* t;
    t = ki; ki = ko; ko = t;
    t = vi; vi = vo; vo = t;
  }
  // sorted slots now in vi (== valsA)
  const int tile_passes = tiles_total <= 256 ? 1 : (tiles_total <= 65536 ? 2 : 3);
  e = launch_pdl(k_duplicate, dim3(L.compact_tiles), dim3(kScanThreads), 0, st, vi, recs, n_visible, tiles_x,
                 tiles_per_view, max_instances, keysC, valsC, st_dup, counters + 5, hist + 4 * 256, n_inst, overflow,
                 tile_passes);
  note_launch();
  if (e != cudaSuccess) return e;
  if ((e = check_launch("k_duplicate")) != cudaSuccess) return e;
  // tile sort: one 8-bit pass per byte of the largest tile key (C -> D -> C ...)
  uint32_t *tki = keysC, *tvi = valsC, *tko = keysD, *tvo = valsD;
  for (int p = 0; p < tile_passes; ++p) {
    e = launch_radix(L.inst_tile, L.inst_tiles > 0 ? L.inst_tiles : 1, st, tki, tvi, tko, tvo, n_inst, max_instances,
                     8 * p, hist + (4 + p) * 256, st_tile + (size_t)p * 256 * L.inst_tiles, counters + 6 + p);
    note_launch();
    if (e != cudaSuccess) return e;
    if ((e = check_launch("k_radix_pass(tile)")) != cudaSuccess) return e;
    uint32_t* t;
    t = tki; tki = tko; tko = t;
    t = tvi; tvi = tvo; tvo = t;
  }
  out->ids = tvi;
  int64_t rb = (max_instances + 1023) / 1024;
  if (rb > 148 * 8) rb = 148 * 8;  // grid-stride: the true I is only known on the device
  e = launch_pdl(k_ranges, dim3((unsigned)(rb > 0 ? rb : 1)), dim3(256), 0, st, (const uint32_t*)tki,
                 (const int64_t*)n_inst, max_instances, ranges);
  note_launch();
  if (e != cudaSuccess) return e;
  if ((e = check_launch("k_ranges")) != cudaSuccess) return e;
  return launch_tile_order(ranges, tiles_total, tiles_per_view, U32(L.order), st);
}

}  // namespace sgs
