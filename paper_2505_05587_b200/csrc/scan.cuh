// scan.cuh — single-pass decoupled look-back helpers (device-only, internal).
#pragma once
#include <stdint.h>

namespace sgs {

constexpr uint64_t kScanFlagAgg = 1ull << 62;
constexpr uint64_t kScanFlagPre = 2ull << 62;
constexpr uint64_t kScanValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) {
  return *reinterpret_cast<const volatile uint64_t*>(p);
}
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}
__device__ __forceinline__ void st_volatile(uint64_t* p, uint64_t v) { *reinterpret_cast<volatile uint64_t*>(p) = v; }
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) { *reinterpret_cast<volatile uint32_t*>(p) = v; }

// Publish a tile's aggregate (tile 0 publishes its inclusive prefix directly).  One lane.
__device__ __forceinline__ void publish_aggregate(uint64_t* status, int tile, uint64_t aggregate) {
  st_volatile(&status[tile], (tile == 0 ? kScanFlagPre : kScanFlagAgg) | aggregate);
}

// Warp-parallel decoupled look-back (one warp) for a tile whose aggregate is already published.
// Returns the exclusive prefix of `tile` and publishes its inclusive prefix.
__device__ __forceinline__ uint64_t lookback_published(uint64_t* status, int tile, uint64_t aggregate) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) return 0;
  uint64_t excl = 0;
  int pred = tile - 1;
  while (true) {
    const int idx = pred - lane;
    uint64_t s = idx >= 0 ? ld_volatile(&status[idx]) : (kScanFlagPre | 0ull);
    while (__any_sync(0xffffffffu, (s >> 62) == 0)) {
      if ((s >> 62) == 0) s = ld_volatile(&status[idx]);
    }
    const uint32_t pre = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    const int stop = pre ? __ffs(pre) - 1 : 31;  // lowest lane = nearest predecessor with a prefix
    uint64_t v = lane <= stop ? (s & kScanValMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (pre) break;
    pred -= 32;
  }
  if (lane == 0) st_volatile(&status[tile], kScanFlagPre | (excl + aggregate));
  return excl;
}

// Publish + look back in one go (one warp).  Returns the exclusive prefix of `tile`.
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* status, int tile, uint64_t aggregate) {
  if ((threadIdx.x & 31) == 0) publish_aggregate(status, tile, aggregate);
  return lookback_published(status, tile, aggregate);
}


}  // namespace sgs
