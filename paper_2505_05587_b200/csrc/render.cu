// render.cu — a3 forward compositing (Eq. eqn:alpha_blend), a4 l1 gradient helper
// (Eq. eqn:loss), a5 backward replay with the splitting-matrix moments (Thm 1 P:L232,
// §4.3).
//
// Work decomposition (B200): one block per 16x16 tile and view, the block -> tile map taken from
// binning.tile_order (bin_sort: longest tile lists first, so the last wave is short), warp-specialised:
//   * one producer warp (forward and backward) stages the tile's depth-ordered splats
//     into a ring of shared-memory buffers (5 in the forward, 3 in the backward) of kBatch splats:
//     the 64-B records are copied with cp.async (ids prefetched two batches ahead), made
//     tile-relative, and given the 8-bit mask of 8x4 sub-blocks their alpha support {m <= tau}
//     reaches (box test refined by an exact per-strip ellipse test).  The forward's consumers record
//     which list entries each warp composited (a per-lane shift register, OR-reduced over the warp
//     every 32 entries) and OR them into the batch's per-splat mask of COMPOSITING sub-blocks, which
//     the producers store as binning.inst_mask once the stage is released; the backward's producer
//     reads it instead of recomputing a geometric mask and copies only the 48 record bytes it needs,
//     so the backward visits exactly the (8x8 block, splat) pairs with a contribution.
//   * forward consumers: 8 warps, one pixel per thread, warp w on the 8x4 sub-block
//     x in 8 (w & 1) .. +7, y in 4 (w >> 1) .. +3;
//   * backward consumers (k_render_bwd2): 4 warps, two pixels per thread, warp w on the 8x8 block
//     (w & 1, w >> 1), lane (lx, ly) on pixels (lx, ly) and (lx, ly + 4), the per-pixel arithmetic
//     on packed f32x2 (fma/add/mul.rn.f32x2): one warp visit per (8x8 block, splat) instead of one
//     per (8x4 sub-block, splat).
// Each consumer compacts a staged batch to the splats whose mask reaches its block (ballots).
// Full/empty mbarriers per buffer replace block-wide barriers, so consumer warps with short lists
// run ahead by up to a ring's depth of batches instead of waiting for the slowest warp (waits:
// try_wait, then parked with a suspend-time hint).  Consumers take four list entries per iteration:
// the four pair tests are independent and are issued before the serial compositing / recursion,
// which is branch-free (predicated) so the four steps need no divergence bookkeeping.
//
// Per-pair arithmetic: the mean is made tile-relative in fp64 before rounding (offsets
// d = x - Pi(p) carry ~1e-7 px error); the conic arrives pre-scaled by log2(e)/2 (a1) so that
//   e = log2(o) - m',  m' = a + dy (b + Qyy' dy),  a = Qxx' dx^2,  b = 2 Qxy' dx,
//   skip if e < log2(alpha_min) (<=> sigma < alpha_min),  sigma = 2^e,  alpha = min(amax, sigma)
// with explicit round-to-nearest operations (scalar in the forward, the same operations per f32x2
// half in the backward), so forward and backward take bit-identical decisions.
//
// Backward: back to front over each pixel's composited prefix (n_contrib from the forward; the
// tile's longest prefix is stored by the forward), T_i recovered as T_{i+1} / (1 - alpha_i)
// (approximate reciprocal; relative error ~1 ulp per step), dL/dalpha_i = T_i sum_ch dL/dC_ch
// (c_ch - B_ch) with B the normalised colour behind (C10), w = dL/dsigma * sigma.  Two phases per
// chunk of list entries (a chunk continues across batch boundaries): the pixel-parallel recursion
// leaves each lane's two-pixel partial sums in shared memory, then lanes grouped per entry sum them
// with the lane positions as compile-time constants, rebuild the 9 moments (w, w d, w d d^T,
// alpha T dL/dC) in the block frame, recentre them on the splat mean and add them with vector REDs
// into moments[view][gid][12].  The splitting matrix needs no per-pair work of its own:
// S_view = P^T (Q M Q - m0 Q) P is formed per Gaussian from these moments (gauss_bwd.cu).
#include <atomic>

#include "common.cuh"

namespace sgs {

SGS_CHECKS_TU(render)

namespace {

constexpr int kConsumers = 8;                       // one pixel per thread, 8 warps per 16x16 tile
constexpr int kFwdProducers = 1;                    // one producer warp: 56 registers for the consumers (2 warps: 48, rematerialisation)
constexpr int kThreadsFwd = 32 * (kConsumers + kFwdProducers);
constexpr int kBatch = 128;                         // splats per staged batch
constexpr int kStages = 3;                          // ring depth (backward: bounded by shared memory)
constexpr int kFwdStages = 5;                       // forward ring depth (slack for unequal consumer warps)
constexpr uint32_t kSuspendNs = 1000000;            // mbarrier try_wait suspend-time hint (ns)

template <int kC>
struct BufferT {
  float4 geo[kBatch];            // (mu_x - ox, mu_y - oy, Qxx', 2 Qxy')   Q' = Q log2(e)/2
  float4 par[kBatch];            // (Qyy', log2(o), -, -)
  float4 col[kBatch];            // (r, g, b, -)
  float* mptr[kBatch];           // backward: &moments[view][gid][0]
  uint32_t mask[kBatch];         // sub-blocks reached by the alpha support
  uint32_t cm[kBatch];           // forward: sub-blocks in which >= 1 pixel composited the splat
  uint32_t cflag[kC][kBatch / 32];   // forward: per consumer, bit t = list entry t was composited
  uint8_t list[kC][kBatch];      // per-consumer compacted lists (written by the consumer)
  int base;                      // list position (relative to the tile start) of slot 0
  int stop;                      // 1: no more batches (forward early termination)
  int cnt;                       // forward: splats in the batch
  int64_t gpos;                  // forward: instance index (into binning.ids) of slot 0
};

// A staged batch: instances [pos, pos + cnt) of binning.ids, list positions trel.. of a tile with
// origin (ox, oy); stoppable: the forward may end the ring here once every consumer has terminated.
struct BatchInfo {
  int64_t pos;
  int cnt, trel;
  double ox, oy;
  bool stoppable;
};
using Buffer = BufferT<kConsumers>;

template <int kS, int kC = kConsumers, int kRaw = 4>
struct SmemT {
  BufferT<kC> buf[kS];
  uint4 raw[kRaw][kBatch];       // producer staging: the next batch's records (cp.async), SoA by 16 B
                                 // (the backward copies 3 of the 4 16-B parts: no extents)
  unsigned long long full[kS], empty[kS];
  int done_warps;
  int stop_flag[2];              // forward: the producers' shared early-exit decision (double-buffered)
};
using SmemFwd = SmemT<kFwdStages>;

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
// Wait for the phase with the given parity to complete: one try_wait without a hint (the phase is
// usually complete already), then try_wait with a suspend-time hint, which parks the warp in hardware
// until the phase completes or the hint elapses.  Measured against polling with an exponential
// __nanosleep back-off (64 ns .. 4 us): the back-off loop executed ~60 failed polls per consumer wait
// in the backward (the sleeps return early), ~9% of its issued instructions; parked waits issue none
// (bwd 1.855 -> 1.844 ms, fwd 0.877 -> 0.874 ms per C2 step).
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity, uint32_t suspend_ns) {
  const uint32_t a = saddr(b);
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  if (ok) return;
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}"
      :
      : "r"(a), "r"(parity), "r"(suspend_ns)
      : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// The pair test shared by forward and backward: e = log2(sigma) (skip if e < log2(alpha_min)).
__device__ __forceinline__ float pair_e(float dx, float dy, const float4 g, const float4 p) {
  const float a = __fmul_rn(__fmul_rn(g.z, dx), dx);
  const float bq = __fmul_rn(g.w, dx);
  const float m = __fmaf_rn(dy, __fmaf_rn(p.x, dy, bq), a);
  return __fsub_rn(p.y, m);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Producer (one warp): batch k covers tile-list positions [first + rel(k), + cnt(k)).  The records
// of batch k + 1 are copied with cp.async (16 x 16 B in flight per lane) and the ids of batch k + 2
// loaded while the warp waits for a free stage, so a batch costs the producer no exposed memory
// round trip once it runs ahead.  Staging a record is then two fp64 subtractions and eight
// interval tests of the padded extents against the 8x4 sub-blocks.
// kFwd: stop early once every consumer warp has terminated (forward early exit).
struct NoPrefetch {
  __device__ __forceinline__ void operator()() const {}
};

template <bool kFwd, int kProd, int kS, int kC = kConsumers, int kRaw = 4, class BatchOf, class Prefetch = NoPrefetch>
__device__ __forceinline__ void run_producer(SmemT<kS, kC, kRaw>& sm, const uint32_t* __restrict__ ids,
                                             const steepgs_splat* __restrict__ vs, int nb, BatchOf batch_of,
                                             float* mom_view, float lmin, uint8_t* __restrict__ inst_mask, int pw,
                                             int lane, int64_t n_g, Prefetch prefetch = Prefetch{}) {
  // producer warp pw of kProd stages the batch slots kk = (q kProd + pw) * 32 + lane
  constexpr int kQ = kBatch / 32 / kProd;
  uint32_t gcur[kQ], gnext[kQ];
  uint32_t mcur[kQ], mnext[kQ];   // backward: the forward's sub-block masks, prefetched with the ids
  auto load_ids = [&](int k, uint32_t* g, uint32_t* mk) {
    BatchInfo bi{0, 0, 0, 0.0, 0.0, false};
    if (k < nb) bi = batch_of(k);
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int kk = (q * kProd + pw) * 32 + lane;
      g[q] = kk < bi.cnt ? __ldg(ids + bi.pos + kk) : 0u;
      if (!kFwd) mk[q] = kk < bi.cnt ? (uint32_t)__ldg(inst_mask + bi.pos + kk) : 0u;
    }
  };
  auto issue = [&](int k, const uint32_t* g) {
    if (k < nb) {
      const BatchInfo bi = batch_of(k);
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int kk = (q * kProd + pw) * 32 + lane;
        if (kk < bi.cnt) {
          const uint4* src = reinterpret_cast<const uint4*>(vs + g[q]);
#pragma unroll
          for (int j = 0; j < (kFwd ? 4 : 3); ++j) cp_async16(&sm.raw[j][kk], src + j);   // bwd: no extents
        }
      }
    }
    cp_async_commit();
  };
  load_ids(0, gcur, mcur);
  issue(0, gcur);
  load_ids(1, gnext, mnext);
  // forward: once the consumers have released a stage, the composited sub-block masks of its batch
  // (cm, ORed in by the consumers) are stored as binning.inst_mask; each producer warp stores the
  // slots it stages, so no other synchronisation is needed
  auto flush = [&](const BufferT<kC>& Bf, int64_t pos0, int cnt0) {
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int kk = (q * kProd + pw) * 32 + lane;
      if (kk < cnt0) inst_mask[pos0 + kk] = (uint8_t)(Bf.cm[kk] & 0xFFu);
    }
  };
  int kend = nb, stopped = 0;
  for (int k = 0; k < nb; ++k) {
    const int s = k % kS;
    if (k >= kS) mbar_wait(&sm.empty[s], ((k / kS) & 1) ^ 1, kSuspendNs);
    BufferT<kC>& B = sm.buf[s];
    if (kFwd && k >= kS) flush(B, B.gpos, B.cnt);   // batch k - kS (read before the named barrier below)
    const BatchInfo bi = batch_of(k);
    int stop = 0;
    if (kFwd) {   // one decision per batch for all producer warps (a split decision would deadlock)
      if (kProd == 1) {
        stop = bi.stoppable && *reinterpret_cast<volatile int*>(&sm.done_warps) == kC;
      } else {
        if (pw == 0 && lane == 0)
          sm.stop_flag[k & 1] = bi.stoppable && *reinterpret_cast<volatile int*>(&sm.done_warps) == kC;
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kProd) : "memory");
        stop = *reinterpret_cast<volatile int*>(&sm.stop_flag[k & 1]);
      }
    }
    const int cnt = bi.cnt;
    const double ox = bi.ox, oy = bi.oy;
    cp_async_wait_all();
    if (!stop) {
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int kk = (q * kProd + pw) * 32 + lane;
        if (kk >= cnt) { B.mask[kk] = 0u; continue; }
        SGS_CHECK((int64_t)gcur[q] < n_g);                           // instance ids index the splats
        const double2 mean = *reinterpret_cast<const double2*>(&sm.raw[0][kk]);
        const float4 a = *reinterpret_cast<const float4*>(&sm.raw[1][kk]);   // conic', log2 o
        const float4 b = *reinterpret_cast<const float4*>(&sm.raw[2][kk]);   // rgb, o
        const float gx = (float)(mean.x - ox), gy = (float)(mean.y - oy);
        B.geo[kk] = make_float4(gx, gy, a.x, a.y);
        B.par[kk] = make_float4(a.z, a.w, 0.0f, 0.0f);
        B.col[kk] = make_float4(b.x, b.y, b.z, 0.0f);
        if (mom_view) B.mptr[kk] = mom_view + (size_t)gcur[q] * 12;
        if (!kFwd) {   // the backward reuses the forward's masks (same splat, same tile)
          B.mask[kk] = mcur[q];
          continue;
        }
        const float4 c = *reinterpret_cast<const float4*>(&sm.raw[3][kk]);   // extents, tau
        uint32_t xb = 0u;
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (gx - c.x <= 8.0f * t + 7.5f && gx + c.x >= 8.0f * t + 0.5f) xb |= 1u << t;
        // per 4-row strip, the x-range of the ellipse {m' <= tau'} over the strip's pixel-centre rows:
        // centre line -b dy / 2a (extremes at the strip ends) +- the half-width at the dy nearest 0,
        // sqrt(4 a tau' - (4ac - b^2) dy^2) / 2a.  Conservative (tau' and the range padded), so only
        // sub-blocks without a pixel in the alpha support are dropped (16% of the AABB's, C2).
        const float tq = fmaf(a.w - lmin, 1.0001f, 1e-4f);
        const float qa = a.x, qb = a.y, qc = a.z;
        const float delta = 4.0f * qa * qc - qb * qb;
        const float inv2a = __fdividef(0.5f, qa), slope = -qb * inv2a;   // approximate: covered by the padding
        uint32_t m = 0u;
#pragma unroll
        for (int t = 0; t < 4; ++t) {   // branch-free: the four strips' tests are predicated
          const bool inb = gy - c.y <= 4.0f * t + 3.5f && gy + c.y >= 4.0f * t + 0.5f;
          const float dy0 = 4.0f * t + 0.5f - gy, dy1 = dy0 + 3.0f;
          const float dym = fminf(fmaxf(0.0f, dy0), dy1);
          const float D = 4.0f * qa * tq - delta * dym * dym;
          const bool ok = inb && D >= 0.0f;
          float sq;
          asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(D));          // inf stays inf (smooth mode)
          const float hw = sq * inv2a * 1.0001f + 0.01f;
          const float x0 = slope * dy0, x1 = slope * dy1;
          const float lo = gx + fminf(x0, x1) - hw, hi = gx + fmaxf(x0, x1) + hw;
          uint32_t xs = 0u;
          if (hi >= 0.5f && lo <= 7.5f) xs |= 1u;
          if (hi >= 8.5f && lo <= 15.5f) xs |= 2u;
          m |= ok ? (xs & xb) << (2 * t) : 0u;
        }
        B.mask[kk] = m;
        B.cm[kk] = 0u;              // the consumers OR in the sub-blocks that composite the splat
      }
    }
    if (pw == 0 && lane == 0) {
      B.base = bi.trel;
      B.stop = stop;
      B.cnt = cnt;
      B.gpos = bi.pos;
    }
    __syncwarp();
    mbar_arrive(&sm.full[s]);
    if (stop) {
      kend = k;
      stopped = 1;
      break;
    }
    if (k == 0) prefetch();   // while the consumers work on the first batch
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      gcur[q] = gnext[q];
      mcur[q] = mnext[q];
    }
    issue(k + 1, gcur);
    load_ids(k + 2, gnext, mnext);
  }
  cp_async_wait_all();
  if (kFwd) {   // the batches still in the ring (the stop batch itself was never consumed)
    for (int kb = max(0, kend - kS + stopped); kb < kend; ++kb) {
      const int s = kb % kS;
      mbar_wait(&sm.empty[s], (kb / kS) & 1, kSuspendNs);
      flush(sm.buf[s], sm.buf[s].gpos, sm.buf[s].cnt);
    }
  }
}

// Consumer: compact the staged batch to the splats whose mask has bit `w` (ascending order, slots
// below `limit`) into the warp's own list; returns the count.
template <int kC>
__device__ __forceinline__ int build_list(const BufferT<kC>& B, uint8_t* __restrict__ list, uint32_t wbits, int lane,
                                          int limit = kBatch) {
  int total = 0;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int q = 0; q < kBatch / 32; ++q) {
    const bool hit = (B.mask[q * 32 + lane] & wbits) != 0u && q * 32 + lane < limit;
    const uint32_t bal = __ballot_sync(0xffffffffu, hit);
    if (hit) list[total + __popc(bal & lt)] = (uint8_t)(q * 32 + lane);
    total += __popc(bal);
  }
  __syncwarp();
  return total;
}

// The (tile, view) a block renders: entry blockIdx of binning.tile_order (bin_sort's order, longest
// lists first; view << 20 | tile).
// kReload: an opaque second load (the forward's epilogue re-reads its tile instead of keeping tile and
// view live through the blend loop, whose 56 registers would otherwise rematerialise ~16 instructions
// per four entries).
template <bool kReload = false>
__device__ __forceinline__ void tile_of_block(const uint32_t* __restrict__ order, int& tile, int& view) {
  const uint32_t* p = order + (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  uint32_t t;
  if (kReload)
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(t) : "l"(p));
  else
    t = __ldg(p);
  view = (int)(t >> 20);
  tile = (int)(t & 0xFFFFFu);
}

template <bool kCount>   // kCount: also count composited / evaluated pairs (the roofline's units)
__global__ void __launch_bounds__(kThreadsFwd, 4) k_render_fwd(const steepgs_splat* __restrict__ splats,
                                                         const uint32_t* __restrict__ ids,
                                                         const uint2* __restrict__ ranges, int64_t n, int W, int H,
                                                         int tiles_x, int tiles_per_view, const RasterK rk,
                                                         float* __restrict__ image, float* __restrict__ final_T,
                                                         int32_t* __restrict__ n_contrib,
                                                         uint32_t* __restrict__ tile_last,
                                                         uint8_t* __restrict__ inst_mask,
                                                         unsigned long long* __restrict__ pair_counts,
                                                         const L1Fused l1, const uint32_t* __restrict__ order) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char fsmem[];
  SmemFwd& sm = *reinterpret_cast<SmemFwd*>(fsmem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int tile, view;
  tile_of_block(order, tile, view);
  SGS_CHECK(tile < tiles_per_view && view < (int)gridDim.y);   // tile_order entries are (view, tile)
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const uint2 rg = ranges[(int64_t)view * tiles_per_view + tile];
  const int nb = (int)((rg.y - rg.x + kBatch - 1) / kBatch);
  if (tid == 0) {
    for (int s = 0; s < kFwdStages; ++s) {
      mbar_init(&sm.full[s], 32 * kFwdProducers);
      mbar_init(&sm.empty[s], 32 * kConsumers);
    }
    sm.done_warps = 0;
  }
  __syncthreads();

  if (warp >= kConsumers) {  // ---------------- producers ----------------
    const int len = (int)(rg.y - rg.x);
#ifndef SGS_FWD_PREFETCH
#define SGS_FWD_PREFETCH 300   // ~half of the 592 resident blocks ahead (150 / 450 / 592 / 1200 measured)
#endif
#if SGS_FWD_PREFETCH > 0
    // Warm L2 for a block about half a wave later (tile_order entry blockIdx + kAhead): its range, the
    // ids of its first batch and their splat records, so that block's start chain (entry -> range ->
    // ids -> records) runs on L2 hits instead of DRAM round trips.
    auto pf = [=]() {
      const int64_t fidx = (int64_t)blockIdx.y * gridDim.x + blockIdx.x + SGS_FWD_PREFETCH;
      if (fidx >= (int64_t)gridDim.x * gridDim.y) return;
      uint32_t e = 0u;
      uint2 frg = make_uint2(0u, 0u);
      if (lane == 0) {
        e = __ldg(order + fidx);
        frg = ranges[(int64_t)(e >> 20) * tiles_per_view + (e & 0xFFFFFu)];
      }
      e = __shfl_sync(0xffffffffu, e, 0);
      frg.x = __shfl_sync(0xffffffffu, frg.x, 0);
      frg.y = __shfl_sync(0xffffffffu, frg.y, 0);
      const int fcnt = min((int)(frg.y - frg.x), kBatch);
      const steepgs_splat* fv = splats + (int64_t)(e >> 20) * n;
#pragma unroll
      for (int q = 0; q < kBatch / 32; ++q) {
        const int kk = q * 32 + lane;
        if (kk < fcnt) {
          const uint32_t g = __ldg(ids + frg.x + kk);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(fv + g));
        }
      }
    };
#else
    auto pf = NoPrefetch{};
#endif
    run_producer<true, kFwdProducers, kFwdStages>(
        sm, ids, splats + (int64_t)view * n, nb,
        [len, rg, ox, oy](int k) {
          return BatchInfo{(int64_t)rg.x + k * kBatch, min(len - k * kBatch, kBatch), k * kBatch, ox, oy, true};
        },
        nullptr, __log2f(rk.alpha_min), inst_mask, warp - kConsumers, lane, n, pf);
    return;
  }

  // ---------------- consumers ----------------
  const int lx = 8 * (warp & 1) + (lane & 7), ly = 4 * (warp >> 1) + (lane >> 3);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = px < W && py < H;
  // pixel centre, tile-relative (Z5).  Opaque (asm) so ptxas keeps them in registers: at 56 registers it
  // otherwise rematerialises them from the thread index inside the blend loop (+6 instructions per four
  // entries, 0.967 vs 0.992 ms per C2 step)
  float fx, fy;
  asm volatile("mov.b32 %0, %1;" : "=f"(fx) : "f"((float)lx + 0.5f));
  asm volatile("mov.b32 %0, %1;" : "=f"(fy) : "f"((float)ly + 0.5f));
  const float lmin = __log2f(rk.alpha_min);                   // -inf in smooth mode
  const float amax = rk.alpha_max, tmin = rk.t_min;
  float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
  int last = 0, ncomp = 0, neval = 0;
  bool done = !inside, warp_done = false;
  for (int k = 0; k < nb; ++k) {
    const int s = k % kFwdStages;
    mbar_wait(&sm.full[s], (k / kFwdStages) & 1, kSuspendNs);
    const Buffer& B = sm.buf[s];
    SGS_CHECK(B.base == k * kBatch);                 // the stage holds batch k (mbarrier ring protocol)
    if (B.stop) break;
    if (!warp_done) {
      uint8_t* lst = sm.buf[s].list[warp];
      const int nl = build_list(B, lst, 1u << warp, lane);
      const int base1 = B.base + 1;
      if (kCount && !done) neval += nl;
      // Two entries per iteration: both pair tests ahead of the serial compositing (as in the bwd).
      // Branch-free (predicated) so the four calls need no divergence bookkeeping; the values are
      // those of the plain C8 loop.
      // Which list entries the warp composited (a warp OR-reduction per four entries into cflag);
      // after the batch they are ORed into the batch's cm[] (sub-blocks with >= 1 composited pixel),
      // which the producers store as binning.inst_mask once the stage is released, so the backward
      // visits exactly the (block, splat) pairs that contribute.
      uint32_t* cfl = sm.buf[s].cflag[warp];
      if (lane < kBatch / 32) cfl[lane] = 0u;
      __syncwarp();
      auto blend = [&](float e, int j) -> bool {
        const bool live = !done && e >= lmin;             // sigma < alpha_min: C8 skip
        const float alpha = fminf(amax, ex2_approx(e));
        const float Tn = __fmul_rn(T, __fsub_rn(1.0f, alpha));
        const bool term = live && Tn < tmin;              // C8 termination
        const bool comp = live && !term;
        done = done || term;
        const float4 c = B.col[j];
        const float aT = __fmul_rn(alpha, T);
        C0 = comp ? __fmaf_rn(aT, c.x, C0) : C0;
        C1 = comp ? __fmaf_rn(aT, c.y, C1) : C1;
        C2 = comp ? __fmaf_rn(aT, c.z, C2) : C2;
        T = comp ? Tn : T;
        last = comp ? base1 + j : last;
        if (kCount) ncomp += comp ? 1 : 0;
        return comp;
      };
      // lb: a shift register of this lane's composited flags (one LEA per entry): after list position
      // t, bit 0 is position t, bit k position t - k.  Every 32 positions (at the top of the loop, lanes
      // converged) and after the batch the warp's OR of the lanes' words is stored to cflag[w], with
      // position 32 w + i at bit 31 - i.
      // the list in words of 32 entries: groups of four, then the word's tail, then the word's flush
      for (int w0 = 0; w0 < nl; w0 += 32) {
        const int tend = min(nl, w0 + 32);
        uint32_t lb = 0u;
        int t = w0;
        for (; t + 3 < tend; t += 4) {
          int jj[4];
          float ee[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            jj[u] = lst[t + u];
            const float4 g = B.geo[jj[u]];
            const float2 p = *reinterpret_cast<const float2*>(&B.par[jj[u]]);
            ee[u] = pair_e(__fsub_rn(fx, g.x), __fsub_rn(fy, g.y), g, make_float4(p.x, p.y, 0.f, 0.f));
          }
          // no skip when this lane is done: blend() composites nothing then (live = !done), and a
          // divergent branch here only costs its reconvergence (0.973 -> 0.962 ms per C2 step)
          bool cb[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) cb[u] = blend(ee[u], jj[u]);
          lb = (lb << 4) | (cb[0] ? 8u : 0u) | (cb[1] ? 4u : 0u) | (cb[2] ? 2u : 0u) | (cb[3] ? 1u : 0u);
        }
        for (; t < tend; ++t) {
          const int ja = lst[t];
          const float4 ga = B.geo[ja];
          const float2 pa = *reinterpret_cast<const float2*>(&B.par[ja]);
          bool c = false;
          if (!done) c = blend(pair_e(__fsub_rn(fx, ga.x), __fsub_rn(fy, ga.y), ga, make_float4(pa.x, pa.y, 0.f, 0.f)), ja);
          lb = (lb << 1) | (uint32_t)c;
        }
        // position w0 + i at bit 31 - i (a partial word is shifted up)
        const uint32_t wb = __reduce_or_sync(0xffffffffu, lb) << ((32 - (tend - w0)) & 31);
        if (lane == 0) cfl[w0 >> 5] = wb;
        if (__all_sync(0xffffffffu, done)) break;   // the rest of the list composites nothing here
      }
      __syncwarp();
      for (int tt = lane; tt < nl; tt += 32)
        if ((cfl[tt >> 5] >> (31 - (tt & 31))) & 1u) atomicOr(&sm.buf[s].cm[lst[tt]], 1u << warp);
      if (__all_sync(0xffffffffu, done)) {
        warp_done = true;
        if (lane == 0) atomicAdd(&sm.done_warps, 1);
      }
    }
    mbar_arrive(&sm.empty[s]);
  }
  // epilogue: the tile is re-read from tile_order (not kept live through the blend loop)
  int etile, eview;
  tile_of_block<true>(order, etile, eview);
  const int epx = (etile % tiles_x) * kTile + lx, epy = (etile / tiles_x) * kTile + ly;
  float ad = 0.0f;   // fused l1: this pixel's sum of |C - C_hat| over the channels
  if (epx < W && epy < H) {
    const int64_t HW = (int64_t)W * H;
    const int64_t pix = (int64_t)epy * W + epx;
    float* img = image + (int64_t)eview * 3 * HW;
    const float out[3] = {__fmaf_rn(T, rk.bg[0], C0), __fmaf_rn(T, rk.bg[1], C1), __fmaf_rn(T, rk.bg[2], C2)};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) img[ch * HW + pix] = out[ch];
    final_T[(int64_t)eview * HW + pix] = T;
    n_contrib[(int64_t)eview * HW + pix] = last;
    if (l1.target || l1.target_u8) {   // a4 fused: dL/dC = scale sign(C - C_hat), the same expression as k_l1_grad
      const int64_t o = (int64_t)eview * 3 * HW + pix;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const float tv = l1.target ? __ldg(l1.target + o + ch * HW)
                                   : __fmul_rn((float)__ldg(l1.target_u8 + o + ch * HW), 1.0f / 255.0f);
        const float r = out[ch] - tv;
        l1.dL[o + ch * HW] = r > 0.0f ? l1.scale : (r < 0.0f ? -l1.scale : 0.0f);
        ad += fabsf(r);
      }
    }
  }
  if (l1.loss) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ad += __shfl_xor_sync(0xffffffffu, ad, o);
    if (lane == 0) atomicAdd(l1.loss + eview, ad * l1.scale);
  }
  {
    const int wl = __reduce_max_sync(0xffffffffu, last);   // the tile's composited prefix, for the backward
    if (lane == 0 && wl > 0) atomicMax(tile_last + (int64_t)eview * tiles_per_view + etile, (uint32_t)wl);
  }
  if (kCount) {
    unsigned long long c = (unsigned long long)ncomp, e = (unsigned long long)neval;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      c += __shfl_xor_sync(0xffffffffu, c, o);
      e += __shfl_xor_sync(0xffffffffu, e, o);
    }
    if (lane == 0) {
      atomicAdd(&pair_counts[0], c);
      atomicAdd(&pair_counts[1], e);
    }
  }
}

__device__ __forceinline__ void red_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// ------------------------------------------------------------------------------------------------
// Backward, two pixels per lane.  Four consumer warps per 16x16 tile, warp w owns the 8x8 block
// (bx, by) = (w & 1, w >> 1); lane (lx, ly) = (lane & 7, lane >> 3) owns pixels a = (lx, ly) and
// b = (lx, ly + 4) of the block (the same column, so the pair test shares dx, a and b q dx).  The
// per-pixel arithmetic runs on packed f32x2 (fma/add/mul.rn.f32x2, sm_100a): the splat's scalars are
// broadcast operands, the two pixels the two halves, so one instruction serves both pixels and the
// values are those of the scalar code (each half is one IEEE round-to-nearest operation).  A warp
// visits a splat once per 8x8 block instead of once per 8x4 sub-block.
// Phase 1 leaves per (entry, lane) the lane's two-pixel partial sums s = w_a + w_b, t = w_b and
// u_ch = aT_a dL/dC_a,ch + aT_b dL/dC_b,ch (w = dL/dsigma sigma); phase 2 (lane e, half h) sums the
// 16 lanes of its half with the lane positions as compile-time constants and rebuilds the 9 moments
// (sum_b's y offset of 4 enters through t).
// ------------------------------------------------------------------------------------------------
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo2(u64 r) { return __uint_as_float((uint32_t)r); }
__device__ __forceinline__ float hi2(u64 r) { return __uint_as_float((uint32_t)(r >> 32)); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 bc2(float a) { return pk2(a, a); }

// pair_e for the two pixels (fx, fy.lo) and (fx, fy.hi): the same operations, in the same order and
// rounding, as pair_e (a = (Qxx' dx) dx, b = 2Qxy' dx, m = fma(dy, fma(Qyy', dy, b), a), e = lo - m).
__device__ __forceinline__ u64 pair_e2(float fx, u64 fy, const float4 g, const float2 p) {
  const float dx = __fsub_rn(fx, g.x);
  const float a = __fmul_rn(__fmul_rn(g.z, dx), dx);
  const float bq = __fmul_rn(g.w, dx);
  const u64 dy = sub2(fy, bc2(g.y));
  const u64 m = fma2(dy, fma2(bc2(p.x), dy, bc2(bq)), bc2(a));
  return sub2(bc2(p.y), m);
}

constexpr int kC2 = 4;                        // consumer warps (8x8 blocks) per tile
template <int kS2>
using Smem2T = SmemT<kS2, kC2, 3>;

template <int kChunk2>
struct BwdScratch2 {
  float4 st[kC2][kChunk2][33];   // (s, t, u0, u1) per (entry, lane); rows padded to 33 (conflict-free phase 2)
  float u2[kC2][kChunk2][33];    // u2 per (entry, lane)
  float2 emean[kC2][kChunk2];    // per chunk entry: the splat mean (tile-relative)
  float* eptr[kC2][kChunk2];     // per chunk entry: &moments[view][gid][0]
};

// kChunk2: list entries per phase-1 -> phase-2 chunk (16: 2 lanes per entry in phase 2, 8: 4 lanes);
// kProd2: producer warps.
template <int kChunk2, int kProd2, int kMinBlocks, int kS2>
__global__ void __launch_bounds__(32 * (kC2 + kProd2), kMinBlocks) k_render_bwd2(const steepgs_splat* __restrict__ splats,
                                                          const uint32_t* __restrict__ ids,
                                                          const uint2* __restrict__ ranges, int64_t n, int W, int H,
                                                          int tiles_x, int tiles_per_view, const RasterK rk,
                                                          const float* __restrict__ final_T,
                                                          const int32_t* __restrict__ n_contrib,
                                                          const float* __restrict__ dL_dimage,
                                                          const uint32_t* __restrict__ tile_last,
                                                          uint8_t* __restrict__ inst_mask,
                                                          float* __restrict__ moments,
                                                          const uint32_t* __restrict__ order) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char dsmem[];
  using Smem2 = Smem2T<kS2>;
  Smem2& sm = *reinterpret_cast<Smem2*>(dsmem);
  BwdScratch2<kChunk2>& sc = *reinterpret_cast<BwdScratch2<kChunk2>*>(dsmem + ((sizeof(Smem2) + 15) & ~size_t(15)));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int tile, view;
  tile_of_block(order, tile, view);
  SGS_CHECK(tile < tiles_per_view && view < (int)gridDim.y);   // tile_order entries are (view, tile)
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const uint2 rg = ranges[(int64_t)view * tiles_per_view + tile];
  const int64_t HW = (int64_t)W * H;
  const int bx = warp & 1, by = warp >> 1;
  const int lx = 8 * bx + (lane & 7), lya = 8 * by + (lane >> 3), lyb = lya + 4;
  const int px = tx * kTile + lx, pya = ty * kTile + lya, pyb = ty * kTile + lyb;
  const bool cons = warp < kC2;
  const bool ina = cons && px < W && pya < H, inb = cons && px < W && pyb < H;
  float Ta = 1.0f, Tb = 1.0f;
  float dla[3] = {0.f, 0.f, 0.f}, dlb[3] = {0.f, 0.f, 0.f};
  int lasta = 0, lastb = 0;
  {
    const float* dl = dL_dimage + (int64_t)view * 3 * HW;
    if (ina) {
      const int64_t pa = (int64_t)pya * W + px;
      Ta = final_T[(int64_t)view * HW + pa];
      lasta = n_contrib[(int64_t)view * HW + pa];
      dla[0] = dl[pa]; dla[1] = dl[HW + pa]; dla[2] = dl[2 * HW + pa];
    }
    if (inb) {
      const int64_t pb = (int64_t)pyb * W + px;
      Tb = final_T[(int64_t)view * HW + pb];
      lastb = n_contrib[(int64_t)view * HW + pb];
      dlb[0] = dl[pb]; dlb[1] = dl[HW + pb]; dlb[2] = dl[2 * HW + pb];
    }
  }
  const int L = (int)__ldg(tile_last + (int64_t)view * tiles_per_view + tile);
  const int nb = (L + kBatch - 1) / kBatch;
  if (tid == 0) {
    for (int st = 0; st < kS2; ++st) {
      mbar_init(&sm.full[st], 32 * kProd2);
      mbar_init(&sm.empty[st], 32 * kC2);
    }
  }
  __syncthreads();
  const int wmax = __reduce_max_sync(0xffffffffu, max(lasta, lastb));

  if (warp >= kC2) {  // ---------------- producers: batches from the back ----------------
    run_producer<false, kProd2, kS2, kC2, 3>(
        sm, ids, splats + (int64_t)view * n, nb,
        [nb, L, rg, ox, oy](int k) {
          const int rel = (nb - 1 - k) * kBatch;
          return BatchInfo{(int64_t)rg.x + rel, min(L - rel, kBatch), rel, ox, oy, false};
        },
        moments + (int64_t)view * n * 12, __log2f(rk.alpha_min), inst_mask, warp - kC2, lane, n);
    return;
  }

  // ---------------- consumers ----------------
  const float fx = (float)lx + 0.5f;
  const u64 fy = pk2((float)lya + 0.5f, (float)lyb + 0.5f);
  const float lmin = __log2f(rk.alpha_min);
  const float amax = rk.alpha_max;
  u64 T2 = pk2(Ta, Tb);
  u64 B0 = bc2(rk.bg[0]), B1 = bc2(rk.bg[1]), B2 = bc2(rk.bg[2]);
  const u64 dl0 = pk2(dla[0], dlb[0]), dl1 = pk2(dla[1], dlb[1]), dl2 = pk2(dla[2], dlb[2]);
  const uint32_t wbits = (1u << (4 * by + bx)) | (1u << (4 * by + 2 + bx));   // the block's two 8x4 strips
  float4(*sst)[33] = sc.st[warp];
  float(*su2)[33] = sc.u2[warp];
  float2* smean = sc.emean[warp];
  float** sptr = sc.eptr[warp];
  const int e2 = lane & (kChunk2 - 1), half = lane / kChunk2;
  const float cxw = (float)(8 * bx + 4), cyw = (float)(8 * by + 4);   // block centre (tile-relative)

  // ---- phase 2 over the chunk's first `ne` rows ----
  auto reduce_chunk = [&](int ne) {
    __syncwarp();
    SGS_CHECK(ne >= 1 && ne <= kChunk2);
    // packed accumulators over the source lanes' (w_a, w_b): P1 = sum, P2 = sum x, P3 = sum x^2, P4 / P5 =
    // sum / sum x over the lanes of the second row (y0' = 1); PU = (u0, u1)
    u64 P1 = 0ull, P2 = 0ull, P3 = 0ull, P4 = 0ull, P5 = 0ull, PU = 0ull;
    float U2 = 0.f;
    const float4* row = sst[e2] + kChunk2 * half;
    const float* row2 = su2[e2] + kChunk2 * half;
#pragma unroll
    for (int i = 0; i < kChunk2; ++i) {   // source lane kChunk2 half + i: x = (i & 7) - 3.5, y0' = i >> 3
      const float4 q = row[i];
      const float xq = (float)(i & 7) - 3.5f;
      const u64 wq = pk2(q.x, q.y);
      P1 = add2(P1, wq);
      P2 = fma2(wq, bc2(xq), P2);
      P3 = fma2(wq, bc2(xq * xq), P3);
      if (i >= 8) {
        P4 = add2(P4, wq);
        P5 = fma2(wq, bc2(xq), P5);
      }
      PU = add2(PU, pk2(q.z, q.w));
      U2 += row2[i];
    }
    const float A = lo2(P1) + hi2(P1), Tt = hi2(P1);           // sum s, sum t   (s = w_a + w_b, t = w_b)
    const float Bx = lo2(P2) + hi2(P2), Tx = hi2(P2);
    const float D = lo2(P3) + hi2(P3);
    const float Cy = lo2(P4) + hi2(P4), Ty = hi2(P4);
    const float E = lo2(P5) + hi2(P5);
    const float U0 = lo2(PU), U1 = hi2(PU);
    // group h's source lanes have y0 = y0' + c_h, c_h = (kChunk2 / 8) h - 3.5 (pixel a; pixel b is y0 + 4)
    const float ch = (float)(kChunk2 / 8) * (float)half - 3.5f;
    float v[12];
    v[0] = A;                                      // sum s
    v[1] = Bx;                                     // sum s x
    v[2] = fmaf(ch, A, Cy);                        // sum s y0
    v[3] = D;                                      // sum s x^2
    v[4] = fmaf(ch, Bx, E);                        // sum s x y0
    v[5] = fmaf(ch, fmaf(ch, A, 2.0f * Cy), Cy);   // sum s y0^2 (y0'^2 = y0')
    v[6] = Tt;                                     // sum t
    v[7] = Tx;                                     // sum t x
    v[8] = fmaf(ch, Tt, Ty);                       // sum t y0
    v[9] = U0; v[10] = U1; v[11] = U2;
#pragma unroll
    for (int o = kChunk2; o < 32; o <<= 1)
#pragma unroll
      for (int q = 0; q < 12; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    bool nz = false;
#pragma unroll
    for (int q = 0; q < 12; ++q) nz |= v[q] != 0.0f;
    if (e2 < ne && half == 0 && nz) {
      // raw moments in the block frame: pixel a at (x, y0), b at (x, y0 + 4); w_b = t
      const float S0 = v[0], Sx = v[1], Sy = fmaf(4.0f, v[6], v[2]);
      const float Sxx = v[3], Sxy = fmaf(4.0f, v[7], v[4]);
      const float Syy = fmaf(16.0f, v[6], fmaf(8.0f, v[8], v[5]));
      const float2 gm = smean[e2];
      const float u = cxw - gm.x, vv = cyw - gm.y;   // d = (x, y) + (u, v)
      const float m1x = fmaf(u, S0, Sx), m1y = fmaf(vv, S0, Sy);
      const float Mxx = fmaf(u, fmaf(u, S0, 2.0f * Sx), Sxx);
      const float Mxy = fmaf(u, m1y, fmaf(vv, Sx, Sxy));
      const float Myy = fmaf(vv, fmaf(vv, S0, 2.0f * Sy), Syy);
      float* mp = sptr[e2];
      red_v4(mp, S0, m1x, m1y, Mxx);
      red_v4(mp + 4, Mxy, Myy, v[9], v[10]);
      atomicAdd(mp + 8, v[11]);
    }
    __syncwarp();
  };

  int fill = 0;   // rows of the current chunk already filled
  for (int k = 0; k < nb; ++k) {
    const int s = k % kS2;
    mbar_wait(&sm.full[s], (k / kS2) & 1, kSuspendNs);
    const BufferT<kC2>& B = sm.buf[s];
    SGS_CHECK(B.base == (nb - 1 - k) * kBatch);      // the stage holds batch k (mbarrier ring protocol)
    uint8_t* lst = sm.buf[s].list[warp];
    const int nl = build_list(B, lst, wbits, lane, wmax - B.base);
    const int lima = lasta - B.base, limb = lastb - B.base;
    for (int t_hi = nl; t_hi > 0;) {
      const int m = min(t_hi, kChunk2 - fill);
      const int t_lo = t_hi - m;
      const int r0 = fill - t_lo;                           // row of list entry t = r0 + t
      if (lane < m) {
        const int j = lst[t_lo + lane];
        smean[fill + lane] = *reinterpret_cast<const float2*>(&B.geo[j]);
        sptr[fill + lane] = B.mptr[j];
      }
      auto recurse = [&](u64 ee, int j, int e) {
        SGS_CHECK(e >= 0 && e < kChunk2 && j < kBatch);
        const float ea = lo2(ee), eb = hi2(ee);
        const bool ha = j < lima && ea >= lmin, hb = j < limb && eb >= lmin;
        const float sa = ha ? ex2_approx(ea) : 0.0f, sb = hb ? ex2_approx(eb) : 0.0f;
        const u64 al = pk2(fminf(amax, sa), fminf(amax, sb));   // 0 for a pixel that does not composite
        const u64 om = sub2(bc2(1.0f), al);
        T2 = mul2(T2, pk2(rcp_approx(lo2(om)), rcp_approx(hi2(om))));   // T_i (rcp(1) = 1: unchanged)
        const float4 c = B.col[j];
        const u64 d0 = sub2(bc2(c.x), B0), d1 = sub2(bc2(c.y), B1), d2 = sub2(bc2(c.z), B2);
        const u64 gs = fma2(dl2, d2, fma2(dl1, d1, mul2(dl0, d0)));
        B0 = fma2(al, d0, B0);                              // B <- alpha c + (1 - alpha) B
        B1 = fma2(al, d1, B1);
        B2 = fma2(al, d2, B2);
        const u64 w = mul2(mul2(T2, gs), pk2(sa, sb));      // dL/dalpha sigma (Z3)
        const u64 aT = mul2(al, T2);
        const u64 p0 = mul2(aT, dl0), p1 = mul2(aT, dl1), p2 = mul2(aT, dl2);   // aT dL/dC per pixel
        sst[e][lane] = make_float4(lo2(w), hi2(w), lo2(p0) + hi2(p0), lo2(p1) + hi2(p1));
        su2[e][lane] = lo2(p2) + hi2(p2);
      };
      int t = t_hi - 1;
      for (; t - 3 >= t_lo; t -= 4) {
        int jj[4];
        u64 ee[4];
#pragma unroll
        for (int uu = 0; uu < 4; ++uu) {
          jj[uu] = lst[t - uu];
          ee[uu] = pair_e2(fx, fy, B.geo[jj[uu]], *reinterpret_cast<const float2*>(&B.par[jj[uu]]));
        }
#pragma unroll
        for (int uu = 0; uu < 4; ++uu) recurse(ee[uu], jj[uu], r0 + t - uu);
      }
      for (; t >= t_lo; --t) {
        const int ja = lst[t];
        recurse(pair_e2(fx, fy, B.geo[ja], *reinterpret_cast<const float2*>(&B.par[ja])), ja, r0 + t);
      }
      fill += m;
      t_hi = t_lo;
      if (fill == kChunk2) {
        reduce_chunk(kChunk2);
        fill = 0;
      }
    }
    __syncwarp();
    mbar_arrive(&sm.empty[s]);
  }
  if (fill > 0) reduce_chunk(fill);
}

__global__ void k_l1_grad(const float* __restrict__ image, const float* __restrict__ target, int64_t count,
                          float scale, float* __restrict__ dL, float* __restrict__ loss) {
  const int view = blockIdx.y;
  const float* a = image + (int64_t)view * count;
  const float* t = target + (int64_t)view * count;
  float* g = dL + (int64_t)view * count;
  float acc = 0.0f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const float r = a[i] - t[i];
    g[i] = r > 0.0f ? scale : (r < 0.0f ? -scale : 0.0f);
    acc += fabsf(r);
  }
  if (loss) {
    __shared__ float s[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
      float x = threadIdx.x < (blockDim.x >> 5) ? s[threadIdx.x] : 0.0f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (threadIdx.x == 0) atomicAdd(loss + view, x * scale);
    }
  }
}

}  // namespace

// Opt a kernel into more than 48 KB of dynamic shared memory on the current device (the attribute is
// per device); `done` records the devices already set (bit per device id < 64).  With mark = false
// the bit is left for a following call on another function of the same group.
static cudaError_t allow_dynamic_smem(std::atomic<uint64_t>& done, const void* fn, size_t bytes, bool mark = false) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && mark && bit) done.fetch_or(bit, std::memory_order_release);
  return e;
}

cudaError_t launch_render_fwd(const steepgs_splat* splats, int64_t n, const steepgs_binning& b, int W, int H,
                              const RasterK& rk, float* image, float* final_T, int32_t* n_contrib,
                              int64_t* pair_counts, cudaStream_t st, const L1Fused& l1) {
  const int tpv = b.tiles_x * b.tiles_y;
  dim3 grid(tpv, b.V);
  if (l1.loss) {
    const cudaError_t e = cudaMemsetAsync(l1.loss, 0, sizeof(float) * (size_t)b.V, st);
    if (e != cudaSuccess) return e;
  }
  {
    static std::atomic<uint64_t> done{0};   // devices whose function attribute is set
    cudaError_t e = allow_dynamic_smem(done, (const void*)k_render_fwd<true>, sizeof(SmemFwd));
    if (e == cudaSuccess) e = allow_dynamic_smem(done, (const void*)k_render_fwd<false>, sizeof(SmemFwd), true);
    if (e != cudaSuccess) return e;
  }
  launch_pdl(pair_counts ? k_render_fwd<true> : k_render_fwd<false>, grid, dim3(kThreadsFwd), sizeof(SmemFwd), st, splats,
             b.ids, reinterpret_cast<const uint2*>(b.ranges), n, W, H, b.tiles_x, tpv, rk, image, final_T, n_contrib,
             b.tile_last, b.inst_mask, reinterpret_cast<unsigned long long*>(pair_counts), l1, b.tile_order);
  note_launch();
  return check_launch("k_render_fwd");
}

cudaError_t launch_l1_grad(const float* image, const float* target, int V, int64_t count, float scale, float* dL,
                           float* loss, cudaStream_t st) {
  if (loss) {
    const cudaError_t e = cudaMemsetAsync(loss, 0, sizeof(float) * (size_t)V, st);
    if (e != cudaSuccess) return e;
  }
  if (count == 0) return cudaSuccess;
  int64_t blocks = (count + 1023) / 1024;
  if (blocks > 1184) blocks = 1184;
  dim3 grid((unsigned)blocks, V);
  k_l1_grad<<<grid, 256, 0, st>>>(image, target, count, scale, dL, loss);
  note_launch();
  return check_launch("k_l1_grad");
}

cudaError_t launch_render_bwd(const steepgs_splat* splats, const steepgs_binning& b, int W, int H,
                              const RasterK& rk, const float* final_T, const int32_t* n_contrib,
                              const float* dL_dimage, int64_t n, float* moments, cudaStream_t st) {
  const int tpv = b.tiles_x * b.tiles_y;
  dim3 grid(tpv, b.V);
  // 8-entry chunks (4 phase-2 lanes per entry), one producer warp, 3-stage ring, 4 blocks per SM: the
  // fastest of the measured configurations (round 2)
  constexpr int kCh = 8, kS2 = kStages;
  using Kern = void (*)(const steepgs_splat*, const uint32_t*, const uint2*, int64_t, int, int, int, int, const RasterK,
                        const float*, const int32_t*, const float*, const uint32_t*, uint8_t*, float*,
                        const uint32_t*);
  const Kern kern = k_render_bwd2<kCh, 1, 4, kS2>;
  const size_t smem2 = ((sizeof(Smem2T<kS2>) + 15) & ~size_t(15)) + sizeof(BwdScratch2<kCh>);
  static std::atomic<uint64_t> done2{0};
  const cudaError_t e2 = allow_dynamic_smem(done2, (const void*)kern, smem2, true);
  if (e2 == cudaSuccess)
    launch_pdl(kern, grid, dim3(32 * (kC2 + 1)), smem2, st, splats, b.ids, reinterpret_cast<const uint2*>(b.ranges), n, W,
               H, b.tiles_x, tpv, rk, final_T, n_contrib, dL_dimage, (const uint32_t*)b.tile_last, b.inst_mask, moments,
               b.tile_order);
  if (e2 != cudaSuccess) return e2;
  note_launch();
  return check_launch("k_render_bwd2");
}

}  // namespace sgs
