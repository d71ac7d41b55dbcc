// render.cu — a3 forward compositing (Eq. eqn:alpha_blend), a4 l1 gradient helper
// (Eq. eqn:loss), a5 backward replay with the splitting-matrix moments (Thm 1 P:L232,
// §4.3).
//
// Work decomposition (B200): one 256-thread block per 16x16 tile and view, one pixel per thread;
// warp w owns the 8x4 sub-block (x: 8 (w & 1) .. +7, y: 4 (w >> 1) .. +3).  The tile's
// depth-ordered splats are staged through shared memory in batches of 256 (one gathered 48-B record
// per thread).  While staging, each splat gets an 8-bit mask of the sub-blocks its alpha support
// {m <= tau} (padded y/x extents sqrt(tau Sigma2D)) can reach; each warp then compacts the batch to
// the splats of its own sub-block with 8 ballots, so it iterates only over splats that can touch its
// 32 pixels (SIMT lanes never evaluate pairs outside the sub-block's candidate set).
//
// Per-pair arithmetic: the mean is made tile-relative in fp64 before rounding (offsets d = x - Pi(p)
// carry ~1e-7 px error); the conic is pre-scaled by log2(e)/2 at staging so that
//   e = log2(o) - m',  m' = a + dy (b + Qyy' dy),  a = Qxx' dx^2,  b = 2 Qxy' dx,
//   skip if e < log2(alpha_min) (<=> sigma < alpha_min),  sigma = exp2(e),  alpha = min(amax, sigma)
// with explicit round-to-nearest intrinsics in one shared function, so forward and backward take
// bit-identical decisions.
//
// Backward: back to front over each pixel's composited prefix (n_contrib from the forward), T_i
// recovered as T_{i+1} / (1 - alpha_i) (fast reciprocal; relative error ~1 ulp per step),
// dL/dalpha_i = T_i sum_ch dL/dC_ch (c_ch - B_ch) with B the normalised colour behind (C10),
// w = dL/dsigma * sigma.  The 9 per-pair values (w, w d, w d d^T, alpha T dL/dC) are reduced across
// the warp with a transposed butterfly (12 shuffles instead of 45) and added with one 9-lane RED per
// (warp, splat) into moments[view][gid][12].  The splitting matrix needs no per-pair work of its own:
// S_view = P^T (Q M Q - m0 Q) P is formed per Gaussian from these moments (gauss_bwd.cu).
#include "common.cuh"

namespace sgs {

namespace {

constexpr int kThreads = 256;          // one pixel per thread, 8 warps per 16x16 tile
constexpr int kBatch = 256;            // splats staged per batch (one per thread)
constexpr float kHalfLog2e = 0.72134752044448170f;  // log2(e) / 2

struct Staged {
  float4* geo;      // (mu_x - ox, mu_y - oy, Qxx', 2 Qxy')   Q' = Q log2(e)/2
  float4* par;      // (Qyy', log2(o), -, -)
  float4* col;      // (r, g, b, -)
  uint32_t* gid;
  uint32_t* mask;   // bit k: alpha support reaches sub-block k (8x4 px)
};

// Stage splat `gid` into slot k: tile-relative mean (fp64 -> fp32), pre-scaled conic, log2(o), and
// the sub-block mask from the padded extents of {m <= tau} (a degenerate det keeps every block).
__device__ __forceinline__ void stage(const steepgs_splat* __restrict__ vs, uint32_t gid, double ox, double oy,
                                      Staged S, int k) {
  const steepgs_splat* sp = vs + gid;
  const double2 mean = *reinterpret_cast<const double2*>(sp);
  const float4 a = *(reinterpret_cast<const float4*>(sp) + 1);
  const float4 b = *(reinterpret_cast<const float4*>(sp) + 2);
  const float gx = (float)(mean.x - ox), gy = (float)(mean.y - oy);
  S.geo[k] = make_float4(gx, gy, __fmul_rn(a.x, kHalfLog2e), __fmul_rn(2.0f * a.y, kHalfLog2e));
  S.par[k] = make_float4(__fmul_rn(a.z, kHalfLog2e), __log2f(a.w), 0.0f, 0.0f);
  S.col[k] = make_float4(b.x, b.y, b.z, 0.0f);
  S.gid[k] = gid;
  const float detq = a.x * a.z - a.y * a.y;
  uint32_t m = 0xFFu;
  if (detq > 0.0f) {
    const float ex = sqrtf(b.w * (a.z / detq)) * 1.001f + 0.01f;
    const float ey = sqrtf(b.w * (a.x / detq)) * 1.001f + 0.01f;
    if (ex == ex && ey == ey) {
      uint32_t xb = 0u, yb = 0u;
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (gx - ex <= 8.0f * q + 7.5f && gx + ex >= 8.0f * q + 0.5f) xb |= 1u << q;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (gy - ey <= 4.0f * q + 3.5f && gy + ey >= 4.0f * q + 0.5f) yb |= 1u << q;
      m = 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (yb & (1u << q)) m |= xb << (2 * q);
    }
  }
  S.mask[k] = m;
}

// Per-warp compaction of the staged batch to the splats whose mask has bit `w`; returns the count.
__device__ __forceinline__ int warp_list(const uint32_t* __restrict__ s_mask, int cnt, int w, int lane,
                                         uint8_t* __restrict__ list) {
  int total = 0;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int c = 0; c < kBatch / 32; ++c) {
    const int j = c * 32 + lane;
    const bool hit = j < cnt && ((s_mask[j] >> w) & 1u);
    const uint32_t bal = __ballot_sync(0xffffffffu, hit);
    if (hit) list[total + __popc(bal & lt)] = (uint8_t)j;
    total += __popc(bal);
  }
  __syncwarp();
  return total;
}

// The pair test shared by forward and backward: returns e = log2(sigma) (skip if e < lmin).
__device__ __forceinline__ float pair_e(float dx, float dy, const float4 g, const float4 p) {
  const float a = __fmul_rn(__fmul_rn(g.z, dx), dx);
  const float bq = __fmul_rn(g.w, dx);
  const float m = __fmaf_rn(dy, __fmaf_rn(p.x, dy, bq), a);
  return __fsub_rn(p.y, m);
}

__global__ void __launch_bounds__(kThreads) k_render_fwd(const steepgs_splat* __restrict__ splats,
                                                         const uint32_t* __restrict__ ids,
                                                         const uint2* __restrict__ ranges, int64_t n, int W, int H,
                                                         int tiles_x, int tiles_per_view, const RasterK rk,
                                                         float* __restrict__ image, float* __restrict__ final_T,
                                                         int32_t* __restrict__ n_contrib,
                                                         unsigned long long* __restrict__ pair_counts) {
  __shared__ float4 s_geo[kBatch], s_par[kBatch], s_col[kBatch];
  __shared__ uint32_t s_gid[kBatch], s_mask[kBatch];
  __shared__ uint8_t s_list[kThreads / 32][kBatch];
  const Staged S{s_geo, s_par, s_col, s_gid, s_mask};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = blockIdx.x, view = blockIdx.y;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int lx = 8 * (warp & 1) + (lane & 7), ly = 4 * (warp >> 1) + (lane >> 3);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = px < W && py < H;
  const float fx = (float)lx + 0.5f, fy = (float)ly + 0.5f;  // pixel centre, tile-relative (Z5)
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const uint2 rg = ranges[(int64_t)view * tiles_per_view + tile];
  const steepgs_splat* vs = splats + (int64_t)view * n;
  const float lmin = __log2f(rk.alpha_min);  // -inf in smooth mode
  float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
  int last = 0, ncomp = 0, neval = 0;
  bool done = !inside;
  uint8_t* mylist = s_list[warp];
  for (uint32_t b = rg.x; b < rg.y; b += kBatch) {
    if (__syncthreads_count(done) == kThreads) break;
    if (b + tid < rg.y) stage(vs, ids[b + tid], ox, oy, S, tid);
    __syncthreads();
    const int cnt = min((int)(rg.y - b), kBatch);
    const int nl = warp_list(s_mask, cnt, warp, lane, mylist);
    for (int t = 0; t < nl; ++t) {
      if (__all_sync(0xffffffffu, done)) break;
      const int j = mylist[t];
      const float4 g = s_geo[j];
      const float4 p = s_par[j];
      if (done) continue;
      ++neval;
      const float e = pair_e(__fsub_rn(fx, g.x), __fsub_rn(fy, g.y), g, p);
      if (e < lmin) continue;                          // sigma < alpha_min: C8 skip
      const float alpha = fminf(rk.alpha_max, exp2f(e));
      const float Tn = __fmul_rn(T, __fsub_rn(1.0f, alpha));
      if (Tn < rk.t_min) { done = true; continue; }    // C8 termination
      const float4 c = s_col[j];
      const float aT = __fmul_rn(alpha, T);
      C0 = __fmaf_rn(aT, c.x, C0);
      C1 = __fmaf_rn(aT, c.y, C1);
      C2 = __fmaf_rn(aT, c.z, C2);
      T = Tn;
      last = (int)(b - rg.x) + j + 1;
      ++ncomp;
    }
  }
  if (inside) {
    const int64_t HW = (int64_t)W * H;
    const int64_t pix = (int64_t)py * W + px;
    float* img = image + (int64_t)view * 3 * HW;
    img[pix] = __fmaf_rn(T, rk.bg[0], C0);
    img[HW + pix] = __fmaf_rn(T, rk.bg[1], C1);
    img[2 * HW + pix] = __fmaf_rn(T, rk.bg[2], C2);
    final_T[(int64_t)view * HW + pix] = T;
    n_contrib[(int64_t)view * HW + pix] = last;
  }
  if (pair_counts) {
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

// Transposed warp reduction of 9 values (see header comment).  After the call, lane l holds in
// v[0] the warp sum of value index slot_of(l) (lanes l and l^1 hold the same value).
template <int NIN, int OFF>
__device__ __forceinline__ void tstage(float* v, bool upper) {
  constexpr int NK = (NIN + 1) / 2;
#pragma unroll
  for (int s = 0; s < NK; ++s) {
    const float hi = (NK + s < NIN) ? v[NK + s] : 0.0f;
    const float keep = upper ? hi : v[s];
    const float send = upper ? v[s] : hi;
    v[s] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
  }
}

__device__ __forceinline__ void reduce9(float* v, int lane) {
  tstage<9, 16>(v, lane & 16);
  tstage<5, 8>(v, lane & 8);
  tstage<3, 4>(v, lane & 4);
  tstage<2, 2>(v, lane & 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
}

__device__ __forceinline__ int slot_of(int lane) {
  int lo = 0, len = 9;
  const int nins[4] = {9, 5, 3, 2};
  const int bits[4] = {16, 8, 4, 2};
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int nk = (nins[s] + 1) / 2;
    if (lane & bits[s]) { lo += nk; len -= nk; }
    else if (len > nk) len = nk;
  }
  return (len >= 1 && (lane & 1) == 0) ? lo : -1;
}

__global__ void __launch_bounds__(kThreads) k_render_bwd(const steepgs_splat* __restrict__ splats,
                                                         const uint32_t* __restrict__ ids,
                                                         const uint2* __restrict__ ranges, int64_t n, int W, int H,
                                                         int tiles_x, int tiles_per_view, const RasterK rk,
                                                         const float* __restrict__ final_T,
                                                         const int32_t* __restrict__ n_contrib,
                                                         const float* __restrict__ dL_dimage,
                                                         float* __restrict__ moments) {
  __shared__ float4 s_geo[kBatch], s_par[kBatch], s_col[kBatch];
  __shared__ uint32_t s_gid[kBatch], s_mask[kBatch];
  __shared__ uint8_t s_list[kThreads / 32][kBatch];
  __shared__ int s_maxlast;
  const Staged S{s_geo, s_par, s_col, s_gid, s_mask};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = blockIdx.x, view = blockIdx.y;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int lx = 8 * (warp & 1) + (lane & 7), ly = 4 * (warp >> 1) + (lane >> 3);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = px < W && py < H;
  const float fx = (float)lx + 0.5f, fy = (float)ly + 0.5f;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const uint2 rg = ranges[(int64_t)view * tiles_per_view + tile];
  const steepgs_splat* vs = splats + (int64_t)view * n;
  const int64_t HW = (int64_t)W * H;
  const int64_t pix = (int64_t)py * W + px;
  const float lmin = __log2f(rk.alpha_min);
  float T = 1.0f, dl0 = 0.0f, dl1 = 0.0f, dl2 = 0.0f;
  int last = 0;
  if (inside) {
    T = final_T[(int64_t)view * HW + pix];
    last = n_contrib[(int64_t)view * HW + pix];
    const float* dl = dL_dimage + (int64_t)view * 3 * HW;
    dl0 = dl[pix]; dl1 = dl[HW + pix]; dl2 = dl[2 * HW + pix];
  }
  if (tid == 0) s_maxlast = 0;
  __syncthreads();
  const int wmax = __reduce_max_sync(0xffffffffu, last);
  if (lane == 0) atomicMax(&s_maxlast, wmax);
  __syncthreads();
  const int L = s_maxlast;
  float B0 = rk.bg[0], B1 = rk.bg[1], B2 = rk.bg[2];
  const int my_slot = slot_of(lane);
  float* mom_view = moments + (int64_t)view * n * 12;
  uint8_t* mylist = s_list[warp];
  const int nb = (L + kBatch - 1) / kBatch;
  for (int bb = nb - 1; bb >= 0; --bb) {
    const uint32_t b = rg.x + (uint32_t)bb * kBatch;
    const int cnt = min(L - bb * kBatch, kBatch);
    __syncthreads();
    if (tid < cnt) stage(vs, ids[b + tid], ox, oy, S, tid);
    __syncthreads();
    const int nl = warp_list(s_mask, cnt, warp, lane, mylist);
    for (int t = nl - 1; t >= 0; --t) {
      const int j = mylist[t];
      const int li = bb * kBatch + j;                  // list position relative to the tile start
      const float4 g = s_geo[j];
      const float4 p = s_par[j];
      float v[9];
      bool contrib = false;
      const float dx = __fsub_rn(fx, g.x), dy = __fsub_rn(fy, g.y);
      if (li < last) {
        const float e = pair_e(dx, dy, g, p);
        if (e >= lmin) {
          contrib = true;
          const float sigma = exp2f(e);
          const float alpha = fminf(rk.alpha_max, sigma);
          const float4 c = s_col[j];
          const float om = 1.0f - alpha;
          T = __fdividef(T, om);                          // T_i (before this splat)
          const float gsum = dl0 * (c.x - B0) + dl1 * (c.y - B1) + dl2 * (c.z - B2);
          const float w = T * gsum * sigma;               // dL/dalpha * sigma (straight-through, Z3)
          B0 = alpha * c.x + om * B0;
          B1 = alpha * c.y + om * B1;
          B2 = alpha * c.z + om * B2;
          const float aT = alpha * T;
          const float wdx = w * dx, wdy = w * dy;
          v[0] = w; v[1] = wdx; v[2] = wdy;
          v[3] = wdx * dx; v[4] = wdx * dy; v[5] = wdy * dy;
          v[6] = aT * dl0; v[7] = aT * dl1; v[8] = aT * dl2;
        }
      }
      if (!__any_sync(0xffffffffu, contrib)) continue;
      if (!contrib) {
#pragma unroll
        for (int q = 0; q < 9; ++q) v[q] = 0.0f;
      }
      reduce9(v, lane);
      if (my_slot >= 0) atomicAdd(mom_view + (int64_t)s_gid[j] * 12 + my_slot, v[0]);
    }
  }
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

cudaError_t launch_render_fwd(const steepgs_splat* splats, int64_t n, const steepgs_binning& b, int W, int H,
                              const RasterK& rk, float* image, float* final_T, int32_t* n_contrib,
                              int64_t* pair_counts, cudaStream_t st) {
  const int tpv = b.tiles_x * b.tiles_y;
  dim3 grid(tpv, b.V);
  k_render_fwd<<<grid, kThreads, 0, st>>>(splats, b.ids, reinterpret_cast<const uint2*>(b.ranges), n, W, H,
                                          b.tiles_x, tpv, rk, image, final_T, n_contrib,
                                          reinterpret_cast<unsigned long long*>(pair_counts));
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
  k_render_bwd<<<grid, kThreads, 0, st>>>(splats, b.ids, reinterpret_cast<const uint2*>(b.ranges), n, W, H,
                                          b.tiles_x, tpv, rk, final_T, n_contrib, dL_dimage, moments);
  note_launch();
  return check_launch("k_render_bwd");
}

}  // namespace sgs
