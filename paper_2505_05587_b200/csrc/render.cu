// render.cu — a3 forward compositing (Eq. eqn:alpha_blend), a4 l1 gradient helper
// (Eq. eqn:loss), a5 backward replay with the splitting-matrix moments (Thm 1 P:L232,
// §4.3).
//
// Work decomposition (B200): one 64-thread block (2 warps) per 16x16 tile and view; each thread owns
// a vertical run of 4 pixels, so warp w covers the 16x8 half-tile of rows 8w..8w+7.  The tile's
// depth-ordered splats are staged through shared memory in batches of 256 (4 gathered 48-B records
// per thread).  While staging, each splat gets a 2-bit mask of the half-tiles its alpha support
// {m <= tau} can reach (its exact y-extent sqrt(tau Sigma2D_yy), padded); a warp skips splats whose
// bit is clear with one warp-uniform test instead of 4 x 32 pixel evaluations.  Every splat that is
// staged is evaluated against 4 pixels per lane, so the per-(warp, splat) fixed cost (shared loads,
// loop control, and in the backward the warp reduction + atomic) is amortised over 128 pixels.
//
// The mean is made tile-relative in fp64 before rounding, so per-pair offsets d = x - Pi(p) carry
// ~1e-7 px error.  The per-pair arithmetic (m, sigma, alpha, skip/termination tests) is written with
// explicit round-to-nearest intrinsics and shared by both kernels, so forward and backward take
// bit-identical decisions.
//
// Backward: back to front over each pixel's composited prefix (n_contrib from the forward), T_i
// recovered as T_{i+1} / (1 - alpha_i) (fast reciprocal; relative error ~1 ulp per step),
// dL/dalpha_i = T_i sum_ch dL/dC_ch (c_ch - B_ch) with B the normalised colour behind (C10),
// w = dL/dsigma * sigma.  The 9 per-pair values (w, w d, w d d^T, alpha T dL/dC) are summed over a
// lane's 4 pixels in registers, reduced across the warp with a transposed butterfly (12 shuffles
// instead of 45) and added with one 9-lane RED per (warp, splat) into moments[view][gid][12].  The
// splitting matrix needs no per-pair work of its own: S_view = P^T (Q M Q - m0 Q) P is formed per
// Gaussian from these moments (gauss_bwd.cu).
#include "common.cuh"

namespace sgs {

namespace {

constexpr int kThreads = 64;           // 2 warps per 16x16 tile
constexpr int kPix = 4;                // pixels per thread (vertical run)
constexpr int kBatch = 256;            // splats staged per batch
constexpr int kLoads = kBatch / kThreads;

// Mahalanobis m = Qxx dx^2 + 2 Qxy dx dy + Qyy dy^2, sigma = o exp(-m/2), alpha = min(amax, sigma).
__device__ __forceinline__ float pair_m(float dx, float dy, float cxx, float cxy2, float cyy) {
  float t = __fmul_rn(cxx, dx);
  t = __fmaf_rn(cxy2, dy, t);
  float m = __fmul_rn(t, dx);
  return __fmaf_rn(__fmul_rn(cyy, dy), dy, m);
}

__device__ __forceinline__ float pair_sigma(float m, float o) { return __fmul_rn(o, __expf(__fmul_rn(-0.5f, m))); }

struct Staged {
  float4* geo;      // (mu_x - ox, mu_y - oy, Qxx, 2 Qxy)
  float4* par;      // (Qyy, o, tau, -)
  float4* col;      // (r, g, b, -)
  uint32_t* gid;
  uint32_t* mask;   // bit w: alpha support reaches half-tile w
};

// Stage splat `gid` into slot k: tile-relative mean (fp64 -> fp32) and the half-tile mask.
__device__ __forceinline__ void stage(const steepgs_splat* __restrict__ vs, uint32_t gid, double ox, double oy,
                                      Staged S, int k) {
  const steepgs_splat* sp = vs + gid;
  const double2 mean = *reinterpret_cast<const double2*>(sp);
  const float4 a = *(reinterpret_cast<const float4*>(sp) + 1);
  const float4 b = *(reinterpret_cast<const float4*>(sp) + 2);
  const float gx = (float)(mean.x - ox), gy = (float)(mean.y - oy);
  S.geo[k] = make_float4(gx, gy, a.x, 2.0f * a.y);
  S.par[k] = make_float4(a.z, a.w, b.w, 0.0f);
  S.col[k] = make_float4(b.x, b.y, b.z, 0.0f);
  S.gid[k] = gid;
  // y-extent of {m <= tau}: sqrt(tau * Sigma2D_yy), Sigma2D_yy = Qxx / det(Q); padded so that every
  // pair the fp32 test m <= tau accepts is kept (a degenerate det keeps both halves).
  const float detq = a.x * a.z - a.y * a.y;
  uint32_t m = 3u;
  if (detq > 0.0f) {
    const float ey = sqrtf(b.w * (a.x / detq)) * 1.001f + 0.01f;
    if (ey == ey) {
      m = 0u;
      if (gy - ey <= 7.5f && gy + ey >= 0.5f) m |= 1u;
      if (gy - ey <= 15.5f && gy + ey >= 8.5f) m |= 2u;
    }
  }
  S.mask[k] = m;
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
  const Staged S{s_geo, s_par, s_col, s_gid, s_mask};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = blockIdx.x, view = blockIdx.y;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int lx = lane & 15, ly0 = warp * 8 + (lane >> 4) * 4;
  const int px = tx * kTile + lx, py0 = ty * kTile + ly0;
  const float fx = (float)lx + 0.5f;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const uint2 rg = ranges[(int64_t)view * tiles_per_view + tile];
  const steepgs_splat* vs = splats + (int64_t)view * n;
  float T[kPix], C0[kPix], C1[kPix], C2[kPix];
  int last[kPix];
  bool done[kPix];
#pragma unroll
  for (int k = 0; k < kPix; ++k) {
    T[k] = 1.0f; C0[k] = C1[k] = C2[k] = 0.0f; last[k] = 0;
    done[k] = !(px < W && py0 + k < H);
  }
  int ncomp = 0, neval = 0;
  const uint32_t wbit = 1u << warp;
  for (uint32_t b = rg.x; b < rg.y; b += kBatch) {
    const bool tdone = done[0] && done[1] && done[2] && done[3];
    if (__syncthreads_count(tdone) == kThreads) break;
#pragma unroll
    for (int l = 0; l < kLoads; ++l) {
      const int k = l * kThreads + tid;
      if (b + k < rg.y) stage(vs, ids[b + k], ox, oy, S, k);
    }
    __syncthreads();
    const int cnt = min((int)(rg.y - b), kBatch);
    if (tdone) continue;
    for (int j = 0; j < cnt; ++j) {
      if (!(s_mask[j] & wbit)) continue;                // half-tile culling (warp-uniform)
      const float4 g = s_geo[j];
      const float4 p = s_par[j];
      const float dx = __fsub_rn(fx, g.x);
#pragma unroll
      for (int k = 0; k < kPix; ++k) {
        if (done[k]) continue;
        ++neval;
        const float dy = __fsub_rn((float)(ly0 + k) + 0.5f, g.y);
        const float m = pair_m(dx, dy, g.z, g.w, p.x);
        if (m > p.z) continue;                          // outside the alpha support (tau)
        const float sigma = pair_sigma(m, p.y);
        const float alpha = fminf(rk.alpha_max, sigma);
        if (alpha < rk.alpha_min) continue;             // C8 skip
        const float Tn = __fmul_rn(T[k], __fsub_rn(1.0f, alpha));
        if (Tn < rk.t_min) { done[k] = true; continue; }  // C8 termination
        const float4 c = s_col[j];
        const float aT = __fmul_rn(alpha, T[k]);
        C0[k] = __fmaf_rn(aT, c.x, C0[k]);
        C1[k] = __fmaf_rn(aT, c.y, C1[k]);
        C2[k] = __fmaf_rn(aT, c.z, C2[k]);
        T[k] = Tn;
        last[k] = (int)(b - rg.x) + j + 1;
        ++ncomp;
      }
    }
  }
  const int64_t HW = (int64_t)W * H;
  float* img = image + (int64_t)view * 3 * HW;
#pragma unroll
  for (int k = 0; k < kPix; ++k) {
    if (!(px < W && py0 + k < H)) continue;
    const int64_t pix = (int64_t)(py0 + k) * W + px;
    img[pix] = __fmaf_rn(T[k], rk.bg[0], C0[k]);
    img[HW + pix] = __fmaf_rn(T[k], rk.bg[1], C1[k]);
    img[2 * HW + pix] = __fmaf_rn(T[k], rk.bg[2], C2[k]);
    final_T[(int64_t)view * HW + pix] = T[k];
    n_contrib[(int64_t)view * HW + pix] = last[k];
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
  __shared__ int s_maxlast;
  const Staged S{s_geo, s_par, s_col, s_gid, s_mask};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = blockIdx.x, view = blockIdx.y;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int lx = lane & 15, ly0 = warp * 8 + (lane >> 4) * 4;
  const int px = tx * kTile + lx, py0 = ty * kTile + ly0;
  const float fx = (float)lx + 0.5f;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const uint2 rg = ranges[(int64_t)view * tiles_per_view + tile];
  const steepgs_splat* vs = splats + (int64_t)view * n;
  const int64_t HW = (int64_t)W * H;
  float T[kPix], dl0[kPix], dl1[kPix], dl2[kPix], B0[kPix], B1[kPix], B2[kPix];
  int last[kPix];
  int mylast = 0;
#pragma unroll
  for (int k = 0; k < kPix; ++k) {
    T[k] = 1.0f; dl0[k] = dl1[k] = dl2[k] = 0.0f; last[k] = 0;
    B0[k] = rk.bg[0]; B1[k] = rk.bg[1]; B2[k] = rk.bg[2];
    if (px < W && py0 + k < H) {
      const int64_t pix = (int64_t)(py0 + k) * W + px;
      T[k] = final_T[(int64_t)view * HW + pix];
      last[k] = n_contrib[(int64_t)view * HW + pix];
      const float* dl = dL_dimage + (int64_t)view * 3 * HW;
      dl0[k] = dl[pix]; dl1[k] = dl[HW + pix]; dl2[k] = dl[2 * HW + pix];
      mylast = max(mylast, last[k]);
    }
  }
  if (tid == 0) s_maxlast = 0;
  __syncthreads();
  const int wmax = __reduce_max_sync(0xffffffffu, mylast);
  if (lane == 0) atomicMax(&s_maxlast, wmax);
  __syncthreads();
  const int L = s_maxlast;
  const int my_slot = slot_of(lane);
  const uint32_t wbit = 1u << warp;
  float* mom_view = moments + (int64_t)view * n * 12;
  const int nb = (L + kBatch - 1) / kBatch;
  for (int bb = nb - 1; bb >= 0; --bb) {
    const uint32_t b = rg.x + (uint32_t)bb * kBatch;
    const int cnt = min(L - bb * kBatch, kBatch);
    __syncthreads();
#pragma unroll
    for (int l = 0; l < kLoads; ++l) {
      const int k = l * kThreads + tid;
      if (k < cnt) stage(vs, ids[b + k], ox, oy, S, k);
    }
    __syncthreads();
    for (int j = cnt - 1; j >= 0; --j) {
      if (!(s_mask[j] & wbit)) continue;                // half-tile culling (warp-uniform)
      const int li = bb * kBatch + j;                   // list position relative to the tile start
      const float4 g = s_geo[j];
      const float4 p = s_par[j];
      const float dx = __fsub_rn(fx, g.x);
      float v[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) v[q] = 0.0f;
      bool contrib = false;
#pragma unroll
      for (int k = 0; k < kPix; ++k) {
        if (li >= last[k]) continue;
        const float dy = __fsub_rn((float)(ly0 + k) + 0.5f, g.y);
        const float m = pair_m(dx, dy, g.z, g.w, p.x);
        if (m > p.z) continue;
        const float sigma = pair_sigma(m, p.y);
        const float alpha = fminf(rk.alpha_max, sigma);
        if (alpha < rk.alpha_min) continue;
        contrib = true;
        const float4 c = s_col[j];
        const float om = 1.0f - alpha;
        T[k] = __fdividef(T[k], om);                        // T_i (before this splat)
        const float gsum = dl0[k] * (c.x - B0[k]) + dl1[k] * (c.y - B1[k]) + dl2[k] * (c.z - B2[k]);
        const float w = T[k] * gsum * sigma;                 // dL/dalpha * sigma (straight-through, Z3)
        B0[k] = alpha * c.x + om * B0[k];
        B1[k] = alpha * c.y + om * B1[k];
        B2[k] = alpha * c.z + om * B2[k];
        const float aT = alpha * T[k];
        const float wdx = w * dx, wdy = w * dy;
        v[0] += w;
        v[1] += wdx;
        v[2] += wdy;
        v[3] += wdx * dx;
        v[4] += wdx * dy;
        v[5] += wdy * dy;
        v[6] += aT * dl0[k];
        v[7] += aT * dl1[k];
        v[8] += aT * dl2[k];
      }
      if (!__any_sync(0xffffffffu, contrib)) continue;
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
