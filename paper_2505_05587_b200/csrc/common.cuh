// common.cuh — internal declarations shared by the sm_100a kernels of libsteepgs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "steepgs.h"

namespace sgs {

// ---- debug-checked build (-DSTEEPGS_CHECKS, libsteepgs_checked.so; tests/test_checked_build.py) ----
// Device-side invariants that compute-sanitizer would otherwise be needed for (ring stage identity
// under the mbarrier protocol, list / row / instance / scatter bounds).  A failed check counts into a
// per-translation-unit device word and records its line; steepgs_debug_checks() reads them.  In the
// release build SGS_CHECK compiles to nothing.
#ifdef STEEPGS_CHECKS
#define SGS_CHECKS_TU(tag)                                                                 \
  static __device__ unsigned int g_sgs_fail[2];                                            \
  cudaError_t checks_io_##tag(unsigned int* out, bool reset) {                            \
    cudaError_t e = cudaMemcpyFromSymbol(out, g_sgs_fail, sizeof(g_sgs_fail));             \
    if (e == cudaSuccess && reset) {                                                       \
      const unsigned int z[2] = {0u, 0u};                                                  \
      e = cudaMemcpyToSymbol(g_sgs_fail, z, sizeof(z));                                    \
    }                                                                                      \
    return e;                                                                              \
  }
#define SGS_CHECK(cond)                                                                    \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      if (atomicAdd(&g_sgs_fail[0], 1u) == 0u) g_sgs_fail[1] = (unsigned int)__LINE__;    \
    }                                                                                      \
  } while (0)
#else
#define SGS_CHECKS_TU(tag)
#define SGS_CHECK(cond) \
  do {                  \
  } while (0)
#endif

constexpr int kTile = 16;          // tile edge in pixels (16x16 = 256 threads per tile block)
constexpr int kMaxViews = 64;      // cameras passed by value in kernel parameters

struct CamPack {                   // by-value kernel parameter (<= 64 * 92 B)
  steepgs_camera cam[kMaxViews];
  float lim[kMaxViews][2];          // guard * (W/2) / fx, guard * (H/2) / fy: the decision chain's
                                    // per-camera cull limits (§3.2), IEEE fp32 on the host
  double dc[kMaxViews][16];         // the camera in fp64 (R row-major, t, fx, fy, cx, cy), widened once on
                                    // the host so the fp64 render values need no per-thread conversions
};

struct RasterK {
  float alpha_min, alpha_max, t_min, dilation;
  float bg[3];
};

inline RasterK raster_k(const steepgs_raster_params* rp) {
  RasterK r;
  r.alpha_min = rp->alpha_min; r.alpha_max = rp->alpha_max; r.t_min = rp->t_min; r.dilation = rp->dilation;
  r.bg[0] = rp->bg[0]; r.bg[1] = rp->bg[1]; r.bg[2] = rp->bg[2];
  return r;
}

// ---- launch bookkeeping (abi.cu) ----
void note_launch(int k = 1);
cudaError_t check_launch(const char* what);

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl may be scheduled while the
// previous kernel of the stream drains its last wave; it executes pdl_wait() (griddepcontrol.wait:
// the previous grid complete and its writes visible) before it reads anything that kernel wrote, and
// pdl_trigger() lets the next kernel's blocks be scheduled once every block of this grid has started.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// kPdl: with the programmatic-stream-serialization attribute (SGS_NO_PDL builds leave it off everywhere).
template <bool kPdl, typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  if (kPdl) {
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
#ifndef SGS_NO_PDL
  return launch_k<true>(kern, grid, block, smem, st, args...);
#else
  return launch_k<false>(kern, grid, block, smem, st, args...);
#endif
}

// ---- launchers (one per .cu) ----
cudaError_t launch_project(const float* params, int64_t ld, int64_t n, const float* sh_rest, int64_t ld_sh,
                           int sh_degree, const CamPack& cams, int V, const RasterK& rk, steepgs_splat* splats,
                           uint32_t* depth_key, uint32_t* tile_rect, int32_t* tiles_touched, cudaStream_t st);
cudaError_t launch_sh_bwd(const float* params, int64_t ld, int64_t n, const float* sh_rest, int64_t ld_sh,
                          int sh_degree, const CamPack& cams, int V, const float* moments, float* grad_S,
                          int64_t ldg, float* grad_sh, int64_t ldg_sh, int accumulate, cudaStream_t st);
cudaError_t launch_adam_planes(float* params, int64_t ld, int planes, int64_t n, const float* grad, int64_t ldg,
                               float* m, float* v, int64_t ldm, const steepgs_adam_params& ap, int64_t step,
                               cudaStream_t st);
size_t loss_ws_bytes(int V, int H, int W);
cudaError_t launch_ssim_loss(const float* image, const float* target, int V, int H, int W, float lam, float scale,
                             float* dL, float* loss, void* ws, cudaStream_t st);
size_t prune_ws_bytes(int64_t n);
cudaError_t launch_prune_decide(const float* logit, int64_t n, float logit_min, int32_t* new_index, int64_t* n_keep,
                                void* ws, size_t ws_bytes, cudaStream_t st);
cudaError_t launch_compact_planes(const float* src, int64_t ld_src, float* dst, int64_t ld_dst, int planes, int64_t n,
                                  const int32_t* new_index, cudaStream_t st);
cudaError_t launch_copy_planes(float* dst, int64_t ld_dst, const float* src, int64_t ld_src, int64_t n, int first,
                               int count, cudaStream_t st);
cudaError_t launch_copy_offspring(float* arr, int64_t ld, int planes, int64_t n, const int32_t* dest,
                                  cudaStream_t st);

// Real spherical harmonics of degree <= D at unit direction d (3DGS ordering and constants; NEXT f3).
template <int D>
__device__ __forceinline__ void sh_basis(const float* d, float* Y) {
  const float x = d[0], y = d[1], z = d[2];
  Y[0] = 0.28209479177387814f;
  if (D < 1) return;
  Y[1] = -0.4886025119029199f * y;
  Y[2] = 0.4886025119029199f * z;
  Y[3] = -0.4886025119029199f * x;
  if (D < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z;
  Y[4] = 1.0925484305920792f * x * y;
  Y[5] = -1.0925484305920792f * y * z;
  Y[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
  Y[7] = -1.0925484305920792f * x * z;
  Y[8] = 0.5462742152960396f * (xx - yy);
  if (D < 3) return;
  Y[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
  Y[10] = 2.890611442640554f * x * y * z;
  Y[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
  Y[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
  Y[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
  Y[14] = 1.445305721320277f * z * (xx - yy);
  Y[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

struct SortWs;  // bin_sort workspace carve-up (sort.cu)
size_t bin_sort_ws_bytes(int64_t n, int V, int tiles, int64_t max_instances);
cudaError_t launch_bin_sort(const uint32_t* depth_key, const uint32_t* tile_rect, const int32_t* tiles_touched,
                            int64_t n, int V, int tiles_x, int tiles_y, void* ws, size_t ws_bytes,
                            int64_t max_instances, steepgs_binning* out, cudaStream_t st);

struct L1Fused {                    // the a4 l1 gradient fused into the forward's epilogue (optional)
  const float* target;              // [V][3][H][W] or nullptr
  float* dL;                        // [V][3][H][W]
  float* loss;                      // [V] or nullptr
  float scale;
  const uint8_t* target_u8;         // [V][3][H][W] 8-bit targets (decoded / 255) instead; both null: off
};
cudaError_t launch_render_fwd(const steepgs_splat* splats, int64_t n, const steepgs_binning& b, int W, int H,
                              const RasterK& rk, float* image, float* final_T, int32_t* n_contrib,
                              int64_t* pair_counts, cudaStream_t st, const L1Fused& l1 = L1Fused{nullptr, nullptr, nullptr, 0.f, nullptr});
cudaError_t launch_l1_grad(const float* image, const float* target, int V, int64_t count, float scale,
                           float* dL, float* loss, cudaStream_t st);
cudaError_t launch_render_bwd(const steepgs_splat* splats, const steepgs_binning& b, int W, int H,
                              const RasterK& rk, const float* final_T, const int32_t* n_contrib,
                              const float* dL_dimage, int64_t n, float* moments, cudaStream_t st);
constexpr int kMaxRanks = 8;        // the fused reduce's peer set (one NVLink / NVSwitch domain)
struct ScatterOut {                 // k_gauss_bwd output redirected to the column owners' partial buffers
  float* peers[kMaxRanks];          // rank q's [R][20][chunk] partial buffer (device / P2P pointers)
  int R, rank;                      // R = 0: the ordinary output into grad_S
  int64_t chunk;
};
struct PeerPtrs {
  float* p[kMaxRanks];
};
cudaError_t launch_gauss_bwd(const float* params, int64_t ld, int64_t n, const CamPack& cams, int V,
                             const RasterK& rk, float* moments, float* grad_S, int64_t ldg, int accumulate,
                             const int32_t* tiles_touched, float* view_grad_stats, cudaStream_t st,
                             const ScatterOut& sc = ScatterOut{{nullptr}, 0, 0, 0});
cudaError_t launch_reduce_bcast(const float* partials, int R, int rank, int64_t n, int64_t chunk, const PeerPtrs& gs,
                                int64_t ldg, int accumulate, cudaStream_t st);

size_t densify_ws_bytes(int64_t n);
cudaError_t launch_densify(float* params, int64_t ld, int64_t n, int64_t capacity, float* grad_S, int64_t ldg,
                           const steepgs_densify_params& dp, uint8_t* mask, int32_t* dest, float* lambda,
                           int64_t* n_split, int32_t* status, void* ws, size_t ws_bytes, cudaStream_t st);

cudaError_t launch_adam(float* params, int64_t ld, int64_t n, const float* grad, int64_t ldg, float* m, float* v,
                        int64_t ldm, const steepgs_adam_params& ap, int64_t step, float* gacc, int gacc_accumulate,
                        cudaStream_t st);
cudaError_t launch_reset_moments(float* m, float* v, int64_t ldm, int64_t n, const uint8_t* mask,
                                 const int64_t* n_split, int mask_value, int planes, int64_t capacity,
                                 cudaStream_t st);

size_t adc_ws_bytes(int64_t n);
cudaError_t launch_adc(float* params, int64_t ld, int64_t n, int64_t capacity, float* grad_S, int64_t ldg,
                       float* stats, int64_t lds, const float* normals, int64_t ldz, const steepgs_adc_params& ap,
                       uint8_t* kind, int32_t* dest, int64_t* n_new, int32_t* status, void* ws, size_t ws_bytes,
                       cudaStream_t st);

}  // namespace sgs
