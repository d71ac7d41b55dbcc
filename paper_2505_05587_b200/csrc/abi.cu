// abi.cu — the extern "C" boundary of libsteepgs (declared in include/steepgs.h): argument
// validation, device check (compute capability 10.x only), launch bookkeeping, error strings.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

// One NVTX range per C-ABI compute call: visible in nsys / ncu --nvtx; a no-op
// (one predictable branch) when no tool is attached.
struct SgsNvtxRange {
  explicit SgsNvtxRange(const char* s) { nvtxRangePushA(s); }
  ~SgsNvtxRange() { nvtxRangePop(); }
};
#define SGS_NVTX(name) SgsNvtxRange sgs_nvtx_range_(name)

namespace sgs {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void note_launch(int k) { g_launches.fetch_add((uint64_t)k, std::memory_order_relaxed); }

cudaError_t check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e;
}

static steepgs_status fail(steepgs_status s, const char* msg) {
  g_last_error = msg;
  return s;
}

static steepgs_status cuda_fail(cudaError_t e, const char* where) {
  if (g_last_error.empty() || g_last_error.find(cudaGetErrorString(e)) == std::string::npos)
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return STEEPGS_ERR_CUDA;
}

static steepgs_status device_ok() {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(STEEPGS_ERR_UNSUPPORTED_DEVICE, "no CUDA device");
  int major = 0;
  e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (e != cudaSuccess || major != 10)
    return fail(STEEPGS_ERR_UNSUPPORTED_DEVICE, "libsteepgs is built for sm_100a (compute capability 10.x) only");
  return STEEPGS_OK;
}

static steepgs_status check_views(const steepgs_camera* cams, int32_t V, CamPack* pack) {
  if (!cams || V < 1 || V > kMaxViews) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "V must be in [1, 64] and cams non-null");
  for (int v = 0; v < V; ++v) {
    if (cams[v].width <= 0 || cams[v].height <= 0 || cams[v].width != cams[0].width || cams[v].height != cams[0].height)
      return fail(STEEPGS_ERR_INVALID_ARGUMENT, "all views need the same positive width/height");
    if (cams[v].width >= 65536 * kTile || cams[v].height >= 65536 * kTile)
      return fail(STEEPGS_ERR_INVALID_ARGUMENT, "image too large");
    if (cams[v].model != 0 && cams[v].model != 1) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "camera model must be 0 or 1");
    if (pack) {
      pack->cam[v] = cams[v];
      // same fp32 operations as the decision chain (MUL(guard, DIV(MUL(0.5, W), fx))), evaluated
      // once per camera; volatile keeps each operation a separately rounded IEEE single op
      volatile float hw = 0.5f * (float)cams[v].width, hh = 0.5f * (float)cams[v].height;
      volatile float qx = hw / cams[v].fx, qy = hh / cams[v].fy;
      volatile float lx = cams[v].guard * qx, ly = cams[v].guard * qy;
      pack->lim[v][0] = lx;
      pack->lim[v][1] = ly;
      for (int k = 0; k < 9; ++k) pack->dc[v][k] = (double)cams[v].R[k];
      for (int k = 0; k < 3; ++k) pack->dc[v][9 + k] = (double)cams[v].t[k];
      pack->dc[v][12] = cams[v].fx; pack->dc[v][13] = cams[v].fy;
      pack->dc[v][14] = cams[v].cx; pack->dc[v][15] = cams[v].cy;
    }
  }
  return STEEPGS_OK;
}

static steepgs_status check_raster(const steepgs_raster_params* rp) {
  if (!rp) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "raster params null");
  if (rp->tile != kTile) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "tile must be 16");
  if (!(rp->alpha_min >= 0.f) || !(rp->alpha_max > 0.f) || !(rp->alpha_max <= 1.f) || !(rp->t_min >= 0.f) ||
      !(rp->dilation >= 0.f))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "raster params out of range");
  return STEEPGS_OK;
}

static bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Binning generations and forward tokens (STEEPGS_ERR_STALE_STATE): bin_sort stamps a fresh
// generation; the forward stores a hash of (generation, splats, n, cameras, raster params); the
// backward recomputes it from its own arguments.
static std::atomic<uint64_t> g_generation{0};
static uint64_t fnv1a(uint64_t h, const void* p, size_t bytes) {
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (size_t k = 0; k < bytes; ++k) h = (h ^ c[k]) * 1099511628211ull;
  return h;
}
static uint64_t fwd_token(const steepgs_binning* b, const steepgs_splat* splats, int64_t n, const steepgs_camera* cams,
                          int32_t V, const steepgs_raster_params* rp) {
  uint64_t h = 14695981039346656037ull;
  h = fnv1a(h, &b->generation, sizeof(b->generation));
  h = fnv1a(h, &splats, sizeof(splats));
  h = fnv1a(h, &n, sizeof(n));
  h = fnv1a(h, &V, sizeof(V));
  h = fnv1a(h, cams, sizeof(steepgs_camera) * (size_t)V);
  h = fnv1a(h, rp, sizeof(*rp));
  return h ? h : 1ull;   // 0 means "no forward"
}
static steepgs_status check_token(const steepgs_binning* b, const steepgs_splat* splats, int64_t n,
                                  const steepgs_camera* cams, int32_t V, const steepgs_raster_params* rp) {
  if (b->fwd_token == 0) return fail(STEEPGS_ERR_STALE_STATE, "render_bwd: no render_fwd on this binning");
  if (b->fwd_token != fwd_token(b, splats, n, cams, V, rp))
    return fail(STEEPGS_ERR_STALE_STATE,
                "render_bwd: the binning was re-sorted, or its forward used other splats / n / cameras / raster params");
  return STEEPGS_OK;
}

static steepgs_status check_binning(const steepgs_binning* b, int32_t V, const steepgs_camera* cams) {
  if (!b || !b->ids || !b->ranges || !b->n_instances || !b->tile_last || !b->inst_mask || !b->tile_order)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "binning null");
  const int tx = (cams[0].width + kTile - 1) / kTile, ty = (cams[0].height + kTile - 1) / kTile;
  if (b->V != V || b->tiles_x != tx || b->tiles_y != ty)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "binning does not match the views of this call");
  return STEEPGS_OK;
}

}  // namespace sgs

using namespace sgs;

#ifdef STEEPGS_CHECKS
namespace sgs {
cudaError_t checks_io_render(unsigned int* out, bool reset);
cudaError_t checks_io_sort(unsigned int* out, bool reset);
cudaError_t checks_io_densify(unsigned int* out, bool reset);
}  // namespace sgs
#endif

extern "C" {

steepgs_status steepgs_debug_checks(int32_t* compiled, uint64_t* failures, uint32_t* first_line, int32_t reset) {
  if (!compiled || !failures || !first_line) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  *failures = 0;
  *first_line = 0;
#ifdef STEEPGS_CHECKS
  *compiled = 1;
  cudaError_t (*io[3])(unsigned int*, bool) = {checks_io_render, checks_io_sort, checks_io_densify};
  for (auto f : io) {
    unsigned int v[2] = {0u, 0u};
    const cudaError_t e = f(v, reset != 0);
    if (e != cudaSuccess) return cuda_fail(e, "steepgs_debug_checks");
    *failures += v[0];
    if (v[0] && !*first_line) *first_line = v[1];
  }
#else
  *compiled = 0;
#endif
  return STEEPGS_OK;
}


const char* steepgs_status_string(steepgs_status s) {
  switch (s) {
    case STEEPGS_OK: return "ok";
    case STEEPGS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case STEEPGS_ERR_WORKSPACE_TOO_SMALL: return "workspace too small";
    case STEEPGS_ERR_CAPACITY: return "capacity exceeded";
    case STEEPGS_ERR_UNSUPPORTED_DEVICE: return "unsupported device (need compute capability 10.x)";
    case STEEPGS_ERR_CUDA: return "CUDA error";
  }
  return "unknown status";
}

const char* steepgs_last_error(void) { return g_last_error.c_str(); }
uint64_t steepgs_launch_count(void) { return g_launches.load(); }
const char* steepgs_version(void) { return "steepgs-b200 0.1 (sm_100a)"; }

steepgs_status steepgs_project(const float* params, int64_t ld, int64_t n, const steepgs_camera* cams, int32_t V,
                               const steepgs_raster_params* rp, steepgs_splat* splats, uint32_t* depth_key,
                               uint32_t* tile_rect, int32_t* tiles_touched, void* stream) {
  SGS_NVTX("steepgs_project");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  CamPack pack;
  if ((s = check_views(cams, V, &pack)) != STEEPGS_OK) return s;
  if ((s = check_raster(rp)) != STEEPGS_OK) return s;
  if (n < 0 || ld < n) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "need 0 <= n <= ld");
  if ((int64_t)V * n >= (1ll << 32)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "V * n must be < 2^32");
  if (n > 0 && (!params || !splats || !depth_key || !tile_rect || !tiles_touched))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned(splats, 16) || !aligned(tile_rect, 8)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "misaligned output");
  const cudaError_t e = launch_project(params, ld, n, nullptr, 0, -1, pack, V, raster_k(rp), splats, depth_key,
                                       tile_rect, tiles_touched, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_project");
}

steepgs_status steepgs_project_sh(const float* params, int64_t ld, int64_t n, const float* sh_rest, int64_t ld_sh,
                                  int32_t sh_degree, const steepgs_camera* cams, int32_t V,
                                  const steepgs_raster_params* rp, steepgs_splat* splats, uint32_t* depth_key,
                                  uint32_t* tile_rect, int32_t* tiles_touched, void* stream) {
  SGS_NVTX("steepgs_project_sh");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  CamPack pack;
  if ((s = check_views(cams, V, &pack)) != STEEPGS_OK) return s;
  if ((s = check_raster(rp)) != STEEPGS_OK) return s;
  if (n < 0 || ld < n) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "need 0 <= n <= ld");
  if (sh_degree < 0 || sh_degree > 3) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "sh_degree must be 0..3");
  if (sh_degree > 0 && n > 0 && (!sh_rest || ld_sh < n)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad sh_rest");
  if ((int64_t)V * n >= (1ll << 32)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "V * n must be < 2^32");
  if (n > 0 && (!params || !splats || !depth_key || !tile_rect || !tiles_touched))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned(splats, 16) || !aligned(tile_rect, 8)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "misaligned output");
  const cudaError_t e = launch_project(params, ld, n, sh_rest, ld_sh, sh_degree, pack, V, raster_k(rp), splats,
                                       depth_key, tile_rect, tiles_touched, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_project_sh");
}

steepgs_status steepgs_sh_bwd(const float* params, int64_t ld, int64_t n, const float* sh_rest, int64_t ld_sh,
                              int32_t sh_degree, const steepgs_camera* cams, int32_t V, const float* moments_ws,
                              float* grad_S, int64_t ldg, float* grad_sh, int64_t ldg_sh, int32_t accumulate,
                              void* stream) {
  SGS_NVTX("steepgs_sh_bwd");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  CamPack pack;
  if ((s = check_views(cams, V, &pack)) != STEEPGS_OK) return s;
  if (n < 0 || ld < n || ldg < n) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "need 0 <= n <= ld, ldg");
  if (sh_degree < 0 || sh_degree > 3) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "sh_degree must be 0..3");
  if (accumulate < 0 || accumulate > 2) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "accumulate must be 0, 1 or 2");
  if (n > 0 && (!params || !moments_ws || !grad_S)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  if (sh_degree > 0 && n > 0 && (!sh_rest || !grad_sh || ld_sh < n || ldg_sh < n))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad sh_rest / grad_sh");
  if (!aligned(moments_ws, 16)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "moments_ws must be 16-byte aligned");
  const cudaError_t e = launch_sh_bwd(params, ld, n, sh_rest, ld_sh, sh_degree, pack, V, moments_ws, grad_S, ldg,
                                      grad_sh, ldg_sh, accumulate, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_sh_bwd");
}

steepgs_status steepgs_adam_step_planes(float* params, int64_t ld, int32_t planes, int64_t n, const float* grad,
                                        int64_t ldg, float* adam_m, float* adam_v, int64_t ldm,
                                        const steepgs_adam_params* ap, int64_t step, void* stream) {
  SGS_NVTX("steepgs_adam_step_planes");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (!ap || step < 1 || n < 0 || planes < 0 || ld < n || ldg < n || ldm < n || !(ap->beta1 >= 0.0 && ap->beta1 < 1.0) ||
      !(ap->beta2 >= 0.0 && ap->beta2 < 1.0) || !(ap->eps > 0.0))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad adam arguments");
  if (n > 0 && planes > 0 && (!params || !grad || !adam_m || !adam_v))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  const cudaError_t e = launch_adam_planes(params, ld, planes, n, grad, ldg, adam_m, adam_v, ldm, *ap, step,
                                           (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_adam_step_planes");
}

steepgs_status steepgs_loss_workspace_size(int32_t V, int32_t height, int32_t width, size_t* bytes) {
  if (!bytes || V < 1 || V > kMaxViews || height <= 0 || width <= 0)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad arguments");
  *bytes = loss_ws_bytes(V, height, width);
  return STEEPGS_OK;
}

steepgs_status steepgs_l1_ssim_grad(const float* image, const float* target, int32_t V, int32_t height, int32_t width,
                                    float lambda_ssim, float scale, float* dL_dimage, float* loss, void* workspace,
                                    size_t ws_bytes, void* stream) {
  SGS_NVTX("steepgs_l1_ssim_grad");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (V < 1 || V > kMaxViews || height <= 0 || width <= 0 || !(lambda_ssim >= 0.f && lambda_ssim <= 1.f))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "need 1 <= V <= 64, H, W > 0, 0 <= lambda <= 1");
  if (!image || !target || !dL_dimage || !workspace) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  if (ws_bytes < loss_ws_bytes(V, height, width)) return fail(STEEPGS_ERR_WORKSPACE_TOO_SMALL, "loss workspace");
  const cudaError_t e = launch_ssim_loss(image, target, V, height, width, lambda_ssim, scale, dL_dimage, loss,
                                         workspace, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_l1_ssim_grad");
}

steepgs_status steepgs_prune_workspace_size(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad arguments");
  *bytes = prune_ws_bytes(n);
  return STEEPGS_OK;
}

steepgs_status steepgs_prune_decide(const float* params, int64_t ld, int64_t n, float logit_min, int32_t* new_index,
                                    int64_t* n_keep, void* workspace, size_t ws_bytes, void* stream) {
  SGS_NVTX("steepgs_prune_decide");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (n < 0 || ld < n || n >= (1ll << 31) || !n_keep || !workspace || (n > 0 && (!params || !new_index)))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad prune arguments");
  if (ws_bytes < prune_ws_bytes(n)) return fail(STEEPGS_ERR_WORKSPACE_TOO_SMALL, "prune workspace too small");
  const cudaError_t e = launch_prune_decide(params + 10 * ld, n, logit_min, new_index, n_keep, workspace, ws_bytes,
                                            (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_prune_decide");
}

steepgs_status steepgs_compact_planes(const float* src, int64_t ld_src, float* dst, int64_t ld_dst, int32_t planes,
                                      int64_t n, const int32_t* new_index, void* stream) {
  SGS_NVTX("steepgs_compact_planes");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (n < 0 || planes < 0 || ld_src < n || ld_dst < n || (n > 0 && planes > 0 && (!src || !dst || !new_index)) ||
      (src == dst && planes > 0 && n > 0))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad compact_planes arguments (out of place only)");
  const cudaError_t e = launch_compact_planes(src, ld_src, dst, ld_dst, planes, n, new_index, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_compact_planes");
}

steepgs_status steepgs_copy_offspring(float* arr, int64_t ld, int32_t planes, int64_t n, const int32_t* dest_index,
                                      void* stream) {
  SGS_NVTX("steepgs_copy_offspring");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (n < 0 || planes < 0 || ld < n || (n > 0 && planes > 0 && (!arr || !dest_index)))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad copy_offspring arguments");
  const cudaError_t e = launch_copy_offspring(arr, ld, planes, n, dest_index, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_copy_offspring");
}

steepgs_status steepgs_bin_sort_workspace_size(int64_t n, int32_t V, int32_t width, int32_t height,
                                               int64_t max_instances, size_t* bytes) {
  if (!bytes || n < 0 || V < 1 || V > kMaxViews || width <= 0 || height <= 0 || max_instances < 0 ||
      max_instances >= (1ll << 31))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad workspace-size arguments");
  const int tiles = ((width + kTile - 1) / kTile) * ((height + kTile - 1) / kTile);
  *bytes = bin_sort_ws_bytes(n, V, tiles, max_instances);
  return STEEPGS_OK;
}

steepgs_status steepgs_bin_sort(const uint32_t* depth_key, const uint32_t* tile_rect, const int32_t* tiles_touched,
                                int64_t n, const steepgs_camera* cams, int32_t V, const steepgs_raster_params* rp,
                                void* workspace, size_t ws_bytes, int64_t max_instances, steepgs_binning* out,
                                void* stream) {
  SGS_NVTX("steepgs_bin_sort");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if ((s = check_views(cams, V, nullptr)) != STEEPGS_OK) return s;
  if ((s = check_raster(rp)) != STEEPGS_OK) return s;
  if (!out || !workspace || n < 0 || max_instances < 0 || max_instances >= (1ll << 31))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad bin_sort arguments");
  if (n > 0 && (!depth_key || !tile_rect || !tiles_touched)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned(workspace, 256)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  const int tx = (cams[0].width + kTile - 1) / kTile, ty = (cams[0].height + kTile - 1) / kTile;
  if ((int64_t)tx * ty * V >= (1 << 24)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "too many tiles");
  size_t need = bin_sort_ws_bytes(n, V, tx * ty, max_instances);
  if (ws_bytes < need) return fail(STEEPGS_ERR_WORKSPACE_TOO_SMALL, "bin_sort workspace too small");
  const cudaError_t e = launch_bin_sort(depth_key, tile_rect, tiles_touched, n, V, tx, ty, workspace, ws_bytes,
                                        max_instances, out, (cudaStream_t)stream);
  out->generation = g_generation.fetch_add(1, std::memory_order_relaxed) + 1;
  out->fwd_token = 0;
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_bin_sort");
}

steepgs_status steepgs_render_fwd(const steepgs_splat* splats, int64_t n, steepgs_binning* b,
                                  const steepgs_camera* cams, int32_t V, const steepgs_raster_params* rp, float* image,
                                  float* final_T, int32_t* n_contrib, int64_t* pair_counts, void* stream) {
  SGS_NVTX("steepgs_render_fwd");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if ((s = check_views(cams, V, nullptr)) != STEEPGS_OK) return s;
  if ((s = check_raster(rp)) != STEEPGS_OK) return s;
  if ((s = check_binning(b, V, cams)) != STEEPGS_OK) return s;
  if (n < 0 || !image || !final_T || !n_contrib || (n > 0 && !splats))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  const cudaError_t e = launch_render_fwd(splats, n, *b, cams[0].width, cams[0].height, raster_k(rp), image, final_T,
                                          n_contrib, pair_counts, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "steepgs_render_fwd");
  b->fwd_token = fwd_token(b, splats, n, cams, V, rp);
  return STEEPGS_OK;
}

steepgs_status steepgs_render_fwd_l1(const steepgs_splat* splats, int64_t n, steepgs_binning* b,
                                     const steepgs_camera* cams, int32_t V, const steepgs_raster_params* rp,
                                     float* image, float* final_T, int32_t* n_contrib, const float* target,
                                     float scale, float* dL_dimage, float* loss, int64_t* pair_counts, void* stream) {
  SGS_NVTX("steepgs_render_fwd_l1");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if ((s = check_views(cams, V, nullptr)) != STEEPGS_OK) return s;
  if ((s = check_raster(rp)) != STEEPGS_OK) return s;
  if ((s = check_binning(b, V, cams)) != STEEPGS_OK) return s;
  if (n < 0 || !image || !final_T || !n_contrib || !target || !dL_dimage || (n > 0 && !splats))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  const L1Fused l1{target, dL_dimage, loss, scale, nullptr};
  const cudaError_t e = launch_render_fwd(splats, n, *b, cams[0].width, cams[0].height, raster_k(rp), image, final_T,
                                          n_contrib, pair_counts, (cudaStream_t)stream, l1);
  if (e != cudaSuccess) return cuda_fail(e, "steepgs_render_fwd_l1");
  b->fwd_token = fwd_token(b, splats, n, cams, V, rp);
  return STEEPGS_OK;
}

steepgs_status steepgs_render_fwd_l1_u8(const steepgs_splat* splats, int64_t n, steepgs_binning* b,
                                        const steepgs_camera* cams, int32_t V, const steepgs_raster_params* rp,
                                        float* image, float* final_T, int32_t* n_contrib, const uint8_t* target,
                                        float scale, float* dL_dimage, float* loss, int64_t* pair_counts,
                                        void* stream) {
  SGS_NVTX("steepgs_render_fwd_l1_u8");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if ((s = check_views(cams, V, nullptr)) != STEEPGS_OK) return s;
  if ((s = check_raster(rp)) != STEEPGS_OK) return s;
  if ((s = check_binning(b, V, cams)) != STEEPGS_OK) return s;
  if (n < 0 || !image || !final_T || !n_contrib || !target || !dL_dimage || (n > 0 && !splats))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  const L1Fused l1{nullptr, dL_dimage, loss, scale, target};
  const cudaError_t e = launch_render_fwd(splats, n, *b, cams[0].width, cams[0].height, raster_k(rp), image, final_T,
                                          n_contrib, pair_counts, (cudaStream_t)stream, l1);
  if (e != cudaSuccess) return cuda_fail(e, "steepgs_render_fwd_l1_u8");
  b->fwd_token = fwd_token(b, splats, n, cams, V, rp);
  return STEEPGS_OK;
}

steepgs_status steepgs_l1_grad(const float* image, const float* target, int32_t V, int64_t count, float scale,
                               float* dL_dimage, float* loss, void* stream) {
  SGS_NVTX("steepgs_l1_grad");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (V < 1 || count < 0 || !image || !target || !dL_dimage) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad l1 arguments");
  const cudaError_t e = launch_l1_grad(image, target, V, count, scale, dL_dimage, loss, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_l1_grad");
}

steepgs_status steepgs_render_bwd_split(const float* params, int64_t ld, int64_t n, const steepgs_splat* splats,
                                        const steepgs_binning* b, const steepgs_camera* cams, int32_t V,
                                        const steepgs_raster_params* rp,
                                        const float* final_T, const int32_t* n_contrib, const float* dL_dimage,
                                        float* moments_ws, float* grad_S, int64_t ldg, int32_t accumulate,
                                        const int32_t* tiles_touched, float* view_grad_stats, void* stream) {
  SGS_NVTX("steepgs_render_bwd_split");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  CamPack pack;
  if ((s = check_views(cams, V, &pack)) != STEEPGS_OK) return s;
  if ((s = check_raster(rp)) != STEEPGS_OK) return s;
  if ((s = check_binning(b, V, cams)) != STEEPGS_OK) return s;
  if (n < 0 || ld < n || ldg < n) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "need 0 <= n <= ld, ldg");
  if ((accumulate & ~7) || (accumulate & 3) == 3)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "accumulate must be 0, 1 or 2 (| 4 after steepgs_sh_bwd)");
  if (view_grad_stats && n > 0 && !tiles_touched)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "view_grad_stats needs tiles_touched");
  if (n > 0 && (!params || !splats || !final_T || !n_contrib || !dL_dimage || !moments_ws || !grad_S))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned(moments_ws, 16)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "moments_ws must be 16-byte aligned");
  if ((s = check_token(b, splats, n, cams, V, rp)) != STEEPGS_OK) return s;
  const RasterK rk = raster_k(rp);
  cudaError_t e = launch_render_bwd(splats, *b, cams[0].width, cams[0].height, rk, final_T, n_contrib, dL_dimage, n,
                                    moments_ws, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "steepgs_render_bwd_split");
  e = launch_gauss_bwd(params, ld, n, pack, V, rk, moments_ws, grad_S, ldg, accumulate, tiles_touched, view_grad_stats,
                       (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_render_bwd_split");
}

steepgs_status steepgs_render_bwd_moments(const steepgs_splat* splats, int64_t n, const steepgs_binning* b,
                                          const steepgs_camera* cams, int32_t V, const steepgs_raster_params* rp,
                                          const float* final_T, const int32_t* n_contrib, const float* dL_dimage,
                                          float* moments_ws, void* stream) {
  SGS_NVTX("steepgs_render_bwd_moments");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if ((s = check_views(cams, V, nullptr)) != STEEPGS_OK) return s;
  if ((s = check_raster(rp)) != STEEPGS_OK) return s;
  if ((s = check_binning(b, V, cams)) != STEEPGS_OK) return s;
  if (n < 0 || (n > 0 && (!splats || !final_T || !n_contrib || !dL_dimage || !moments_ws)))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned(moments_ws, 16)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "moments_ws must be 16-byte aligned");
  if ((s = check_token(b, splats, n, cams, V, rp)) != STEEPGS_OK) return s;
  const cudaError_t e = launch_render_bwd(splats, *b, cams[0].width, cams[0].height, raster_k(rp), final_T, n_contrib,
                                          dL_dimage, n, moments_ws, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_render_bwd_moments");
}

steepgs_status steepgs_gauss_bwd_split(const float* params, int64_t ld, int64_t n, const steepgs_camera* cams,
                                       int32_t V, const steepgs_raster_params* rp,
                                       float* moments_ws, float* grad_S, int64_t ldg, int32_t accumulate,
                                       const int32_t* tiles_touched, float* view_grad_stats, void* stream) {
  SGS_NVTX("steepgs_gauss_bwd_split");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  CamPack pack;
  if ((s = check_views(cams, V, &pack)) != STEEPGS_OK) return s;
  if ((s = check_raster(rp)) != STEEPGS_OK) return s;
  if (n < 0 || ld < n || ldg < n) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "need 0 <= n <= ld, ldg");
  if ((accumulate & ~7) || (accumulate & 3) == 3)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "accumulate must be 0, 1 or 2 (| 4 after steepgs_sh_bwd)");
  if (view_grad_stats && n > 0 && !tiles_touched)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "view_grad_stats needs tiles_touched");
  if (n > 0 && (!params || !moments_ws || !grad_S)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned(moments_ws, 16)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "moments_ws must be 16-byte aligned");
  const cudaError_t e = launch_gauss_bwd(params, ld, n, pack, V, raster_k(rp), moments_ws, grad_S, ldg, accumulate,
                                         tiles_touched, view_grad_stats, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_gauss_bwd_split");
}

steepgs_status steepgs_scatter_chunk(int64_t n, int32_t R, int64_t* chunk) {
  if (!chunk || n < 0 || R < 1 || R > kMaxRanks) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad scatter arguments");
  const int64_t c = (n + R - 1) / R;
  *chunk = ((c + 31) / 32) * 32;   // owners' column ranges start on 128-B boundaries
  return STEEPGS_OK;
}

steepgs_status steepgs_gauss_bwd_scatter(const float* params, int64_t ld, int64_t n, const steepgs_camera* cams,
                                         int32_t V, const steepgs_raster_params* rp, float* moments_ws,
                                         const uint64_t* peer_partials, int32_t R, int32_t rank, int64_t chunk,
                                         void* stream) {
  SGS_NVTX("steepgs_gauss_bwd_scatter");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  CamPack pack;
  if ((s = check_views(cams, V, &pack)) != STEEPGS_OK) return s;
  if ((s = check_raster(rp)) != STEEPGS_OK) return s;
  if (n < 0 || ld < n || R < 1 || R > kMaxRanks || rank < 0 || rank >= R || !peer_partials)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad scatter arguments");
  int64_t need = 0;
  steepgs_scatter_chunk(n, R, &need);
  if (chunk != need) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "chunk must be steepgs_scatter_chunk(n, R)");
  if (n > 0 && (!params || !moments_ws)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned(moments_ws, 16)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "moments_ws must be 16-byte aligned");
  ScatterOut sc{};
  for (int q = 0; q < R; ++q) {
    sc.peers[q] = reinterpret_cast<float*>(peer_partials[q]);
    if (!sc.peers[q]) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null peer partial buffer");
  }
  sc.R = R; sc.rank = rank; sc.chunk = chunk;
  const cudaError_t e = launch_gauss_bwd(params, ld, n, pack, V, raster_k(rp), moments_ws, nullptr, 0, 0, nullptr,
                                         nullptr, (cudaStream_t)stream, sc);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_gauss_bwd_scatter");
}

steepgs_status steepgs_reduce_bcast(const float* partials, int32_t R, int32_t rank, int64_t n, int64_t chunk,
                                    const uint64_t* peer_grad_S, int64_t ldg, int32_t accumulate, void* stream) {
  SGS_NVTX("steepgs_reduce_bcast");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (n < 0 || R < 1 || R > kMaxRanks || rank < 0 || rank >= R || !peer_grad_S || ldg < n || (accumulate & ~3) ||
      accumulate == 3)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad reduce arguments");
  int64_t need = 0;
  steepgs_scatter_chunk(n, R, &need);
  if (chunk != need) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "chunk must be steepgs_scatter_chunk(n, R)");
  if (n > 0 && !partials) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  PeerPtrs gs{};
  for (int q = 0; q < R; ++q) {
    gs.p[q] = reinterpret_cast<float*>(peer_grad_S[q]);
    if (!gs.p[q]) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null peer grad_S");
  }
  const cudaError_t e = launch_reduce_bcast(partials, R, rank, n, chunk, gs, ldg, accumulate, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_reduce_bcast");
}

steepgs_status steepgs_adc_workspace_size(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad arguments");
  *bytes = adc_ws_bytes(n);
  return STEEPGS_OK;
}

steepgs_status steepgs_densify_adc(float* params, int64_t ld, int64_t n, int64_t capacity, float* grad_S,
                                   int64_t ldg, float* view_grad_stats, const float* normals, int64_t ldz,
                                   const steepgs_adc_params* ap, uint8_t* kind, int32_t* dest_index,
                                   int64_t* n_new, int32_t* status, void* workspace, size_t ws_bytes,
                                   void* stream) {
  SGS_NVTX("steepgs_densify_adc");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (!ap || n < 0 || capacity < n || ld < capacity || ldg < capacity || ldz < n || capacity > INT32_MAX ||
      !(ap->scale_factor > 0.f) || !(ap->denom > 0.f))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad adc arguments (need n <= capacity <= ld, ldg; ldz >= n)");
  if (!n_new || !status || !workspace || (n > 0 && (!params || !grad_S || !view_grad_stats || !normals || !kind ||
                                                    !dest_index)))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  const cudaError_t e = launch_adc(params, ld, n, capacity, grad_S, ldg, view_grad_stats, ldg, normals, ldz, *ap, kind,
                                   dest_index, n_new, status, workspace, ws_bytes, (cudaStream_t)stream);
  if (e == cudaErrorInvalidValue) return fail(STEEPGS_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_densify_adc");
}

steepgs_status steepgs_adam_step(float* params, int64_t ld, int64_t n, const float* grad_S, int64_t ldg,
                                 float* adam_m, float* adam_v, int64_t ldm, const steepgs_adam_params* ap,
                                 int64_t step, float* gacc, int32_t gacc_accumulate, void* stream) {
  SGS_NVTX("steepgs_adam_step");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (!ap || step < 1 || n < 0 || ld < n || ldg < n || ldm < n || !(ap->beta1 >= 0.0 && ap->beta1 < 1.0) ||
      !(ap->beta2 >= 0.0 && ap->beta2 < 1.0) || !(ap->eps > 0.0) || (gacc_accumulate & ~1))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad adam arguments");
  if (n > 0 && (!params || !grad_S || !adam_m || !adam_v)) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  const cudaError_t e = launch_adam(params, ld, n, grad_S, ldg, adam_m, adam_v, ldm, *ap, step, gacc,
                                    gacc_accumulate, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_adam_step");
}

steepgs_status steepgs_reset_moments(float* adam_m, float* adam_v, int64_t ldm, int64_t n,
                                     const uint8_t* split_mask, const int64_t* n_split, int32_t mask_value,
                                     int32_t planes, void* stream) {
  SGS_NVTX("steepgs_reset_moments");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (!adam_m || !adam_v || !n_split || n < 0 || ldm < n || (n > 0 && !split_mask) || mask_value < 1 ||
      mask_value > 255 || planes < 0)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad reset_moments arguments");
  const cudaError_t e = launch_reset_moments(adam_m, adam_v, ldm, n, split_mask, n_split, mask_value, planes, ldm,
                                            (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_reset_moments");
}

steepgs_status steepgs_copy_planes(float* dst, int64_t ld_dst, const float* src, int64_t ld_src, int64_t n,
                                   int32_t first, int32_t count, void* stream) {
  SGS_NVTX("steepgs_copy_planes");
  if (!dst || !src || n < 0 || ld_dst < n || ld_src < n || first < 0 || count < 0)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad copy_planes arguments");
  if (n == 0 || count == 0) return STEEPGS_OK;
  const cudaError_t e = launch_copy_planes(dst, ld_dst, src, ld_src, n, first, count, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_copy_planes");
}

steepgs_status steepgs_densify_workspace_size(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "bad densify workspace arguments");
  *bytes = densify_ws_bytes(n);
  return STEEPGS_OK;
}

steepgs_status steepgs_densify(float* params, int64_t ld, int64_t n, int64_t capacity, float* grad_S, int64_t ldg,
                               const steepgs_densify_params* dp, uint8_t* split_mask, int32_t* dest_index,
                               float* lambda_min, int64_t* n_split, int32_t* status, void* workspace,
                               size_t ws_bytes, void* stream) {
  SGS_NVTX("steepgs_densify");
  steepgs_status s;
  if ((s = device_ok()) != STEEPGS_OK) return s;
  if (!dp || !(dp->denom > 0.f) || dp->gate < 0 || dp->gate > 2)
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "densify params: denom > 0, gate in {0, 1, 2}");
  if (n < 0 || capacity < n || ld < capacity || ldg < capacity || capacity >= (1ll << 31))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "need 0 <= n <= capacity <= ld, ldg < 2^31");
  if (!params || !grad_S || !n_split || !status || !workspace || (n > 0 && (!split_mask || !dest_index)))
    return fail(STEEPGS_ERR_INVALID_ARGUMENT, "null pointer");
  if (ws_bytes < densify_ws_bytes(n)) return fail(STEEPGS_ERR_WORKSPACE_TOO_SMALL, "densify workspace too small");
  const cudaError_t e = launch_densify(params, ld, n, capacity, grad_S, ldg, *dp, split_mask, dest_index, lambda_min,
                                       n_split, status, workspace, ws_bytes, (cudaStream_t)stream);
  return e == cudaSuccess ? STEEPGS_OK : cuda_fail(e, "steepgs_densify");
}

steepgs_status steepgs_densify_host_count(float* params, int64_t ld, int64_t n, int64_t capacity, float* grad_S,
                                          int64_t ldg, const steepgs_densify_params* dp, uint8_t* split_mask,
                                          int32_t* dest_index, float* lambda_min, int64_t* n_split, int32_t* status,
                                          void* workspace, size_t ws_bytes, int64_t* n_split_host, void* stream) {
  SGS_NVTX("steepgs_densify_host_count");
  if (!n_split_host) return fail(STEEPGS_ERR_INVALID_ARGUMENT, "n_split_host null");
  steepgs_status s = steepgs_densify(params, ld, n, capacity, grad_S, ldg, dp, split_mask, dest_index, lambda_min,
                                     n_split, status, workspace, ws_bytes, stream);
  if (s != STEEPGS_OK) return s;
  int64_t ns = 0;
  int32_t st = 0;
  cudaError_t e = cudaMemcpyAsync(&ns, n_split, sizeof ns, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&st, status, sizeof st, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "steepgs_densify_host_count");
  *n_split_host = ns;
  return st == 0 ? STEEPGS_OK : fail(STEEPGS_ERR_CAPACITY, "n + n_split > capacity");
}

}  // extern "C"
