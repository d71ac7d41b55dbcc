// optim.cu — NEXT f1: the Algorithm-1 optimiser step ("update each Gaussian parameters via
// standard gradient descent"; 3DGS trains with Adam) fused over the 14 SoA parameter planes, and the
// Adam-state reset of densified Gaussians.  Bound: HBM (7 x 4 B per parameter per step).
#include <math.h>

#include "common.cuh"

namespace sgs {

namespace {

__constant__ int kGroupOfPlane[14] = {0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 3, 4, 4, 4};

struct AdamK {
  float lr[5];
  float b1, omb1, b2, omb2, eps, bc1, bc2;
};

__global__ void __launch_bounds__(256) k_adam(float* __restrict__ params, int64_t ld, int64_t n,
                                              const float* __restrict__ grad, int64_t ldg, float* __restrict__ m,
                                              float* __restrict__ v, int64_t ldm, const AdamK ap,
                                              float* __restrict__ gacc, int gacc_acc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int k = 0; k < 14; ++k) {
    const float g = grad[k * ldg + i];
    const float mk = ap.b1 * m[k * ldm + i] + ap.omb1 * g;
    const float vk = ap.b2 * v[k * ldm + i] + ap.omb2 * (g * g);
    m[k * ldm + i] = mk;
    v[k * ldm + i] = vk;
    const float mh = mk / ap.bc1, vh = vk / ap.bc2;
    params[k * ld + i] -= ap.lr[kGroupOfPlane[k]] * mh / (sqrtf(vh) + ap.eps);
    if (gacc && k < 3) gacc[k * ldm + i] = gacc_acc ? gacc[k * ldm + i] + g : g;
  }
}

__global__ void __launch_bounds__(256) k_reset_moments(float* __restrict__ m, float* __restrict__ v, int64_t ldm,
                                                       int64_t n, const uint8_t* __restrict__ mask,
                                                       const int64_t* __restrict__ n_split, int mask_value,
                                                       int planes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t end = n + *n_split;
  if (i >= end || (i < n && mask[i] != mask_value)) return;
  for (int k = 0; k < planes; ++k) {
    m[k * ldm + i] = 0.0f;
    v[k * ldm + i] = 0.0f;
  }
}

}  // namespace

cudaError_t launch_adam(float* params, int64_t ld, int64_t n, const float* grad, int64_t ldg, float* m, float* v,
                        int64_t ldm, const steepgs_adam_params& ap, int64_t step, float* gacc, int gacc_accumulate,
                        cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  AdamK k;
  for (int g = 0; g < 5; ++g) k.lr[g] = (float)ap.lr[g];
  k.b1 = (float)ap.beta1;
  k.omb1 = (float)(1.0 - ap.beta1);
  k.b2 = (float)ap.beta2;
  k.omb2 = (float)(1.0 - ap.beta2);
  k.eps = (float)ap.eps;
  k.bc1 = (float)(1.0 - pow(ap.beta1, (double)step));
  k.bc2 = (float)(1.0 - pow(ap.beta2, (double)step));
  k_adam<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(params, ld, n, grad, ldg, m, v, ldm, k, gacc, gacc_accumulate);
  note_launch();
  return check_launch("k_adam");
}

cudaError_t launch_reset_moments(float* m, float* v, int64_t ldm, int64_t n, const uint8_t* mask,
                                 const int64_t* n_split, int mask_value, int planes, int64_t capacity,
                                 cudaStream_t st) {
  if (capacity == 0) return cudaSuccess;
  k_reset_moments<<<(unsigned)((capacity + 255) / 256), 256, 0, st>>>(m, v, ldm, n, mask, n_split, mask_value, planes);
  note_launch();
  return check_launch("k_reset_moments");
}

}  // namespace sgs
