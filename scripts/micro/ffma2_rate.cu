// Microbenchmark: issue rate of FFMA (3-register form) vs FFMA2 (fma.rn.f32x2, sm_100a) vs FADD2/FMUL2
// and MUFU.EX2 on one B200 SM set.  Prints lane-FLOP/clk/SM for each.  (scripts/micro)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t pk(float a, float b){ uint64_t r; asm volatile("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(uint64_t r){ float a,b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a+b; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c){ uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
constexpr int ITER = 4096;
__global__ void k_ffma(float* out, float s, float t) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  float b = s, c = t;
  for (int i = 0; i < ITER; ++i) {
    a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
    a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_ffma_rr(float* out, float s, float t) {   // all three operands distinct registers per op
  float a[8], b[8], c[8];
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x + j; b[j] = s + j; c[j] = t - j; }
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b[j], c[j]);
  }
  float r = 0; for (int j = 0; j < 8; ++j) r += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_ffma2(float* out, float s, float t) {
  uint64_t a0 = pk(threadIdx.x, 1), a1 = pk(2, 3), a2 = pk(4, 5), a3 = pk(6, 7);
  uint64_t b = pk(s, s + 1), c = pk(t, t + 1);
  for (int i = 0; i < ITER; ++i) {
    a0 = fma2(a0, b, c); a1 = fma2(a1, b, c); a2 = fma2(a2, b, c); a3 = fma2(a3, b, c);
    a0 = fma2(a0, b, c); a1 = fma2(a1, b, c); a2 = fma2(a2, b, c); a3 = fma2(a3, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = lo(a0) + lo(a1) + lo(a2) + lo(a3);
}
__global__ void k_ffma2_bc(float* out, float s, float t) {   // scalar-broadcast b, c (the raster's form)
  uint64_t a0 = pk(threadIdx.x, 1), a1 = pk(2, 3), a2 = pk(4, 5), a3 = pk(6, 7), a4 = pk(8, 9), a5 = pk(1, 2), a6 = pk(3, 4), a7 = pk(5, 6);
  uint64_t b = pk(s, s), c = pk(t, t);
  for (int i = 0; i < ITER; ++i) {
    a0 = fma2(a0, b, c); a1 = fma2(a1, b, c); a2 = fma2(a2, b, c); a3 = fma2(a3, b, c);
    a4 = fma2(a4, b, c); a5 = fma2(a5, b, c); a6 = fma2(a6, b, c); a7 = fma2(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = lo(a0) + lo(a1) + lo(a2) + lo(a3) + lo(a4) + lo(a5) + lo(a6) + lo(a7);
}
__global__ void k_ex2(float* out, float s) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  for (int i = 0; i < ITER; ++i) {
    float y0, y1, y2, y3;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(a1));
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y2) : "f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y3) : "f"(a3));
    a0 = y0 * s; a1 = y1 * s; a2 = y2 * s; a3 = y3 * s;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int blocks = p.multiProcessorCount * 4, threads = 512;
  float* out; cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* nm, auto launch, double flops_per_thread_iter) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    double ops = flops_per_thread_iter * ITER * (double)blocks * threads;
    double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / p.multiProcessorCount;
    printf("%-28s %8.3f ms  %8.1f lane-ops/clk/SM (at the %d MHz nominal clock)\n", nm, ms, per_clk_sm, clk / 1000);
  };
  run("FFMA (shared b,c)", [&] { k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 8);
  run("FFMA (3 distinct regs)", [&] { k_ffma_rr<<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 8);
  run("FFMA2 (packed b,c)", [&] { k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 16);
  run("FFMA2 (broadcast b,c)", [&] { k_ffma2_bc<<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 16);
  run("MUFU.EX2 (+FMUL)", [&] { k_ex2<<<blocks, threads>>>(out, 0.5f); }, 4);
  printf("SMs %d\n", p.multiProcessorCount);
  return 0;
}
