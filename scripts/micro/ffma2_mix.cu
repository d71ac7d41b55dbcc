// Does FFMA2 free issue slots in mixed code?  A: 8 FFMA + 8 ALU (LOP3/IADD) per iteration;
// B: 4 FFMA2 (the same 8 FMAs per lane) + the same 8 ALU; C: 8 ALU only; D: 8 FFMA only; E: 4 FFMA2 only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t pk(float a, float b){ uint64_t r; asm volatile("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(uint64_t r){ float a,b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a+b; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c){ uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint32_t alu(uint32_t x, uint32_t y){ uint32_t d; asm volatile("{\n\t.reg .u32 t;\n\tshr.u32 t, %1, 1;\n\tadd.u32 %0, t, %2;\n\t}" : "=r"(d) : "r"(x), "r"(y)); return d; }
constexpr int ITER = 4096;
template <int MODE>
__global__ void k(float* out, float s, float t) {
  float a[8]; uint64_t p[4]; uint32_t u[8];
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x + j; u[j] = threadIdx.x * (j + 1); }
  for (int j = 0; j < 4; ++j) p[j] = pk(threadIdx.x + j, j);
  const uint64_t b = pk(s, s), c = pk(t, t);
  const uint32_t y = (uint32_t)(s * 1000);
  for (int i = 0; i < ITER; ++i) {
    if (MODE == 0 || MODE == 3) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], s, t);
    }
    if (MODE == 1 || MODE == 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) p[j] = fma2(p[j], b, c);
    }
    if (MODE <= 2) {
#pragma unroll
      for (int j = 0; j < 8; ++j) u[j] = alu(u[j], u[(j + 3) & 7]);
    }
  }
  float r = 0; for (int j = 0; j < 8; ++j) r += a[j] + (float)u[j];
  for (int j = 0; j < 4; ++j) r += lo(p[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int blocks = p.multiProcessorCount * 4, threads = 512;
  float* out; cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* nm, auto launch, double winst_per_iter) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    double wi = winst_per_iter * ITER * (double)blocks * threads / 32;
    printf("%-34s %8.3f ms  %6.2f warp-inst/clk/SMSP at 1965 MHz\n", nm, ms, wi / (ms * 1e-3) / 1965e6 / (p.multiProcessorCount * 4));
  };
  run("A: 8 FFMA + 8 ALU (LEA.HI)", [&] { k<0><<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 16);
  run("B: 4 FFMA2 + 8 ALU", [&] { k<1><<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 12);
  run("C: 8 ALU", [&] { k<2><<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 8);
  run("D: 8 FFMA", [&] { k<3><<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 8);
  run("E: 4 FFMA2", [&] { k<4><<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 4);
  return 0;
}
