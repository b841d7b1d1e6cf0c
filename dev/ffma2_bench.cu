// Throughput of FFMA vs FFMA2 (fma.rn.f32x2) vs MUFU.TANH per SM (dev microbench).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8]; unsigned long long p[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i; float2 f = make_float2(a[i], a[i] + 1); p[i] = *reinterpret_cast<unsigned long long*>(&f); }
  const float b = 0.999f, c = 1e-4f;
  float2 bb = make_float2(b, b), cc = make_float2(c, c);
  unsigned long long b2 = *reinterpret_cast<unsigned long long*>(&bb), c2 = *reinterpret_cast<unsigned long long*>(&cc);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fmaf(a[i], a[i] * 0.f + b, c);
      if (MODE == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(b2), "l"(c2));
      if (MODE == 2) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 3) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) { float2 f = *reinterpret_cast<float2*>(&p[i]); s += a[i] + f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(const char* name, float* d, int ops_per_inst) {
  int iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<148 * 4, 512>>>(d, iters);
  cudaEventRecord(e0);
  k<MODE><<<148 * 4, 512>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warp_insts = 148.0 * 4 * 16 * iters * 8;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-8s %.3f ms  warp-inst/cycle/SM = %.2f  (lane-ops/cycle/SM = %.1f)\n", name, ms,
         warp_insts / 148 / cycles, warp_insts / 148 / cycles * 32 * ops_per_inst);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 4 * 512 * 4);
  run<0>("ffma", d, 1); run<1>("ffma2", d, 2); run<2>("tanh", d, 1); run<3>("ex2", d, 1);
  return 0;
}
