// tcgen05.mma issue/throughput microbenchmark (one CTA per SM, one issuing thread).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2509_22681_b200/csrc/ptx.cuh"
using namespace flame;
template <int N, bool TS>
__global__ void bench(int n_mma, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const bool leader = ptx::elect_one();
    const uint32_t a = ptx::smem_u32(smem), b = a + 65536;
    constexpr uint32_t idesc = ptx::make_idesc_bf16(128, N, 0, 0);
    unsigned long long t0 = clock64();
    if (leader) {
      for (int i = 0; i < n_mma; ++i) {
        const int k = i & 3;
        if (TS) ptx::mma_bf16_ts(tmem + 256, tmem + k * 8, ptx::make_desc_sw128(b + k * 32, 16, 1024), idesc, 1u);
        else ptx::mma_bf16_ss(tmem + 256, ptx::make_desc_sw128(a + k * 32, 16, 1024), ptx::make_desc_sw128(b + k * 32, 16, 1024), idesc, 1u);
      }
      ptx::mma_commit(&bar);
    }
    __syncwarp();
    unsigned long long t1 = clock64();
    ptx::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (leader && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}
template <int N, bool TS>
void run(int ctas) {
  unsigned long long* d; cudaMalloc(&d, 16); unsigned long long h[2];
  auto k = bench<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int n = 4096;
  k<<<ctas, 128, 160 * 1024>>>(n, d); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<<<ctas, 128, 160 * 1024>>>(n, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  double flops = 2.0 * 128 * N * 16 * n * ctas;
  printf("N=%3d %s ctas=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma, %.1f TFLOP/s  err=%s\n", N, TS ? "TS" : "SS", ctas,
         double(h[0]) / n, double(h[1]) / n, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<64, false>(1); run<128, false>(1); run<256, false>(1); run<64, true>(1); run<128, true>(1);
  run<64, false>(148); run<128, false>(148); run<256, false>(148); run<64, true>(148); run<256, true>(148);
  return 0;
}
