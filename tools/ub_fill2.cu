// Microbenchmark (diagnostics, round 2): is the issue cost of cp.async.bulk per thread or per warp? One warp per
// SM; K lanes each issue a 4-KB bulk copy per round (one mbarrier per round, D rounds in flight), L2-resident.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ub_fill2 tools/ub_fill2.cu && tools/ub_fill2
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../paper_2604_06370_b200/csrc/sm100.cuh"
using namespace fkv::sm100;
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__global__ void __launch_bounds__(32, 1) run(const uint8_t* g, int K, int D, int W, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[8];
  const int lane = threadIdx.x;
  if (lane < 8) mbar_init(smem_u32(&bar[lane]), 1);
  fence_mbar_init();
  __syncwarp();
  const uint8_t* src = g + (size_t)blockIdx.x * (256 << 10);
  uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int s = it % D;
    const uint32_t b = smem_u32(&bar[s]);
    if (it >= D) { mbar_wait(b, ph[s]); ph[s] ^= 1; }
    if (lane == 0) mbar_expect_tx(b, (uint32_t)K * W);
    __syncwarp();
    if (lane < K) bulk_g2s(smem_u32(smem) + (uint32_t)(s * K + lane) * W, src + ((it * K + lane) % 64) * W, W, b);
    __syncwarp();
  }
  for (int s = 0; s < D; ++s) mbar_wait(smem_u32(&bar[s]), ph[s]);
  if (lane == 0) { out[2 * blockIdx.x] = clock64() - t0; out[2 * blockIdx.x + 1] = (long long)iters * K * W; }
}
int main() {
  uint8_t* g; cudaMalloc(&g, 148u << 18); cudaMemset(g, 1, 148u << 18);
  long long* d; cudaMalloc(&d, 148 * 16);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int W : {4096, 2048}) for (int D : {1, 2, 4}) for (int K : {1, 2, 4, 8, 16}) {
    if ((size_t)D * K * W > 196 * 1024) continue;
    const int iters = 2000 / K + 8;
    run<<<148, 32, 200 * 1024>>>(g, K, D, W, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[296]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0, by = 0; for (int i = 0; i < 148; ++i) cyc += h[2 * i], by += h[2 * i + 1];
    printf("W %5d B D %d lanes %2d: %6.1f B/clk/SM, %6.0f cycles per op-round, %5.0f cycles per op %s\n", W, D, K,
           by / cyc, cyc / 148 / iters, cyc / 148 / iters / K * D, cudaGetErrorString(e));
  }
  return 0;
}
