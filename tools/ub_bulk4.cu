// Microbenchmark (diagnostics, round 2): TMA-engine operation rate per SM. W warps (lane 0 each) issue 1D bulk
// copies of S bytes into private ring slots (one mbarrier per slot, `inflight` slots per warp) from an
// L2-resident source (every CTA reads the same 8 MiB window); reported: ops per SM per 1000 cycles and B/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ub_bulk4 tools/ub_bulk4.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../paper_2604_06370_b200/csrc/sm100.cuh"
using namespace fkv::sm100;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void wait_spin(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}

__global__ void __launch_bounds__(512, 1) run(const uint8_t* src, int W, int S, int inflight, int n_ops,
                                              long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[16][16];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int w = 0; w < 16; ++w)
      for (int i = 0; i < 16; ++i) mbar_init(smem_u32(&bar[w][i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  if (wid < W && lane == 0) {
    const uint32_t region = 196608 / W;  // bytes of smem per warp
    for (int i = 0; i < n_ops; ++i) {
      const int sl = i % inflight;
      if (i >= inflight) wait_spin(smem_u32(&bar[wid][sl]), ((i / inflight) - 1) & 1);
      mbar_expect_tx(smem_u32(&bar[wid][sl]), S);
      const uint32_t dst = smem_u32(smem) + wid * region + (sl * S) % (region - S + 1);
      bulk_g2s(dst, src + ((size_t)(wid * 7919 + i) * S) % (8u << 20), S, smem_u32(&bar[wid][sl]));
    }
    for (int i = n_ops - inflight; i < n_ops; ++i) wait_spin(smem_u32(&bar[wid][i % inflight]), (i / inflight) & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  uint8_t* src;
  cudaMalloc(&src, 16 << 20);
  cudaMemset(src, 1, 16 << 20);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
  for (int S : {2048, 4096, 16384})
    for (int W : {1, 2, 4, 8}) {
      const int inflight = 8;
      if (W * inflight * S > 196608 * 4) continue;
      const int n_ops = 512;
      run<<<148, 512, 196608>>>(src, W, S, inflight, 32, d);
      cudaDeviceSynchronize();
      run<<<148, 512, 196608>>>(src, W, S, inflight, n_ops, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      const double ops = (double)W * n_ops;
      printf("op %5d B, %d issuing warps: %.1f cycles per op per SM, %.1f B/clk/SM %s\n", S, W, avg / ops,
             ops * S / avg, cudaGetErrorString(e));
    }
  return 0;
}
