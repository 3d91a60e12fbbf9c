// Microbenchmark (diagnostics, round 2): costs seen by one issuing thread on B200.
//   (a) mbarrier try_wait on an already-completed phase, (b) arrive.expect_tx, (c) issue of one 4-KB bulk copy,
//   (d) latency of one 4-KB bulk copy (L2 hit), (e) ld.global L2-hit latency, (f) 1D bulk ops: 1..32 in flight
//   per thread, one barrier per op vs one per 8 ops. One CTA (unloaded) and 148 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ub_lat tools/ub_lat.cu
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

__global__ void __launch_bounds__(128, 1) run(const uint8_t* src, int inflight, int per_bar, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[64];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 64; ++i) mbar_init(smem_u32(&bar[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long r[8];
  const uint32_t b0 = smem_u32(&bar[63]);
  // (b) arrive.expect_tx (0 bytes -> completes phase 0 of bar 63)
  long long t = clock64();
  mbar_expect_tx(b0, 0);
  r[1] = clock64() - t;
  // (a) try_wait on the completed phase
  t = clock64();
  wait_spin(b0, 0);
  r[0] = clock64() - t;
  // (c)+(d) one 4-KB bulk copy: issue cost and completion latency
  const uint32_t b1 = smem_u32(&bar[62]);
  mbar_expect_tx(b1, 4096);
  t = clock64();
  bulk_g2s(smem_u32(smem), src + 4096 * blockIdx.x % (1 << 20), 4096, b1);
  r[2] = clock64() - t;
  wait_spin(b1, 0);
  r[3] = clock64() - t;
  // (e) ld.global latency (L2 hit: the line was just copied by the bulk op)
  t = clock64();
  const uint32_t v = *(volatile const uint32_t*)(src + 4096 * blockIdx.x % (1 << 20) + 64);
  r[4] = clock64() - t + (v == 12345);
  // (f) stream 256 x 4 KB ops, `inflight` ring slots, per_bar ops per barrier
  const int n = 256;
  const int slots = inflight / per_bar;
  t = clock64();
  for (int i = 0; i < n; i += per_bar) {
    const int k = (i / per_bar) % slots, round = (i / per_bar) / slots;
    if (round > 0) wait_spin(smem_u32(&bar[k]), (round - 1) & 1);
    mbar_expect_tx(smem_u32(&bar[k]), 4096 * per_bar);
    for (int j = 0; j < per_bar; ++j)
      bulk_g2s(smem_u32(smem) + ((i + j) % inflight) * 4096, src + ((size_t)(i + j) * 4096 + blockIdx.x * 65536) % (8 << 20),
               4096, smem_u32(&bar[k]));
  }
  for (int k = 0; k < slots; ++k) {
    const int last = (n / per_bar) - slots + k;
    wait_spin(smem_u32(&bar[last % slots]), (last / slots) & 1);
  }
  r[5] = (clock64() - t) / n;
  for (int i = 0; i < 6; ++i) out[blockIdx.x * 8 + i] = r[i];
}

int main() {
  uint8_t* src;
  cudaMalloc(&src, 8 << 20);
  cudaMemset(src, 1, 8 << 20);
  long long* d;
  cudaMalloc(&d, 148 * 8 * 8);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int grid : {1, 148})
    for (int inflight : {1, 4, 8, 16, 32})
      for (int per_bar : {1, 8}) {
        if (per_bar > inflight) continue;
        run<<<grid, 128, 160 * 1024>>>(src, inflight, per_bar, d);
        cudaDeviceSynchronize();
        run<<<grid, 128, 160 * 1024>>>(src, inflight, per_bar, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148 * 8];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double a[6] = {0, 0, 0, 0, 0, 0};
        for (int b = 0; b < grid; ++b)
          for (int i = 0; i < 6; ++i) a[i] += h[b * 8 + i];
        for (int i = 0; i < 6; ++i) a[i] /= grid;
        printf("grid %3d inflight %2d ops/barrier %d: try_wait(done) %.0f, expect_tx %.0f, bulk issue %.0f, bulk 4KB "
               "latency %.0f, ld L2 latency %.0f | stream: %.0f cycles per 4-KB op (%.1f B/clk) %s\n",
               grid, inflight, per_bar, a[0], a[1], a[2], a[3], a[4], a[5], 4096.0 / a[5], cudaGetErrorString(e));
      }
  return 0;
}
