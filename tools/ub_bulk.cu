// Microbenchmark (diagnostics, round 2): 1D bulk-copy (cp.async.bulk, TMA engine) streaming into shared memory.
// 148 CTAs, one producer warp issuing `chunk`-byte copies into a ring of `ring` bytes (mbarrier complete_tx),
// one consumer warp releasing slots. `share` CTAs read identical addresses (L2 reuse), else distinct (HBM stream).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ub_bulk tools/ub_bulk.cu
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
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void wait_any(int mode, uint32_t bar, uint32_t parity) {
  if (mode) wait_spin(bar, parity); else mbar_wait(bar, parity);
}
__global__ void __launch_bounds__(64, 1) run(const uint8_t* src, size_t src_bytes, int chunk, int nslots, int per_op,
                                             int n_chunks, int share, int spin) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[64], empty[64];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nslots; ++i) { mbar_init(smem_u32(&full[i]), 1); mbar_init(smem_u32(&empty[i]), 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int grp = blockIdx.x / share;
  const size_t per_cta = (size_t)n_chunks * chunk;
  const uint8_t* base = src + ((size_t)grp * per_cta) % (src_bytes - per_cta);
  if (wid == 0 && lane == 0) {
    for (int i = 0; i < n_chunks; ++i) {
      const int s = i % nslots, ph = (i / nslots) & 1;
      if (i >= nslots) wait_any(spin, smem_u32(&empty[s]), ph ^ 1);
      mbar_expect_tx(smem_u32(&full[s]), chunk);
      for (int o = 0; o < chunk; o += per_op)
        bulk_g2s(smem_u32(smem + (size_t)s * chunk + o), base + (size_t)i * chunk + o, per_op, smem_u32(&full[s]));
    }
  } else if (wid == 1 && lane == 0) {
    for (int i = 0; i < n_chunks; ++i) {
      const int s = i % nslots, ph = (i / nslots) & 1;
      wait_any(spin, smem_u32(&full[s]), ph);
      mbar_arrive(smem_u32(&empty[s]));
    }
  }
}

int main() {
  const size_t bytes = (size_t)4 << 30;
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct V { int chunk, ring_kb, per_op, share, spin; };
  const V vs[] = {{4096, 128, 4096, 1, 0},   {4096, 128, 4096, 1, 1},   {16384, 128, 16384, 1, 1},
                  {32768, 128, 32768, 1, 1}, {32768, 192, 32768, 1, 1}, {32768, 128, 4096, 1, 1},
                  {4096, 64, 4096, 1, 1},    {4096, 128, 4096, 2, 1},   {4096, 128, 4096, 8, 1},
                  {4096, 192, 4096, 16, 1},  {32768, 128, 32768, 2, 1}, {32768, 128, 32768, 8, 1},
                  {32768, 192, 32768, 16, 1}, {16384, 192, 16384, 16, 1}, {16384, 192, 16384, 1, 1}};
  for (const V& v : vs) {
    const int nslots = v.ring_kb * 1024 / v.chunk;
    const int n_chunks = (int)((64ll << 20) / v.chunk);  // 64 MiB per CTA
    run<<<148, 64, v.ring_kb * 1024>>>(src, bytes, v.chunk, nslots, v.per_op, 64, v.share, v.spin);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    run<<<148, 64, v.ring_kb * 1024>>>(src, bytes, v.chunk, nslots, v.per_op, n_chunks, v.share, v.spin);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tb = 148.0 * n_chunks * v.chunk / (ms * 1e-3) / 1e12;
    printf("spin %d chunk %6d B ring %3d KB op %6d B share %2d: %.2f TB/s delivered to SMs (%.2f TB/s unique) %s\n", v.spin, v.chunk,
           v.ring_kb, v.per_op, v.share, tb, tb / v.share, cudaGetErrorString(err));
  }
  return 0;
}
