// Microbenchmark (diagnostics, round 2): can 4-KB shared-memory fills (residual pages) reach the SM's L2 ingest
// rate?  32-KB slots, each filled by 8 x 4 KB pieces: one lane issuing 8 bulk copies, 8 lanes issuing one each,
// 2 producer warps, or LDGSTS (cp.async 16 B by a whole warp, cp.async.mbarrier.arrive.noinc).
// `share` CTAs read identical addresses (L2 hits after the first reader).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ub_bulk3 tools/ub_bulk3.cu
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

// mode 0: lane 0 issues 8 ops per slot; 1: lanes 0..7 one op each; 2: warps 0,1 alternate slots (lane 0 each);
// 3: LDGSTS by warp 0 (16 B per lane per op); 4: two LDGSTS warps alternate slots
__global__ void __launch_bounds__(128, 1) run(const uint8_t* src, size_t src_bytes, int nslots, int n_chunks,
                                              int share, int mode, int page_stride) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[64], empty[64];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunk = 32768;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nslots; ++i) {
      mbar_init(smem_u32(&full[i]), mode >= 3 ? 32 : 1);
      mbar_init(smem_u32(&empty[i]), 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int grp = blockIdx.x / share;
  // pages of a slot are scattered: page k of chunk i at (i * 8 + k) * page_stride
  const size_t span = (size_t)n_chunks * 8 * page_stride;
  const uint8_t* base = src + ((size_t)grp * 1315423911ull * 4096) % (src_bytes - span);
  const int n_prod = (mode == 2 || mode == 4) ? 2 : 1;
  if (wid < n_prod) {
    for (int i = wid; i < n_chunks; i += n_prod) {
      const int s = i % nslots, ph = (i / nslots) & 1;
      if (i >= nslots) wait_spin(smem_u32(&empty[s]), ph ^ 1);
      if (mode <= 2) {
        if (lane == 0) mbar_expect_tx(smem_u32(&full[s]), chunk);
        __syncwarp();
        if (mode == 1) {
          if (lane < 8)
            bulk_g2s(smem_u32(smem + (size_t)s * chunk + lane * 4096), base + ((size_t)i * 8 + lane) * page_stride, 4096,
                     smem_u32(&full[s]));
        } else if (lane == 0) {
          for (int k = 0; k < 8; ++k)
            bulk_g2s(smem_u32(smem + (size_t)s * chunk + k * 4096), base + ((size_t)i * 8 + k) * page_stride, 4096,
                     smem_u32(&full[s]));
        }
      } else {
        for (int k = 0; k < 8; ++k) {
          const uint8_t* g = base + ((size_t)i * 8 + k) * page_stride;
          const uint32_t d = smem_u32(smem + (size_t)s * chunk + k * 4096);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d + (c * 32 + lane) * 16),
                         "l"(g + (c * 32 + lane) * 16)
                         : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&full[s])) : "memory");
      }
    }
  } else if (wid == 3 && lane == 0) {
    for (int i = 0; i < n_chunks; ++i) {
      const int s = i % nslots, ph = (i / nslots) & 1;
      wait_spin(smem_u32(&full[s]), ph);
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
  const char* names[] = {"1 lane x 8 bulk", "8 lanes x 1 bulk", "2 warps x 8 bulk", "LDGSTS 1 warp", "LDGSTS 2 warps"};
  for (int share : {1, 8})
    for (int stride : {4096, 65536})
      for (int mode = 0; mode < 5; ++mode) {
        const int nslots = 4;  // 128 KB ring
        const int n_chunks = 2048;
        run<<<148, 128, nslots * 32768>>>(src, bytes, nslots, 64, share, mode, stride);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        run<<<148, 128, nslots * 32768>>>(src, bytes, nslots, n_chunks, share, mode, stride);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double tb = 148.0 * n_chunks * 32768 / (ms * 1e-3) / 1e12;
        printf("%-18s share %d page stride %6d: %.2f TB/s delivered (%.1f B/clk/SM at 1.965 GHz) %s\n", names[mode],
               share, stride, tb, tb * 1e12 / 148 / 1.965e9, cudaGetErrorString(err));
      }
  return 0;
}
