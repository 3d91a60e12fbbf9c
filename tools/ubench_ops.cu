// Microbenchmark (diagnostics): full-chip TMA throughput vs op size / box shape, >= 128 KB in flight per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_ops tools/ubench_ops.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../paper_2604_06370_b200/csrc/sm100.cuh"
#include "../paper_2604_06370_b200/csrc/tma_host.hpp"
using namespace fkv::sm100;
struct Maps { CUtensorMap m; };
// kind 0: 2D box; 1: 3D box; 2: 1D bulk of `bytes`; 3: cp.async 16B by 32 lanes (bytes per op)
__global__ void run(const __grid_constant__ Maps mp, const uint8_t* base, int64_t rows, int kind, int bytes, int box_rows,
                    int ops_per_stage, int stages, int iters) {
  const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[8];
  const int stage_bytes = ops_per_stage * bytes;
  if (threadIdx.x == 0) { for (int i = 0; i < stages; ++i) mbar_init(smem_u32(&full[i]), kind == 3 ? blockDim.x : 1); fence_mbar_init(); }
  __syncthreads();
  if (kind != 3 && threadIdx.x != 0) return;
  for (int i = 0; i < iters + stages; ++i) {
    if (i >= stages) mbar_wait(smem_u32(&full[i % stages]), ((i / stages) - 1) & 1);
    if (i >= iters) continue;
    const int s = i % stages;
    const uint32_t bar = smem_u32(&full[s]);
    if (kind != 3) mbar_expect_tx(bar, stage_bytes);
    for (int o = 0; o < ops_per_stage; ++o) {
      const int64_t r = (((int64_t)blockIdx.x * 7919 + (int64_t)i * 37 + o * 101) * box_rows) % rows;
      const uint32_t dst = smem_u32(smem) + s * stage_bytes + o * bytes;
      if (kind == 0) tma_load_2d(dst, &mp.m, 0, (int)r, bar);
      else if (kind == 1) tma_load_3d(dst, &mp.m, 0, (int)r, 0, bar);
      else if (kind == 2) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst), "l"(base + r * 256), "r"(bytes), "r"(bar) : "memory");
      else {
        for (int c = wid * 32 + lane; c < bytes / 16; c += 32 * nw)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + c * 16), "l"(base + r * 256 + c * 16) : "memory");
      }
    }
    if (kind == 3) asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
  }
}
int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  const int nsm = prop.multiProcessorCount;
  const size_t big = (size_t)2 << 30;
  void* buf; cudaMalloc(&buf, big); cudaMemset(buf, 0, big);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const uint64_t rows_big = big / 256;
  struct C { const char* name; int kind, bytes, box_rows, box_cols; } cs[] = {
      {"3D {64,128,2} 32KB", 1, 32768, 128, 64}, {"3D {64,64,2} 16KB", 1, 16384, 64, 64},
      {"2D {64,128} 16KB", 0, 16384, 128, 64}, {"2D {64,64} 8KB", 0, 8192, 64, 64},
      {"2D {16,128} 4KB (32B rows)", 0, 4096, 128, 16}, {"2D {64,32} 4KB", 0, 4096, 32, 64},
      {"1D bulk 32KB", 2, 32768, 128, 0}, {"1D bulk 16KB", 2, 16384, 64, 0}, {"1D bulk 4KB", 2, 4096, 16, 0},
      {"cp.async 4KB", 3, 4096, 16, 0}, {"cp.async 32KB", 3, 32768, 128, 0}};
  for (int foot = 0; foot < 2; ++foot)
  for (int nwarps : {1, 2, 4})
  for (auto c : cs) {
    if (c.kind != 3 && nwarps > 1) continue;
    const uint64_t rows = foot ? rows_big : (32ull << 20) / 256;  // 32 MB: L2-resident
    Maps mp;
    if (c.kind == 1) mp.m = fkv::make_tmap_3d_bf16_halves(buf, rows, c.box_rows);
    else if (c.kind == 0) mp.m = fkv::make_tmap_2d_bf16(buf, rows, 128, 256, c.box_cols, c.box_rows, c.box_cols == 64 ? 128 : 32);
    for (int inflight_kb : {96, 192}) {
      const int stages = 3;
      int ops = inflight_kb * 1024 / stages / c.bytes; if (ops < 1) ops = 1;
      const int iters = 150;
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        run<<<nsm, 32 * nwarps, stages * ops * c.bytes>>>(mp, (const uint8_t*)buf, rows - 256, c.kind, c.bytes, c.box_rows, ops, stages, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
      }
      const double bytes = (double)nsm * iters * ops * c.bytes;
      printf("%s w%d %-28s ring %3d KB (%2d ops/stage): %6.0f GB/s  %6.1f ns/op/SM  %s\n", foot ? "HBM" : "L2 ", nwarps, c.name, stages * ops * c.bytes / 1024, ops,
             bytes / best / 1e6, best * 1e6 / (iters * ops), cudaGetErrorString(cudaGetLastError()));
    }
  }
}
