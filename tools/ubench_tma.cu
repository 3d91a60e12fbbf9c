// Microbenchmark (diagnostics): full-chip TMA tensor-box streaming in the shape the decode kernel uses.
// Per tile: one 3D box {64,128,2} bf16 (32 KB, SW128) from "K", one from "V", and n_res 2D boxes {16,128} (4 KB, SW32).
// stages-deep ring, consumer frees a stage as soon as it lands (no compute). footprint selects L2-resident vs HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tma tools/ubench_tma.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../paper_2604_06370_b200/csrc/sm100.cuh"
#include "../paper_2604_06370_b200/csrc/tma_host.hpp"
using namespace fkv::sm100;
struct Maps { CUtensorMap kb, vb, rr; };
__global__ void stream(const __grid_constant__ Maps m, int64_t rows_b, int64_t rows_r, int tiles, int stages, int n_res,
                       int same, int kv, const void* rrbase) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[8];
  const int stage_bytes = (kv ? 65536 : 0) + n_res * 4096;
  if (threadIdx.x == 0) { for (int i = 0; i < stages; ++i) mbar_init(smem_u32(&full[i]), 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int grp = same > 0 ? blockIdx.x / same : blockIdx.x;
  for (int i = 0; i < tiles + stages; ++i) {
    if (i >= stages) mbar_wait(smem_u32(&full[i % stages]), ((i / stages) - 1) & 1);
    if (i >= tiles) continue;
    const int s = i % stages;
    const uint32_t bar = smem_u32(&full[s]);
    const uint32_t dst = smem_u32(smem) + s * stage_bytes - (kv ? 0 : 65536);
    const int64_t tb = (((int64_t)grp * 7919 + (int64_t)i * 37) * 128) % rows_b;
    mbar_expect_tx(bar, (kv ? 65536 : 0) + n_res * 4096);
    if (kv) {
      tma_load_3d(dst, &m.kb, 0, (int)tb, 0, bar);
      tma_load_3d(dst + 32768, &m.vb, 0, (int)tb, 0, bar);
    }
    for (int r = 0; r < n_res; ++r) {
      const int64_t tr = (((int64_t)blockIdx.x * 104729 + (int64_t)i * 53 + r * 977) * 128) % rows_r;
      if (same < 0) {
        const void* src = (const uint8_t*)rrbase + tr * 32;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst + 65536 + r * 4096), "l"(src), "r"(4096), "r"(bar) : "memory");
      } else {
        tma_load_2d(dst + 65536 + r * 4096, &m.rr, 0, (int)tr, bar);
      }
    }
  }
}

__device__ __forceinline__ uint32_t cl_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t mapa_(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void cl_sync() { asm volatile("barrier.cluster.arrive.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tma3_mc(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar, uint16_t mask) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3, %4}], [%5], %6;\n"
               :: "r"(dst), "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "h"(mask) : "memory");
}
// K/V boxes of 128 keys split in csz row-slices, slice k loaded by rank k and multicast to the cluster
__global__ void stream_mc(const __grid_constant__ Maps m, int64_t rows_b, int tiles, int stages, int csz) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  const uint32_t rank = cl_rank();
  if (threadIdx.x == 0) { for (int i = 0; i < stages; ++i) { mbar_init(smem_u32(&full[i]), 1); mbar_init(smem_u32(&empty[i]), csz); } fence_mbar_init(); }
  cl_sync();
  if (threadIdx.x == 0) {
    const int grp = blockIdx.x / csz;
    const int rows = 128 / csz;
    for (int i = 0; i < tiles + stages; ++i) {
      const int c = i - (stages - 1);
      if (c >= 0 && c < tiles) {   // consume tile c: wait, then release it in every rank
        mbar_wait(smem_u32(&full[c % stages]), (c / stages) & 1);
        for (int q = 0; q < csz; ++q)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" :: "r"(mapa_(smem_u32(&empty[c % stages]), q)) : "memory");
      }
      if (i >= tiles) continue;
      const int s = i % stages;
      if (i >= stages) mbar_wait(smem_u32(&empty[s]), ((i / stages) - 1) & 1);
      const uint32_t bar = smem_u32(&full[s]);
      const uint32_t dst = smem_u32(smem) + s * 65536;
      const int64_t tb = (((int64_t)grp * 7919 + (int64_t)i * 37) * 128) % rows_b;
      mbar_expect_tx(bar, 65536);
      // rank's slice: rows [rank*rows, +rows) of both halves -> smem offset rank*rows*128 within each 16 KB half
      tma3_mc(dst + rank * rows * 128, &m.kb, 0, (int)tb + rank * rows, 0, bar, (uint16_t)((1u << csz) - 1));
      tma3_mc(dst + 32768 + rank * rows * 128, &m.vb, 0, (int)tb + rank * rows, 0, bar, (uint16_t)((1u << csz) - 1));
    }
  }
  __syncwarp();
  cl_sync();
}
int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  const int nsm = prop.multiProcessorCount;
  const size_t big = (size_t)3 << 30;
  void *kb, *vb, *rr;
  cudaMalloc(&kb, big); cudaMalloc(&vb, big); cudaMalloc(&rr, (size_t)1 << 30);
  cudaMemset(kb, 0, big); cudaMemset(vb, 0, big); cudaMemset(rr, 0, (size_t)1 << 30);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int foot : {0, 1}) {
    const uint64_t rows_b = foot ? big / 256 : (16ull << 20) / 256;    // 16 MB x2 (L2) or 3 GB x2 (HBM)
    const uint64_t rows_r = foot ? ((1ull << 30) / 32) : (8ull << 20) / 32;
    Maps m;
    m.kb = fkv::make_tmap_3d_bf16_halves(kb, rows_b, 128);
    m.vb = fkv::make_tmap_3d_bf16_halves(vb, rows_b, 128);
    m.rr = fkv::make_tmap_2d_bf16(rr, rows_r, 16, 32, 16, 128, 32);
    struct C { int stages, n_res, same, kv, grid_mult; } cs[] = {
        {2, 4, 0, 1, 1}, {3, 0, 0, 1, 1}, {3, 4, 0, 1, 1}, {4, 0, 0, 1, 1}, {6, 0, 0, 1, 1}, {2, 4, 4, 1, 1},
        {3, 0, 4, 1, 1}, {6, 0, 4, 1, 1}, {6, 0, 8, 1, 1}, {4, 8, 0, 0, 1}, {4, 16, 0, 0, 1}, {2, 32, 0, 0, 1}, {3, 16, 0, 0, 1}, {3, 16, -1, 0, 1}, {2, 32, -1, 0, 1}, {2, 0, 0, 1, 2},
        {1, 8, 0, 1, 2}};
    for (auto c : cs) {
      const int stage_bytes = (c.kv ? 65536 : 0) + c.n_res * 4096;
      if (c.stages * stage_bytes > 220 * 1024 / c.grid_mult) continue;
      const int tiles = 200, grid = nsm * c.grid_mult;
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        stream<<<grid, 32, c.stages * stage_bytes>>>(m, rows_b, rows_r, tiles, c.stages, c.n_res, c.same, c.kv, rr);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
      }
      cudaError_t err = cudaGetLastError();
      const double bytes = (double)grid * tiles * ((c.kv ? 65536 : 0) + c.n_res * 4096);
      printf("%s stages %d n_res %2d same %d kv %d ctas/SM %d: %.0f GB/s delivered (%.1f us) %s\n", foot ? "HBM" : "L2 ",
             c.stages, c.n_res, c.same, c.kv, c.grid_mult, bytes / best / 1e6, best * 1e3, cudaGetErrorString(err));
    }

    for (int csz = 0; csz < 0; ++csz) {
      for (int stages : {3}) {
        CUtensorMap kb2 = fkv::make_tmap_3d_bf16_halves(kb, rows_b, 128 / csz);
        CUtensorMap vb2 = fkv::make_tmap_3d_bf16_halves(vb, rows_b, 128 / csz);
        Maps m2 = m; m2.kb = kb2; m2.vb = vb2;
        cudaFuncSetAttribute(stream_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        const int tiles = 200, grid = (nsm / csz) * csz;
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(grid); cfg.blockDim = dim3(32); cfg.dynamicSmemBytes = stages * 65536;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(e0);
          cudaLaunchKernelEx(&cfg, stream_mc, m2, (int64_t)rows_b, tiles, stages, csz);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          if (rep && ms < best) best = ms;
        }
        const double bytes = (double)grid * tiles * 65536;
        printf("%s MULTICAST csz %d stages %d: %.0f GB/s delivered, %.0f GB/s source (%.1f us) %s\n", foot ? "HBM" : "L2 ", csz, stages,
               bytes / best / 1e6, bytes / csz / best / 1e6, best * 1e3, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
}
