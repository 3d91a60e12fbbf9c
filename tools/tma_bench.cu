// Microbenchmark (diagnostics, not part of the library): per-SM throughput of
// TMA 2D boxes vs 1D bulk copies of the sizes used by the tcgen05 kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench tools/tma_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#include "../paper_2604_06370_b200/csrc/sm100.cuh"
#include "../paper_2604_06370_b200/csrc/tma_host.hpp"

using namespace fkv::sm100;

__device__ __forceinline__ void bulk_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// mode 0: 2D TMA box {bc cols, br rows} (bf16); mode 1: 1D bulk of `bytes`
__global__ void bench(const __grid_constant__ CUtensorMap map, const uint8_t* base, int mode, int bc, int br,
                      int bytes, int iters, int64_t rows_total, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[4];
  const int stages = 4;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long t0 = clock64();
  const int64_t per_op_rows = br;
  int64_t row = (int64_t)blockIdx.x * 4099 * per_op_rows;
  for (int i = 0; i < iters; ++i) {
    const int s = i % stages;
    if (i >= stages) mbar_wait(smem_u32(&bars[s]), ((i / stages) - 1) & 1);
    const uint32_t dst = smem_u32(smem) + s * 32768;
    mbar_expect_tx(smem_u32(&bars[s]), mode == 0 ? bc * br * 2 : bytes);
    row = (row + per_op_rows * 7) % (rows_total - per_op_rows);
    if (mode == 0)
      tma_load_2d(dst, &map, 0, (int)row, smem_u32(&bars[s]));
    else
      bulk_1d(dst, base + ((int64_t)row * 256 % ((int64_t)rows_total * 256 - bytes)) / 1024 * 1024, bytes,
              smem_u32(&bars[s]));
  }
  for (int i = iters - stages; i < iters; ++i) mbar_wait(smem_u32(&bars[i % stages]), (i / stages) & 1);
  out[blockIdx.x] = clock64() - t0;
}

int main() {
  const int64_t rows = 1 << 22;  // 4M rows x 256 B = 1 GiB
  uint8_t* buf;
  cudaMalloc(&buf, rows * 256);
  cudaMemset(buf, 1, rows * 256);
  long long* out;
  cudaMalloc(&out, 148 * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 1024);
  struct Cfg { int mode, bc, br, sw, bytes; const char* name; };
  std::vector<Cfg> cfgs = {{0, 64, 64, 128, 0, "2D 64x64 SW128 (8KB)"},   {0, 64, 128, 128, 0, "2D 64x128 SW128 (16KB)"},
                           {0, 16, 64, 32, 0, "2D 16x64 SW32 (2KB)"},     {0, 16, 128, 32, 0, "2D 16x128 SW32 (4KB)"},
                           {1, 0, 8, 0, 2048, "1D 2KB"},                  {1, 0, 32, 0, 8192, "1D 8KB"},
                           {1, 0, 64, 0, 16384, "1D 16KB"},               {1, 0, 128, 0, 32768, "1D 32KB"}};
  for (auto& c : cfgs) {
    CUtensorMap m;
    if (c.mode == 0) {
      const int cols = c.sw == 128 ? 128 : 16;
      m = fkv::make_tmap_2d_bf16(buf, c.sw == 128 ? rows : rows * 8, cols, cols * 2, c.bc, c.br, c.sw);
    } else {
      m = fkv::make_tmap_2d_bf16(buf, rows, 128, 256, 64, 64, 128);
    }
    const int iters = 2000;
    const int rows_total = (int)(c.mode == 0 && c.sw == 32 ? (rows * 8 > 2000000000 ? 2000000000 : rows * 8) : rows);
    bench<<<148, 32, 4 * 32768 + 1024>>>(m, buf, c.mode, c.bc, c.br, c.bytes, iters, rows_total, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<<<148, 32, 4 * 32768 + 1024>>>(m, buf, c.mode, c.bc, c.br, c.bytes, iters, rows_total, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> h(148);
    cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (auto v : h) mx = v > mx ? v : mx;
    const double op_bytes = c.mode == 0 ? c.bc * c.br * 2.0 : c.bytes;
    printf("%-26s %7.1f us  %6.1f cyc/op  %6.1f B/cyc/SM  %7.2f TB/s chip  (err %s)\n", c.name, ms * 1e3,
           (double)mx / iters, op_bytes * iters / mx, op_bytes * iters * 148 / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
