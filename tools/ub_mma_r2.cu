// Microbenchmark (diagnostics, round 2): tcgen05.mma cycles per instruction vs N, with the issue loop
// separated from the tensor-pipe time (clock after the last issue vs after the commit lands).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ub_mma_r2 tools/ub_mma_r2.cu
// Variants: descriptors precomputed in registers (no per-MMA descriptor arithmetic), one issuing thread,
// 64 MMAs per commit, 1 CTA or 148 CTAs, SS (A, B in smem) and TS (A in TMEM), optional cta_group::2 pairs.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../paper_2604_06370_b200/csrc/sm100.cuh"
using namespace fkv::sm100;

template <int N, int MODE>  // MODE 0: SS, A advances over 8 K-steps; 1: SS same A/B every MMA; 2: TS; 3: SS M=64
__global__ void __launch_bounds__(128, 1) run(int n_iter, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int wid = threadIdx.x >> 5;
  if (wid == 0) tmem_alloc(smem_u32(&tbase), 512);
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  for (int i = threadIdx.x; i < 128 * 1024 / 16; i += blockDim.x)
    ((uint4*)smem)[i] = make_uint4(0x3f803f80u ^ (i * 2654435761u & 0x00ff00ffu), 0x3f003f00u, 0xbf803f80u, i);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase, sb = smem_u32(smem);
  long long t0 = 0, t1 = 0, t2 = 0;
  if (threadIdx.x == 32) {
    const uint32_t id = idesc_bf16(MODE == 3 ? 64 : 128, N, false, false);
    uint64_t da[8], db[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int ss = MODE == 1 ? 0 : s;
      da[s] = make_desc(sb + (ss >> 2) * 16384 + (ss & 3) * 32, 16, 1024, SWZ_128);
      db[s] = make_desc(sb + 65536 + (ss >> 2) * 32768 + (ss & 3) * 32, 16, 1024, SWZ_128);
    }
    t0 = clock64();
    for (int i = 0; i < n_iter; ++i) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (MODE == 2)
          mma_ts(tm, tm + 256 + 8 * (s & 3), db[s], id, 1u);
        else if (MODE == 4)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tm),
                       "l"(da[s]), "l"(db[s]), "r"(id), "r"(1u), "r"(0xffff0000u), "r"(~0u), "r"(~0u), "r"(~0u));
        else
          mma_ss(tm, da[s], db[s], id, 1u);
      }
    }
    t1 = clock64();
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tm, 512);
}

template <int N, int MODE>
void go(int grid, const char* name) {
  long long* d;
  cudaMalloc(&d, 296 * 16);
  cudaFuncSetAttribute(run<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int n_iter = 256;  // 2048 MMAs
  run<N, MODE><<<grid, 128, 128 * 1024>>>(n_iter, d);  // warm
  cudaDeviceSynchronize();
  run<N, MODE><<<grid, 128, 128 * 1024>>>(n_iter, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, grid * 16, cudaMemcpyDeviceToHost);
  double iss = 0, tot = 0;
  for (int i = 0; i < grid; ++i) iss += h[2 * i], tot += h[2 * i + 1];
  iss /= grid; tot /= grid;
  const int M = MODE == 3 ? 64 : 128;
  printf("%-28s grid=%3d M=%3d N=%3d: issue %.1f cyc/MMA, total %.1f cyc/MMA (guide floor %d) %s\n", name, grid, M, N,
         iss / (n_iter * 8), tot / (n_iter * 8), 128 * N / 256, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int grid : {148}) {
    go<16, 0>(grid, "SS advancing");
    go<32, 0>(grid, "SS advancing");
    go<64, 0>(grid, "SS advancing");
    go<128, 0>(grid, "SS advancing");
    go<256, 0>(grid, "SS advancing");
    go<64, 1>(grid, "SS same operands");
    go<128, 1>(grid, "SS same operands");
    go<256, 1>(grid, "SS same operands");
    go<16, 2>(grid, "TS");
    go<64, 2>(grid, "TS");
    go<128, 2>(grid, "TS");
    go<256, 2>(grid, "TS");
    go<16, 4>(grid, "SS lane-masked");
    go<128, 4>(grid, "SS lane-masked");
    go<256, 4>(grid, "SS lane-masked");
  }
  return 0;
}
