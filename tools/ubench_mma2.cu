// Microbenchmark (diagnostics): is the ~120-cycle cost of a tcgen05.mma (N <= 128) per issuing warp or per SM?
// W warps issue n MMAs each (M = 128, K = 16, SS, N given) into their own accumulators; per-SM cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma2 tools/ubench_mma2.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../paper_2604_06370_b200/csrc/sm100.cuh"
using namespace fkv::sm100;
__global__ void run(int n, int N, int W, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bars[4];
  const int wid = threadIdx.x >> 5;
  if (wid == 0) tmem_alloc(smem_u32(&tbase), 512);
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bars[i]), 1); fence_mbar_init(); }
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) ((uint4*)smem)[i] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase, sb = smem_u32(smem);
  long long t0 = clock64();
  if (wid >= 1 && wid <= W) {
    const uint32_t id = idesc_bf16(128, N, false, false);
    const uint64_t da = make_desc(sb, 16, 1024, SWZ_128), db = make_desc(sb + 65536, 16, 1024, SWZ_128);
    const uint32_t dcol = tm + (uint32_t)((wid - 1) * 128);
    for (int i = 0; i < n; i += 8) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const uint64_t a = da + (uint64_t)((((s >> 2) * 16384 + (s & 3) * 32)) >> 4);
        const uint64_t b = db + (uint64_t)((((s >> 2) * 8192 + (s & 3) * 32)) >> 4);
        asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dcol), "l"(a), "l"(b),
                     "r"(id), "r"((uint32_t)(i + s > 0)));
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&bars[wid - 1])) : "memory");
    mbar_wait(smem_u32(&bars[wid - 1]), 0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (wid == 0) tmem_dealloc(tm, 512);
}
int main() {
  long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int W : {1, 2, 3})
    for (int N : {64, 128}) {
      const int n = 2048;
      run<<<148, 160, 96 * 1024>>>(n, N, W, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      printf("W=%d issuing warps N=%3d: %.1f cycles per MMA per SM (%s)\n", W, N, avg / (n * W), cudaGetErrorString(e));
    }
}
