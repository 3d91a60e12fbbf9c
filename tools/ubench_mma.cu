// Microbenchmark (diagnostics): tcgen05.mma throughput per SM for the decode kernel's shapes
// (M = 128, N = 16..256, K = 16 per instruction; SS with K-major SW128 / MN-major operands; TS with A in TMEM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma tools/ubench_mma.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../paper_2604_06370_b200/csrc/sm100.cuh"
using namespace fkv::sm100;
__global__ void run(int n_mma, int N, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int wid = threadIdx.x >> 5;
  if (wid == 0) tmem_alloc(smem_u32(&tbase), 512);
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) ((uint4*)smem)[i] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase, sb = smem_u32(smem);
  long long t0 = 0, t1 = 0;
  if (mode >= 3 && wid == 1) {  // warp-wide issue with elect.sync, descriptors = base + constant
    const uint32_t id = idesc_bf16(mode == 9 ? 64 : 128, N, false, false);
    const uint64_t da = make_desc(sb, 16, 1024, SWZ_128), db = make_desc(sb + 65536, 16, 1024, SWZ_128);
    t0 = clock64();
    for (int i = 0; i < n_mma; i += 8) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const uint64_t a = da + (uint64_t)((((s >> 2) * 16384 + (s & 3) * 32)) >> 4);
        const uint64_t b = db + (uint64_t)((((s >> 2) * 8192 + (s & 3) * 32)) >> 4);
        if (mode == 3 || mode >= 5) {
          const int chains = mode == 3 ? 1 : (mode == 5 ? 2 : (mode == 6 ? 4 : (mode == 9 ? 1 : 8)));
          const uint32_t dcol = tm + (uint32_t)((s % chains) * (N > 64 ? 128 : 64));
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dcol), "l"(a), "l"(b),
                       "r"(id), "r"((uint32_t)(i + s > 0)));
        }
        else if (mode == 4)
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm),
                       "r"(tm + 256 + 8 * (s & 3)), "l"(b), "r"(id), "r"((uint32_t)(i + s > 0)));
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&bar)) : "memory");
    mbar_wait(smem_u32(&bar), 0);
    t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;

  } else if (mode < 3 && threadIdx.x == 0) {
    const uint32_t id = idesc_bf16(128, N, mode == 2, mode == 2);
    t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const uint32_t s = (i & 7);
      if (mode == 0)        // A K-major SW128 (keys x d), B K-major SW128 (rows x d): S^T = K Q^T
        mma_ss(tm, make_desc(sb + (s >> 2) * 16384 + (s & 3) * 32, 16, 1024, SWZ_128),
               make_desc(sb + 65536 + (s >> 2) * 8192 + (s & 3) * 32, 16, 1024, SWZ_128), id, i > 0);
      else if (mode == 2)   // A MN-major (V^T: d x keys), B MN-major (P^T): O^T = V^T P^T
        mma_ss(tm, make_desc(sb + s * 2048, 16384, 1024, SWZ_128), make_desc(sb + 98304 + s * 2048, 16384, 1024, SWZ_128),
               id, i > 0);
      else                  // TS: A from TMEM (cols 256..), B K-major SW128
        mma_ts(tm, tm + 256 + 8 * (s & 3), make_desc(sb + 65536 + (s >> 2) * 8192 + (s & 3) * 32, 16, 1024, SWZ_128), id,
               i > 0);
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tm, 512);
}
int main() {
  long long* d; cudaMalloc(&d, 296 * 8);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const char* names[10] = {"SS K-major/K-major (S^T = K Q^T)", "TS (A in TMEM)", "SS MN-major/MN-major (O^T = V^T P^T)",
                          "warp-issued SS, 1 chain", "warp-issued TS", "warp-issued SS, 2 chains", "warp-issued SS, 4 chains",
                          "warp-issued SS, 8 chains", "unused", "M=64 SS, 1 chain"};
  for (int mode : {9, 3})
    for (int N : {16, 32, 64, 128}) {
      if (mode == 7 && N > 64) continue;
      int n = 4096;
      run<<<148, 128, 160 * 1024>>>(4096, N, mode, d);
      cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      printf("%-40s N=%3d: %.1f cycles/MMA (floor %d) %s\n", names[mode], N, avg / n, 128 * N / 256,
             cudaGetErrorString(cudaGetLastError()));
    }
}
