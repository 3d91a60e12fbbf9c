// Self-tests of the tcgen05/TMEM/TMA building blocks used by ra_tc.cu:
// every operand layout of the ResidualAttention tcgen05 kernel is exercised
// on a small GEMM and compared against a reference by the caller
// (tests/test_gpu_selftest.py). Diagnostic entry point fkv_selftest_umma.
#include <cuda_bf16.h>

#include "../../include/forkkv.h"
#include "sm100.cuh"
#include "tma_host.hpp"

namespace fkv {
namespace {
using namespace sm100;

struct SelfTest {
  int test, M, N, K;
};

// A: [M][K] bf16 row-major, B: [N][K] bf16 row-major, D: [M][N] fp32.
__global__ void __launch_bounds__(128, 1) umma_selftest_kernel(SelfTest t, const __nv_bfloat16* A,
                                                               const __nv_bfloat16* B, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  uint8_t* sA = smem;
  uint8_t* sB = smem + 64 * 1024;
  const int M = t.M, N = t.N, K = t.K;
  if (wid == 0) tmem_alloc(smem_u32(&tmem_base), 512);
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  // ---- fill smem operands in the layout under test ----
  bool a_mn = false, b_mn = false;
  int aW = 8, bW = 8;
  uint32_t a_lbo = 16, a_sbo = 1024, a_kblk = 0, b_lbo = 16, b_sbo = 1024, b_kblk = 0;
  uint32_t a_kstep = 32, b_kstep = 32;  // bytes per 16-element K step (within an atom column)
  switch (t.test) {
    case 0:  // K-major SW128 A and B (S^T = K_base Q^T)
      a_kblk = M * 128; b_kblk = N * 128; break;
    case 1:  // MN-major SW128 A and B (O^T = V^T P^T)
      a_mn = b_mn = true; a_lbo = K * 128; b_lbo = K * 128; a_kstep = b_kstep = 2048; break;
    case 2:  // A K-major SW32 (R_k, K=16), B MN-major SW128 (B_k [r][d]) (K_lora = R_k B_k)
      aW = 2; a_sbo = 256; b_mn = true; b_lbo = K * 128; b_kstep = 2048; break;
    case 3:  // A MN-major SW32 (R_v^T, owner blocks of 16 at LBO), B MN-major SW128 (P^T)
      a_mn = true; aW = 2; a_lbo = K * 32; a_sbo = 256; a_kstep = 512; b_mn = true; b_lbo = K * 128;
      b_kstep = 2048; break;
    case 6:  // A K-major SW32 (R_k, K=16), B MN-major SW64 (permuted B_k quarter blocks, N = 32 per atom)
      aW = 2; a_sbo = 256; b_mn = true; bW = 4; b_lbo = K * 64; b_sbo = 512; b_kstep = 1024; break;
    case 4:  // A in TMEM (bf16 packed), B K-major SW128 (S_res = K_lora Q_o^T)
      b_kblk = N * 128; break;
    default: break;
  }
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const uint32_t off = a_mn ? mnmajor_off(m, k, aW, a_lbo, a_sbo) : kmajor_off(m, k, aW, a_sbo, a_kblk);
    *(__nv_bfloat16*)(sA + off) = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const uint32_t off = b_mn ? mnmajor_off(n, k, bW, b_lbo, b_sbo) : kmajor_off(n, k, bW, b_sbo, b_kblk);
    *(__nv_bfloat16*)(sB + off) = B[i];
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t d_tmem = tbase;          // columns [0, N)
  const uint32_t a_tmem = tbase + 256;    // columns [256, 256 + K/2)
  if (t.test == 4) {
    // thread = row m = 32*wid + lane writes its K values packed (2 per column)
    const int m = 32 * wid + lane;
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float lo = __bfloat162float(A[m * K + 2 * (c0 + j)]);
        const float hi = __bfloat162float(A[m * K + 2 * (c0 + j) + 1]);
        r[j] = pack_bf16x2(lo, hi);
      }
      FKV_TMEM_ST16(a_tmem + ((uint32_t)(32 * wid) << 16) + c0, r);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16(M, N, a_mn, b_mn);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int s = 0; s < K / 16; ++s) {
      uint32_t aoff, boff;
      if (a_mn) aoff = s * a_kstep;
      else aoff = (s * 16 / (8 * aW)) * a_kblk + (s * 16 % (8 * aW)) * 2;
      if (b_mn) boff = s * b_kstep;
      else boff = (s * 16 / (8 * bW)) * b_kblk + (s * 16 % (8 * bW)) * 2;
      const uint64_t bd = make_desc(b0 + boff, b_lbo, b_sbo, bW == 8 ? SWZ_128 : (bW == 4 ? SWZ_64 : SWZ_32));
      if (t.test == 4) {
        mma_ts(d_tmem, a_tmem + 8 * s, bd, idesc, s > 0);
      } else {
        const uint64_t ad = make_desc(a0 + aoff, a_lbo, a_sbo, aW == 8 ? SWZ_128 : SWZ_32);
        mma_ss(d_tmem, ad, bd, idesc, s > 0);
      }
    }
    mma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  const int m = 32 * wid + lane;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    FKV_TMEM_LD32(d_tmem + ((uint32_t)(32 * wid) << 16) + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 32 && c0 + j < N; ++j) D[m * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tbase, 512);
}

// TMA SW128 box {64 cols, 64 rows} vs the kmajor_off layout formula.
__global__ void tma_selftest_kernel(const __grid_constant__ CUtensorMap map, const __nv_bfloat16* G, int cols,
                                    int row0, int col0, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(smem_u32(&bar), 64 * 64 * 2);
    tma_load_2d(smem_u32(smem), &map, col0, row0, smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  int bad = 0;
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
    const int r = i / 64, c = i % 64;
    const __nv_bfloat16 v = *(const __nv_bfloat16*)(smem + kmajor_off(r, c, 8, 1024, 0));
    if (__bfloat16_as_ushort(v) != __bfloat16_as_ushort(G[(int64_t)(row0 + r) * cols + col0 + c])) ++bad;
  }
  atomicAdd(D, (float)bad);
}

}  // namespace
}  // namespace fkv

extern "C" fkv_status fkv_selftest_umma(int32_t test, const void* A, const void* B, float* D, int32_t M, int32_t N,
                                        int32_t K, void* stream) {
  using namespace fkv;
  cudaStream_t s = (cudaStream_t)stream;
  if (test == 5) {
    // A: [M rows][K cols] global bf16; TMA box at (row 64, col 64) when it fits
    try {
      CUtensorMap m = make_tmap_2d_bf16(A, (uint64_t)M, (uint64_t)K, (uint64_t)K * 2, 64, 64, 128);
      cudaMemsetAsync(D, 0, sizeof(float), s);
      tma_selftest_kernel<<<1, 128, 64 * 64 * 2 + 1024, s>>>(m, (const __nv_bfloat16*)A, K, M - 64, K - 64, D);
    } catch (...) {
      return FKV_E_CUDA;
    }
    return cudaGetLastError() == cudaSuccess ? FKV_OK : FKV_E_CUDA;
  }
  if (test < 0 || test > 6 || test == 5 || M != 128 || N < 16 || N > 256 || N % 16 || K < 16 || K > 128 || K % 16)
    return FKV_E_INVALID;
  const int smem = 128 * 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  SelfTest t{test, M, N, K};
  umma_selftest_kernel<<<1, 128, smem, s>>>(t, (const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D);
  return cudaGetLastError() == cudaSuccess ? FKV_OK : FKV_E_CUDA;
}
