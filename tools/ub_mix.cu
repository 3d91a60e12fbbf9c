// Microbenchmark (diagnostics, round 2): tensor-pipe cycles per attention tile for the MMA instruction mixes of
// the rows-on-lanes kernel, alone and with the shared-memory / TMEM traffic the real kernel adds around them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ub_mix tools/ub_mix.cu && tools/ub_mix
// One CTA per SM (148), warp 1 lane 0 issues `n_tiles` tiles of the chosen mix back to back (one commit per tile);
// optional background: warp 2 streams 32-KB bulk copies from an L2-resident buffer into shared memory (the ring
// fills), warps 4-7 loop tcgen05.ld 128 columns + tcgen05.st 64 columns (the softmax's TMEM traffic).
#include <cuda.h>
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
__device__ __forceinline__ void mma_ss_m(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc, uint4 dis) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc), "r"(dis.x), "r"(dis.y), "r"(dis.z), "r"(dis.w));
}

constexpr uint32_t OFF_Q = 0, OFF_QT = 32768, OFF_K = 36864, OFF_RK = 102400, OFF_BG = 167936;
constexpr uint32_t SMEM = OFF_BG + 32768 + 1024;

// MIX 0: current rows kernel per 128 keys: 8 SS (SW128, N=128) + 8 SS masked (SW32, N=128) + 8 x (TS MN-SW128 N=128
//        + TS MN-SW32 N=128)                                                          = 32 instructions / 128 keys
// MIX 1: N=256 per 256 keys: 8 SS (SW128, N=256) + 8 SS masked (SW32, N=256) + 16 TS (B MN-SW32, N=256)
//                                                                                     = 32 instructions / 256 keys
// MIX 2: as 1 with the PV B operand MN-SW128 (V | R_v atoms of 64 columns)
// MIX 3: only 8 SS SW128 N=256 (S base)          MIX 4: only 8 SS SW32 masked N=256 (S residual)
// MIX 5: only 16 TS MN-SW32 N=256 (PV)            MIX 6: only 16 TS MN-SW128 N=256
// MIX 7: only 8 SS SW128 N=128                    MIX 8: 8 SS (SW128, N=128) + 8 SS masked (SW32, N=128) + 8 TS N=256
template <int MIX>
__global__ void __launch_bounds__(256, 1) run(int n_tiles, int bg, const uint8_t* gsrc, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, bgbar[2];
  __shared__ volatile int stop;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (wid == 0) tmem_alloc(smem_u32(&tbase), 512);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init(smem_u32(&bgbar[0]), 1);
    mbar_init(smem_u32(&bgbar[1]), 1);
    stop = 0;
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (int)(SMEM - 1024) / 16; i += blockDim.x)
    ((uint4*)smem)[i] = make_uint4(0x3f803f80u ^ (i * 2654435761u & 0x00ff00ffu), 0x3f003f00u, 0xbf803f80u, 0x3e803e80u);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase, sb = smem_u32(smem);
  if (wid == 1 && lane == 0) {
    const uint32_t qa = sb + OFF_Q, qt = sb + OFF_QT, kb = sb + OFF_K, rk = sb + OFF_RK;
    const uint4 none = make_uint4(0, 0, 0, 0), msk = make_uint4(0xffff0000u, ~0u, ~0u, ~0u);
    const long long t0 = clock64();
    for (int t = 0; t < n_tiles; ++t) {
      if (MIX == 0 || MIX == 7 || MIX == 8) {
        const uint32_t idS = idesc_bf16(128, 128, false, false);
        for (int k = 0; k < 8; ++k)
          mma_ss_m(tm, make_desc(qa + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, SWZ_128),
                   make_desc(kb + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, SWZ_128), idS, k != 0, none);
        if (MIX != 7)
          for (int s = 0; s < 8; ++s)
            mma_ss_m(tm, make_desc(qt, 16, 256, SWZ_32), make_desc(rk + 4096u * s, 16, 256, SWZ_32), idS, 1u, msk);
        if (MIX == 0) {
          const uint32_t idV = idesc_bf16(128, 128, false, true);
          for (int k = 0; k < 8; ++k) {
            mma_ts(tm + 256, tm + 8 * k, make_desc(kb + 2048u * k, 16384, 1024, SWZ_128), idV, 1u);
            mma_ts(tm + 384, tm + 8 * k, make_desc(rk + 512u * k, 4096, 256, SWZ_32), idV, 1u);
          }
        } else if (MIX == 8) {
          const uint32_t idV = idesc_bf16(128, 256, false, true);
          for (int k = 0; k < 8; ++k) mma_ts(tm + 256, tm + 8 * k, make_desc(kb + 512u * k, 2048, 256, SWZ_32), idV, 1u);
        }
      } else {
        const uint32_t idS = idesc_bf16(128, 256, false, false);
        if (MIX == 1 || MIX == 2 || MIX == 3)
          for (int k = 0; k < 8; ++k)
            mma_ss_m(tm, make_desc(qa + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, SWZ_128),
                     make_desc(kb + (k >> 2) * 32768 + (k & 3) * 32, 16, 1024, SWZ_128), idS, k != 0, none);
        if (MIX == 1 || MIX == 2 || MIX == 4)
          for (int s = 0; s < 8; ++s)
            mma_ss_m(tm, make_desc(qt, 16, 256, SWZ_32), make_desc(rk + 8192u * s, 16, 256, SWZ_32), idS, 1u, msk);
        const uint32_t idV = idesc_bf16(128, 256, false, true);
        if (MIX == 1 || MIX == 5)
          for (int k = 0; k < 16; ++k)  // 4 units of 64 keys: [16 atom columns of 16][64 keys][32 B]
            mma_ts(tm + 256, tm + 8 * k, make_desc(kb + (k >> 2) * 32768 + 512u * (k & 3), 2048, 256, SWZ_32), idV,
                   1u);
        if (MIX == 2 || MIX == 6)
          for (int k = 0; k < 16; ++k)  // [4 atom columns of 64][64 keys][128 B]
            mma_ts(tm + 256, tm + 8 * k, make_desc(kb + (k >> 2) * 32768 + 2048u * (k & 3), 8192, 1024, SWZ_128),
                   idV, 1u);
      }
    }
    const long long t1 = clock64();
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    const long long t2 = clock64();
    out[blockIdx.x * 4] = t1 - t0;
    out[blockIdx.x * 4 + 1] = t2 - t0;
    stop = 1;
  } else if (wid == 2 && lane == 0 && (bg & 1)) {
    // ring fills: 32-KB bulk copies, 2 in flight, from an L2-resident 8 MiB window
    long long bytes = 0;
    uint32_t ph[2] = {0, 0};
    int i = 0;
    const long long t0 = clock64();
    for (int s = 0; s < 2; ++s) {
      mbar_expect_tx(smem_u32(&bgbar[s]), 32768);
      bulk_g2s(sb + OFF_BG + (s ? 0 : 0), gsrc + (size_t)((blockIdx.x * 7 + i++) % 256) * 32768, 32768,
               smem_u32(&bgbar[s]));
    }
    while (!stop) {
      const int s = i & 1;
      mbar_wait(smem_u32(&bgbar[s]), ph[s]);
      ph[s] ^= 1;
      bytes += 32768;
      mbar_expect_tx(smem_u32(&bgbar[s]), 32768);
      bulk_g2s(sb + OFF_BG, gsrc + (size_t)((blockIdx.x * 7 + i++) % 256) * 32768, 32768, smem_u32(&bgbar[s]));
    }
    for (int s = 0; s < 2; ++s) mbar_wait(smem_u32(&bgbar[(i + s) & 1]), ph[(i + s) & 1]);
    out[blockIdx.x * 4 + 2] = bytes;
    out[blockIdx.x * 4 + 3] = clock64() - t0;
  } else if (wid >= 2 && (bg & 8)) {
    // mbarrier spinners: 6 warps polling a barrier phase that completes only at the end (like the kernel's waiting
    // roles); bit 16 of bg: back off with nanosleep between polls
    __shared__ __align__(8) uint64_t never;
    if (threadIdx.x == 64) { mbar_init(smem_u32(&never), 1); fence_mbar_init(); }
    __syncwarp();
    uint32_t ok = 0;
    while (!stop) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(ok) : "r"(smem_u32(&never)), "r"(0u) : "memory");
      if (bg & 16) __nanosleep(64);
    }
    if (ok == 7) out[0] = 1;
  } else if (wid >= 4 && (bg & 4)) {
    // softmax-like ALU / MUFU load on every SMSP (warps 4-7), no TMEM traffic
    float a = threadIdx.x * 1e-3f, b2 = 0.f;
    while (!stop) {
#pragma unroll 16
      for (int i = 0; i < 64; ++i) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a));
        b2 = fmaf(y, 0.999f, b2);
        a = fmaf(a, 1.0001f, 1e-7f);
      }
    }
    if (b2 == 12345.f) out[0] = 1;
  } else if (wid >= 4 && (bg & 2)) {
    const uint32_t lb = (uint32_t)(32 * (wid - 4)) << 16;
    while (!stop) {
      uint32_t r[128];
      FKV_TMEM_LD32(tm + lb + 0, (r + 0));
      FKV_TMEM_LD32(tm + lb + 32, (r + 32));
      FKV_TMEM_LD32(tm + lb + 64, (r + 64));
      FKV_TMEM_LD32(tm + lb + 96, (r + 96));
      tmem_ld_wait();
      uint32_t pk[64];
#pragma unroll
      for (int c = 0; c < 64; ++c) pk[c] = r[2 * c] ^ r[2 * c + 1];
      FKV_TMEM_ST16(tm + lb + 0, (pk + 0));
      FKV_TMEM_ST16(tm + lb + 16, (pk + 16));
      FKV_TMEM_ST16(tm + lb + 32, (pk + 32));
      FKV_TMEM_ST16(tm + lb + 48, (pk + 48));
      tmem_st_wait();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tm, 512);
}

template <int MIX>
void go(int bg, const uint8_t* gsrc, const char* name, int keys) {
  long long* d;
  cudaMalloc(&d, 148 * 32);
  cudaMemset(d, 0, 148 * 32);
  cudaFuncSetAttribute(run<MIX>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int n_tiles = 64;
  run<MIX><<<148, 256, SMEM>>>(n_tiles, bg, gsrc, d);
  cudaDeviceSynchronize();
  run<MIX><<<148, 256, SMEM>>>(n_tiles, bg, gsrc, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double iss = 0, tot = 0, by = 0, bc = 0;
  for (int i = 0; i < 148; ++i) iss += h[4 * i], tot += h[4 * i + 1], by += h[4 * i + 2], bc += h[4 * i + 3];
  iss /= 148; tot /= 148;
  printf("%-44s bg=%d: %7.0f cyc/tile (%5.0f per 128 keys), issue %7.0f; bg fill %.1f B/clk/SM %s\n", name, bg,
         tot / n_tiles, tot / n_tiles * 128 / keys, iss / n_tiles, bc > 0 ? by / bc : 0.0, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  uint8_t* g;
  cudaMalloc(&g, 8 << 20);
  cudaMemset(g, 1, 8 << 20);
  for (int bg : {0, 8, 24}) {
    go<0>(bg, g, "cur: S8+R8 N128 SS, PV 8x(TS128 SW128+SW32)", 128);
    go<1>(bg, g, "N256: S8+R8 SS, PV 16 TS MN-SW32", 256);
    go<2>(bg, g, "N256: S8+R8 SS, PV 16 TS MN-SW128", 256);
    go<8>(bg, g, "mixed: S8+R8 N128 SS, PV 8 TS N256 SW32", 128);
    go<3>(bg, g, "only S 8 SS SW128 N256", 256);
    go<4>(bg, g, "only R 8 SS SW32 masked N256", 256);
    go<5>(bg, g, "only PV 16 TS MN-SW32 N256", 256);
    go<6>(bg, g, "only PV 16 TS MN-SW128 N256", 256);
    go<7>(bg, g, "only S 8 SS SW128 N128", 128);
  }
  return 0;
}
