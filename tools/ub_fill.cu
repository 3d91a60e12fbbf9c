// Microbenchmark (diagnostics, round 2): per-SM shared-memory fill rate vs bytes in flight, the question behind
// the rows kernel's load pipeline. 148 CTAs (one per SM) each stream their own slice of a buffer far larger
// than L2 (HBM-bound, cold) or a small window (L2-resident), with
//   mode 0: 1D bulk copies (cp.async.bulk) of S bytes, D slots in flight, issued by one thread
//   mode 1: the same issued round-robin by W warps (lane 0 each; D slots per warp)
//   mode 2: 16-byte cp.async by W full warps (D slots of S bytes per warp, completion via cp.async.mbarrier)
// Reports B/clk/SM and the chip-wide TB/s at the measured SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ub_fill tools/ub_fill.cu && tools/ub_fill
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
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_inc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}

constexpr int kMaxSlots = 64;

__global__ void __launch_bounds__(256, 1) fill(const uint8_t* g, size_t slice, int S, int D, int W, int mode,
                                               int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[kMaxSlots];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < kMaxSlots) mbar_init(smem_u32(&bar[threadIdx.x]), mode == 2 ? 1 : 1);
  fence_mbar_init();
  __syncthreads();
  const uint8_t* src = g + (size_t)blockIdx.x * slice;
  const size_t nchunks = slice / S;
  long long t0 = clock64();
  if (wid < W) {
    // warp wid owns slots [wid * D, wid * D + D)
    uint32_t ph[kMaxSlots / 1];
    for (int i = 0; i < D; ++i) ph[i] = 0;
    size_t c = wid;
    const int n = iters;
    for (int it = 0; it < n; ++it) {
      const int s = it % D;
      const int slot = wid * D + s;
      const uint32_t dst = smem_u32(smem) + (uint32_t)slot * S;
      const uint32_t b = smem_u32(&bar[slot]);
      if (it >= D) {
        mbar_wait(b, ph[s]);
        ph[s] ^= 1;
      }
      const uint8_t* p = src + (c % nchunks) * S;
      c += W;
      if (mode == 2) {
        for (int o = lane * 16; o < S; o += 512) cp_async16(dst + o, p + o);
        cp_async_arrive_inc(b);
        __syncwarp();
        if (lane == 0) mbar_arrive(b);
      } else if (lane == 0) {
        mbar_expect_tx(b, S);
        bulk_g2s(dst, p, S, b);
      }
      __syncwarp();
    }
    for (int s = 0; s < D && s < n; ++s) {
      const int slot = wid * D + s;
      mbar_wait(smem_u32(&bar[slot]), ph[s]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = clock64() - t0;
    out[2 * blockIdx.x + 1] = (long long)iters * W * S;
  }
}

int main() {
  const size_t big = (size_t)148 * (24u << 20);   // 24 MiB per SM: 3.5 GB, far beyond L2
  uint8_t* g;
  cudaMalloc(&g, big);
  cudaMemset(g, 1, big);
  long long* d;
  cudaMalloc(&d, 148 * 16);
  cudaFuncSetAttribute(fill, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  struct Cfg { int S, D, W, mode; };
  const Cfg cfgs[] = {{32768, 1, 1, 0}, {32768, 2, 1, 0}, {32768, 4, 1, 0}, {32768, 6, 1, 0},
                      {4096, 8, 1, 0},  {4096, 16, 1, 0}, {4096, 32, 1, 0}, {4096, 48, 1, 0},
                      {16384, 4, 1, 0}, {16384, 8, 1, 0}, {16384, 12, 1, 0},
                      {4096, 8, 4, 1},  {4096, 12, 4, 1}, {32768, 1, 4, 1}, {32768, 1, 6, 1},
                      {4096, 4, 4, 2},  {4096, 8, 4, 2},  {4096, 12, 4, 2}, {16384, 2, 4, 2}, {16384, 3, 4, 2}};
  for (int win = 0; win < 2; ++win) {
    const size_t slice = win == 0 ? (24u << 20) : (256u << 10);   // HBM stream vs L2-resident 256 KB per SM
    for (const Cfg& c : cfgs) {
      if ((size_t)c.S * c.D * c.W > 196 * 1024 || c.D * c.W > kMaxSlots) continue;
      const int iters = (int)((win == 0 ? (16u << 20) : (16u << 20)) / ((size_t)c.S * c.W));
      fill<<<148, 256, 200 * 1024>>>(g, slice, c.S, c.D, c.W, c.mode, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[296];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0, by = 0;
      for (int i = 0; i < 148; ++i) cyc += h[2 * i], by += h[2 * i + 1];
      const double bpc = by / cyc;
      printf("%s mode %d S %6d D %2d W %d inflight %4d KB: %6.1f B/clk/SM  (%5.2f TB/s at %d MHz) %s\n",
             win == 0 ? "HBM" : "L2 ", c.mode, c.S, c.D, c.W, c.S * c.D * c.W / 1024, bpc,
             bpc * 148 * clk_khz * 1e3 / 1e12, clk_khz / 1000, cudaGetErrorString(e));
    }
  }
  return 0;
}
