// Microbenchmark (diagnostics, round 2): can a cluster multicast feed an SM faster than its own loads when G CTAs
// read the same tiles (the keys-on-lanes kernel streams each 128-key base tile into the 4 CTAs of its kv head)?
// 148 CTAs in clusters of G; every group streams ONE slice (shared by its G CTAs) chunk by chunk, D slots in flight.
//   mode 0: every CTA loads every chunk itself (one thread, cp.async.bulk) -- today's pattern
//   mode 1: chunk i is loaded by CTA (i % G) with .multicast::cluster into all G CTAs (same smem offset; each CTA's
//           own mbarrier gets complete_tx); a slot is refilled once all G CTAs released it (remote arrives on the
//           issuing CTA's empty barrier)
// Consumers are instant (wait full -> release). Reports received B/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ub_mcast tools/ub_mcast.cu && tools/ub_mcast
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2604_06370_b200/csrc/sm100.cuh"
using namespace fkv::sm100;

constexpr int kMaxSlots = 16;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_mc(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                            uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __launch_bounds__(128, 1) mc(const uint8_t* g, size_t slice, int S, int D, int G, int mode, int iters,
                                              long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kMaxSlots], empty[kMaxSlots];
  const uint32_t rank = cta_rank();
  if (threadIdx.x < kMaxSlots) {
    mbar_init(smem_u32(&full[threadIdx.x]), 1);
    mbar_init(smem_u32(&empty[threadIdx.x]), G);
  }
  fence_mbar_init();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cluster_sync();
  const uint8_t* src = g + (size_t)(blockIdx.x / G) * slice;
  const size_t nchunks = slice / S;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    uint32_t fph[kMaxSlots] = {}, eph[kMaxSlots] = {};
    // chunk i -> slot i % D; mode 1: issued by CTA i % G into every CTA
    int issued = 0;
    for (int i = 0; i < iters; ++i) {
      // issue ahead: keep up to D chunks in flight
      while (issued < iters && issued < i + D) {
        const int s = issued % D;
        const uint32_t dst = smem_u32(smem) + (uint32_t)s * S;
        const uint8_t* p = src + (size_t)(issued % nchunks) * S;
        if (mode == 0) {
          if (issued >= D) { mbar_wait(smem_u32(&empty[s]), eph[s]); eph[s] ^= 1; }
          mbar_expect_tx(smem_u32(&full[s]), S);
          bulk_g2s(dst, p, S, smem_u32(&full[s]));
        } else {
          // every CTA expects the chunk on its own full barrier; the issuer first waits until all G released slot s
          mbar_expect_tx(smem_u32(&full[s]), S);
          if ((uint32_t)(issued % G) == rank) {
            if (issued >= D) { mbar_wait(smem_u32(&empty[s]), eph[s]); eph[s] ^= 1; }
            bulk_g2s_mc(dst, p, S, smem_u32(&full[s]), (uint16_t)((1u << G) - 1));
          }
        }
        ++issued;
      }
      const int s = i % D;
      mbar_wait(smem_u32(&full[s]), fph[s]);
      fph[s] ^= 1;
      // release: mode 0 locally (count G: arrive G times), mode 1 to the CTA that issues the slot's next chunk
      if (mode == 0) {
        for (int k = 0; k < G; ++k) mbar_arrive(smem_u32(&empty[s]));
      } else {
        const uint32_t nxt = (uint32_t)((i + D) % G);
        arrive_remote(mapa(smem_u32(&empty[s]), nxt));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = clock64() - t0;
    out[2 * blockIdx.x + 1] = (long long)iters * S;
  }
  cluster_sync();
}

int main() {
  const size_t slice = 24u << 20;
  const size_t big = (size_t)148 * slice;
  uint8_t* g;
  cudaMalloc(&g, big);
  cudaMemset(g, 1, big);
  long long* d;
  cudaMalloc(&d, 148 * 16);
  cudaFuncSetAttribute(mc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(mc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  struct Cfg { int S, D, G, mode; };
  const Cfg cfgs[] = {{32768, 4, 1, 0}, {32768, 4, 2, 0}, {32768, 4, 2, 1}, {32768, 4, 4, 0}, {32768, 4, 4, 1},
                      {16384, 8, 4, 0}, {16384, 8, 4, 1}, {32768, 6, 4, 0}, {32768, 6, 4, 1}, {16384, 12, 4, 1},
                      {32768, 6, 2, 1}, {16384, 12, 2, 1}};
  for (const Cfg& c : cfgs) {
    const int grid = 148 / c.G * c.G;
    const int iters = (int)((64u << 20) / (size_t)c.S);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(128);
    lc.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&lc, mc, (const uint8_t*)g, slice, c.S, c.D, c.G, c.mode, iters, d);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    long long h[296] = {};
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0, by = 0;
    for (int i = 0; i < grid; ++i) cyc += h[2 * i], by += h[2 * i + 1];
    const double bpc = by / cyc;
    printf("mode %d (%s) G %d S %6d D %2d: received %6.1f B/clk/SM (%5.2f TB/s into smem; HBM-side %5.2f TB/s) %s\n",
           c.mode, c.mode ? "multicast" : "own loads", c.G, c.S, c.D, bpc, bpc * grid * clk_khz * 1e3 / 1e12,
           bpc * grid * clk_khz * 1e3 / 1e12 / c.G, cudaGetErrorString(e));
  }
  return 0;
}
