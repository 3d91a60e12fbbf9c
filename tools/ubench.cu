// Microbenchmarks (diagnostics, not part of the library) for the design of the
// decode kernel: TMEM load/store bandwidth per SM, TMA bulk bandwidth from L2
// and from HBM at full chip, and TMA multicast across a cluster.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench tools/ubench.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2604_06370_b200/csrc/sm100.cuh"

using namespace fkv::sm100;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);       \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

// ---------------- TMEM bandwidth ----------------
// every warp w reads (mode 0) / writes (mode 1) 32 lanes (lane quarter w%4) x 32 columns per op
__global__ void tmem_bw(int iters, int mode, int cols_per_op, long long* out, uint32_t* sink) {
  __shared__ uint32_t tbase;
  const int wid = threadIdx.x >> 5;
  if (wid == 0) tmem_alloc(smem_u32(&tbase), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)((wid >> 2) * 64 % 512);
  uint32_t acc = 0;
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * i;
  __syncthreads();
  const long long t0 = clock64();
  if (mode == 0) {
    for (int it = 0; it < iters; ++it) {
      FKV_TMEM_LD32(tm, r);
      FKV_TMEM_LD32(tm + 32, (r));
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= r[i];
    }
  } else {
    for (int it = 0; it < iters; ++it) {
      FKV_TMEM_ST16(tm, r);
      FKV_TMEM_ST16(tm + 16, (r + 16));
      FKV_TMEM_ST16(tm + 32, r);
      FKV_TMEM_ST16(tm + 48, (r + 16));
      tmem_st_wait();
      r[0] += it;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tbase, 512);
}

// ---------------- TMA bulk bandwidth ----------------
__device__ __forceinline__ void bulk_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_1d_mc(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                           uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
      "%4;\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
}

// each CTA streams `tiles` tiles of `tile_bytes`; tile i of CTA b at ((b*7919 + i*stride_tiles) % n_tiles_total)
// csz > 1: the cluster shares tile i (same address for all ranks); rank k loads bytes [k*tb/csz, (k+1)*tb/csz)
// multicast to every rank.  stages x tile_bytes of smem.
__global__ void tma_bw(const uint8_t* src, int64_t n_tiles_total, int tile_bytes, int tiles, int csz, int stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[8];
  const uint32_t rank = csz > 1 ? cluster_rank() : 0;
  const int cid = blockIdx.x / csz;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_mbar_init();
  }
  if (csz > 1) cluster_sync_all(); else __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t part = tile_bytes / csz;
    for (int i = 0; i < tiles; ++i) {
      const int s = i % stages;
      if (i >= stages) mbar_wait(smem_u32(&bars[s]), ((i / stages) - 1) & 1);
      const int64_t t = ((int64_t)cid * 7919 + (int64_t)i * 131) % n_tiles_total;
      const uint8_t* g = src + t * tile_bytes;
      const uint32_t bar = smem_u32(&bars[s]);
      mbar_expect_tx(bar, tile_bytes);
      if (csz == 1) {
        for (uint32_t o = 0; o < (uint32_t)tile_bytes; o += 16384)
          bulk_1d(smem_u32(smem) + s * tile_bytes + o, g + o, min(16384, tile_bytes - (int)o), bar);
      } else {
        bulk_1d_mc(smem_u32(smem) + s * tile_bytes + rank * part, g + rank * part, part, bar,
                   (uint16_t)((1u << csz) - 1));
      }
      if (csz > 1 && s == stages - 1) {
        // keep the ranks within one ring of each other (a peer must not receive phase k+1 bytes before k completed)
        mbar_wait(bar, (i / stages) & 1);
        for (int q = 0; q < stages - 1; ++q) {
          const int ii = i - (stages - 1) + q;
          if (ii >= 0) mbar_wait(smem_u32(&bars[q]), (ii / stages) & 1);
        }
      }
    }
    for (int i = (tiles > stages ? tiles - stages : 0); i < tiles; ++i)
      mbar_wait(smem_u32(&bars[i % stages]), (i / stages) & 1);
  }
  if (csz > 1) {
    __syncwarp();
    // the stage barrier loop above does not sync the cluster; a final sync keeps smem alive until peers finish
    cluster_sync_all();
  }
}

// multicast pipeline with cross-CTA "empty" barriers (the production pattern):
// mc=1: rank k loads part k of tile i multicast to all ranks; mc=0: every rank loads the whole
// tile itself (unicast, same addresses as its peers at about the same time).
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
__global__ void tma_bw_mc(const uint8_t* src, int64_t n_tiles_total, int tile_bytes, int tiles, int csz, int stages,
                          int mc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x / csz;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), mc ? csz : 1);
    }
    fence_mbar_init();
  }
  cluster_sync_all();
  if (threadIdx.x == 0) {
    const uint32_t part = mc ? tile_bytes / csz : tile_bytes;
    for (int i = 0; i < tiles; ++i) {
      const int s = i % stages;
      if (i >= stages) mbar_wait(smem_u32(&empty[s]), ((i / stages) - 1) & 1);
      const int64_t t = ((int64_t)cid * 7919 + (int64_t)i * 131) % n_tiles_total;
      const uint8_t* g = src + t * tile_bytes;
      const uint32_t bar = smem_u32(&full[s]);
      mbar_expect_tx(bar, tile_bytes);
      if (mc) {
        bulk_1d_mc(smem_u32(smem) + s * tile_bytes + rank * part, g + rank * part, part, bar,
                   (uint16_t)((1u << csz) - 1));
      } else {
        for (uint32_t o = 0; o < (uint32_t)tile_bytes; o += 16384)
          bulk_1d(smem_u32(smem) + s * tile_bytes + o, g + o, min(16384, tile_bytes - (int)o), bar);
      }
      // consumer side (same thread): wait for the oldest outstanding stage, then free it in every rank
      const int c = i - (stages - 2);
      if (c >= 0) {
        const int cs = c % stages;
        mbar_wait(smem_u32(&full[cs]), (c / stages) & 1);
        if (mc) {
          for (int q = 0; q < csz; ++q) mbar_arrive_remote(mapa(smem_u32(&empty[cs]), q));
        } else {
          mbar_arrive(smem_u32(&empty[cs]));
        }
      }
    }
    for (int c = tiles - (stages - 2); c < tiles; ++c) {
      if (c < 0) continue;
      const int cs = c % stages;
      mbar_wait(smem_u32(&full[cs]), (c / stages) & 1);
      if (mc)
        for (int q = 0; q < csz; ++q) mbar_arrive_remote(mapa(smem_u32(&empty[cs]), q));
    }
  }
  __syncwarp();
  cluster_sync_all();
}

int main() {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const int nsm = prop.multiProcessorCount;
  printf("device %s, %d SMs, clock %d kHz\n", prop.name, nsm, prop.clockRate);
  long long* d_out;
  uint32_t* d_sink;
  CK(cudaMalloc(&d_out, 4096 * sizeof(long long)));
  CK(cudaMalloc(&d_sink, 4096 * 1024 * sizeof(uint32_t)));
  // TMEM bandwidth: 1 CTA per SM, W warps
  for (int mode = 0; mode < 2; ++mode) {
    for (int W : {1, 4, 8, 16}) {
      const int iters = 2000;
      tmem_bw<<<nsm, 32 * W>>>(iters, mode, 32, d_out, d_sink);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      std::vector<long long> h(nsm);
      CK(cudaMemcpy(h.data(), d_out, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
      double cyc = 0;
      for (auto v : h) cyc += v;
      cyc /= nsm;
      const double bytes = (double)iters * W * 32 * 64 * 4;  // 64 columns x 32 lanes x 4 B per warp-iteration
      printf("TMEM %s: %2d warps/SM: %.1f B/cycle/SM (%.0f cycles)\n", mode ? "st" : "ld", W, bytes / cyc, cyc);
    }
  }
  // TMA bandwidth
  const size_t big = (size_t)4 << 30;
  uint8_t* src;
  CK(cudaMalloc(&src, big));
  CK(cudaMemset(src, 1, big));
  CK(cudaFuncSetAttribute(tma_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(tma_bw_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(tma_bw_mc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (size_t footprint : {(size_t)48 << 20, big}) {
    for (int tb : {16384, 32768}) {
      for (int cfgi = 0; cfgi < 9; ++cfgi) {
        const int csz = (int[]){1, 2, 4, 8, 16, 2, 4, 8, 1}[cfgi];
        const int mc = cfgi >= 1 && cfgi <= 4;
        const int stages = cfgi == 8 ? 6 : 4;
        if (stages * tb > 200 * 1024) continue;
        const int64_t ntiles = footprint / tb;
        const int tiles = footprint > ((size_t)1 << 30) ? 400 : 1600;
        const int grid = csz == 1 ? nsm : (nsm / csz) * csz;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(32);
        cfg.dynamicSmemBytes = stages * tb;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = csz;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        float best = 1e30f;
        bool ok = true;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaEventRecord(e0));
          cudaError_t err;
          err = cudaLaunchKernelEx(&cfg, tma_bw_mc, (const uint8_t*)src, ntiles, tb, tiles, csz, stages, mc);
          if (err != cudaSuccess) {
            printf("  launch csz=%d failed: %s\n", csz, cudaGetErrorString(err));
            cudaGetLastError();
            ok = false;
            break;
          }
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (rep > 0 && ms < best) best = ms;
        }
        if (!ok) continue;
        const double delivered = (double)grid * tiles * tb;
        const double l2reads = mc ? delivered / csz : delivered;
        printf("TMA footprint %5zu MB tile %5d csz %2d mc %d stages %d grid %3d: delivered %.0f GB/s (to smem), source reads %.0f GB/s, %.1f us\n",
               footprint >> 20, tb, csz, mc, stages, grid, delivered / best / 1e6, l2reads / best / 1e6, best * 1e3);
      }
    }
  }
  return 0;
}
