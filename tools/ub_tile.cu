// Microbenchmark (diagnostics, round 2): the rows kernel's per-tile load pattern alone (no MMA / softmax), to
// find the fastest way to fill the 5 x 32 KB ring: per tile one K unit (32 KB), one R_k unit (8 x 4 KB pages),
// one V unit (32 KB), one R_v unit (8 x 4 KB), consumed in that order by a consumer thread that frees each unit
// as soon as it lands. 148 CTAs, one per SM. Sources: base pages in a 2 GB pool (HBM-streamed: every CTA pair
// reads the same base tile, like the two row blocks of a kv head), residual pages in a 32 MB pool (L2-resident,
// like the head-shared residual).
//   mode 0: K, V by one TMA-engine bulk op each (issuing thread per kind), residual by 8 lanes of one warp (bulk)
//   mode 1: as 0, residual by cp.async 16 B from 2 warps (R_k warp, R_v warp)
//   mode 2: as 0, residual by cp.async 16 B from 4 warps (2 per plane, half the slots each)
//   mode 3: everything by cp.async 16 B: 8 warps (2 per unit kind)
//   mode 4: as 0 but K and V each split into 4 x 8 KB bulk ops from 4 lanes
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ub_tile tools/ub_tile.cu && tools/ub_tile
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

constexpr int kNU = 5;
constexpr uint32_t kUnit = 32768;

__device__ __forceinline__ uint64_t hash(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// unit u: kind = u % 4 (0 K, 1 R_k, 2 V, 3 R_v), tile = u / 4
__global__ void __launch_bounds__(512, 1) run(const uint8_t* base, const uint8_t* res, int n_tiles, int mode,
                                             long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kNU], empty[kNU];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_res_warps = mode == 1 ? 1 : (mode == 2 ? 2 : 0);  // per plane
  if (threadIdx.x == 0) {
    for (int i = 0; i < kNU; ++i) {
      // arrivals per phase: TMA units 1; cp.async units: issuing warps' lane 0
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t sb = smem_u32(smem);
  const int pair = blockIdx.x >> 1;  // CTAs 2i, 2i+1 read the same base tiles
  const int n_units = 4 * n_tiles;
  long long t0 = clock64();
  auto base_src = [&](int tile, int kind) {
    const uint64_t pg = (uint64_t)(pair * n_tiles + tile) % 32768;  // 32768 pages x 32 KB = 1 GB per plane
    return base + (size_t)(kind == 2 ? 1 : 0) * (1ull << 30) + pg * kUnit;
  };
  auto res_src = [&](int tile, int kind, int slot) {
    const uint64_t pg = hash((uint64_t)(blockIdx.x % 16) * 7919 + tile * 8 + slot) % 4096;  // 16 MB per plane
    return res + (size_t)(kind == 3 ? 1 : 0) * (16u << 20) + pg * 4096;
  };
  if (wid == 0) {
    // consumer: units in order; frees each as soon as it is full
    if (lane == 0)
      for (int u = 0; u < n_units; ++u) {
        const int s = u % kNU;
        mbar_wait(smem_u32(&full[s]), (u / kNU) & 1);
        mbar_arrive(smem_u32(&empty[s]));
      }
  } else {
    // producers: warp 1 K, warp 2 V, warp 3 residual (bulk); warps 4.. cp.async helpers per mode
    for (int u = 0; u < n_units; ++u) {
      const int kind = u & 3, tile = u >> 2, s = u % kNU;
      const uint32_t dst = sb + s * kUnit, fb = smem_u32(&full[s]);
      bool mine;
      if (mode == 3) mine = wid >= 4 && wid < 12 && ((wid - 4) >> 1) == kind;
      else if (kind == 0) mine = wid == 1;
      else if (kind == 2) mine = wid == 2;
      else if (mode == 0 || mode == 4) mine = wid == 3;
      else mine = wid >= 4 && wid < 4 + 2 * n_res_warps && ((wid - 4) / n_res_warps) == (kind == 3 ? 1 : 0);
      if (!mine) continue;
      mbar_wait(smem_u32(&empty[s]), ((u / kNU) & 1) ^ 1);
      if (kind == 0 || kind == 2) {
        const uint8_t* src = base_src(tile, kind);
        if (mode == 3) {
          const int part = (wid - 4) & 1;  // two warps, 16 KB each
          for (int o = part * 16384 + lane * 16; o < (part + 1) * 16384; o += 512) cp_async16(dst + o, src + o);
          cp_async_arrive_inc(fb);
          __syncwarp();
          named_bar_sync(2 + kind, 64);  // both warps' pending arrivals registered before the one expected arrival
          if (lane == 0 && part == 0) mbar_arrive(fb);
        } else if (mode == 4) {
          if (lane == 0) mbar_expect_tx(fb, kUnit);
          __syncwarp();
          if (lane < 4) bulk_g2s(dst + lane * 8192, src + lane * 8192, 8192, fb);
        } else if (lane == 0) {
          mbar_expect_tx(fb, kUnit);
          bulk_g2s(dst, src, kUnit, fb);
        }
      } else {
        if (mode == 0 || mode == 4) {
          if (lane == 0) mbar_expect_tx(fb, kUnit);
          __syncwarp();
          if (lane < 8) bulk_g2s(dst + lane * 4096, res_src(tile, kind, lane), 4096, fb);
        } else {
          const int nw = mode == 3 ? 2 : n_res_warps;
          const int part = mode == 3 ? ((wid - 4) & 1) : ((wid - 4) % n_res_warps);
          const int s0 = part * 8 / nw, s1 = (part + 1) * 8 / nw;
          for (int sl = s0; sl < s1; ++sl) {
            const uint8_t* src = res_src(tile, kind, sl);
            for (int o = lane * 16; o < 4096; o += 512) cp_async16(dst + sl * 4096 + o, src + o);
          }
          cp_async_arrive_inc(fb);
          __syncwarp();
          if (nw > 1) named_bar_sync(2 + kind, 32 * nw);
          if (lane == 0 && part == 0) mbar_arrive(fb);
        }
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  uint8_t *base, *res;
  cudaMalloc(&base, 2ull << 30);
  cudaMalloc(&res, 32u << 20);
  cudaMemset(base, 1, 2ull << 30);
  cudaMemset(res, 2, 32u << 20);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const size_t smem = kNU * kUnit;
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int n_tiles = 64;
  const char* names[] = {"K,V bulk 1 op each; residual 8 lanes bulk", "residual cp.async 1 warp/plane",
                         "residual cp.async 2 warps/plane", "all cp.async 2 warps/unit kind",
                         "K,V 4 x 8KB bulk from 4 lanes; residual 8 lanes bulk"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      run<<<148, 512, smem>>>(base, res, n_tiles, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0, mx = 0;
      for (int i = 0; i < 148; ++i) avg += h[i], mx = h[i] > mx ? h[i] : mx;
      avg /= 148;
      if (rep == 1)
        printf("mode %d %-52s: %6.0f cycles/tile (max CTA %6.0f), %5.1f B/clk/SM  %s\n", mode, names[mode],
               avg / n_tiles, mx / n_tiles, 131072.0 * n_tiles / avg, cudaGetErrorString(e));
    }
  }
  return 0;
}
