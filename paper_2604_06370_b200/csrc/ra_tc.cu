// Grouped ResidualAttention on 5th-generation tensor cores (tcgen05 + TMEM +
// TMA), bf16 in / fp32 accumulate, d = 128, r = 16: the hot loop of §8(a)
// row a5 for items whose rows share a base-page segment.
//
// One CTA = one plan item: kv head h, key range [k0, k1) of a base-page
// segment shared by all its query rows, up to 4 "slots" of 16 rows; a slot
// belongs to one residual owner (adapter + residual pages), consecutive slots
// of one owner form a group. The key tile (128 keys) sits on the TMEM lanes
// (M = keys), the CTA's 64 query rows on N, so per-owner residual terms are
// plain N-slices of the same accumulator:
//
//   Stage 1 (Alg1.332-336)   S^T  = K_base Q^T                    [tcgen05 SS]
//     DEFERRED (paper):      KL   = R_k,g B_k,g for one half of d; B_k's
//                            columns are permuted so a half holds the RoPE
//                            pairs (i, i+64)                       [tcgen05 SS]
//                            key warps: KL <- RoPE_t(KL) in fp32x2, bf16
//                            written back in place in TMEM       [tcgen05.ld/st]
//                            S^T[:, rows of g] += KL Q_g^T       [tcgen05 TS]
//     NONE (north-star split): S^T[:, rows of g] += R_k,g (Q_g B_k,g^T)^T [SS]
//   Stage 2 (Alg1.338-346)   key warps: one online softmax per query row
//                            (a column of S^T), lazily rescaled; P^T -> smem
//                            O^T  += V_base^T P^T                [tcgen05 SS]
//                            A^T  += [R_v,0..3 ; 1]^T P^T        [tcgen05 SS]
//                            (the all-ones slot accumulates the row sums l)
//   Stage 3 (Alg1.348-350)   in the combine kernel (late V fusion, Eq.4).
//
// 12 warps: warpgroup 2 = control (warp 8 TMA producer, 9/10 S-side MMA issuers (10 also allocates
// TMEM), 11 PV-side MMA issuer; setmaxnreg.dec; high warp ids win the issue arbiter), warpgroups 0, 1
// = key warps (thread = TMEM lane = key of the tile; WG1 owns d-half 0 of the
// K_lora rebuild and query columns 0..31, WG2 d-half 1 and columns 32..63;
// setmaxnreg.inc).  Buffers: K_base x1 (released right after S^T), R_k x2,
// V_base x2, R_v x2.
#include <cuda_bf16.h>

#include <cstddef>
#include <cstdint>

#include "kernels.hpp"
#include "sm100.cuh"

namespace fkv {
namespace k {
namespace {
using namespace sm100;

constexpr int kD = 128, kR = 16, kTile = 128, kRows = 64, kSlots = 4;
// shared memory map (bytes from the 1024-aligned dynamic smem base)
constexpr uint32_t OFF_KB = 0;                       // K_base [2 d-halves][128 keys][128 B]  32 KB
constexpr uint32_t OFF_RK = 32768;                   // R_k x2 stages x 4 slots x 4 KB       32 KB
constexpr uint32_t OFF_V = 65536;                    // V_base x2 stages                      64 KB
constexpr uint32_t OFF_RV = 131072;                  // R_v x2 stages x 5 slots (slot 4 = 1)  40 KB
constexpr uint32_t kRvStage = 5 * 4096;
constexpr uint32_t OFF_Q = OFF_RV + 2 * kRvStage;    // Q rows, K-major SW128               16 KB
constexpr uint32_t OFF_BK = OFF_Q + 16384;           // B_k slots (DEFERRED) | q~ (NONE)     16 KB
constexpr uint32_t OFF_P = OFF_BK + 16384;           // P^T [128 keys][64 rows]             16 KB
constexpr uint32_t OFF_MISC = OFF_P + 16384;
constexpr uint32_t kSmemBytes = OFF_MISC + 3072;
// TMEM columns
// S^T is split in two accumulators: S0 = K_base Q^T + the d-half-0 residual terms (key warpgroup 0),
// S1 = the d-half-1 residual terms (key warpgroup 1); the softmax adds them.
constexpr uint32_t T_S = 0, T_S1 = 64, T_O = 128, T_A = 192, T_KL = 256;  // KL: [wg][4 bufs] x 32 columns
constexpr int kKlBufs = 4;

struct Misc {
  uint64_t kbfull, kbempty, rkfull[2], rkempty[2], vfull[2], vempty[2], sfull[2], sfree, klfull[2][kKlBufs], klready[2][kKlBufs],
      pfull, pvdone;
  alignas(16) float m_run[kRows];
  alignas(16) float alpha[kRows];
  float red[2][4][32];
  alignas(16) int32_t pos[kRows];
  int32_t g_first[kSlots], g_cnt[kSlots];
  int32_t slot_res[kSlots], slot_ad[kSlots];
  int32_t n_groups, n_slots, causal;
  uint32_t tmem_base;
};
static_assert(sizeof(Misc) <= 3072, "misc");
constexpr int kNumBars = 31;
static_assert(offsetof(Misc, m_run) >= kNumBars * 8 && offsetof(Misc, m_run) % 16 == 0, "barriers");

struct TcMaps {
  CUtensorMap kb, vb, rk, rv;
};

__device__ __forceinline__ bool bar_or(uint32_t id, uint32_t n, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, %2, %3, p;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

// ---- packed fp32x2 helpers (FFMA2 / FMUL2 on sm_100) ----
__device__ __forceinline__ uint64_t f2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void uf2(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint32_t pack2(uint64_t v) {
  float a, b;
  uf2(v, a, b);
  return pack_bf16x2(a, b);
}
__device__ __forceinline__ float ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// diagnostics: clock64 stamp of pipeline event e for tile j of CTA dbg_block
__device__ __forceinline__ void ev(const AttnParams& p, int e, int j) {
  if (p.dbg && (int)blockIdx.x == p.dbg_block && j < 256) p.dbg[e * 256 + j] = clock64();
}

// permuted B_k column n' -> d, in 32-column quarter blocks b = 2w + q (w = d-half of key warpgroup w,
// q = quarter): block b holds d = 32w + 16q + [0, 16) followed by the RoPE partners d + 64.
__device__ __forceinline__ int perm_d(int n) {
  const int b = n >> 5, c = n & 31;
  return 32 * (b >> 1) + 16 * (b & 1) + (c < 16 ? c : 64 + c - 16);
}

__global__ void __launch_bounds__(384, 1) ra_tc_kernel(const __grid_constant__ TcMaps maps, AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  Misc& ms = *reinterpret_cast<Misc*>(smem + OFF_MISC);
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (sbase & 1023) __trap();
  if (tid == 0) ev(p, 20, 0);
  const DevItem it = p.items[blockIdx.x];
  const int h = it.kv_head;
  const int k0 = it.key_begin, k1 = it.key_end;
  const int n_tiles = (k1 - k0 + kTile - 1) / kTile;
  const int P = p.P;
  const bool deferred = p.rope_mode == FKV_ROPE_DEFERRED;

  // ---------------- setup ----------------
  if (tid == 0) {
    ms.n_slots = it.n_warps;
    int ng = 0, causal = 0;
    for (int o = 0; o < it.n_warps; ++o) {
      const DevWarp w = p.warps[it.warp_off + o];
      ms.slot_res[o] = w.res_off;
      ms.slot_ad[o] = w.adapter_slot;
      if (o > 0 && w.res_off == ms.slot_res[o - 1] && w.adapter_slot == ms.slot_ad[o - 1]) {
        ms.g_cnt[ng - 1]++;
      } else {
        ms.g_first[ng] = o; ms.g_cnt[ng] = 1; ++ng;
      }
      for (int i = 0; i < w.n_rows; ++i)
        if (p.rows[w.row_off + i].pos < k1 - 1) causal = 1;
    }
    ms.n_groups = ng;
    ms.causal = causal;
    uint64_t* bars = &ms.kbfull;
    for (int i = 0; i < kNumBars; ++i) mbar_init(smem_u32(bars + i), 1);
    mbar_init(smem_u32(&ms.sfree), 256);
    if (p.rope_mode == FKV_ROPE_DEFERRED) {  // both S-side issuers release R_k
      mbar_init(smem_u32(&ms.rkempty[0]), 2);
      mbar_init(smem_u32(&ms.rkempty[1]), 2);
    }
    mbar_init(smem_u32(&ms.pfull), 256);
    for (int w = 0; w < 2; ++w)
      for (int b = 0; b < kKlBufs; ++b) mbar_init(smem_u32(&ms.klready[w][b]), 128);
    fence_mbar_init();
  }
  if (wid == 10) tmem_alloc(smem_u32(&ms.tmem_base), 512);
  if (tid < kRows) {
    ms.m_run[tid] = -INFINITY;
    const int o = tid >> 4, i = tid & 15;
    int pos = -1;
    if (o < it.n_warps) {
      const DevWarp w = p.warps[it.warp_off + o];
      if (i < w.n_rows) pos = p.rows[w.row_off + i].pos;
    }
    ms.pos[tid] = pos;
  }
  // Q rows -> K-major SW128 (B operand of S^T = K Q^T); zero rows for padding
  for (int c = tid; c < kRows * 16; c += 384) {
    const int row = c >> 4, ch = c & 15;
    const int o = row >> 4, i = row & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (o < it.n_warps) {
      const DevWarp w = p.warps[it.warp_off + o];
      if (i < w.n_rows) {
        const DevRow rw = p.rows[w.row_off + i];
        v = __ldg((const uint4*)((const __nv_bfloat16*)p.Q +
                                 ((int64_t)(p.seqs[rw.seq].q_row0 + rw.qi) * p.hq + rw.qh) * kD) + ch);
      }
    }
    *(uint4*)(smem + OFF_Q + kmajor_off(row, ch * 8, 8, 1024, 8192)) = v;
  }
  // all-ones R_v slot 4 of both stages: A^T lanes 64..79 accumulate the row sums l
  for (int c = tid; c < 2 * 256; c += 384)
    *(uint4*)(smem + OFF_RV + (c >> 8) * kRvStage + 4 * 4096 + (c & 255) * 16) =
        make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  __syncthreads();
  const int n_groups = ms.n_groups, n_slots = ms.n_slots;
  if (deferred) {
    // B_k^h of each slot, columns permuted, MN-major SW64 [quarter block][16 r][32]
    for (int c = tid; c < n_slots * kR * (kD / 8); c += 384) {
      const int o = c / (kR * 16), e = c % (kR * 16), jj = e >> 4, n8 = (e & 15) * 8;
      const __nv_bfloat16* Bk = (const __nv_bfloat16*)p.adapters[2 * ms.slot_ad[o]] +
                                (int64_t)p.layer * p.adapter_layer_stride + (int64_t)h * kR * kD + jj * kD;
      // 8 consecutive permuted columns n8..n8+7 map to 8 consecutive d
      const uint4 v = __ldg((const uint4*)(Bk + perm_d(n8)));
      *(uint4*)(smem + OFF_BK + o * 4096 + mnmajor_off(n8, jj, 4, 1024, 512)) = v;
    }
  } else {
    // q~ = Q B_k^T per row (the north-star split), bf16, K-major SW32
    for (int c = tid; c < kRows * kR; c += 384) {
      const int row = c >> 4, jj = c & 15, o = row >> 4;
      float acc = 0.f;
      if (o < n_slots) {
        const __nv_bfloat16* Bk = (const __nv_bfloat16*)p.adapters[2 * ms.slot_ad[o]] +
                                  (int64_t)p.layer * p.adapter_layer_stride + (int64_t)h * kR * kD + jj * kD;
        for (int d8 = 0; d8 < kD; d8 += 8) {
          const uint4 qv = *(const uint4*)(smem + OFF_Q + kmajor_off(row, d8, 8, 1024, 8192));
          const uint4 bv = __ldg((const uint4*)(Bk + d8));
          const __nv_bfloat162* q2 = (const __nv_bfloat162*)&qv;
          const __nv_bfloat162* b2 = (const __nv_bfloat162*)&bv;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 a = __bfloat1622float2(q2[e]), b = __bfloat1622float2(b2[e]);
            acc += a.x * b.x + a.y * b.y;
          }
        }
      }
      *(__nv_bfloat16*)(smem + OFF_BK + kmajor_off(row, jj, 2, 256, 0)) = __float2bfloat16_rn(acc);
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = ms.tmem_base;
  if (tid == 0) ev(p, 21, 0);

  if (wid >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (wid == 8 && lane == 0) {
      // ================= TMA producer =================
      tma_prefetch_desc(&maps.kb); tma_prefetch_desc(&maps.vb);
      tma_prefetch_desc(&maps.rk); tma_prefetch_desc(&maps.rv);
      const int64_t brow_l = (int64_t)p.layer * p.nb;  // 2D views: row = ((layer*NB + page)*Hkv + h)*P
      const int64_t rrow_l = (int64_t)p.layer * p.nr;  //                 (layer*NR + page)*P
      const int pages = kTile / P;
      auto row_of = [&](int t, bool base) -> int {  // 2D-view row of the page holding key t (clamped)
        const int slot = (t < k1 ? t : k0) / P;
        if (base) return (int)(((brow_l + p.base_pages[it.base_off + slot]) * p.hkv + h) * P);
        return slot;
      };
      auto prefetch = [&](int j) {  // L2 prefetch of every box of tile j (hides DRAM latency)
        if (j >= n_tiles) return;
        const int t0 = k0 + j * kTile;
        for (int q = 0; q < pages; ++q) {
          const int t = t0 + q * P;
          if (t >= k1) break;
          const int row = row_of(t, true), slot = row_of(t, false);
          if (P == 128) {  // base K/V only: the single-buffered K_base is the latency-critical stream
            tma_prefetch_l2_3d(&maps.kb, 0, row, 0);
            tma_prefetch_l2_3d(&maps.vb, 0, row, 0);
          } else {
            tma_prefetch_l2(&maps.kb, 0, row); tma_prefetch_l2(&maps.kb, 64, row);
            tma_prefetch_l2(&maps.vb, 0, row); tma_prefetch_l2(&maps.vb, 64, row);
          }
          (void)slot;
        }
      };
      auto issue_rk = [&](int j) {
        const int st = j & 1, t0 = k0 + j * kTile;
        ev(p, 0, j);
        const uint32_t bar = smem_u32(&ms.rkfull[st]);
        mbar_expect_tx(bar, n_groups * kTile * kR * 2);
        for (int q = 0; q < pages; ++q) {
          const int slot = row_of(t0 + q * P, false);
          for (int g = 0; g < n_groups; ++g) {
            const int o = ms.g_first[g];
            const int rp = p.res_pages[ms.slot_res[o] + slot];
            tma_load_2d(sbase + OFF_RK + st * 16384 + o * 4096 + q * P * 32, &maps.rk, 0, (int)((rrow_l + rp) * P),
                        bar);
          }
        }
      };
      auto issue_kb = [&](int j) {
        const int t0 = k0 + j * kTile;
        ev(p, 1, j);
        const uint32_t bar = smem_u32(&ms.kbfull);
        mbar_expect_tx(bar, kTile * kD * 2);
        if (P == 128) {
          tma_load_3d(sbase + OFF_KB, &maps.kb, 0, row_of(t0, true), 0, bar);
        } else {
          for (int q = 0; q < pages; ++q) {
            const int row = row_of(t0 + q * P, true);
            tma_load_2d(sbase + OFF_KB + q * P * 128, &maps.kb, 0, row, bar);
            tma_load_2d(sbase + OFF_KB + 16384 + q * P * 128, &maps.kb, 64, row, bar);
          }
        }
      };
      auto issue_v = [&](int j) {
        const int st = j & 1, t0 = k0 + j * kTile;
        ev(p, 2, j);
        const uint32_t bar = smem_u32(&ms.vfull[st]);
        mbar_expect_tx(bar, kTile * kD * 2 + n_slots * kTile * kR * 2);
        for (int q = 0; q < pages; ++q) {
          const int t = t0 + q * P;
          const int row = row_of(t, true), slot = row_of(t, false);
          if (P == 128) {
            tma_load_3d(sbase + OFF_V + st * 32768, &maps.vb, 0, row, 0, bar);
          } else {
            tma_load_2d(sbase + OFF_V + st * 32768 + q * P * 128, &maps.vb, 0, row, bar);
            tma_load_2d(sbase + OFF_V + st * 32768 + 16384 + q * P * 128, &maps.vb, 64, row, bar);
          }
          for (int o = 0; o < n_slots; ++o) {
            const int rp = p.res_pages[ms.slot_res[o] + slot];
            tma_load_2d(sbase + OFF_RV + st * kRvStage + o * 4096 + q * P * 32, &maps.rv, 0,
                        (int)((rrow_l + rp) * P), bar);
          }
        }
      };
      // three independent streams, each issued as soon as its buffer is free
      const int kPrefetch = p.tc_prefetch;
      for (int j = 0; j < kPrefetch; ++j) prefetch(j);

      int nrk = 0, nkb = 0, nv = 0;
      while (nrk < n_tiles || nkb < n_tiles || nv < n_tiles) {
        bool progress = false;
        if (nrk < n_tiles && (nrk < 2 || mbar_test(smem_u32(&ms.rkempty[nrk & 1]), ((nrk >> 1) - 1) & 1))) {
          issue_rk(nrk);
          if (kPrefetch) prefetch(nrk + kPrefetch);
          ++nrk;
          progress = true;
        }
        if (nkb < nrk && (nkb < 1 || mbar_test(smem_u32(&ms.kbempty), (nkb - 1) & 1))) {
          issue_kb(nkb);
          ++nkb;
          progress = true;
        }
        if (nv < nrk && (nv < 2 || mbar_test(smem_u32(&ms.vempty[nv & 1]), ((nv >> 1) - 1) & 1))) {
          issue_v(nv);
          ++nv;
          progress = true;
        }
        if (!progress) __nanosleep(64);  // yield issue slots to the key warps
      }
    } else if ((wid == 9 || (wid == 10 && deferred)) && lane == 0) {
      // ================= S-side MMA issuers =================
      // warp 1: S0 = K_base Q^T (+ NONE residual, or the d-half-0 DEFERRED units of key warpgroup 0)
      // warp 2: S1 = the d-half-1 DEFERRED units of key warpgroup 1
      const int w = wid - 9;
      const uint32_t sacc = tm + (w ? T_S1 : T_S);
      const uint32_t id_s = idesc_bf16(128, kRows, false, false);
      const uint32_t id_rb = idesc_bf16(128, 32, false, true);
      int Uw = 0;  // this warpgroup's K_lora unit counter (buffer = U % kKlBufs)
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        const uint32_t rk = sbase + OFF_RK + st * 16384;
        mbar_wait_sleep(smem_u32(&ms.rkfull[st]), (j >> 1) & 1);
        tc_fence_after();
        if (w == 0) ev(p, 3, j);
        const int n_units = deferred ? 2 * n_groups : 0;  // unit k = q * n_groups + g (quarter-major)
        auto rb = [&](int k) {  // KL[w][b] (fp32, 32 cols) = R_k,g B_k,g[:, quarter block 2w + q]
          const int q = k / n_groups, g = k % n_groups, o = ms.g_first[g];
          const int b = (Uw + k) % kKlBufs;
          const uint64_t ad = make_desc(rk + o * 4096, 16, 256, SWZ_32);
          const uint64_t bd = make_desc(sbase + OFF_BK + o * 4096 + (2 * w + q) * 1024, 1024, 512, SWZ_64);
          mma_ss(tm + T_KL + 128 * w + 32 * b, ad, bd, id_rb, 0);
          mma_commit(smem_u32(&ms.klfull[w][b]));
        };
        auto ts = [&](int k) {  // S_w^T[:, rows of g] += RoPE(KL)[bf16, in place] Q_g^T over the unit's 32 d
          const int q = k / n_groups, g = k % n_groups, o = ms.g_first[g], cnt = ms.g_cnt[g];
          const int U = Uw + k, b = U % kKlBufs;
          mbar_wait_sleep(smem_u32(&ms.klready[w][b]), (U / kKlBufs) & 1);
          tc_fence_after();
          const uint32_t id = idesc_bf16(128, 16 * cnt, false, false);
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) {
            const int d = 64 * s2 + 32 * w + 16 * q;
            const uint64_t bd =
                make_desc(sbase + OFF_Q + (d >> 6) * 8192 + 2048 * o + (d & 63) * 2, 16, 1024, SWZ_128);
            // S1 has no base term: the first K-step of each group's first unit initialises it
            mma_ts(sacc + 16 * o, tm + T_KL + 128 * w + 32 * b + 8 * s2, bd, id, (w == 0 || q > 0 || s2 > 0));
          }
        };
        for (int k = 0; k < n_units && k < kKlBufs; ++k) rb(k);
        if (w == 0) mbar_wait_sleep(smem_u32(&ms.kbfull), j & 1);
        if (j > 0) mbar_wait_sleep(smem_u32(&ms.sfree), (j - 1) & 1);
        tc_fence_after();
        if (w == 0) {
          ev(p, 4, j);
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const uint64_t ad = make_desc(sbase + OFF_KB + (s >> 2) * 16384 + (s & 3) * 32, 16, 1024, SWZ_128);
            const uint64_t bd = make_desc(sbase + OFF_Q + (s >> 2) * 8192 + (s & 3) * 32, 16, 1024, SWZ_128);
            mma_ss(tm + T_S, ad, bd, id_s, s > 0);
          }
          mma_commit(smem_u32(&ms.kbempty));
        }
        if (deferred) {
          for (int k = 0; k < n_units; ++k) {
            ts(k);
            if (k + kKlBufs < n_units) rb(k + kKlBufs);
          }
          Uw += n_units;
        } else {
          for (int g = 0; g < n_groups; ++g) {
            const int o = ms.g_first[g], cnt = ms.g_cnt[g];
            const uint64_t ad = make_desc(rk + o * 4096, 16, 256, SWZ_32);
            const uint64_t bd = make_desc(sbase + OFF_BK + o * 512, 16, 256, SWZ_32);
            mma_ss(tm + T_S + 16 * o, ad, bd, idesc_bf16(128, 16 * cnt, false, false), 1);
          }
        }
        if (w == 0) ev(p, 5, j);
        mma_commit(smem_u32(&ms.sfull[w]));
        mma_commit(smem_u32(&ms.rkempty[st]));
      }
    } else if (wid == 11 && lane == 0) {
      // ================= PV-side MMA issuer =================
      const uint32_t id_pv = idesc_bf16(128, kRows, true, true);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        mbar_wait_sleep(smem_u32(&ms.pfull), j & 1);
        mbar_wait_sleep(smem_u32(&ms.vfull[st]), (j >> 1) & 1);
        tc_fence_after();
        ev(p, 6, j);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint64_t bd = make_desc(sbase + OFF_P + s * 2048, 16384, 1024, SWZ_128);
          const uint64_t ad = make_desc(sbase + OFF_V + st * 32768 + s * 2048, 16384, 1024, SWZ_128);
          mma_ss(tm + T_O, ad, bd, id_pv, (j > 0 || s > 0));
        }
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint64_t bd = make_desc(sbase + OFF_P + s * 2048, 16384, 1024, SWZ_128);
          const uint64_t ad = make_desc(sbase + OFF_RV + st * kRvStage + s * 512, 4096, 256, SWZ_32);
          mma_ss(tm + T_A, ad, bd, id_pv, (j > 0 || s > 0));
        }
        mma_commit(smem_u32(&ms.pvdone));
        mma_commit(smem_u32(&ms.vempty[st]));
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    // ================= key warps =================
    const int w = wid >> 2;                        // key warpgroup 0/1
    const int kl = tid - 128 * w;                  // key within the tile == TMEM lane
    const uint32_t lb = (uint32_t)(32 * (wid & 3)) << 16;
    const int cb = 32 * w;                         // this group's query columns [cb, cb + 32)
    const uint32_t bar_id = 1 + w;                 // named barrier of this warpgroup
    const bool causal = ms.causal != 0;
    const uint64_t sc2 = f2(p.scale_log2, p.scale_log2);
    int U = 0;
    // RoPE rows of this key for the next tile, frequencies [32w, 32w + 32), prefetched one tile ahead
    float4 rc[8], rs[8];
    auto load_rope = [&](int jj) {
      const int tt = min(k0 + jj * kTile + kl, k1 - 1);
      const float4* cp = (const float4*)(p.rope_cos + (int64_t)tt * (kD / 2) + 32 * w);
      const float4* sp = (const float4*)(p.rope_sin + (int64_t)tt * (kD / 2) + 32 * w);
#pragma unroll
      for (int q = 0; q < 8; ++q) { rc[q] = __ldg(cp + q); rs[q] = __ldg(sp + q); }
    };
    if (deferred) load_rope(0);
    for (int j = 0; j < n_tiles; ++j) {
      const int t = k0 + j * kTile + kl;
      const bool tvalid = t < k1;
      if (kl == 0) ev(p, 7 + 6 * w, j);
      if (deferred) {
        for (int q = 0; q < 2; ++q) {
          // quarter q: frequencies 32w + 16q + [0, 16)
          uint64_t C[8], S[8], NS[8];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float4 a = rc[4 * q + e], bq = rs[4 * q + e];
            C[2 * e] = f2(a.x, a.y); C[2 * e + 1] = f2(a.z, a.w);
            S[2 * e] = f2(bq.x, bq.y); S[2 * e + 1] = f2(bq.z, bq.w);
            NS[2 * e] = f2(-bq.x, -bq.y); NS[2 * e + 1] = f2(-bq.z, -bq.w);
          }
          // two units per step: one TMEM load/store round trip and one barrier wait for both
          for (int g = 0; g < n_groups; g += 2) {
            const int nu = (g + 1 < n_groups) ? 2 : 1;
            uint32_t x[2][16], y[2][16], lh[2][16];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (u < nu) {
                const int b = (U + u) % kKlBufs;
                mbar_wait_sleep(smem_u32(&ms.klfull[w][b]), ((U + u) / kKlBufs) & 1);
              }
            }
            tc_fence_after();
            if (kl == 0 && g == 0 && q == 0) ev(p, 8 + 6 * w, j);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (u < nu) {
                const uint32_t kt = tm + T_KL + 128 * w + 32 * ((U + u) % kKlBufs) + lb;
                FKV_TMEM_LD16(kt, x[u]);
                FKV_TMEM_LD16(kt + 16, y[u]);
              }
            }
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 2; ++u) {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const uint64_t X = f2(__uint_as_float(x[u][2 * e]), __uint_as_float(x[u][2 * e + 1]));
                const uint64_t Y = f2(__uint_as_float(y[u][2 * e]), __uint_as_float(y[u][2 * e + 1]));
                lh[u][e] = pack2(fma2(Y, NS[e], mul2(X, C[e])));       // x cos - y sin  (d)
                lh[u][8 + e] = pack2(fma2(X, S[e], mul2(Y, C[e])));    // x sin + y cos  (d + 64)
              }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (u < nu) {
                const uint32_t kt = tm + T_KL + 128 * w + 32 * ((U + u) % kKlBufs) + lb;
                FKV_TMEM_ST16(kt, lh[u]);
              }
            }
            tmem_st_wait();
            tc_fence_before();
#pragma unroll
            for (int u = 0; u < 2; ++u)
              if (u < nu) mbar_arrive(smem_u32(&ms.klready[w][(U + u) % kKlBufs]));
            U += nu;
          }
        }
        if (j + 1 < n_tiles) load_rope(j + 1);
      }
      // ---- online softmax over this group's 32 query columns (Alg1.339-341) ----
      if (kl == 0) ev(p, 9 + 6 * w, j);
      mbar_wait_sleep(smem_u32(&ms.sfull[0]), j & 1);
      if (deferred) mbar_wait_sleep(smem_u32(&ms.sfull[1]), j & 1);
      tc_fence_after();
      if (kl == 0) ev(p, 10 + 6 * w, j);
      uint32_t sr[32];
      FKV_TMEM_LD32(tm + T_S + cb + lb, sr);
      if (deferred) {
        uint32_t s1[32];
        FKV_TMEM_LD32(tm + T_S1 + cb + lb, s1);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) sr[c] = __float_as_uint(__uint_as_float(sr[c]) + __uint_as_float(s1[c]));
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(smem_u32(&ms.sfree));
      uint64_t x2[16];
      float mx = -INFINITY;
      {
        const float4* mp = (const float4*)&ms.m_run[cb];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 m4 = mp[q];
          const uint64_t s01 = f2(__uint_as_float(sr[4 * q]), __uint_as_float(sr[4 * q + 1]));
          const uint64_t s23 = f2(__uint_as_float(sr[4 * q + 2]), __uint_as_float(sr[4 * q + 3]));
          x2[2 * q] = fma2(s01, sc2, f2(-m4.x, -m4.y));
          x2[2 * q + 1] = fma2(s23, sc2, f2(-m4.z, -m4.w));
        }
        if (causal || !tvalid) {
          const int4* pp = (const int4*)&ms.pos[cb];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int4 p4 = pp[q];
            float a, b2, c, d;
            uf2(x2[2 * q], a, b2);
            uf2(x2[2 * q + 1], c, d);
            if (!tvalid || t > p4.x) a = -INFINITY;
            if (!tvalid || t > p4.y) b2 = -INFINITY;
            if (!tvalid || t > p4.z) c = -INFINITY;
            if (!tvalid || t > p4.w) d = -INFINITY;
            x2[2 * q] = f2(a, b2);
            x2[2 * q + 1] = f2(c, d);
          }
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float a, b2;
          uf2(x2[q], a, b2);
          mx = max3(mx, a, b2);
        }
      }
      // lazy rescaling: only when some score exceeds the running max by > 2^8
      if (bar_or(bar_id, 128, mx > 8.0f)) {
        if (kl == 0) ev(p, 19, j + 128 * w);
        float v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const bool ok = tvalid && (!causal || t <= ms.pos[cb + c]);
          v[c] = ok ? __uint_as_float(sr[c]) * p.scale_log2 : -INFINITY;
        }
#pragma unroll
        for (int step = 0; step < 5; ++step) {
          const int off = 16 >> step, half = 16 >> step;
          const bool up = lane & off;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const float send = up ? v[i] : v[i + half];
            const float keep = up ? v[i + half] : v[i];
            v[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, off));
          }
        }
        if (kl == 0) ev(p, 23 + w, j);
        ms.red[w][wid & 3][lane] = v[0];  // lane l holds column cb + l
        named_bar_sync(bar_id, 128);
        if (kl == 0) ev(p, 29 + w, j);
        bool resc = false;
        if (kl < 32) {
          const int c = cb + kl;
          const float cm = fmaxf(fmaxf(ms.red[w][0][kl], ms.red[w][1][kl]), fmaxf(ms.red[w][2][kl], ms.red[w][3][kl]));
          const float mo = ms.m_run[c];
          const float mn = fmaxf(mo, cm);
          float al = 1.f;
          if (mn != mo) {
            al = mo == -INFINITY ? 0.f : ex2(mo - mn);
            resc = mo != -INFINITY;
          }
          ms.alpha[c] = al;
          ms.m_run[c] = mn;
        }
        if (kl == 0) ev(p, 27 + w, j);
        if (bar_or(bar_id, 128, resc) && j > 0) {
          // rescale this group's columns of O^T and A^T by alpha
          mbar_wait_sleep(smem_u32(&ms.pvdone), (j - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const uint32_t base = tm + (part ? T_A : T_O) + cb + lb;
            uint32_t r[32];
            FKV_TMEM_LD32(base, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * ms.alpha[cb + i]);
            FKV_TMEM_ST16(base, r);
            FKV_TMEM_ST16(base + 16, (r + 16));
          }
          tmem_st_wait();
          tc_fence_before();
        }
        if (kl == 0) ev(p, 25 + w, j);
        // recompute with the updated running max (a column with no visible key keeps -inf -> p = 0)
        const float* mr = &ms.m_run[cb];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float m0 = mr[2 * q], m1 = mr[2 * q + 1];
          const bool ok0 = tvalid && (!causal || t <= ms.pos[cb + 2 * q]);
          const bool ok1 = tvalid && (!causal || t <= ms.pos[cb + 2 * q + 1]);
          const float x0 = ok0 ? __uint_as_float(sr[2 * q]) * p.scale_log2 - (m0 == -INFINITY ? 0.f : m0) : -INFINITY;
          const float x1 = ok1 ? __uint_as_float(sr[2 * q + 1]) * p.scale_log2 - (m1 == -INFINITY ? 0.f : m1)
                               : -INFINITY;
          x2[q] = f2(x0, x1);
        }
      }
      // P^T row of this key (bf16, MN-major SW128), columns [cb, cb + 32)
      uint32_t pk[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        float a, b2;
        uf2(x2[q], a, b2);
        pk[q] = pack_bf16x2(ex2(a), ex2(b2));
      }
      if (kl == 0) ev(p, 11 + 6 * w, j);
      if (j > 0) mbar_wait_sleep(smem_u32(&ms.pvdone), (j - 1) & 1);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch)
        *(uint4*)(smem + OFF_P + mnmajor_off(cb + ch * 8, kl, 8, 16384, 1024)) =
            make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      fence_async_smem();
      mbar_arrive(smem_u32(&ms.pfull));
      if (kl == 0) ev(p, 12 + 6 * w, j);
    }
    // ---- epilogue: partial entries [m, l, acc[128], acc_r[16]] for columns [cb, cb+32) ----
    mbar_wait_sleep(smem_u32(&ms.pvdone), (n_tiles - 1) & 1);
    tc_fence_after();
    uint32_t o_[32], a_[32];
    FKV_TMEM_LD32(tm + T_O + cb + lb, o_);
    FKV_TMEM_LD32(tm + T_A + cb + lb, a_);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int c = cb + i, o = c >> 4, r = c & 15;
      if (o < n_slots) {
        const DevWarp wd = p.warps[it.warp_off + o];
        if (r < wd.n_rows) {
          float* ent = p.ws + (int64_t)(wd.entry_off + r) * p.entry_stride;
          ent[2 + kl] = __uint_as_float(o_[i]);                    // acc[d = kl]
          if ((kl >> 4) == o) ent[2 + kD + (kl & 15)] = __uint_as_float(a_[i]);  // acc_r[j] of this row's owner
          if (kl == 64) {
            ent[0] = ms.m_run[c];
            ent[1] = __uint_as_float(a_[i]);                      // l (all-ones slot)
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) ev(p, 22, 0);
  if (wid == 10) tmem_dealloc(tm, 512);
}

}  // namespace

cudaError_t launch_attention_tc(const AttnParams& p, const void* maps, cudaStream_t s) {
  if (p.n_items == 0) return cudaSuccess;
  if (p.d != kD || p.r != kR || p.dtype != FKV_DTYPE_BF16 || (kTile % p.P) || p.P < 8) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ra_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  ra_tc_kernel<<<p.n_items, 384, kSmemBytes, s>>>(*(const TcMaps*)maps, p);
  return cudaGetLastError();
}

size_t tc_maps_bytes() { return sizeof(TcMaps); }

}  // namespace k
}  // namespace fkv
