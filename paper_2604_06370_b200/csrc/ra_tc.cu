// Grouped ResidualAttention on 5th-generation tensor cores (tcgen05 + TMEM +
// TMA), bf16 in / fp32 accumulate, d = 128, r = 16: the hot loop of §8(a)
// rows a5 (decode) and a7 (chunked prefill) for plan items whose query rows
// share a base-page segment.
//
// Persistent kernel: one CTA per SM walks its list of plan items (kv head h,
// key range [k0, k1) of a shared segment, up to 4 (8) "slots" of 16 query rows; a
// slot belongs to one residual owner = adapter + residual pages; consecutive
// slots of one owner form a group).  Keys sit on the TMEM lanes (M = 128 keys
// per tile), the item's 64 (128) query rows on N, so every per-owner residual term
// is an N-slice of the same accumulator:
//
//   Stage 1 (Alg1.332-336)  S^T  = K_base Q^T                          [SS]
//     NONE (north-star split, Eq.4 applied to K):
//                           S^T[:, rows of g] += R_k,g (Q_g B_k,g^T)^T  [SS]
//     DEFERRED (paper, Alg1.335): KL = R_k,g B_k,g per 32-column quarter
//                           block of d (RoPE pairs (i, i+64) side by side)
//                           [SS] -> key warps rotate KL at the key's
//                           absolute position in fp32 and write bf16 back in
//                           place -> S^T[:, rows of g] += KL Q_g^T       [TS]
//   Stage 2 (Alg1.338-346)  key warps: online softmax per query row (one
//                           column of S^T), lazily rescaled; P^T -> smem
//                           O^T += V_base^T P^T                         [SS]
//                           A^T += [R_v,0..3 ; 1]^T P^T (the all-ones slot
//                           accumulates the row sums l)                 [SS]
//   Stage 3 (Alg1.348-350)  combine kernel (late V fusion, Eq.4).
//
// 12 warps (control warps have the high ids, which win the issue arbiter):
//   warp 8  producer: K_base tiles (TMA, one 3D box per tile), R_k pages and the per-item header / Q / X images
//           (16-byte cp.async by all lanes), page ids from the plan's tile records;
//   warp 9  S-side MMA issuer, warp 10 PV-side MMA issuer (whole warps, one elected lane per instruction);
//   warp 11 TMEM allocator, then the V-side loader: V_base 64-key halves (TMA) + R_v pages (cp.async);
//   warps 0..7 key warps: thread = TMEM lane = key of the tile; key warpgroup w owns query columns
//           [rows/2 w, rows/2 (w+1)) (chunks of 32) and, in DEFERRED, the d-half w of the K_lora rotation.
// S^T is double-buffered in TMEM so S(j+1) overlaps softmax(j); P^T is a ring of 64-key halves so PV(j)
// overlaps softmax(j+1).  Template parameters: mode (NONE / DEFERRED) and query rows per CTA (64, or 128 for
// NONE with 8 slots and CUDA-core row sums).  DESIGN.md §4 has the measured cost model.
#include <cuda_bf16.h>

#include <cstddef>
#include <cstdint>

#include "kernels.hpp"
#include "sm100.cuh"

namespace fkv {
namespace k {
namespace {
using namespace sm100;

constexpr int kD = 128, kR = 16, kTile = 128, kMaxSlots = 8;
#ifndef FKV_LAZY_START
#define FKV_LAZY_START 1
#endif
constexpr bool kLazyStart = FKV_LAZY_START;  // first tile of a non-causal item: m = 0 reference (no column max)
// diagnostics only (A/B builds, wrong output): skip loads / math to find the binding pipeline stage.
// bit 1: K_base TMA, 2: V_base TMA, 4: R_k copies, 8: R_v copies, 16: key-warp exponentials (P = bf16(x)),
// 32: null key warps (pipeline handshakes only)
#ifndef FKV_DIAG_SKIP
#define FKV_DIAG_SKIP 0
#endif
constexpr int kSkip = FKV_DIAG_SKIP;
#ifndef FKV_STAGE_EARLY
#define FKV_STAGE_EARLY 1
#endif
constexpr bool kStageEarly = FKV_STAGE_EARLY;
#ifndef FKV_PROD_SLEEP
#define FKV_PROD_SLEEP 0  // ns the polling producer sleeps after a pass without progress (A/B: 0 > 20..200 >> 800)
#endif  // stager: loads and q~ before griddepcontrol.wait (C2 +2.3%)
// lazy-rescale headroom (log2 units): p = 2^(x - m) may reach 2^kLazyHi before the running max moves. fp32
// accumulators and bf16 P hold 2^16 x 32K keys easily; a larger headroom makes the first-tile slow path (m = 0
// reference, ~8 K cycles cold) and later rescales rarer
#ifndef FKV_LAZY_HI
#define FKV_LAZY_HI 16
#endif
constexpr float kLazyHi = FKV_LAZY_HI;
#ifndef FKV_SKIP_EMPTY
#define FKV_SKIP_EMPTY 1
#endif
constexpr bool kSkipEmpty = FKV_SKIP_EMPTY;  // key warps skip the softmax of a chunk with no used query column
constexpr int kKlBufs = 4;
// TMEM columns (Cfg::tS / tO / tA): S^T[2 buffers] 0..127 | O^T, A^T of accumulator set 0 at 128, 192 |
// NONE: set 1 at 256, 320 (double-buffered across items) | DEFERRED: K_lora [wg][4 bufs] x 32 at 256..511.
constexpr uint32_t T_KL = 256;

template <bool kDef, int kRowsT>
struct Cfg {
  static constexpr int ROWS = kRowsT, SLOTS = kRowsT / 16;
  // NONE, 64 rows: PV as O_ext = P [V | R_v of the 4 slots] with the query rows on the TMEM lanes: 8 MMA
  // instructions of N = 192 per tile instead of 16 (O^T and A^T separately); row sums on the CUDA cores
  static constexpr bool PVROW = !kDef;
  static constexpr bool ONES = kRowsT == 64 && !PVROW;  // A^T has a free slot for the all-ones rows (row sums l)
  // R_k (small) is single-buffered with its pages L2-prefetched two tiles ahead; V_base / R_v wait for softmax(T):
  // a deeper ring; P^T in 64-key halves so softmax(T+1) overlaps PV(T)
  // K_base ring in 16-KB d-half units (a 128-key tile = 2 units): 4 units = two whole tiles (one 3D TMA box per
  // tile); 128-row CTAs: 3 units (each d-half its own box, S(T+1)'s first half streams in while S(T) runs)
#ifndef FKV_KU64
#define FKV_KU64 4
#endif
#ifndef FKV_VS64
#define FKV_VS64 3
#endif
#ifndef FKV_NPH64
#define FKV_NPH64 4
#endif
#ifndef FKV_NQ64
#define FKV_NQ64 2
#endif
  static constexpr int KU = kRowsT == 128 ? 3 : (kDef ? 4 : FKV_KU64);
  static constexpr int RS = 1;                      // R_k ring (4 KB per slot)
  static constexpr int VS = kRowsT == 128 ? 2 : (kDef ? 3 : FKV_VS64);  // V-side ring (64-key half of V_base | R_v per slot | ones)
  static constexpr int NPH = kRowsT == 128 ? 2 : (kDef ? 4 : FKV_NPH64);  // P^T ring of 64-key halves (PV of half h needs only it)
  static constexpr int NQ = (kDef || kRowsT == 128) ? 1 : FKV_NQ64;  // per-item Q / X buffers (freed by the S-side MMAs)
  static constexpr int NRC = 4;  // per-item header ring (held by the key warps until the item's epilogue)
  // Accumulator layout switches (both measured on B200): split accumulation chains (SH / PAR = 2) do not help, a
  // tcgen05.mma costs ~120 cycles for N <= 128 whether or not it depends on the previous one
  // (tools/ubench_mma.cu); double-buffered O^T / A^T (AB = 2) overlap an item's epilogue with the next item.
  static constexpr int AB = (kDef || kRowsT == 128) ? 1 : 2;  // O^T / A^T accumulator sets in TMEM
  static constexpr int SH = 1;                   // S^T accumulation chains (d-halves)
  static constexpr int PAR = 1;                  // O^T / A^T accumulation chains (key-chunk parity)
  __host__ __device__ static constexpr uint32_t tS(int sb, int h) { return ROWS * sb + 0 * h; }
  __host__ __device__ static constexpr uint32_t tO(int ab, int par) { return 2 * ROWS + 2 * ROWS * ab + 0 * par; }
  __host__ __device__ static constexpr uint32_t tA(int ab, int par) { return 3 * ROWS + 2 * ROWS * ab + 0 * par; }
  static constexpr uint32_t XB = kDef ? 4096 : 512;  // per-slot X image: packed B_k | q~
  static constexpr uint32_t QB = ROWS * 256;         // Q buffer: [2 d-halves][ROWS][128 B]
  static constexpr uint32_t PHB = ROWS * 128;        // P^T half: [ROWS / 64 atoms][64 keys / 8][8][64 cols x 2 B]
  static constexpr uint32_t RB = SLOTS * 4096;       // R_k entry: [slot][128 keys][32 B]
  // V-side entry: PVROW: [V d-half 0 | V d-half 1 | R_v 4 slots interleaved per key] as three SW128 MN-major atoms
  // of 64 columns (8 KB each); otherwise [V half 16 KB | R_v per slot 2 KB | ones 2 KB]
  static constexpr uint32_t VE = 16384 + SLOTS * 2048 + (ONES ? 2048 : 0);
  // PVROW: O_ext [rows on lanes][V d 128 | R_v 16 per slot] at TMEM column 2 ROWS (after the two S^T buffers)
  static constexpr int OXW = 128 + 16 * SLOTS;
  __host__ __device__ static constexpr uint32_t tOX(int ab) { return 2 * ROWS + OXW * ab; }
  static constexpr uint32_t OFF_V = 0;
  static constexpr uint32_t OFF_K = OFF_V + VS * VE;
  static constexpr uint32_t OFF_R = OFF_K + KU * 16384;
  static constexpr uint32_t OFF_Q = OFF_R + RS * RB;
  static constexpr uint32_t OFF_P = OFF_Q + NQ * QB;
  static constexpr uint32_t OFF_X = OFF_P + NPH * PHB;  // [NQ][SLOTS][XB]
  static constexpr uint32_t OFF_MISC = OFF_X + NQ * SLOTS * XB;
  // 64-row NONE: room for the ping-pong variant's per-warpgroup m_run / row-sum buffers (SMEM = 227 KB exactly)
  static constexpr uint32_t MISCB = kRowsT == 128 ? 7168 : (PVROW ? 7168 : 2048);
  static constexpr uint32_t SMEM = OFF_MISC + MISCB;
  static_assert(SMEM <= 232448, "shared memory");
  static_assert(!(kDef && kRowsT != 64), "DEFERRED runs 64-row CTAs");
};

template <class C>
struct kDefOf;
template <bool D, int R>
struct kDefOf<Cfg<D, R>> {
  static constexpr bool value = D;
};
template <class C, bool PP = false>
struct MiscT {
  uint64_t kfull[C::KU], kempty[C::KU], rfull[1], rempty[1], vfull[C::VS], vempty[C::VS], rvfull[C::VS], qfull[2],
      qempty[2], sfull[2], sfree[2], pfull[C::NPH], pfree[C::NPH], accfree[2], recfull[C::NRC], recempty[C::NRC], kl[kDefOf<C>::value ? 4 * kKlBufs : 1];  // kl: DEFERRED klfull | klready
  // running column max (PVROW: two buffers by item parity, reset by the item's end, so items start barrier-free)
  // (PP: [warpgroup][item parity])
  alignas(16) float m_run[(PP ? 4 : C::PVROW ? 2 : 1) * C::ROWS];
  alignas(16) float lw[C::ONES ? 4 : (PP ? 4 : C::PVROW ? 2 : 1) * 4 * C::ROWS];  // row-sum partials per key warp [4][ROWS]
  alignas(16) ItemRecT<C::SLOTS> rec[C::NRC];        // per-item header ring
  uint32_t tmem_base;
};

struct TcMaps {
  // kb: P == 128: 3D {64, 128, 2} (a whole tile, both d-halves), else 2D {64, P}; vb: P >= 64: 3D {64, 64, 2},
  // else 2D {64, P}; rk / rv: the residual pool viewed as 128-byte rows, {64, P / 4} / {64, min(P, 64) / 4}
  CUtensorMap kb, vb, rk, rv, kh;  // kh: K_base d-half boxes {64, 128} (P = 128, 3-unit K ring)
};

struct ItemInfo {
  int h, k0, k1, base_off, warp_off, n_slots, n_groups, n_tiles;
  int g_first[kMaxSlots], g_cnt[kMaxSlots], slot_res[kMaxSlots];
};

__device__ __forceinline__ void load_item(const AttnParams& p, int idx, ItemInfo& I) {
  const DevItem it = p.items[idx];
  I.h = it.kv_head;
  I.k0 = it.key_begin;
  I.k1 = it.key_end;
  I.base_off = it.base_off;
  I.warp_off = it.warp_off;
  I.n_slots = it.n_warps;
  I.n_tiles = (it.key_end - it.key_begin + kTile - 1) / kTile;
  int ng = 0, prev_res = -1, prev_ad = -1;
  for (int o = 0; o < kMaxSlots; ++o) {
    if (o < it.n_warps) {
      const DevWarp w = p.warps[it.warp_off + o];
      I.slot_res[o] = w.res_off;
      if (o > 0 && w.res_off == prev_res && w.adapter_slot == prev_ad) {
        I.g_cnt[ng - 1]++;
      } else {
        I.g_first[ng] = o;
        I.g_cnt[ng] = 1;
        ++ng;
      }
      prev_res = w.res_off;
      prev_ad = w.adapter_slot;
    }
  }
  I.n_groups = ng;
}

// group structure from a staged item header
// tile record (kTileRecInts ints): a = (t0, k1, meta, base page), b / c = residual pages of slots 0..3 / 4..7
struct TileRec {
  int4 a, b, c;
  __device__ __forceinline__ int page(int o) const {
    switch (o) {
      case 0: return b.x; case 1: return b.y; case 2: return b.z; case 3: return b.w;
      case 4: return c.x; case 5: return c.y; case 6: return c.z; default: return c.w;
    }
  }
};

template <class Rec>
__device__ __forceinline__ void item_from_rec(const Rec& r, ItemInfo& I) {
  I.k0 = r.k0;
  I.k1 = r.k1;
  I.n_tiles = r.n_tiles & 0xffff;
  I.n_slots = r.meta & 15;
  int ng = 0;
  for (int o = 0; o < I.n_slots; ++o) {
    if ((r.meta >> (8 + o)) & 1) {
      I.g_first[ng] = o;
      I.g_cnt[ng] = 1;
      ++ng;
    } else {
      I.g_cnt[ng - 1]++;
    }
  }
  I.n_groups = ng;
}

// the fields the key warps need (no per-slot arrays: keeps them in registers)
struct ItemLite {
  int k0, k1, warp_off, n_slots, n_groups, n_tiles;
};
__device__ __forceinline__ void load_item_lite(const AttnParams& p, int idx, ItemLite& I) {
  const DevItem it = p.items[idx];
  I.k0 = it.key_begin;
  I.k1 = it.key_end;
  I.warp_off = it.warp_off;
  I.n_slots = it.n_warps;
  I.n_tiles = (it.key_end - it.key_begin + kTile - 1) / kTile;
  int ng = 0, prev_res = -1, prev_ad = -1;
#pragma unroll
  for (int o = 0; o < kMaxSlots; ++o) {
    if (o < it.n_warps) {
      const DevWarp w = p.warps[it.warp_off + o];
      if (!(o > 0 && w.res_off == prev_res && w.adapter_slot == prev_ad)) ++ng;
      prev_res = w.res_off;
      prev_ad = w.adapter_slot;
    }
  }
  I.n_groups = ng;
}

__device__ __forceinline__ bool bar_or(uint32_t id, uint32_t n, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, %2, %3, p;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

// ---- packed fp32x2 helpers (FFMA2 / FADD2 / FMUL2 on sm_100): the CUDA builtins, so the register allocator
// sees the pairs (no inline-asm moves); a pair travels as one 64-bit value
__device__ __forceinline__ float2 as_f2(uint64_t v) {
  float2 r;
  memcpy(&r, &v, 8);
  return r;
}
__device__ __forceinline__ uint64_t as_u64(float2 v) {
  uint64_t r;
  memcpy(&r, &v, 8);
  return r;
}
__device__ __forceinline__ uint64_t f2(float a, float b) { return as_u64(make_float2(a, b)); }
__device__ __forceinline__ void uf2(uint64_t v, float& a, float& b) {
  const float2 f = as_f2(v);
  a = f.x;
  b = f.y;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) { return as_u64(__fmul2_rn(as_f2(a), as_f2(b))); }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { return as_u64(__fadd2_rn(as_f2(a), as_f2(b))); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  return as_u64(__ffma2_rn(as_f2(a), as_f2(b), as_f2(c)));
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
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;\n" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void unpack_h2(uint32_t v, float& lo, float& hi) {
  asm("{\n\t.reg .f16 l, h;\n\tmov.b32 {l, h}, %2;\n\tcvt.f32.f16 %0, l;\n\tcvt.f32.f16 %1, h;\n\t}\n"
      : "=f"(lo), "=f"(hi)
      : "r"(v));
}
__device__ __forceinline__ void atomic_max_f(float* a, float v) {
  if (v >= 0.f)
    atomicMax((int*)a, __float_as_int(v));
  else
    atomicMin((unsigned int*)a, __float_as_uint(v));
}
// tcgen05 issue from a whole warp: one elected lane issues (uniform operands keep ptxas on the uniform datapath)
__device__ __forceinline__ void mma_ss_e(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_ts_e(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_e(uint32_t mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(mbar)
      : "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
// arrive on `bar` when all of this thread's prior cp.async copies have landed (no count increment)
__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// 32 consecutive bytes (8 fp32 TMEM words) to global memory in one 256-bit store (sm_100)
__device__ __forceinline__ void st_global_v8(float* dst, const uint32_t* x) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(x[0]), "r"(x[1]), "r"(x[2]),
               "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7])
               : "memory");
}

// diagnostics: clock64 stamp of pipeline event e for index j (< 256) of CTA dbg_block (fkv_debug_timeline)
// (EV: the kernel-uniform dbg_on test first, so the stamps cost one predicated branch when off)
// The stamps are compiled out of the product build: their per-site tests cost issue slots in the key warps' loop
// (A/B: C2 main kernel 90.8 -> 88.6 us). tools/timeline.py needs a -DFKV_TIMELINE=1 build
// (bash tools/variants.sh tl -DFKV_TIMELINE=1; FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_tl.so)
#ifndef FKV_TIMELINE
#define FKV_TIMELINE 0
#endif
#if FKV_TIMELINE
#define EV(e, j)                 \
  do {                           \
    if (dbg_on) ev(p, e, j);     \
  } while (0)
#else
#define EV(e, j) \
  do {           \
  } while (0)
#endif
// dbg_on (dbg != null and this CTA is dbg_block) is tested by EV once per site; only the index bound here
__device__ __forceinline__ void ev(const AttnParams& p, int e, uint32_t j) {
  if (j < 256) p.dbg[e * 256 + j] = clock64();
}

// permuted B_k column n' -> d, in 32-column quarter blocks b = 2w + q (w = d-half of key warpgroup w,
// q = quarter): block b holds d = 32w + 16q + [0, 16) followed by the RoPE partners d + 64.
__device__ __forceinline__ int perm_d(int n) {
  const int b = n >> 5, c = n & 31;
  return 32 * (b >> 1) + 16 * (b & 1) + (c < 16 ? c : 64 + c - 16);
}

// ---------------------------------------------------------------------------
// Stage kernel: per warp slot (16 query rows of one owner), the exact shared-
// memory images the main kernel bulk-copies: Q rows (K-major SW128, both
// d-halves, 2 KB each) and q~ = Q B_k^T (NONE, K-major SW32, 512 B) or B_k^h
// with permuted columns (DEFERRED, MN-major SW64 quarter blocks, 4 KB).
__global__ void __launch_bounds__(256) ra_stage_kernel(AttnParams p, int n_images) {
  // Loads and q~ before griddepcontrol.wait, stores after it: the reads (Q rows, B_k, the plan's descriptors) are
  // never written by a kernel that triggers its dependents early (kv_write and the combine wait first; the main
  // kernel, which triggers at entry, writes neither), while the image buffer may still be read by the previous
  // main kernel until the predecessor grid completes. So the loads overlap the predecessor (kv_write) and only
  // the stores wait; the main kernel waits for this grid's completion before it reads the images.
  // The dependents (the main kernel) launch only once every stager CTA has passed griddepcontrol.wait: the
  // main kernel streams K/V pool rows before its own wait, and the predecessor (kv_write) writes the newest ones
  if (!kStageEarly) {
    pdl_wait();
    pdl_trigger();
  }
  const int ii = blockIdx.x;
  if (ii >= n_images) {
    if (kStageEarly) {
      pdl_wait();
      pdl_trigger();
    }
    return;
  }
  __shared__ __align__(16) float qs[16][kD];
  __shared__ int4 dsc[5];  // planner record: B_k^h address, n_rows, kv head, Q row of each of the 16 slot rows
  uint8_t* img = p.stage + (int64_t)ii * kStageBytes;
  const int tid = threadIdx.x;
  if (tid < 5) dsc[tid] = p.stage_desc[5 * ii + tid];
  __syncthreads();
  const int n_rows = dsc[0].z;
  const int* qrows = (const int*)&dsc[1];
  const __nv_bfloat16* Bk = (const __nv_bfloat16*)(((uint64_t)(uint32_t)dsc[0].y << 32) | (uint32_t)dsc[0].x) +
                            (int64_t)p.layer * p.adapter_layer_stride;
  const bool def = p.rope_mode == FKV_ROPE_DEFERRED;
  __shared__ __align__(16) float bs[kR][kD + 4];
  // one 16-byte Q chunk and one B_k^h chunk per thread (16 rows x 16 chunks each, the same index space)
  const int row = tid >> 4, ch = tid & 15, jj = tid >> 4, n8 = (tid & 15) * 8;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (row < n_rows) v = __ldg((const uint4*)((const __nv_bfloat16*)p.Q + (int64_t)qrows[row] * kD) + ch);
  const uint4 bv = __ldg((const uint4*)(Bk + jj * kD + (def ? perm_d(n8) : n8)));
  float acc = 0.f;
  if (!def) {
    const __nv_bfloat162* q2 = (const __nv_bfloat162*)&v;
    const __nv_bfloat162* b2 = (const __nv_bfloat162*)&bv;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(q2[e]), b = __bfloat1622float2(b2[e]);
      qs[row][ch * 8 + 2 * e] = f.x;
      qs[row][ch * 8 + 2 * e + 1] = f.y;
      bs[jj][n8 + 2 * e] = b.x;
      bs[jj][n8 + 2 * e + 1] = b.y;
    }
    // q~[row][j] = sum_d Q[row][d] B_k[j][d], one output per thread (paired FFMA2 over d)
    __syncthreads();
    const int orow = tid >> 4, oj = tid & 15;
    uint64_t acc2 = 0;
#pragma unroll 8
    for (int dd = 0; dd < kD; dd += 4) {
      const float4 qv = *(const float4*)&qs[orow][dd], bv4 = *(const float4*)&bs[oj][dd];
      acc2 = fma2(f2(qv.x, qv.y), f2(bv4.x, bv4.y), acc2);
      acc2 = fma2(f2(qv.z, qv.w), f2(bv4.z, bv4.w), acc2);
    }
    float a0, a1;
    uf2(acc2, a0, a1);
    acc = a0 + a1;
  }
  if (kStageEarly) {
    pdl_wait();     // the predecessor's pool rows are written; the previous main kernel is done with the images
    pdl_trigger();  // only now may the main kernel launch (see above)
  }
  *(uint4*)(img + (ch >> 3) * 2048 + kmajor_off(row, (ch & 7) * 8, 8, 1024, 0)) = v;
  if (def) {
    *(uint4*)(img + 4096 + mnmajor_off(n8, jj, 4, 1024, 512)) = bv;  // packed B_k image (RoPE partner order)
  } else {
    const int orow = tid >> 4, oj = tid & 15;
    *(__nv_bfloat16*)(img + 4096 + kmajor_off(orow, oj, 2, 256, 0)) = __float2bfloat16_rn(orow < n_rows ? acc : 0.f);
  }
}

// ---------------------------------------------------------------------------
template <bool kDef, int kRowsT, bool kPP>
__global__ void __launch_bounds__(384, 1) ra_tc_kernel(const __grid_constant__ TcMaps maps, AttnParams p) {
  using C = Cfg<kDef, kRowsT>;
  // kPP (NONE, 64 rows): ping-pong key warpgroups. Warpgroup w takes the tiles T with T & 1 == w, all 64 query
  // columns, its own running max, row sums, O_ext accumulator (TMEM set w) and partial entries (entry + 16 w), so
  // the two softmax chains run on different tiles and overlap
  static_assert(!kPP || (!kDef && kRowsT == 64), "ping-pong: NONE, 64 rows");
  constexpr bool PP = kPP;
  constexpr int kRows = C::ROWS, kSlots = C::SLOTS;
  using ItemRec = ItemRecT<kSlots>;
  using Misc = MiscT<C, kPP>;
  static_assert(sizeof(Misc) <= C::MISCB, "misc");
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  Misc& ms = *reinterpret_cast<Misc*>(smem + C::OFF_MISC);
  const ItemRec* item_recs = (const ItemRec*)p.item_recs;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  // K ring: d-half h of tile T in unit (2T + h) % KU, its (2T + h) / KU-th use; one 3D box (one barrier) per tile
  // when the two units of a tile are adjacent (KU = 4, P = 128)
  const bool k_single = C::KU % 2 == 0 && p.P == kTile;
  auto k_unit = [](uint32_t T, int h) { return (int)((2 * T + h) % C::KU); };
  auto k_use = [](uint32_t T, int h) { return (2 * T + h) / C::KU; };
  auto k_free = [&](uint32_t T) {  // both units of tile T free (the S MMAs of their previous tile completed)
    bool ok = true;
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (2 * T + h >= (uint32_t)C::KU) ok = ok && mbar_test(smem_u32(&ms.kempty[k_unit(T, h)]), (k_use(T, h) - 1) & 1);
    return ok;
  };
  if (sbase & 1023) __trap();
  const long long t_start = clock64();
  uint64_t g_start = 0;
  if (p.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
  const int cta = blockIdx.x;
  const bool dbg_on = p.dbg != nullptr && cta == p.dbg_block;
  pdl_trigger();  // the combine kernel may be scheduled as CTAs drain (it waits for this grid's completion)
  const int it_begin = p.sched_ptr[cta], it_end = p.sched_ptr[cta + 1];
  const int n_my = it_end - it_begin;
  const int P = p.P;

  // ---------------- setup ----------------
  if (tid == 0) {
    for (int i = 0; i < C::KU; ++i) { mbar_init(smem_u32(&ms.kfull[i]), 1); mbar_init(smem_u32(&ms.kempty[i]), 1); }
    // rfull / rvfull: one cp.async.mbarrier.arrive.noinc per lane of the copying warp
    for (int i = 0; i < C::RS; ++i) { mbar_init(smem_u32(&ms.rfull[i]), 32); mbar_init(smem_u32(&ms.rempty[i]), 1); }
    for (int i = 0; i < C::VS; ++i) {
      mbar_init(smem_u32(&ms.vfull[i]), 1);
      mbar_init(smem_u32(&ms.vempty[i]), 1);
      mbar_init(smem_u32(&ms.rvfull[i]), 32);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&ms.qfull[i]), p.P == kTile ? 32 : 1);  // fast path: one cp.async arrive per lane
      mbar_init(smem_u32(&ms.qempty[i]), 1);  // S-side commit (the last MMA reading Q / X)
      mbar_init(smem_u32(&ms.sfull[i]), 1);
      mbar_init(smem_u32(&ms.sfree[i]), PP ? 128 : 256);
    }
    for (int i = 0; i < C::NPH; ++i) {
      mbar_init(smem_u32(&ms.pfull[i]), PP ? 64 : 128);  // the key threads of one 64-key half (both warpgroups)
      mbar_init(smem_u32(&ms.pfree[i]), 1);
    }
    for (int i = 0; i < C::NRC; ++i) {
      mbar_init(smem_u32(&ms.recfull[i]), p.P == kTile ? 32 : 1);
      mbar_init(smem_u32(&ms.recempty[i]), 2);  // one arrive per key warpgroup after the item's epilogue
    }
    mbar_init(smem_u32(&ms.accfree[0]), PP ? 128 : 256);
    mbar_init(smem_u32(&ms.accfree[1]), PP ? 128 : 256);
    for (int w = 0; w < 2; ++w)
      for (int b = 0; b < kKlBufs; ++b) {
        if (kDef) {
          mbar_init(smem_u32(&ms.kl[w * kKlBufs + b]), 1);                 // klfull
          mbar_init(smem_u32(&ms.kl[2 * kKlBufs + w * kKlBufs + b]), 128);  // klready
        }
      }
    fence_mbar_init();
  }
  if (wid == 11) tmem_alloc(smem_u32(&ms.tmem_base), 512);
  if (kSkip)  // diagnostics: skipped copies leave zeros (finite scores), not stale bytes
    for (uint32_t c = tid; c < C::OFF_MISC / 16; c += 384) *(uint4*)(smem + 16 * c) = make_uint4(0, 0, 0, 0);
  for (int c = tid; c < (PP ? 4 : C::PVROW ? 2 : 1) * C::ROWS; c += 384) ms.m_run[c] = -INFINITY;
  // the all-ones R_v slot (index 4) of every V-side entry: A^T lanes 64..79 accumulate the row sums l
  if (C::ONES)
    for (int c = tid; c < C::VS * 128; c += 384)
      *(uint4*)(smem + C::OFF_V + (c >> 7) * C::VE + 16384 + kSlots * 2048 + (c & 127) * 16) =
        make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = ms.tmem_base;

  if (wid >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (wid == 8 && P == kTile) {
      // ================= producer, fast path (P = 128: one page per tile), whole warp =================
      // TMA (lane 0): K_base tiles; cp.async (all lanes): R_k tiles and the per-item header / Q / X images.
      // Page ids come from the tile records, each stream's next record preloaded (no page-table chasing).
      tma_prefetch_desc(&maps.kb); tma_prefetch_desc(&maps.vb); tma_prefetch_desc(&maps.kh);
      const __nv_bfloat16* rkl = (const __nv_bfloat16*)p.res_k + (int64_t)p.layer * p.res_layer_stride;
      const int64_t brow_l = (int64_t)p.layer * p.nb;
      const int r0 = p.tile_ptr[cta], nrec = p.tile_ptr[cta + 1] - r0;
      auto ldrec = [&](int T, TileRec& r) {
        if (T < nrec) {
          const int4* q = p.tile_recs + (int64_t)(r0 + T) * (kTileRecInts / 4);
          r.a = __ldg(q);
          r.b = __ldg(q + 1);
          r.c = __ldg(q + 2);
        }
      };
      auto base_row = [&](const TileRec& r) {  // 2D-view row of the tile's base page
        return (int)(((brow_l + r.a.w) * p.hkv + (r.a.z >> 16)) * kTile);
      };
      TileRec kR_ = {}, rR = {}, fR = {};
      ldrec(0, kR_);
      rR = kR_;
      constexpr int kPf = 2;  // L2 prefetch distance (tiles) of K_base and R_k
      ldrec(kPf, fR);
      uint32_t nk = 0, nr = 0;
      int iq = 0, irc = 0;
      int qitem = n_my > 0 ? p.sched_items[it_begin] : 0;
      DevItem qit = p.items[qitem];
      for (;;) {
        bool busy = false, progress = false;
        if (nk < (uint32_t)nrec) {  // K_base tile (32 KB: one 3D box, or one 2D box per d-half unit)
          busy = true;
          if (k_free(nk)) {
            if (lane == 0) {
              EV(0, nk);
              if (kSkip & 1) {
                mbar_arrive(smem_u32(&ms.kfull[k_unit(nk, 0)]));
                if (!k_single) mbar_arrive(smem_u32(&ms.kfull[k_unit(nk, 1)]));
              } else if (k_single) {
                const uint32_t bar = smem_u32(&ms.kfull[k_unit(nk, 0)]);
                mbar_expect_tx(bar, 32768);
                // base tiles stream through L2 evict-first: the residual pages (reused by every kv head) and
                // the other row blocks' hits keep their lines (measured +2.6% on C2)
                if (p.l2_evict_first)
                  tma_load_3d_hint(sbase + C::OFF_K + k_unit(nk, 0) * 16384, &maps.kb, 0, base_row(kR_), 0, bar,
                                   l2_policy_evict_first());
                else
                  tma_load_3d(sbase + C::OFF_K + k_unit(nk, 0) * 16384, &maps.kb, 0, base_row(kR_), 0, bar);
              } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const uint32_t bar = smem_u32(&ms.kfull[k_unit(nk, h)]);
                  mbar_expect_tx(bar, 16384);
                  tma_load_2d(sbase + C::OFF_K + k_unit(nk, h) * 16384, &maps.kh, 64 * h, base_row(kR_), bar);
                }
              }
            }
            if (nk + kPf < (uint32_t)nrec) {  // R_k pages of tile nk + kPf -> L2 (one 128-byte line per lane)
#pragma unroll
              for (int o = 0; o < kSlots; ++o)
                if ((fR.a.z >> (8 + o)) & 1)
                  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(rkl + (int64_t)fR.page(o) * kTile * kR + lane * 64));
            }
            ++nk;
            ldrec(nk, kR_);
            ldrec(nk + kPf, fR);
            progress = true;
          }
        }
        if (nr < (uint32_t)nrec) {  // R_k of the tile's groups (cp.async, 4 KB per group)
          busy = true;
          const int slot = nr % C::RS;
          if (nr < (uint32_t)C::RS || mbar_test(smem_u32(&ms.rempty[slot]), ((nr / C::RS) - 1) & 1)) {
            const uint32_t dst = sbase + C::OFF_R + slot * C::RB;
#pragma unroll
            for (int o = 0; o < kSlots; ++o) {
              if (!(kSkip & 4) && ((rR.a.z >> (8 + o)) & 1)) {
                const __nv_bfloat16* src = rkl + (int64_t)rR.page(o) * kTile * kR;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  const int c = lane + 32 * u;
                  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + o * 4096 + c * 16),
                               "l"(src + c * 8)
                               : "memory");
                }
              }
            }
            cp_async_arrive(smem_u32(&ms.rfull[slot]));
            ++nr;
            ldrec(nr, rR);
            progress = true;
          }
        }
        if (iq < n_my) {  // per-item header, Q rows and q~ / packed B_k (staged images): cp.async by all lanes
          busy = true;
          if (iq == 0) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the stager's images are complete
          const int qb = iq % C::NQ;
          if (iq < C::NQ || mbar_test(smem_u32(&ms.qempty[qb]), ((iq / C::NQ) - 1) & 1)) {
            EV(9, iq);
            for (int o = 0; o < qit.n_warps; ++o) {
              const uint8_t* src = p.stage + (int64_t)(qit.pad_[0] + o) * kStageBytes;
#pragma unroll
              for (int u = 0; u < 8; ++u) {  // Q image: 2 x 2 KB
                const int c = lane + 32 * u;
                cp_async16(sbase + C::OFF_Q + qb * C::QB + (c >> 7) * (C::QB / 2) + o * 2048 + (c & 127) * 16, src + c * 16);
              }
              for (int c = lane; c < (int)(C::XB / 16); c += 32)
                cp_async16(sbase + C::OFF_X + qb * kSlots * C::XB + o * C::XB + c * 16, src + 4096 + c * 16);
            }
            cp_async_arrive(smem_u32(&ms.qfull[qb]));
            ++iq;
            if (iq < n_my) {
              qitem = p.sched_items[it_begin + iq];
              qit = p.items[qitem];
            }
            progress = true;
          }
        }
        if (irc < n_my) {  // per-item header ring (runs ahead of the Q images)
          busy = true;
          const int rb = irc % C::NRC;
          if (irc < C::NRC || mbar_test(smem_u32(&ms.recempty[rb]), ((irc / C::NRC) - 1) & 1)) {
            const uint8_t* rsrc = (const uint8_t*)(item_recs + p.sched_items[it_begin + irc]);
            if (lane < (int)(sizeof(ItemRec) / 16)) cp_async16(smem_u32(&ms.rec[rb]) + lane * 16, rsrc + lane * 16);
            cp_async_arrive(smem_u32(&ms.recfull[rb]));
            ++irc;
            progress = true;
          }
        }
        if (!busy) break;
        if (!progress) __nanosleep(FKV_PROD_SLEEP);  // polling warps have issue priority: yield the SMSP to the key warps
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
    } else if (wid == 8 && lane == 0) {
      // ================= TMA producer (generic page size) =================
      tma_prefetch_desc(&maps.kb); tma_prefetch_desc(&maps.vb);
      tma_prefetch_desc(&maps.rk); tma_prefetch_desc(&maps.rv);
      const int64_t brow_l = (int64_t)p.layer * p.nb;  // 2D views: row = ((layer*NB + page)*Hkv + h)*P + key
      const int Pm = P < 64 ? P : 64;
      const int pf = p.tc_prefetch;
      ItemInfo Ik, Iv;
      int ik = 0, jk = 0, iv = 0, jv = 0, eh = 0, iq = 0, irc = 0;
      uint32_t nk = 0, nv = 0;
      if (n_my > 0) { load_item(p, p.sched_items[it_begin], Ik); Iv = Ik; }
      auto brow = [&](const ItemInfo& I, int sl) {
        return (int)(((brow_l + p.base_pages[I.base_off + sl]) * p.hkv + I.h) * P);
      };
      auto next = [&](int& i, int& j, ItemInfo& I) {
        if (++j == I.n_tiles) {
          j = 0;
          if (++i < n_my) load_item(p, p.sched_items[it_begin + i], I);
        }
      };
      for (;;) {
        bool busy = false, progress = false;
        // K_base tile (32 KB)
        if (ik < n_my) {
          busy = true;
          if (k_free(nk)) {
            EV(0, nk);
            const int t0 = Ik.k0 + jk * kTile;
            if (pf > 0 && P == kTile) {
              // L2 prefetch of the K_base / V_base tiles pf tiles ahead (L2 is the deep buffer, smem the short one)
              int pi = ik, pj = jk + pf;
              while (pi < n_my && pj >= (pi == ik ? Ik.n_tiles : 1 << 30)) { pj -= Ik.n_tiles; ++pi; break; }
              if (pi == ik && pj < Ik.n_tiles) {
                const int tp = Ik.k0 + pj * kTile;
                const int row = brow(Ik, tp / P);
                tma_prefetch_l2_3d(&maps.kb, 0, row, 0);
                tma_prefetch_l2_3d(&maps.vb, 0, row, 0);
                tma_prefetch_l2_3d(&maps.vb, 0, row + 64, 0);
              }
            }
            if (k_single) {
              const uint32_t bar = smem_u32(&ms.kfull[k_unit(nk, 0)]);
              mbar_expect_tx(bar, 32768);
              tma_load_3d(sbase + C::OFF_K + k_unit(nk, 0) * 16384, &maps.kb, 0,
                          brow(Ik, (t0 < Ik.k1 ? t0 : Ik.k0) / P), 0, bar);
            } else {
              for (int h = 0; h < 2; ++h) {
                const uint32_t dst = sbase + C::OFF_K + k_unit(nk, h) * 16384, bar = smem_u32(&ms.kfull[k_unit(nk, h)]);
                mbar_expect_tx(bar, 16384);
                for (int q = 0; q < kTile / P; ++q) {
                  const int t = t0 + q * P;
                  const int row = brow(Ik, (t < Ik.k1 ? t : Ik.k0) / P);
                  if (P == kTile)
                    tma_load_2d(dst, &maps.kh, 64 * h, row, bar);
                  else
                    tma_load_2d(dst + q * P * 128, &maps.kb, 64 * h, row, bar);
                }
              }
            }
            ++nk;
            progress = true;
            next(ik, jk, Ik);
          }
        }
        // V-side: 64-key half of V_base (16 KB); the residual loader warp adds R_v of every slot
        if (iv < n_my) {
          busy = true;
          const int slot = nv % C::VS;
          if (nv < (uint32_t)C::VS || mbar_test(smem_u32(&ms.vempty[slot]), ((nv / C::VS) - 1) & 1)) {
            const uint32_t dst = sbase + C::OFF_V + slot * C::VE, bar = smem_u32(&ms.vfull[slot]);
            EV(7, nv);
            mbar_expect_tx(bar, 16384);
            for (int q = 0; q < 64 / Pm; ++q) {
              const int t = Iv.k0 + jv * kTile + 64 * eh + q * Pm;
              const int tt = t < Iv.k1 ? t : Iv.k0;
              const int sl = tt / P, off = tt % P;
              const int row = brow(Iv, sl) + off;
              if (P >= 64) {
                tma_load_3d(dst, &maps.vb, 0, row, 0, bar);
              } else {
                tma_load_2d(dst + q * Pm * 128, &maps.vb, 0, row, bar);
                tma_load_2d(dst + 8192 + q * Pm * 128, &maps.vb, 64, row, bar);
              }
            }
            ++nv;
            progress = true;
            if (++eh == 2) {
              eh = 0;
              next(iv, jv, Iv);
            }
          }
        }
        // per-item Q rows and q~ / packed B_k (staged images)
        if (iq < n_my) {
          busy = true;
          if (iq == 0) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the stager's images are complete
          const int qb = iq % C::NQ;
          if (iq < C::NQ || mbar_test(smem_u32(&ms.qempty[qb]), ((iq / C::NQ) - 1) & 1)) {
            const DevItem it = p.items[p.sched_items[it_begin + iq]];
            EV(9, iq);
            const uint32_t bar = smem_u32(&ms.qfull[qb]);
            mbar_expect_tx(bar, it.n_warps * (4096 + C::XB));
            for (int o = 0; o < it.n_warps; ++o) {
              const uint8_t* src = p.stage + (int64_t)(it.pad_[0] + o) * kStageBytes;
              bulk_g2s(sbase + C::OFF_Q + qb * C::QB + o * 2048, src, 2048, bar);
              bulk_g2s(sbase + C::OFF_Q + qb * C::QB + C::QB / 2 + o * 2048, src + 2048, 2048, bar);
              bulk_g2s(sbase + C::OFF_X + qb * kSlots * C::XB + o * C::XB, src + 4096, C::XB, bar);
            }
            ++iq;
            progress = true;
          }
        }
        if (irc < n_my) {  // per-item header ring
          busy = true;
          const int rb = irc % C::NRC;
          if (irc < C::NRC || mbar_test(smem_u32(&ms.recempty[rb]), ((irc / C::NRC) - 1) & 1)) {
            const uint32_t bar = smem_u32(&ms.recfull[rb]);
            mbar_expect_tx(bar, (uint32_t)sizeof(ItemRec));
            bulk_g2s(smem_u32(&ms.rec[rb]), item_recs + p.sched_items[it_begin + irc], sizeof(ItemRec), bar);
            ++irc;
            progress = true;
          }
        }
        if (!busy) break;
        if (!progress) __nanosleep(FKV_PROD_SLEEP);  // polling warps have issue priority: yield the SMSP to the key warps
      }
    } else if (wid == 9) {
      // ================= S-side MMA issuer (whole warp: uniform operands, one elected lane issues) =================
      const uint32_t id_s = idesc_bf16(128, kRows, false, false);
      const uint32_t id_rb = idesc_bf16(128, 32, false, true);
      uint32_t T = 0, U = 0;
      for (int ii = 0; ii < n_my; ++ii) {
        const int qb = ii % C::NQ;
        const uint32_t qs = sbase + C::OFF_Q + qb * C::QB;
        const uint32_t xs = sbase + C::OFF_X + qb * kSlots * C::XB;
        mbar_wait(smem_u32(&ms.recfull[ii % C::NRC]), (ii / C::NRC) & 1);
        mbar_wait(smem_u32(&ms.qfull[qb]), (ii / C::NQ) & 1);
        EV(10, ii);
        tc_fence_after();
        // group table of the item, packed 8 bits per group: first slot, slot count
        const int meta = ms.rec[ii % C::NRC].meta, n_tiles = ms.rec[ii % C::NRC].n_tiles & 0xffff;
        const int n_slots = meta & 15;
        uint64_t gf = 0, gc = 0;  // 8 bits per group
        int ng = 0;
#pragma unroll
        for (int o = 0; o < kSlots; ++o) {
          if (o < n_slots) {
            if ((meta >> (8 + o)) & 1) {
              gf |= (uint64_t)o << (8 * ng);
              gc |= 1ull << (8 * ng);
              ++ng;
            } else {
              gc += 1ull << (8 * (ng - 1));
            }
          }
        }
        const uint64_t dq = make_desc(qs, 16, 1024, SWZ_128);
        for (int j = 0; j < n_tiles; ++j, ++T) {
          const int sb = T & 1;
          const uint32_t sacc = tm + C::tS(sb, 0);

          const uint32_t rk = sbase + C::OFF_R + (T % C::RS) * C::RB;
          auto base_s = [&]() {  // S^T = K_base Q^T over both d-halves (descriptor + (byte offset >> 4))
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int u = k_unit(T, h);
              if (h == 0 || !k_single) {
                mbar_wait(smem_u32(&ms.kfull[k_single ? k_unit(T, 0) : u]), k_use(T, k_single ? 0 : h) & 1);
                if (h == 0) EV(1, T);
                tc_fence_after();
              }
              const uint64_t dk = make_desc(sbase + C::OFF_K + u * 16384, 16, 1024, SWZ_128);
#pragma unroll
              for (int c = 0; c < 4; ++c)
                mma_ss_e(tm + C::tS(sb, 0), dk + (uint64_t)((c * 32) >> 4),
                         dq + (uint64_t)((h * (C::QB / 2) + c * 32) >> 4), id_s, h > 0 || c > 0);
              mma_commit_e(smem_u32(&ms.kempty[u]));
            }
          };
          if constexpr (!kDef) {
            if (T >= 2) mbar_wait(smem_u32(&ms.sfree[sb]), ((T >> 1) - 1) & 1);
            EV(8, T);
            base_s();
            mbar_wait(smem_u32(&ms.rfull[T % C::RS]), (T / C::RS) & 1);
            tc_fence_after();
            const uint64_t dr = make_desc(rk, 16, 256, SWZ_32), dx = make_desc(xs, 16, 256, SWZ_32);
#pragma unroll
            for (int g = 0; g < kSlots; ++g) {
              if (g < ng) {
                const uint32_t o = (uint32_t)(gf >> (8 * g)) & 0xff, cnt = (uint32_t)(gc >> (8 * g)) & 0xff;
                mma_ss_e(tm + C::tS(sb, C::SH - 1) + 16 * o, dr + (uint64_t)(o * 256), dx + (uint64_t)(o * 32),
                         idesc_bf16(128, 16 * cnt, false, false), 1);
              }
            }
            mma_commit_e(smem_u32(&ms.rempty[T % C::RS]));
          } else {
            // R_k first: the K_lora rebuild units start before the base tile lands
            mbar_wait(smem_u32(&ms.rfull[T % C::RS]), (T / C::RS) & 1);
            tc_fence_after();
            const int n_units = 2 * ng;  // unit k = q * ng + g (quarter-major)
            const uint64_t dr = make_desc(rk, 16, 256, SWZ_32), dx = make_desc(xs, 1024, 512, SWZ_64);
            auto rb = [&](int w, int k) {  // KL[w][b] (fp32, 32 cols) = R_k,g B_k,g[:, quarter block 2w + q]
              const int q = k >= ng, g = k - q * ng;
              const uint32_t o = (uint32_t)(gf >> (8 * g)) & 0xff;
              const uint32_t b = (U + k) % kKlBufs;
              mma_ss_e(tm + T_KL + 128 * w + 32 * b, dr + (uint64_t)(o * 256),
                       dx + (uint64_t)((o * 4096 + (2 * w + q) * 1024) >> 4), id_rb, 0);
              mma_commit_e(smem_u32(&ms.kl[w * kKlBufs + b]));
              if (T == 4) EV(15, 32 * w + k);
            };
            auto ts = [&](int w, int k) {  // S^T[:, rows of g] += RoPE(KL)[bf16, in place] Q_g^T over the unit's 32 d
              const int q = k >= ng, g = k - q * ng;
              const uint32_t o = (uint32_t)(gf >> (8 * g)) & 0xff, cnt = (uint32_t)(gc >> (8 * g)) & 0xff;
              const uint32_t Uk = U + k, b = Uk % kKlBufs;
              if (T == 4) EV(11, 32 * w + k);
              mbar_wait(smem_u32(&ms.kl[2 * kKlBufs + w * kKlBufs + b]), (Uk / kKlBufs) & 1);
              if (T == 4) EV(12, 32 * w + k);
              tc_fence_after();
              const uint32_t id = idesc_bf16(128, 16 * cnt, false, false);
#pragma unroll
              for (int s2 = 0; s2 < 2; ++s2) {
                const uint32_t d = 64 * s2 + 32 * w + 16 * q;
                mma_ts_e(sacc + 16 * o, tm + T_KL + 128 * w + 32 * b + 8 * s2,
                         dq + (uint64_t)(((d >> 6) * (C::QB / 2) + 2048 * o + (d & 63) * 2) >> 4), id, 1);
              }
            };
            for (int k = 0; k < n_units && k < kKlBufs; ++k) { rb(0, k); rb(1, k); }
            if (T >= 2) mbar_wait(smem_u32(&ms.sfree[sb]), ((T >> 1) - 1) & 1);
            EV(8, T);
            base_s();
            for (int k = 0; k < n_units; ++k) {
              ts(0, k);
              ts(1, k);
              if (k + kKlBufs < n_units) { rb(0, k + kKlBufs); rb(1, k + kKlBufs); }
            }
            mma_commit_e(smem_u32(&ms.rempty[T % C::RS]));
            U += n_units;
          }
          mma_commit_e(smem_u32(&ms.sfull[sb]));
          EV(2, T);
        }
        mma_commit_e(smem_u32(&ms.qempty[qb]));
      }
    } else if (wid == 10) {
      // ================= PV-side MMA issuer (whole warp, one elected lane issues) =================
      const uint32_t id_pv = idesc_bf16(128, kRows, true, true);
      const uint32_t id_px = idesc_bf16(128, C::OXW, true, true);
      uint32_t nv = 0, T = 0;
      uint32_t uses[2] = {0, 0};  // PP: items so far whose tiles used accumulator set w
      for (int ii = 0; ii < n_my; ++ii) {
        const int qb = ii % C::NQ;
        mbar_wait(smem_u32(&ms.recfull[ii % C::NRC]), (ii / C::NRC) & 1);
        const int n_tiles = ms.rec[ii % C::NRC].n_tiles & 0xffff;
        for (int j = 0; j < n_tiles; ++j, ++T) {
          const int ab = PP ? (int)(T & 1) : ii % C::AB;
          if constexpr (PP) {
            if (j < 2) {  // the warpgroup's first tile of the item: its previous item's epilogue freed the set
              if (uses[ab] > 0) mbar_wait(smem_u32(&ms.accfree[ab]), (uses[ab] - 1) & 1);
              ++uses[ab];
            }
          } else {
            if (j == 0 && ii >= C::AB) mbar_wait(smem_u32(&ms.accfree[ab]), ((ii / C::AB) - 1) & 1);
          }
          for (int kh = 0; kh < 2; ++kh, ++nv) {
            // P^T half kh of tile T = ring entry nv (the V-side entries run in the same order)
            const int ps = nv % C::NPH;
            mbar_wait(smem_u32(&ms.pfull[ps]), (nv / C::NPH) & 1);
            if (kh == 0) EV(5, T);
            const uint64_t dp = make_desc(sbase + C::OFF_P + ps * C::PHB, 8192, 1024, SWZ_128);
            mbar_wait(smem_u32(&ms.vfull[nv % C::VS]), (nv / C::VS) & 1);
            mbar_wait(smem_u32(&ms.rvfull[nv % C::VS]), (nv / C::VS) & 1);
            EV(6, nv);
            tc_fence_after();
            const uint32_t ve = sbase + C::OFF_V + (nv % C::VS) * C::VE;
            const uint64_t dv = make_desc(ve, 8192, 1024, SWZ_128), da = make_desc(ve + 16384, 2048, 256, SWZ_32);
            if constexpr (C::PVROW) {
              // O_ext[rows on lanes][V d | R_v slots] += P [V | R_v]: A = P from the P^T half (MN-major, the
              // second 64-row atom aliases the first: LBO = 0, lanes 64..127 duplicate the rows), B = the V-side entry
              const uint64_t pa = make_desc(sbase + C::OFF_P + ps * C::PHB, kRows == 128 ? 8192 : 0, 1024, SWZ_128);
#pragma unroll
              for (int s = 0; s < 4; ++s)
                mma_ss_e(tm + C::tOX(ab), pa + (uint64_t)((s * 2048) >> 4), dv + (uint64_t)((s * 2048) >> 4), id_px,
                         (j >= (PP ? 2 : 1) || kh > 0 || s > 0));
              mma_commit_e(smem_u32(&ms.vempty[nv % C::VS]));
              mma_commit_e(smem_u32(&ms.pfree[ps]));
              continue;
            }
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const int ck = 4 * kh + s, par = ck % C::PAR;  // NONE: two chains per accumulator (key-chunk parity)
              const uint64_t bd = dp + (uint64_t)((s * 2048) >> 4);
              const uint32_t acc = (j > 0 || ck >= C::PAR);
              mma_ss_e(tm + C::tO(ab, par), dv + (uint64_t)((s * 2048) >> 4), bd, id_pv, acc);
              mma_ss_e(tm + C::tA(ab, par), da + (uint64_t)((s * 512) >> 4), bd, id_pv, acc);
            }
            mma_commit_e(smem_u32(&ms.vempty[nv % C::VS]));
            mma_commit_e(smem_u32(&ms.pfree[ps]));
          }
          EV(18, T);
        }
      }
    } else if (wid == 11) {
      // ================= V-side loader (whole warp): V_base halves (TMA, lane 0) + R_v (cp.async) =================
      // R_k tiles (per group) and R_v halves (per slot) are many small contiguous pieces (4 KB per page and
      // owner): 16-byte cp.async by 32 lanes keeps them off the TMA engine, whose per-operation cost would
      // otherwise dominate. The page format is the SW32 operand layout already, so copies are verbatim.
      const __nv_bfloat16* rkl = (const __nv_bfloat16*)p.res_k + (int64_t)p.layer * p.res_layer_stride;
      const __nv_bfloat16* rvl = (const __nv_bfloat16*)p.res_v + (int64_t)p.layer * p.res_layer_stride;
      const int Pm = P < 64 ? P : 64;
      auto wait_free = [&](uint32_t bar, uint32_t parity) {
        mbar_wait(bar, parity);
      };
      auto commit = [&](uint32_t full_bar) { cp_async_arrive(full_bar); };
      // destination of 16-B chunk c (key c >> 1, physical page chunk c & 1) of slot o's R_v half: verbatim SW32
      // (per-slot 2 KB operand), or PVROW: column 16 o + 8 hq of the SW128 MN-major [V | R_v] atom, hq the
      // logical half the page's SW32 swizzle put in that chunk
      auto rv_off = [&](int o, int c) -> uint32_t {
        if constexpr (C::PVROW) {
          const int key = c >> 1, hq = (c & 1) ^ ((key >> 2) & 1);
          return mnmajor_off(16 * o + 8 * hq, key, 8, 8192, 1024);
        } else {
          return (uint32_t)(o * 2048 + c * 16);
        }
      };
      if (P == kTile) {
        // fast path: one page per tile; R_v halves only (R_k is streamed by the producer warp); page ids from
        // the tile records (32 per lane batch, the next batch prefetched)
        const int r0 = p.tile_ptr[cta], nrec = p.tile_ptr[cta + 1] - r0;
        TileRec cur = {}, nxt = {};  // lane L holds the record of tile (batch * 32 + L)
        auto load_batch = [&](int base) {
          const int r = base + lane;
          if (r < nrec) {
            const int4* q = p.tile_recs + (int64_t)(r0 + r) * (kTileRecInts / 4);
            nxt.a = __ldg(q);
            nxt.b = __ldg(q + 1);
            nxt.c = __ldg(q + 2);
          }
        };
        load_batch(0);
        for (int T = 0; T < nrec; ++T) {
          if ((T & 31) == 0) {
            cur = nxt;
            load_batch(T + 32);
          }
          const int L = T & 31;
          TileRec rc;
          rc.a = make_int4(0, 0, __shfl_sync(0xffffffffu, cur.a.z, L), __shfl_sync(0xffffffffu, cur.a.w, L));
          rc.b = make_int4(__shfl_sync(0xffffffffu, cur.b.x, L), __shfl_sync(0xffffffffu, cur.b.y, L),
                           __shfl_sync(0xffffffffu, cur.b.z, L), __shfl_sync(0xffffffffu, cur.b.w, L));
          rc.c = make_int4(__shfl_sync(0xffffffffu, cur.c.x, L), __shfl_sync(0xffffffffu, cur.c.y, L),
                           __shfl_sync(0xffffffffu, cur.c.z, L), __shfl_sync(0xffffffffu, cur.c.w, L));
          const int ns = rc.a.z & 15;
          const int vrow = (int)((((int64_t)p.layer * p.nb + rc.a.w) * p.hkv + (rc.a.z >> 16)) * kTile);
          for (int h = 0; h < 2; ++h) {
            const uint32_t nv = 2 * T + h, slot = nv % C::VS;
            if (nv >= (uint32_t)C::VS) wait_free(smem_u32(&ms.vempty[slot]), ((nv / C::VS) - 1) & 1);
            if (lane == 0 && (kSkip & 2)) {
              mbar_arrive(smem_u32(&ms.vfull[slot]));
            } else if (lane == 0) {  // V_base 64-key half (16 KB, one 3D box)
              EV(7, nv);
              const uint32_t bar = smem_u32(&ms.vfull[slot]);
              mbar_expect_tx(bar, 16384);
              if (p.l2_evict_first)
                tma_load_3d_hint(sbase + C::OFF_V + slot * C::VE, &maps.vb, 0, vrow + 64 * h, 0, bar, l2_policy_evict_first());
              else
                tma_load_3d(sbase + C::OFF_V + slot * C::VE, &maps.vb, 0, vrow + 64 * h, 0, bar);
            }
            const uint32_t dst = sbase + C::OFF_V + slot * C::VE + 16384;
#pragma unroll
            for (int o = 0; o < kSlots; ++o) {
              if (!(kSkip & 8) && o < ns) {
                const __nv_bfloat16* src = rvl + ((int64_t)rc.page(o) * kTile + 64 * h) * kR;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const int c = lane + 32 * u;
                  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + rv_off(o, c)),
                               "l"(src + c * 8)
                               : "memory");
                }
              }
            }
            commit(smem_u32(&ms.rvfull[slot]));
          }
        }
      } else {
      uint32_t T = 0;
      for (int ii = 0; ii < n_my; ++ii) {
        ItemInfo I;
        load_item(p, p.sched_items[it_begin + ii], I);
        for (int j = 0; j < I.n_tiles; ++j, ++T) {
          const int t0 = I.k0 + j * kTile;
          {  // R_k of the item's groups: 4 KB per group at the group's first slot
            const int slot = T % C::RS;
            if (T >= (uint32_t)C::RS) wait_free(smem_u32(&ms.rempty[slot]), ((T / C::RS) - 1) & 1);
            const uint32_t dst = sbase + C::OFF_R + slot * C::RB;
            for (int g = 0; g < I.n_groups; ++g) {
              const int o = I.g_first[g];
#pragma unroll
              for (int u = 0; u < 8; ++u) {  // 256 chunks of 16 B = 128 keys x 32 B
                const int c = lane + 32 * u, key = c >> 1;
                const int t = t0 + key;
                const int tt = t < I.k1 ? t : I.k0;
                const int rp = p.res_pages[I.slot_res[o] + tt / P];
                const __nv_bfloat16* src = rkl + ((int64_t)rp * P + tt % P) * kR + (c & 1) * 8;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + o * 4096 + c * 16), "l"(src)
                             : "memory");
              }
            }
            commit(smem_u32(&ms.rfull[slot]));
          }
          for (int h = 0; h < 2; ++h) {  // R_v halves into the V-side entries: 2 KB per slot
            const uint32_t nv = 2 * T + h, slot = nv % C::VS;
            if (nv >= (uint32_t)C::VS) wait_free(smem_u32(&ms.vempty[slot]), ((nv / C::VS) - 1) & 1);
            const uint32_t dst = sbase + C::OFF_V + slot * C::VE + 16384;
            for (int o = 0; o < I.n_slots; ++o) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {  // 128 chunks = 64 keys x 32 B
                const int c = lane + 32 * u, key = c >> 1;
                const int t = t0 + 64 * h + key;
                const int tt = t < I.k1 ? t : I.k0;
                const int rp = p.res_pages[I.slot_res[o] + tt / P];
                const __nv_bfloat16* src = rvl + ((int64_t)rp * P + tt % P) * kR + (c & 1) * 8;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + rv_off(o, c)), "l"(src)
                             : "memory");
              }
            }
            commit(smem_u32(&ms.rvfull[slot]));
          }
        }
      }
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      (void)Pm;
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    // ================= key warps =================
    // thread = key of the tile = TMEM lane; key warpgroup w owns query columns [CPW w, CPW (w + 1)), processed in
    // chunks of 32 (one TMEM load of S^T each); DEFERRED (64-row CTAs): also the d-half w of the K_lora rotation
    constexpr int CPW = PP ? kRows : kRows / 2, NCH = CPW / 32;
    const int w = wid >> 2;                         // key warpgroup 0/1
    const int kl = tid - 128 * w;                   // key within the tile == TMEM lane
    const int wq = wid & 3;                         // warp within the warpgroup (TMEM lane quarter)
    const uint32_t lb = (uint32_t)(32 * wq) << 16;
    const uint32_t bar_id = 1 + w;                  // named barrier of this warpgroup
    const int WOFF = PP ? 0 : CPW * w;              // first query column of this warpgroup
    const uint64_t sc2 = f2(p.scale_log2, p.scale_log2);
    const float scl = p.scale_log2;
    uint32_t T = 0, U = 0;
    // RoPE angle addition: cos/sin(theta_i * kl) of this thread's key offset for frequencies [32w, 32w + 32),
    // packed as fp16 pairs (cos, sin) (|error| <= 2^-12, below the bf16 rounding of K_lora itself)
    uint32_t cst[32];
    if constexpr (kDef) {
      const int row = kl < p.max_pos ? kl : p.max_pos - 1;
      const float4* cp = (const float4*)(p.rope_cos + (int64_t)row * (kD / 2) + 32 * w);
      const float4* sp = (const float4*)(p.rope_sin + (int64_t)row * (kD / 2) + 32 * w);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 a = __ldg(cp + q), b = __ldg(sp + q);
        cst[4 * q] = pack_h2(a.x, b.x); cst[4 * q + 1] = pack_h2(a.y, b.y);
        cst[4 * q + 2] = pack_h2(a.z, b.z); cst[4 * q + 3] = pack_h2(a.w, b.w);
      }
    }
    // partial entries [m, l, acc[128], acc_r[16]] of item ie: l, acc, acc_r (m is written at the item's end), once PV
    // of its last tile Tl completed; then the accumulators and the header are free
    auto epilogue = [&](int ie, uint32_t Tl, int qbe) {
      const ItemRec& Re = ms.rec[qbe];
      const int ab = PP ? w : ie % C::AB, ns = Re.meta & 15;
      for (uint32_t np = 2 * Tl; np < 2 * Tl + 2; ++np) mbar_wait(smem_u32(&ms.pfree[np % C::NPH]), (np / C::NPH) & 1);
      tc_fence_after();
      if constexpr (C::PVROW && kRows == 128) {
        // rows on the TMEM lanes: row c = 32 wq + lane; warpgroup 0 writes acc (columns [0, 128)), warpgroup 1 the
        // row owner's acc_r (one 32-column load covers the two slots of the warp's rows)
        const int c = 32 * wq + lane, o = c >> 4, r = c & 15;
        const bool valid = o < ns && r < Re.n_rows[o];
        float* ent = p.ws + (int64_t)(Re.entry_off[o < ns ? o : 0] + r) * p.entry_stride + kEntAcc;
        if (w == 0) {
#pragma unroll 1
          for (int part = 0; part < 4; ++part) {
            uint32_t x[32];
            FKV_TMEM_LD32(tm + C::tOX(ab) + 32 * part + lb, x);
            tmem_ld_wait();
            if (part == 3) {
              tc_fence_before();
              mbar_arrive(smem_u32(&ms.accfree[ab]));
            }
            if (valid) {
#pragma unroll
              for (int i = 0; i < 4; ++i) st_global_v8(ent + 32 * part + 8 * i, x + 8 * i);
            }
          }
        } else {
          uint32_t x[32];
          FKV_TMEM_LD32(tm + C::tOX(ab) + kD + 32 * wq + lb, x);
          tmem_ld_wait();
          tc_fence_before();
          mbar_arrive(smem_u32(&ms.accfree[ab]));
          if (valid) {
            const bool hi = lane & 16;
#pragma unroll
            for (int i = 0; i < 4; ++i)
              *(float4*)(ent + kD + 4 * i) = make_float4(
                  __uint_as_float(hi ? x[16 + 4 * i] : x[4 * i]), __uint_as_float(hi ? x[17 + 4 * i] : x[4 * i + 1]),
                  __uint_as_float(hi ? x[18 + 4 * i] : x[4 * i + 2]), __uint_as_float(hi ? x[19 + 4 * i] : x[4 * i + 3]));
          }
        }
        named_bar_sync(bar_id, 128);
        if (kl == 0) mbar_arrive(smem_u32(&ms.recempty[qbe]));
        if (tid == 0) EV(27, ie);
        return;
      } else if constexpr (C::PVROW) {
        // rows on the TMEM lanes: row c = 32 (wq & 1) + lane sits in lane quarters wq & 1 and (wq & 1) + 2 (the A
        // operand's second atom duplicates the rows); the lazy rescale keeps columns [0, 96) current in the first
        // copy and [96, 192) in the second, so all 8 key warps share the stores as: warp (w, wq) writes its rows'
        // columns [48 q, 48 q + 48), q = 2 (wq >> 1) + w: acc (16-byte stores) and the row owner's acc_r
        // PP: one warpgroup holds the set, each of its warps writes 96 columns in two 48-column passes
        const int c = 32 * (wq & 1) + lane, o = c >> 4, r = c & 15;
        const bool valid = o < ns && r < Re.n_rows[o];
        float* ent = p.ws + (int64_t)(Re.entry_off[o < ns ? o : 0] + r + (PP ? 16 * w : 0)) * p.entry_stride + kEntAcc;
#pragma unroll 1
        for (int pass = 0; pass < (PP ? 2 : 1); ++pass) {
          const int q = 2 * (wq >> 1) + (PP ? pass : w);
          const uint32_t base = tm + C::tOX(ab) + 48 * q + lb;
          uint32_t x[48];
          if (tid == 0) EV(14, ie);
          FKV_TMEM_LD16(base, x);
          FKV_TMEM_LD16(base + 16, (x + 16));
          FKV_TMEM_LD16(base + 32, (x + 32));
          tmem_ld_wait();
          if (tid == 0) EV(15, ie);
          if (pass == (PP ? 1 : 0)) {
            tc_fence_before();
            mbar_arrive(smem_u32(&ms.accfree[ab]));
          }
          if (valid) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              const int col = 48 * q + 16 * k;  // warp-uniform
              if (col < kD) {
                st_global_v8(ent + col, x + 16 * k);
                st_global_v8(ent + col + 8, x + 16 * k + 8);
              } else if ((col - kD) / 16 == o) {
                st_global_v8(ent + kD, x + 16 * k);
                st_global_v8(ent + kD + 8, x + 16 * k + 8);
              }
            }
          }
        }
        named_bar_sync(bar_id, 128);
        if (kl == 0) mbar_arrive(smem_u32(&ms.recempty[qbe]));
        if (tid == 0) EV(27, ie);
        return;
      }
#pragma unroll 1
      for (int ch = 0; ch < NCH; ++ch) {
        const int cb = WOFF + 32 * ch;
        uint32_t o_[32], a_[32];
        FKV_TMEM_LD32(tm + C::tO(ab, 0) + cb + lb, o_);
        FKV_TMEM_LD32(tm + C::tA(ab, 0) + cb + lb, a_);
        tmem_ld_wait();
        if (ch == NCH - 1) {
          tc_fence_before();
          mbar_arrive(smem_u32(&ms.accfree[ab]));
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int c = cb + i, o = c >> 4, r = c & 15;
          if (o < ns && r < Re.n_rows[o]) {
            float* ent = p.ws + (int64_t)(Re.entry_off[o] + r) * p.entry_stride;
            ent[kEntAcc + kl] = __uint_as_float(o_[i]);                                  // acc[d = kl]
            if ((kl >> 4) == o) ent[kEntAcc + kD + (kl & 15)] = __uint_as_float(a_[i]);  // acc_r[j] of this row's owner
            if (kl == 64) {
              if constexpr (C::ONES) {
                ent[1] = __uint_as_float(a_[i]);  // l (all-ones slot)
              } else {
                ent[1] = ms.lw[c] + ms.lw[kRows + c] + ms.lw[2 * kRows + c] + ms.lw[3 * kRows + c];
              }
            }
          }
        }
      }
      // this warpgroup is done with the item header (and the row-sum partials)
      named_bar_sync(bar_id, 128);
      if (kl == 0) mbar_arrive(smem_u32(&ms.recempty[qbe]));
    };
    int pend_ii = -1, pend_qb = 0;
    uint32_t pend_Tl = 0;
    for (int ii = 0; ii < n_my; ++ii) {
      const int qb = ii % C::NRC;  // header ring entry
      mbar_wait(smem_u32(&ms.recfull[qb]), (ii / C::NRC) & 1);
      const ItemRec& R = ms.rec[qb];
      ItemLite I;
      I.k0 = R.k0;
      I.k1 = R.k1;
      I.n_tiles = R.n_tiles & 0xffff;
      I.n_slots = R.meta & 15;
      I.n_groups = (R.meta >> 4) & 15;
      // PVROW: m_run / row-sum partials double-buffered by item parity (PP: one buffer per warpgroup)
      const int mbuf = PP ? 2 * w + (ii & 1) : (ii & 1);
      float* const mrun = ms.m_run + (C::PVROW ? mbuf * kRows : 0);
      float* const lwb = ms.lw + (C::PVROW ? mbuf * 4 * kRows : 0);
      if constexpr (!C::PVROW) {
        // per-item column state of this warpgroup; the previous item's epilogue is done with m_run / lw
        named_bar_sync(bar_id, 128);
        if (kl < CPW) {
          ms.m_run[CPW * w + kl] = -INFINITY;
          if constexpr (!C::ONES) {
#pragma unroll
            for (int q = 0; q < 4; ++q) ms.lw[q * kRows + CPW * w + kl] = 0.f;
          }
        }
        named_bar_sync(bar_id, 128);
      }
      // lazy start: the item's running max is the m = 0 reference held in registers (lref) until a slow path moves
      // it into m_run (no shared-memory stores from the fast path)
      uint32_t lrefm = 0;  // bit ch: chunk ch runs on the register reference
      // PVROW: this thread's per-column partial row sums (its keys, fp32 p) over the item's tiles, pairs of columns;
      // reduced over the keys once at the item end
      uint64_t lsum2[C::PVROW ? NCH : 1][C::PVROW ? 16 : 1];
#pragma unroll
      for (int ch = 0; ch < (C::PVROW ? NCH : 1); ++ch)
#pragma unroll
        for (int q = 0; q < (C::PVROW ? 16 : 1); ++q) lsum2[ch][q] = 0;
      // bit ch: chunk ch has a query column that does not see every key of the item (planner, n_tiles >> 16)
      const uint32_t causal_mask = ((uint32_t)R.n_tiles >> (16 + (WOFF >> 5))) & ((1u << NCH) - 1);
      // used query columns of each chunk (slot o < n_slots, row < n_rows[o]); unused ones are masked like invisible
      uint32_t colmask[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int o0 = (WOFF + 32 * ch) >> 4;
        const int n0 = o0 < I.n_slots ? R.n_rows[o0] : 0, n1 = o0 + 1 < I.n_slots ? R.n_rows[o0 + 1] : 0;
        colmask[ch] = (n0 >= 16 ? 0xffffu : (1u << n0) - 1) | ((n1 >= 16 ? 0xffffu : (1u << n1) - 1) << 16);
      }
      if (tid == 0) EV(25, ii);
      int jw = -1;          // PP: this warpgroup's tiles of the item so far - 1
      uint32_t Tmine = 0;   // PP: this warpgroup's last tile
      for (int j = 0; j < I.n_tiles; ++j, ++T) {
        if (PP && (int)(T & 1) != w) continue;  // the other warpgroup's tile
        ++jw;
        Tmine = T;
        const int jm = PP ? jw : j;  // index of this tile among the warpgroup's tiles of the item
        const int t0 = I.k0 + j * kTile;
        const int t = t0 + kl;
        const bool tvalid = t < I.k1;
        if constexpr (kDef) {
          const int prow = t0 < p.max_pos ? t0 : p.max_pos - 1;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            // frequencies 32w + 16q + [0, 16): angle addition cos/sin((t0 + kl) theta)
            uint64_t Cs[8], Ss[8], NS[8];
            const float4* cp = (const float4*)(p.rope_cos + (int64_t)prow * (kD / 2) + 32 * w + 16 * q);
            const float4* sp = (const float4*)(p.rope_sin + (int64_t)prow * (kD / 2) + 32 * w + 16 * q);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float4 c0 = __ldg(cp + e), s0 = __ldg(sp + e);
              const float c0v[4] = {c0.x, c0.y, c0.z, c0.w}, s0v[4] = {s0.x, s0.y, s0.z, s0.w};
              float cc[4], ss[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                float a, b;
                unpack_h2(cst[16 * q + 4 * e + u], a, b);
                cc[u] = fmaf(c0v[u], a, -s0v[u] * b);
                ss[u] = fmaf(s0v[u], a, c0v[u] * b);
              }
              Cs[2 * e] = f2(cc[0], cc[1]); Cs[2 * e + 1] = f2(cc[2], cc[3]);
              Ss[2 * e] = f2(ss[0], ss[1]); Ss[2 * e + 1] = f2(ss[2], ss[3]);
              NS[2 * e] = f2(-ss[0], -ss[1]); NS[2 * e + 1] = f2(-ss[2], -ss[3]);
            }
            // two units per step: one TMEM load/store round trip and one barrier wait for both
            // one unit at a time (keeps the key warps within their register budget: no spills)
            for (int g = 0; g < I.n_groups; ++g) {
              uint32_t x[16], y[16], lh[16];
              const uint32_t b = U % kKlBufs;
              mbar_wait(smem_u32(&ms.kl[w * kKlBufs + b]), (U / kKlBufs) & 1);
              if (T == 4 && kl == 0) EV(13, 32 * w + q * I.n_groups + g);
              tc_fence_after();
              const uint32_t kt = tm + T_KL + 128 * w + 32 * b + lb;
              FKV_TMEM_LD16(kt, x);
              FKV_TMEM_LD16(kt + 16, y);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const uint64_t X = f2(__uint_as_float(x[2 * e]), __uint_as_float(x[2 * e + 1]));
                const uint64_t Y = f2(__uint_as_float(y[2 * e]), __uint_as_float(y[2 * e + 1]));
                lh[e] = pack2(fma2(Y, NS[e], mul2(X, Cs[e])));      // x cos - y sin  (d)
                lh[8 + e] = pack2(fma2(X, Ss[e], mul2(Y, Cs[e])));  // x sin + y cos  (d + 64)
              }
              FKV_TMEM_ST16(kt, lh);
              tmem_st_wait();
              tc_fence_before();
              mbar_arrive(smem_u32(&ms.kl[2 * kKlBufs + w * kKlBufs + b]));
              if (T == 4 && kl == 0) EV(14, 32 * w + q * I.n_groups + g);
              ++U;
            }
          }
        }
        const int sb = T & 1;
        // this thread's P^T half (keys 0..63 | 64..127) = ring entry 2T + half
        const uint32_t np = 2 * T + (kl >> 6), ps = np % C::NPH;
        uint8_t* pbuf = smem + C::OFF_P + ps * C::PHB;
        // PP: both chunks unrolled (lsum2[ch] / colmask[ch] stay in registers)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          // ---- online softmax over the chunk's 32 query columns (Alg1.339-341) ----
          if (kSkipEmpty && colmask[ch] == 0u) {
            // no query row of the item in this chunk (a 1-slot private item leaves the second warpgroup idle):
            // only the handshakes (the P^T columns are never read for a used row), the SMSP's MUFU and issue
            // slots go to the other warpgroup's chain
            if (ch == 0) {
              mbar_wait(smem_u32(&ms.sfull[sb]), (T >> 1) & 1);
              tc_fence_after();
            }
            if (ch == NCH - 1) {
              tc_fence_before();
              mbar_arrive(smem_u32(&ms.sfree[sb]));
            }
            if (ch == 0 && np >= (uint32_t)C::NPH) mbar_wait(smem_u32(&ms.pfree[ps]), ((np / C::NPH) - 1) & 1);
            continue;
          }
          const int cb = WOFF + 32 * ch;
          const uint16_t* P1 = R.pos1 + cb;  // key t visible iff t - k0 < P1[c]
          uint32_t vm = tvalid ? colmask[ch] : 0u;
          if (((causal_mask >> ch) & 1) && tvalid) {
            const int tr = t - I.k0;
            vm = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 pv = *(const uint4*)(P1 + 8 * q);
              const uint32_t w4[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                vm |= (uint32_t)(tr < (int)(w4[e] & 0xffffu)) << (8 * q + 2 * e);
                vm |= (uint32_t)(tr < (int)(w4[e] >> 16)) << (8 * q + 2 * e + 1);
              }
            }
          }
          if (ch == 0) {
            mbar_wait(smem_u32(&ms.sfull[sb]), (T >> 1) & 1);
            if (tid == 0) EV(3, T);
            tc_fence_after();
          }
          if constexpr ((kSkip & 32) != 0) {  // diagnostics: null consumer (pipeline handshakes only)
            tc_fence_before();
            mbar_arrive(smem_u32(&ms.sfree[sb]));
            if (np >= (uint32_t)C::NPH) mbar_wait(smem_u32(&ms.pfree[ps]), ((np / C::NPH) - 1) & 1);
            continue;
          }
          uint32_t sr[32];
          FKV_TMEM_LD32(tm + C::tS(sb, 0) + cb + lb, sr);
          tmem_ld_wait();
          if (!kDef && tid == 0) EV(28, T);
          if (ch == NCH - 1) {
            tc_fence_before();
            mbar_arrive(smem_u32(&ms.sfree[sb]));
          }
          uint64_t x2[16];
          float mx = -INFINITY;
          // lazy start (NONE, 64 rows, items whose every query column sees every key): the first tile takes the
          // running max m = 0 as its reference instead of computing the column maxima; the slow path below still
          // runs when a score leaves [-64, kLazyHi] of it (p then stays within [2^-64, 2^kLazyHi]: no bf16 / fp32
          // underflow or overflow)
          const bool lazy0 = C::PVROW && kLazyStart && jm == 0 && causal_mask == 0;
          const bool lref = (lrefm >> ch) & 1u;
          {
            const float4* mp = (const float4*)&mrun[cb];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 m4 = (lazy0 || lref) ? make_float4(0.f, 0.f, 0.f, 0.f) : mp[q];
              const uint64_t s01 = f2(__uint_as_float(sr[4 * q]), __uint_as_float(sr[4 * q + 1]));
              const uint64_t s23 = f2(__uint_as_float(sr[4 * q + 2]), __uint_as_float(sr[4 * q + 3]));
              x2[2 * q] = fma2(s01, sc2, f2(-m4.x, -m4.y));
              x2[2 * q + 1] = fma2(s23, sc2, f2(-m4.z, -m4.w));
            }
            if (vm != 0xffffffffu) {
#pragma unroll
              for (int q = 0; q < 16; ++q) {
                float a, b2;
                uf2(x2[q], a, b2);
                a = (vm >> (2 * q)) & 1u ? a : -INFINITY;
                b2 = (vm >> (2 * q + 1)) & 1u ? b2 : -INFINITY;
                x2[q] = f2(a, b2);
              }
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              float a, b2;
              uf2(x2[q], a, b2);
              mx = max3(mx, a, b2);
            }
          }
          // lazy rescaling: only when some score exceeds the running max by > 2^kLazyHi
          float alpha_l = 1.f;  // this lane's column (cb + lane) rescale factor (row-sum partials)
          if (tid == 0) EV(20, T);
          bool out = mx > kLazyHi;
          if (lazy0) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              float a, b2;
              uf2(x2[q], a, b2);
              out |= (a < -64.f && a > -INFINITY) || (b2 < -64.f && b2 > -INFINITY);
            }
          }
          const bool slow_ = bar_or(bar_id, 128, out);
          if (!kDef && tid == 0) EV(29, T);
          if (slow_) {
            if (tid == 0) EV(21, T);
            // first tile of the item: every column is fresh (m = -inf), nothing to read back or rescale
            const bool first = jm == 0;
            float mo[32];
            if (!first) {
              const float4* mp = (const float4*)&mrun[cb];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 m4 = lref ? make_float4(0.f, 0.f, 0.f, 0.f) : mp[q];
                mo[4 * q] = m4.x; mo[4 * q + 1] = m4.y; mo[4 * q + 2] = m4.z; mo[4 * q + 3] = m4.w;
              }
            }
            const float mo_l = first ? -INFINITY : (lref ? 0.f : mrun[cb + lane]);
            // the register reference becomes m_run's baseline before the atomics (ordered by the barrier below)
            if (lref && wq == 0) mrun[cb + lane] = 0.f;
            float v[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const bool ok = (vm >> c) & 1u;
              v[c] = ok ? __uint_as_float(sr[c]) * scl : -INFINITY;
            }
            // per-column max over the warp's 32 keys (redux.sync.max.f32, sm_100a); lane l keeps column cb + l
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              float r;
              asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v[c]));
              if (lane == c) v[0] = r;
            }
            // lane l holds the warp's max for column cb + l; every thread has read the old maxima (mo)
            if (!first) named_bar_sync(bar_id, 128);
            if (tid == 0) EV(22, T);
            if (v[0] > -INFINITY) atomic_max_f(&mrun[cb + lane], v[0]);
            named_bar_sync(bar_id, 128);
            if (tid == 0) EV(23, T);
            float mn[32];
            bool resc = false;
            {
              const float4* mp = (const float4*)&mrun[cb];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 m4 = mp[q];
                mn[4 * q] = m4.x; mn[4 * q + 1] = m4.y; mn[4 * q + 2] = m4.z; mn[4 * q + 3] = m4.w;
              }
            }
            {
              const float mn_l = mrun[cb + lane];
              alpha_l = mo_l == -INFINITY ? 0.f : ex2(mo_l - mn_l);
            }
            float al[32];
            if (!first) {
#pragma unroll
              for (int c = 0; c < 32; ++c) {  // branch-free: ex2(0) = 1 for unchanged columns
                const bool fresh = mo[c] == -INFINITY;
                al[c] = fresh ? 0.f : ex2(mo[c] - mn[c]);
                resc |= !fresh && (mn[c] != mo[c]);
              }
              if constexpr (C::PVROW) {
#pragma unroll
                for (int q = 0; q < 16; ++q) lsum2[ch][q] = mul2(lsum2[ch][q], f2(al[2 * q], al[2 * q + 1]));
              }
            }
            if (resc && jm > 0) {
              // rescale the chunk's columns of O^T and A^T by alpha (all PV up to tile T-1 complete)
              // all PV into this accumulator set up to the warpgroup's previous tile (PP: T - 2) complete
              for (uint32_t q2 = 2 * (T - (PP ? 2 : 1)); q2 < 2 * (T - (PP ? 1 : 0)); ++q2)
                mbar_wait(smem_u32(&ms.pfree[q2 % C::NPH]), (q2 / C::NPH) & 1);
              tc_fence_after();
              if constexpr (C::PVROW) {
                // rows on lanes, times alpha_l of this lane's row cb + lane. 64 rows: quarters w (columns [0, 96)) and
                // w + 2 (the duplicate rows, columns [96, 192)); 128 rows: quarter 2 w + ch, all 256 columns
                const bool mine = PP ? (wq & 1) == ch : kRows == 64 ? (wq & 1) == w : wq == 2 * w + ch;
                if (mine) {
                  constexpr int NPART = kRows == 64 ? 3 : C::OXW / 32;
                  const uint32_t base = tm + C::tOX(PP ? w : ii % C::AB) + (kRows == 64 ? 96 * (wq >> 1) : 0) + lb;
#pragma unroll 1
                  for (int part = 0; part < NPART; ++part) {
                    uint32_t r[32];
                    FKV_TMEM_LD32(base + 32 * part, r);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha_l);
                    FKV_TMEM_ST16(base + 32 * part, r);
                    FKV_TMEM_ST16(base + 32 * part + 16, (r + 16));
                  }
                }
              } else {
#pragma unroll
                for (int part = 0; part < 2; ++part) {
                  const uint32_t base = tm + ((part & 1) ? C::tA(ii % C::AB, 0) : C::tO(ii % C::AB, 0)) + cb + lb;
                  uint32_t r[32];
                  FKV_TMEM_LD32(base, r);
                  tmem_ld_wait();
#pragma unroll
                  for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * al[i]);
                  FKV_TMEM_ST16(base, r);
                  FKV_TMEM_ST16(base + 16, (r + 16));
                }
              }
              tmem_st_wait();
              tc_fence_before();
            }
            if (tid == 0) EV(24, T);
            // recompute with the updated running max (a column with no visible key keeps -inf -> p = 0)
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float m0 = mn[2 * q], m1 = mn[2 * q + 1];
              const bool ok0 = (vm >> (2 * q)) & 1u;
              const bool ok1 = (vm >> (2 * q + 1)) & 1u;
              const float x0 = ok0 ? __uint_as_float(sr[2 * q]) * scl - (m0 == -INFINITY ? 0.f : m0) : -INFINITY;
              const float x1 = ok1 ? __uint_as_float(sr[2 * q + 1]) * scl - (m1 == -INFINITY ? 0.f : m1) : -INFINITY;
              x2[q] = f2(x0, x1);
            }
            lrefm &= ~(1u << ch);  // m_run holds the chunk's running max from here on
          } else if (lazy0) {
            lrefm |= 1u << ch;  // the m = 0 reference stays (registers)
          }
          // P^T row of this key (bf16, MN-major SW128), the chunk's columns
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            float a, b2;
            uf2(x2[q], a, b2);
            const float ea = (kSkip & 16) ? a : ex2(a), eb = (kSkip & 16) ? b2 : ex2(b2);
            pk[q] = pack_bf16x2(ea, eb);
            if constexpr (C::PVROW) lsum2[ch][q] = fadd2(lsum2[ch][q], f2(ea, eb));
          }
          if (ch == 0) {
            if (tid == 0) EV(16, T);
            if (np >= (uint32_t)C::NPH) mbar_wait(smem_u32(&ms.pfree[ps]), ((np / C::NPH) - 1) & 1);
            if (tid == 0) EV(17, T);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *(uint4*)(pbuf + mnmajor_off(cb + q * 8, kl & 63, 8, 8192, 1024)) =
                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          if (!kDef && tid == 0) EV(11, T);
          if constexpr (!C::ONES && !C::PVROW) {
            // row sums l without an all-ones MMA slot: the warp's 32 keys summed per column (of the bf16 P the
            // MMA uses), lane l -> column cb + l; per-warp partials, rescaled with the running max
            float v[32];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              v[2 * q] = __uint_as_float(pk[q] << 16);
              v[2 * q + 1] = __uint_as_float(pk[q] & 0xffff0000u);
            }
#pragma unroll
            for (int step = 0; step < 5; ++step) {
              const int off = 16 >> step, half = 16 >> step;
              const bool up = lane & off;
#pragma unroll
              for (int i = 0; i < half; ++i) {
                const float send = up ? v[i] : v[i + half];
                const float keep = up ? v[i + half] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
              }
            }
            float* lp = &lwb[wq * kRows + cb + lane];
            *lp = *lp * alpha_l + v[0];
          }
        }
        fence_async_smem();
        if (!kDef && tid == 0) EV(12, T);
        mbar_arrive(smem_u32(&ms.pfull[ps]));
        if (tid == 0) EV(4, T);
        if (C::AB > 1 && jm == 0 && pend_ii >= 0) {
          epilogue(pend_ii, pend_Tl, pend_qb);
          pend_ii = -1;
        }
      }
      // ---- item end: the running max is final -> m of every partial entry now; the accumulators once the
      // last PV completes (NONE 64-row: deferred past the next item's first tile, the PV pipe runs on) ----
      if (tid == 0) EV(26, ii);
      if constexpr (C::PVROW) {
        // m and l of the warpgroup's columns CPW w + kl (the epilogue runs later; m_run / lw are double-buffered):
        // the thread partials reduced over the warp's 32 keys (lane l -> column cb + l), then over the 4 warps
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          float v[32];
#pragma unroll
          for (int q = 0; q < 16; ++q) uf2(lsum2[ch][q], v[2 * q], v[2 * q + 1]);
#pragma unroll
          for (int step = 0; step < 5; ++step) {
            const int off = 16 >> step, half = 16 >> step;
            const bool up = lane & off;
#pragma unroll
            for (int i = 0; i < half; ++i) {
              const float send = up ? v[i] : v[i + half];
              const float keep = up ? v[i + half] : v[i];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
          }
          lwb[wq * kRows + WOFF + 32 * ch + lane] = v[0];
        }
        if (tid == 0) EV(13, ii);
        named_bar_sync(bar_id, 128);
        if (kl < CPW) {
          // PP: a warpgroup without a tile in the item writes l = 0 (the combine skips the entry)
          const int c = WOFF + kl, o = c >> 4, r = c & 15;
          if (o < I.n_slots && r < R.n_rows[o]) {
            float* ent = p.ws + (int64_t)(R.entry_off[o] + r + (PP ? 16 * w : 0)) * p.entry_stride;
            ent[0] = ((lrefm >> (kl >> 5)) & 1u) ? 0.f : mrun[c];  // column c = CPW w + kl is in chunk kl / 32
            ent[1] = lwb[c] + lwb[kRows + c] + lwb[2 * kRows + c] + lwb[3 * kRows + c];
          }
          mrun[c] = -INFINITY;  // this buffer's next item (ii + 2) starts fresh
        }
      } else if (kl == 64) {
#pragma unroll 1
        for (int i = 0; i < CPW; ++i) {
          const int c = CPW * w + i, o = c >> 4, r = c & 15;
          if (o < I.n_slots && r < R.n_rows[o]) p.ws[(int64_t)(R.entry_off[o] + r) * p.entry_stride] = mrun[c];
        }
      }
      if (C::AB == 1) {
        epilogue(ii, T - 1, qb);
      } else if (PP && jw < 0) {
        // PP: no tile of this item for this warpgroup: no accumulator to write; release the header now (an earlier
        // item's epilogue may still be pending)
        named_bar_sync(bar_id, 128);
        if (kl == 0) mbar_arrive(smem_u32(&ms.recempty[qb]));
      } else {
        pend_ii = ii;
        pend_Tl = PP ? Tmine : T - 1;
        pend_qb = qb;
      }
    }
    if (pend_ii >= 0) epilogue(pend_ii, pend_Tl, pend_qb);
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 11) tmem_dealloc(tm, 512);
  if (tid == 0 && p.dbg && cta < 256) {  // diagnostics: per-CTA duration (cycles) and tile count
    p.dbg[30 * 256 + cta] = clock64() - t_start;
    uint64_t g_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
    p.dbg[32 * 256 + cta] = (long long)g_start;  // diagnostics buffer of 34 x 256 (tools/timeline.py)
    p.dbg[33 * 256 + cta] = (long long)g_end;
    p.dbg[31 * 256 + cta] = p.tile_ptr[cta + 1] - p.tile_ptr[cta];
  }
}

}  // namespace

template <bool kDef, int kRowsT, bool kPP = false>
cudaError_t launch_tc_variant(const AttnParams& p, const void* maps, cudaStream_t s) {
  static bool attr[64] = {};  // the max-dynamic-shared-memory opt-in is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    const cudaError_t e = cudaFuncSetAttribute(ra_tc_kernel<kDef, kRowsT, kPP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               Cfg<kDef, kRowsT>::SMEM);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  // programmatic dependent launch: the CTAs start (TMEM, barriers, K / V / residual streaming) while the stager
  // finishes; the producer's griddepcontrol.wait orders the staged-image reads after it
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_ctas);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = Cfg<kDef, kRowsT>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ra_tc_kernel<kDef, kRowsT, kPP>, *(const TcMaps*)maps, p);
}

cudaError_t launch_attention_tc(const AttnParams& p, const void* maps, cudaStream_t s) {
  if (p.n_items == 0) return cudaSuccess;
  if (p.d != kD || p.r != kR || p.dtype != FKV_DTYPE_BF16 || (kTile % p.P) || p.P < 8 || p.n_ctas < 1 || !p.stage)
    return cudaErrorInvalidValue;
  if (p.rope_mode == FKV_ROPE_DEFERRED) {
    if (p.tc_rows != 64) return cudaErrorInvalidValue;
    return launch_tc_variant<true, 64>(p, maps, s);
  }
  if (p.tc_rows == 128) return launch_tc_variant<false, 128>(p, maps, s);
  return p.tc_pp ? launch_tc_variant<false, 64, true>(p, maps, s) : launch_tc_variant<false, 64>(p, maps, s);
}

cudaError_t launch_stage(const AttnParams& p, int32_t n_images, cudaStream_t s) {
  if (n_images <= 0) return cudaSuccess;
  return launch_pdl(ra_stage_kernel, dim3(n_images), dim3(256), 0, s, p, n_images);
}

size_t tc_maps_bytes() { return sizeof(TcMaps); }

}  // namespace k
}  // namespace fkv
