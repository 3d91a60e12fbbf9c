// ResidualAttention on 5th-generation tensor cores, query rows on the TMEM lanes (bf16 in / fp32 accumulate,
// d = 128, r = 16): the hot loop of §8(a) rows a5 (decode) and a7 (chunked prefill), NONE residual-RoPE mode
// (the north-star split, C-1). One persistent CTA per SM walks a static list of plan items
// (rows.hpp); every item holds up to 128 query rows (TMEM lane = row) and a sequence of 128-key tiles.
//
// Per tile (Alg1.332-346 with the split of Eq.4 applied to K and V):
//   S       = Q K_base^T                                  8 x tcgen05.mma M=128 N=keys K=16   [SS]
//   S      += q~_s R_k,s^T   for every residual slot s     1 x MMA per slot, output lanes = the slot's rows
//             (q~ = Q B_k^T per row, computed once per item on the CUDA cores of the aux warpgroup)
//   softmax: per row (thread = lane), lazily rescaled online max (threshold 2^8), P (bf16) back into TMEM
//   O      += P V_base                                    TS MMA (A = P from TMEM), N = 128
//   A_r    += P [R_v,0 | ... | R_v,n-1]                    TS MMA, N = 16 n (stacked slots; each row keeps its
//                                                           own slot's 16 columns, Eq.4 late fusion)
// The combine kernel merges the per-item partials (m, l, O, A_r) and applies O = (acc + acc_r B_v) / l
// (Alg1.348-350) once per output row.
//
// Warp roles (384 threads):
//   warps 0-3  softmax (thread = row = TMEM lane)
//   warp  4    MMA issuer (one thread)
//   warp  5    K_base loader (TMA tensor boxes), warp 7 V_base loader
//   warp  6    R_k and R_v loader (bulk copies of residual pages: the page format is the SW32 operand)
//   warps 8-11 aux: q~ of the next item, Q image of the next item (cp.async), epilogue (TMEM -> partial entries)
//
// Shared memory: Q image 32 KB (SW128 K-major) | q~ images 2 x 4 KB (SW32 K-major) | ring of kNU 16-KB units
// (per tile, in MMA consumption order: K d-half 0, K d-half 1, R_k slots 0-3, [R_k slots 4-7] for S; V keys
// 0-63, R_v keys 0-63, [V keys 64-127, R_v keys 64-127] for PV) | barriers, per-row (m, l) hand-off.
// TMEM (512 columns): S/P buffer 0 [0,128), S/P buffer 1 [128,256), O [256,384), A_r [384,512).
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "kernels.hpp"
#include "rows.hpp"
#include "sm100.cuh"

namespace fkv {
namespace k {
namespace {
using namespace sm100;

constexpr int kNU = 6;  // ring slots
constexpr uint32_t kUnit = 32768;
constexpr uint32_t OFF_QT = 0, OFF_RING = 8192;  // q~ images 2 x 4 KB; the item's Q rows live in TMEM
constexpr uint32_t OFF_BAR = OFF_RING + kNU * kUnit;
// TMEM columns: S/P buffers [0, 256), O [256, 384), A_r [384, 448) (slot s at 16 (s % 4): slots 0-3 and 4-7 share
// the columns through two lane-masked MMAs), Q of the current item [448, 512) (bf16 pairs, the A operand of S)
constexpr uint32_t T_O = 256, T_AR = 384, T_Q = 448;
constexpr int kThreads = 384;
constexpr int kRingConsumers = 9;  // item-queue readers: 4 softmax warps, MMA issuer, K, V, R_k, R_v loaders

struct Bars {
  uint64_t full[kNU], empty[kNU];
  uint64_t s_full[2], p_full[2], o_done, o_final, o_free, q_full, q_empty, qt_full[2], ml_full[2];
  uint32_t tmem_base;
  uint32_t pad_;
  float2 ml[2][kRowsLanes];
  uint64_t ring_full[4], ring_empty[4];  // the CTA's item queue (dynamic schedule, see the aux warpgroup)
  int ring_id[4];
  int issued[kNU];  // per ring slot: the last unit whose MMAs the issuer has issued (monotonic; see ring_wait_free)
  int prog[16];  // diagnostics: per-role progress counters (reported by the deadlock watchdog)
};
// epilogue staging: per aux warp, 8 partial entries of 152 floats (+1 pad word against bank conflicts), so that
// the entries leave as coalesced 128-byte stores instead of 32 rows x 608-byte strides per warp instruction
constexpr int kEpiRows = 8, kEpiStride = 153;
constexpr uint32_t OFF_EPI = (OFF_BAR + (uint32_t)sizeof(Bars) + 127u) & ~127u;
constexpr uint32_t kSmemBytes = OFF_EPI + 4u * kEpiRows * kEpiStride * 4u;
static_assert(kSmemBytes <= 232448, "shared memory");

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
// arrive on `bar` once this thread's prior cp.async copies have landed (pending count +1 now, -1 then)
__device__ __forceinline__ void cp_async_arrive_inc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
// D (+)= A[smem] B[smem]; lanes with a set bit in `dis` keep their D (disable-output-lane)
__device__ __forceinline__ void mma_ss_m(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc, uint4 dis) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc), "r"(dis.x), "r"(dis.y), "r"(dis.z), "r"(dis.w));
}
// issued by the whole MMA warp, one elected lane executes: the operands are warp-uniform, so ptxas keeps them on the
// uniform datapath (a single-lane issuer got an ELECT / R2UR.BROADCAST waterfall loop around every MMA)
__device__ __forceinline__ void mma_ss_me(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc, uint4 dis) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc), "r"(dis.x), "r"(dis.y), "r"(dis.z), "r"(dis.w));
}
__device__ __forceinline__ void mma_ts_me(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc, uint4 dis) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc), "r"(dis.x), "r"(dis.y), "r"(dis.z), "r"(dis.w));
}
__device__ __forceinline__ void mma_commit_e(uint32_t mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(mbar)
      : "memory");
}
// D (+)= A[tmem] B[smem], lane-masked
__device__ __forceinline__ void mma_ts_m(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc, uint4 dis) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc), "r"(dis.x), "r"(dis.y), "r"(dis.z), "r"(dis.w));
}
// mbarrier phase wait: try_wait without a suspend-time hint (the hinted form compiles to NANOSLEEP.SYNCS with a
// 1 ms hint whose wake-up latency cost several microseconds per wait on B200)
// With FKV_HANG_DIAG set, a wait that spins for ~2^27 polls records (block, warp, lane, barrier offset, parity,
// site) into host-mapped memory (fkv_debug_hang_report) and traps, turning a pipeline deadlock into a located error.
__device__ __noinline__ void hang_trap(uint32_t bar, uint32_t parity, long long* hang, int site) {
  extern __shared__ __align__(1024) uint8_t smem[];
  hang[0] = 1;
  hang[1] = blockIdx.x;
  hang[2] = threadIdx.x;
  hang[3] = (long long)(bar - smem_u32(smem));
  hang[4] = parity;
  hang[5] = site;
  const volatile int* pr = reinterpret_cast<const volatile int*>(smem + OFF_BAR + offsetof(Bars, prog));
  for (int i = 0; i < 16; ++i) hang[8 + i] = pr[i];
  __threadfence_system();
  __trap();
}
__device__ __forceinline__ void wait_bar_(uint32_t bar, uint32_t parity, long long* hang, int site) {
  uint32_t ok;
  uint32_t n = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (__builtin_expect(!ok && ++n == (1u << 27), 0) && hang != nullptr) hang_trap(bar, parity, hang, site);
  } while (!ok);
}
#define wait_bar(bar, parity) wait_bar_((bar), (parity), p.hang, __LINE__)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// diagnostics timeline (fkv_debug_timeline): event ev, index i -> dbg[ev * 512 + i] = clock64 of CTA dbg_block
template <bool kDbg>
__device__ __forceinline__ void stamp_(const RowsParams& p, int ev, int i) {
  if (kDbg && (int)blockIdx.x == p.dbg_block && i < 512) p.dbg[ev * 512 + i] = clock64();
}
#define stamp stamp_<kDbg>


template <bool kDbg>
__global__ void __launch_bounds__(kThreads, 1)
    ra_rows_kernel(const __grid_constant__ RowsParams p, const __grid_constant__ RowsMaps maps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const long long t_start = clock64();
  Bars& B = *reinterpret_cast<Bars*>(smem + OFF_BAR);
  const uint32_t sb = smem_u32(smem);
  if (tid == 0) {
    for (int i = 0; i < kNU; ++i) {
      mbar_init(smem_u32(&B.full[i]), 1);
      mbar_init(smem_u32(&B.empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&B.s_full[i]), 1);
      mbar_init(smem_u32(&B.p_full[i]), 4);
      mbar_init(smem_u32(&B.qt_full[i]), 4);
      mbar_init(smem_u32(&B.ml_full[i]), 4);
    }
    mbar_init(smem_u32(&B.o_done), 1);
    mbar_init(smem_u32(&B.o_final), 1);
    mbar_init(smem_u32(&B.o_free), 4);
    mbar_init(smem_u32(&B.q_full), 4);
    mbar_init(smem_u32(&B.q_empty), 1);
    for (int i = 0; i < kNU; ++i) B.issued[i] = -1000;
    for (int i = 0; i < 4; ++i) {
      mbar_init(smem_u32(&B.ring_full[i]), 1);
      mbar_init(smem_u32(&B.ring_empty[i]), kRingConsumers);
    }
    fence_mbar_init();
  }
  // zero the operand buffers once: stale shared memory must hold finite values (keys beyond a ragged tile
  // and empty Q rows are multiplied by zero probabilities / never read, but NaN * 0 would poison a row)
  for (uint32_t i = tid; i < OFF_BAR / 16; i += kThreads) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  // the kernel is a programmatic dependent launch: the pools (kv_write) and Q are the predecessor's outputs, and
  // the predecessor may be another instance of this kernel still holding the SM's tensor memory
  pdl_wait();
  if (wid == 4) tmem_alloc(smem_u32(&B.tmem_base), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = B.tmem_base;
  // ---- the CTA's item queue ------------------------------------------------------------------------------
  // Items are taken dynamically from a global queue (p.sched_items in the planner's cost order, a counter in the
  // workspace): the aux warpgroup takes item k + 1 at the start of item k and publishes it in a 4-entry ring;
  // every other role reads the ring (ring_get blocks, ring_try does not) and releases an item when it is done
  // with it (kRingConsumers arrivals: the 4 softmax warps, the MMA issuer, the K, V and residual loaders). id -1
  // = the queue is exhausted.
  auto ring_get = [&](int k) -> int {
    wait_bar(smem_u32(&B.ring_full[k & 3]), (k >> 2) & 1);
    return *reinterpret_cast<volatile int*>(&B.ring_id[k & 3]);
  };
  auto ring_release = [&](int k) { mbar_arrive(smem_u32(&B.ring_empty[k & 3])); };
  // A producer may refill slot u % kNU once unit u - kNU has been consumed (its MMAs completed: `empty`). The
  // issuer consumes the S-stream and PV-stream units out of order, so a slot's `empty` barrier can lag two
  // phases behind a producer, and a parity wait alone would then pass early (aliasing). The monotonic
  // `issued` word removes the ambiguity: once the issuer has issued unit u - kNU, every earlier phase of the slot
  // has completed (unit u - kNU could only be loaded after u - 2 kNU was consumed), so the parity names one phase.
  auto slot_wait_free = [&](uint32_t u) {
    const uint32_t s_ = u % kNU;
    if (u >= (uint32_t)kNU) {
      uint32_t n = 0;
      while (*reinterpret_cast<volatile int*>(&B.issued[s_]) < (int)u - kNU) {
        if (++n == (1u << 27) && p.hang != nullptr) hang_trap(smem_u32(&B.issued[s_]), u, p.hang, __LINE__);
      }
    }
    wait_bar(smem_u32(&B.empty[s_]), ((u / kNU) & 1) ^ 1);
  };
  // Walk the CTA's ring units in producer order. Over the CTA's flat tile sequence j = 0..N-1 (all items) the
  // 32-KB units of tile j are K 4j, R_k 4j+1, V 4j+2, R_v 4j+3 (unit u uses ring slot u % kNU). With kNU = 6 every
  // unit reuses the slot of a unit consumed more than a tile earlier: K(j) and R_k(j) those of V(j-2) and R_v(j-2),
  // V(j) and R_v(j) those of K(j-1) and R_k(j-1), so both halves of a tile load while the previous tile computes
  // (the MMA issuer consumes the S and PV streams out of order; `slot_wait_free` keeps the slot parity unambiguous).
  // f(kind, u, item, t, tile, n_tiles_of_item, next): kind 0 = K, 1 = V, 2 = R_k, 3 = R_v of tile t of the
  // item-th item; `next` = the next tile (-1 none, -2 not known yet). rel(item) once an item is no longer
  // referenced.
  auto walk = [&](auto&& f, auto&& rel) {
    int id = ring_get(0);
    if (id < 0) return;
    int k = 0, t0 = __ldg(&p.items[id].tile0), n = __ldg(&p.items[id].n_tiles);
    int j = 0;  // flat tile index
    for (;;) {
      int nid = -1, nt0 = -1, nn = 0;
      for (int t = 0; t < n; ++t, ++j) {
        int tn = t0 + t + 1;
        if (t + 1 == n) {
          // the next item may not be published yet (it is published after the epilogue of item k - 1, which waits
          // for this item's V side): only peek here (-2 = unknown) and block after the tile's units
          tn = -2;
          if (mbar_test(smem_u32(&B.ring_full[(k + 1) & 3]), ((k + 1) >> 2) & 1)) {
            const int pid = *reinterpret_cast<volatile int*>(&B.ring_id[(k + 1) & 3]);
            tn = pid >= 0 ? __ldg(&p.items[pid].tile0) : -1;
          }
        }
        f(0, (uint32_t)(4 * j), k, t, t0 + t, n, tn);
        f(2, (uint32_t)(4 * j + 1), k, t, t0 + t, n, tn);
        f(1, (uint32_t)(4 * j + 2), k, t, t0 + t, n, tn);
        f(3, (uint32_t)(4 * j + 3), k, t, t0 + t, n, tn);
        if (t + 1 == n) {
          rel(k);
          nid = ring_get(k + 1);
          if (nid >= 0) {
            nt0 = __ldg(&p.items[nid].tile0);
            nn = __ldg(&p.items[nid].n_tiles);
          }
        }
      }
      if (nid < 0) break;
      ++k;
      t0 = nt0;
      n = nn;
    }
  };
  // register budget per warpgroup (setmaxnreg at the top of each role): softmax 224, loaders / MMA 104, aux 176
  // (x 128 threads = 64512 registers = the CTA allocation of 168 x 384: more would deadlock setmaxnreg.inc; a
  // warpgroup going below the launch count of 168 must use .dec: .inc to a lower count is an illegal instruction).
  // Dependent grids (the combine kernel, or the next instance of this kernel) are released only after every
  // warpgroup has moved its registers (named barrier 1 below): registers freed by setmaxnreg.dec must not be
  // handed to a co-scheduled CTA of another grid before our setmaxnreg.inc claims them (observed on B200 as a
  // hang / launch failure when the trigger came earlier or at the very end).
  auto release_dependents = [&]() {
    named_bar_sync(1, kThreads);
    pdl_trigger();
  };

  if (wid < 4) {
    // ============================ softmax warpgroup: thread = query row = TMEM lane ============================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    release_dependents();
    const uint32_t lane_base = (uint32_t)(32 * wid) << 16;
    const int row = tid;
    int g = 0;
    for (int io = 0;; ++io) {
      const int id = ring_get(io);
      if (id < 0) break;
      const RItem it = p.items[id];
      const RRow rr = p.rows[it.row0 + row];
      float m_run = -INFINITY, l = 0.f;
      RTile T = p.tiles[it.tile0];
      for (int t = 0; t < it.n_tiles; ++t, ++g) {
        const uint32_t lw = __ldg(&p.wus[T.wu].lanes[wid]);
        const int b = g & 1;
        RTile Tn;
        if (t + 1 < it.n_tiles) Tn = p.tiles[it.tile0 + t + 1];
        if (lane == 0) B.prog[wid] = g;
        wait_bar(smem_u32(&B.s_full[b]), (g >> 1) & 1);
        if (tid == 0) stamp(p, 4, g);
        tc_fence_after();
        if (lw != 0u && !(p.flags & 32)) {  // diagnostics: bit 5 skips the softmax work
          const bool active = (lw >> lane) & 1u;
          const uint32_t ts = tm + lane_base + 128u * b;
          uint32_t sr[128];
          FKV_TMEM_LD32(ts + 0, (sr + 0));
          FKV_TMEM_LD32(ts + 32, (sr + 32));
          FKV_TMEM_LD32(ts + 64, (sr + 64));
          FKV_TMEM_LD32(ts + 96, (sr + 96));
          tmem_ld_wait();
          int limit = T.n_keys;
          if (T.flags & kTileCausal) limit = min(limit, rr.pos - T.key0 + 1);
          if (__any_sync(0xffffffffu, limit < 128)) {
#pragma unroll
            for (int c = 0; c < 128; ++c)
              if (c >= limit) sr[c] = __float_as_uint(-INFINITY);
          }
          float mx;
          {
            float m4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float a = __uint_as_float(sr[32 * q]);
#pragma unroll
              for (int c = 1; c < 31; c += 2)
                a = max3(a, __uint_as_float(sr[32 * q + c]), __uint_as_float(sr[32 * q + c + 1]));
              m4[q] = fmaxf(a, __uint_as_float(sr[32 * q + 31]));
            }
            mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * p.scale_log2;
          }
          const bool need = active && mx > m_run + 8.f;
          const bool resc = need && m_run != -INFINITY;
          const float m_new = need ? mx : m_run;
          const float alpha = resc ? ex2(m_run - m_new) : 1.f;
          if (__any_sync(0xffffffffu, resc)) {
            // O and A_r of this warp's rows were last written by PV of the previous tile
            wait_bar(smem_u32(&B.o_done), (g - 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c0 = 0; c0 < 192; c0 += 32) {
              uint32_t o[32];
              FKV_TMEM_LD32(tm + lane_base + T_O + c0, o);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
              FKV_TMEM_ST16(tm + lane_base + T_O + c0, o);
              FKV_TMEM_ST16(tm + lane_base + T_O + c0 + 16, (o + 16));
              tmem_st_wait();
            }
          }
          if (active) {
            m_run = m_new;
            l *= alpha;
          }
          // p = 2^(s * scale_log2 - m): packed fp32x2 FMA, MUFU ex2, bf16 pairs back into the S columns
          const float2 sl2 = make_float2(p.scale_log2, p.scale_log2);
          const float2 nm2 = make_float2(-m_run, -m_run);
          float2 acc2 = make_float2(0.f, 0.f);
          uint32_t pk[64];
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), sl2, nm2);
            x.x = ex2(x.x);
            x.y = ex2(x.y);
            acc2 = __fadd2_rn(acc2, x);
            pk[c] = pack_bf16x2(x.x, x.y);
          }
          FKV_TMEM_ST16(ts + 0, (pk + 0));
          FKV_TMEM_ST16(ts + 16, (pk + 16));
          FKV_TMEM_ST16(ts + 32, (pk + 32));
          FKV_TMEM_ST16(ts + 48, (pk + 48));
          tmem_st_wait();
          if (active) l += acc2.x + acc2.y;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&B.p_full[b]));
        if (tid == 0) stamp(p, 5, g);
        if (t + 1 < it.n_tiles) T = Tn;
      }
      B.ml[io & 1][row] = make_float2(m_run, l);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(smem_u32(&B.ml_full[io & 1]));
        ring_release(io);
      }
    }
  } else if (wid < 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 104;\n" ::: "memory");
    release_dependents();
    if (wid == 4) {
      // ============================ MMA issuer (whole warp, one elected lane issues) ============================
      // Two streams over the CTA's flat tile sequence, issued in whichever order their inputs arrive:
      //   S(k)  = Q K^T + q~ R_k^T        needs K(k), R_k(k) (and the item's Q / q~ images at its first tile);
      //           S(k) may run at most one tile ahead of PV (S buffer k & 1 holds P(k-2) until PV(k-2) is issued);
      //   PV(k) = O += P V, A_r += P R_v  needs softmax(k) done, V(k), R_v(k) (and the epilogue of the previous
      //           item done at an item's first tile).
      // A late K tile then no longer holds up a PV whose data is ready (and vice versa), so ring slots are freed
      // as soon as their MMAs can run. Ring units of tile k (producer order, see walk): K at 2 * ck(k), R_k next;
      // V at 2 * cv(k), R_v next, with ck(0) = 0, ck(k) = 2k - 1, cv(k) = 2k + 2, cv(N - 1) = 2N - 1.
      {
        struct Cur {  // position in the CTA's flat tile sequence; its item comes from the ring (non-blocking)
          int k = 0, id = 0, t = 0, n = 0, t0 = 0;
          bool loaded = false;
        };
        auto try_load = [&](Cur& c) -> bool {
          if (c.loaded) return true;
          if (!mbar_test(smem_u32(&B.ring_full[c.k & 3]), (c.k >> 2) & 1)) return false;
          c.id = *reinterpret_cast<volatile int*>(&B.ring_id[c.k & 3]);
          c.loaded = true;
          if (c.id >= 0) {
            c.t0 = __ldg(&p.items[c.id].tile0);
            c.n = __ldg(&p.items[c.id].n_tiles);
          }
          return true;
        };
        auto advance = [&](Cur& c) -> bool {  // true when c left its item
          if (++c.t < c.n) return false;
          c.t = 0;
          ++c.k;
          c.loaded = false;
          return true;
        };
        Cur cs, cp;
        int ks = 0, kp = 0;  // flat indices of the next S / PV tile
        const uint4 none = make_uint4(0, 0, 0, 0);
        // the next S tile's record, WU lanes and per-slot lane masks, loaded right after the previous S was issued
        // (their global-load latency overlaps the wait for the tile's data); S(k) hands (n_keys, n_slots, flags,
        // lanes) to PV(k) in registers by parity
        int s_nk = 0, s_ns = 0, s_fl = 0, s_wu = 0;
        uint4 s_ml[kRowsMaxSlots];
        auto load_s = [&](const Cur& c) {
          const RTile* Tp = p.tiles + c.t0 + c.t;
          s_nk = __ldg(&Tp->n_keys);
          s_ns = __ldg(&Tp->n_slots);
          s_fl = __ldg(&Tp->flags);
          const int wu = __ldg(&Tp->wu);
          s_wu = wu;
#pragma unroll
          for (int sl = 0; sl < kRowsMaxSlots; ++sl)
            s_ml[sl] = __ldg(reinterpret_cast<const uint4*>(p.wus[wu].slot_lanes[sl]));
        };
        int pv_nk0 = 0, pv_nk1 = 0, pv_ns0 = 0, pv_ns1 = 0, pv_fl0 = 0, pv_fl1 = 0, pv_wu0 = 0, pv_wu1 = 0;
        bool s_rec = false;  // s_* hold the record of cs's tile
        uint32_t spins = 0;
        for (;;) {
          if (try_load(cp) && cp.id < 0) break;  // PV stream done: every tile issued
          bool did = false;
          if (ks <= kp + 1 && try_load(cs) && cs.id >= 0) {
            if (!s_rec) {
              load_s(cs);
              s_rec = true;
            }
            const uint32_t uk = (uint32_t)(4 * ks), ur = uk + 1;
            const bool first = cs.t == 0;
            bool ready = mbar_test(smem_u32(&B.full[uk % kNU]), (uk / kNU) & 1) &&
                         mbar_test(smem_u32(&B.full[ur % kNU]), (ur / kNU) & 1);
            if (ready && first)
              ready = mbar_test(smem_u32(&B.q_full), cs.k & 1) &&
                      mbar_test(smem_u32(&B.qt_full[cs.k & 1]), (cs.k >> 1) & 1);
            if (ready) {
              // ------------------------- S = Q K^T + q~ R_k^T -------------------------
              const int n_keys = s_nk, n_slots = s_ns;
              if (ks & 1) { pv_nk1 = s_nk; pv_ns1 = s_ns; pv_fl1 = s_fl; pv_wu1 = s_wu; }
              else { pv_nk0 = s_nk; pv_ns0 = s_ns; pv_fl0 = s_fl; pv_wu0 = s_wu; }
              stamp(p, 0, ks);
              if (first) stamp(p, 8, cs.k);
              tc_fence_after();
              // Q rows (cp.async) and q~ (st.shared) of a new item are generic-proxy writes; residual pages come by
              // bulk copy (async proxy) unless FKV_ROWS_FLAGS bit 0 selects cp.async
              if (first || (p.flags & 1)) fence_async_smem();
              const int nsk = (n_keys + 15) & ~15;
              const uint32_t idS = idesc_bf16(128, nsk, false, false);
              const uint32_t dS = tm + 128u * (ks & 1);
              const uint32_t kb = sb + OFF_RING + (uk % kNU) * kUnit;
#pragma unroll
              for (int k = 0; k < 8; ++k)
                mma_ts_me(dS, tm + T_Q + 8u * k, make_desc(kb + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, SWZ_128),
                          idS, k != 0, none);
              mma_commit_e(smem_u32(&B.empty[uk % kNU]));
              *reinterpret_cast<volatile int*>(&B.issued[uk % kNU]) = (int)uk;
              const uint32_t qt = sb + OFF_QT + 4096u * (cs.k & 1);
              const uint32_t rb = sb + OFF_RING + (ur % kNU) * kUnit;
              const int nsl = (p.flags & 8) ? 0 : n_slots;  // diagnostics: bit 3 skips the residual S MMAs
#pragma unroll
              for (int sl = 0; sl < kRowsMaxSlots; ++sl)
                if (sl < nsl)
                  mma_ss_me(dS, make_desc(qt, 16, 256, SWZ_32), make_desc(rb + 4096u * sl, 16, 256, SWZ_32), idS, 1u,
                           make_uint4(~s_ml[sl].x, ~s_ml[sl].y, ~s_ml[sl].z, ~s_ml[sl].w));
              mma_commit_e(smem_u32(&B.empty[ur % kNU]));
              *reinterpret_cast<volatile int*>(&B.issued[ur % kNU]) = (int)ur;
              mma_commit_e(smem_u32(&B.s_full[ks & 1]));
              stamp(p, 1, ks);
              if (cs.t == cs.n - 1) mma_commit_e(smem_u32(&B.q_empty));
              ++ks;
              advance(cs);
              s_rec = false;
              if (try_load(cs) && cs.id >= 0) {
                load_s(cs);  // the next S tile's record: its latency overlaps the wait for its data
                s_rec = true;
              }
              did = true;
            }
          }
          if (!did && kp < ks) {
            const uint32_t uv = (uint32_t)(4 * kp + 2), urv = uv + 1;
            const int b = kp & 1;
            bool ready = mbar_test(smem_u32(&B.p_full[b]), (kp >> 1) & 1) &&
                         mbar_test(smem_u32(&B.full[uv % kNU]), (uv / kNU) & 1) &&
                         mbar_test(smem_u32(&B.full[urv % kNU]), (urv / kNU) & 1);
            if (ready && cp.t == 0 && cp.k > 0) ready = mbar_test(smem_u32(&B.o_free), (cp.k - 1) & 1);
            if (ready) {
              // ------------------------- O += P V ; A_r += P R_v -------------------------
              const int n_keys = b ? pv_nk1 : pv_nk0, n_slots = b ? pv_ns1 : pv_ns0;
              const uint32_t acc0 = ((b ? pv_fl1 : pv_fl0) & kTileFirst) ? 0u : 1u;
              const int pwu = b ? pv_wu1 : pv_wu0;
              const uint4 lw = __ldg(reinterpret_cast<const uint4*>(p.wus[pwu].lanes));  // L1: S read these lines
              stamp(p, 2, kp);
              tc_fence_after();
              if (p.flags & 1) fence_async_smem();  // residual pages by cp.async (diagnostics)
              const uint4 dis = make_uint4(~lw.x, ~lw.y, ~lw.z, ~lw.w);
              const uint32_t idV = idesc_bf16(128, 128, false, true);
              // A_r: slots 0-3 (columns 16 s) and slots 4-7 (columns 16 (s - 4)) into the same 64 columns, each MMA
              // writing only its slots' lanes
              const uint4 mlo = __ldg(reinterpret_cast<const uint4*>(p.wus[pwu].lanes_lo));
              const uint4 mhi = __ldg(reinterpret_cast<const uint4*>(p.wus[pwu].lanes_hi));
              const uint4 dlo = make_uint4(~mlo.x, ~mlo.y, ~mlo.z, ~mlo.w), dhi = make_uint4(~mhi.x, ~mhi.y, ~mhi.z, ~mhi.w);
              const uint32_t idR0 = idesc_bf16(128, 16 * min(n_slots, 4), false, true);
              const uint32_t idR1 = idesc_bf16(128, 16 * max(n_slots - 4, 1), false, true);
              const int nk = (n_keys + 15) >> 4;
              const uint32_t pa = tm + 128u * b;
              const uint32_t vb = sb + OFF_RING + (uv % kNU) * kUnit, rvb = sb + OFF_RING + (urv % kNU) * kUnit;
              for (int k = 0; k < nk; ++k) {
                const uint32_t acc = k ? 1u : acc0;
                const uint32_t a = pa + 8u * k;
                mma_ts_me(tm + T_O, a, make_desc(vb + 2048u * k, 16384, 1024, SWZ_128), idV, acc, dis);
                if (!(p.flags & 16)) {  // diagnostics: bit 4 skips the R_v MMAs
                  mma_ts_me(tm + T_AR, a, make_desc(rvb + 512u * k, 4096, 256, SWZ_32), idR0, acc, dlo);
                  if (n_slots > 4)
                    mma_ts_me(tm + T_AR, a, make_desc(rvb + 4u * 4096u + 512u * k, 4096, 256, SWZ_32), idR1, acc, dhi);
                }
              }
              mma_commit_e(smem_u32(&B.empty[uv % kNU]));
              mma_commit_e(smem_u32(&B.empty[urv % kNU]));
              *reinterpret_cast<volatile int*>(&B.issued[uv % kNU]) = (int)uv;
              *reinterpret_cast<volatile int*>(&B.issued[urv % kNU]) = (int)urv;
              mma_commit_e(smem_u32(&B.o_done));
              stamp(p, 3, kp);
              if (cp.t == cp.n - 1) mma_commit_e(smem_u32(&B.o_final));
              ++kp;
              const int kprev = cp.k;
              if (advance(cp) && lane == 0) ring_release(kprev);
              did = true;
            }
          }
          if (!did) {
            B.prog[4] = ks * 1000 + kp;
            if (++spins == (1u << 28) && p.hang != nullptr) hang_trap(0, ks * 1000 + kp, p.hang, __LINE__);
          }
        }
      }
    } else if (wid == 5) {
      // ======= K_base (lane 0) and V_base (lane 1) tiles: one TMA box {64 d, 128 keys, 2 d-halves} per tile =======
      // (P = 128; per-page 2D boxes otherwise). Each lane runs its own walk over its kind's units (one issuing thread
      // streams ~45 B/clk at most, tools/ub_fill.cu: K and V get a thread each); the next tile's record is read one
      // step ahead (its latency overlaps the wait for a free ring slot).
      if (lane < 2) {
        const int my_kind = lane;  // 0 = K, 1 = V
        int kt = 0;
        const int P = p.P;
        const int ppt = 128 / P;  // pages per tile
        const CUtensorMap* m3 = my_kind == 0 ? &maps.k3d : &maps.v3d;
        const CUtensorMap* m2 = my_kind == 0 ? &maps.k2d : &maps.v2d;
        int c_pg = -1, c_h = 0, c_nk = 0, c_bo = 0;
        bool have = false;
        walk([&](int kind, uint32_t u, int, int, int ti, int, int tn) {
          if (kind != my_kind) return;
          if (!have) {
            const RTile* T0 = p.tiles + ti;
            c_pg = __ldg(&T0->base_page); c_h = __ldg(&T0->kv_head); c_nk = __ldg(&T0->n_keys);
            c_bo = __ldg(&T0->base_off);
          }
          int n_pg = -1, n_h = 0, n_nk = 0, n_bo = 0;
          if (tn >= 0) {
            const RTile* Tn = p.tiles + tn;
            n_pg = __ldg(&Tn->base_page); n_h = __ldg(&Tn->kv_head); n_nk = __ldg(&Tn->n_keys);
            n_bo = __ldg(&Tn->base_off);
          }
          const int64_t hrow = (int64_t)c_h * P;
          const uint32_t s_ = u % kNU;
          B.prog[5 + my_kind] = (int)u;
          slot_wait_free(u);
          stamp(p, my_kind == 0 ? 6 : 15, kt);
          const uint32_t dst = sb + OFF_RING + s_ * kUnit;
          if (P == 128) {
            const bool ld = c_pg >= 0 && !(p.flags & 128);  // diagnostics: bit 7 skips the base copies
            mbar_expect_tx(smem_u32(&B.full[s_]), ld ? 32768u : 0u);
            if (ld)
              tma_load_3d(dst, m3, 0, (int)(p.base_rows_layer + (int64_t)c_pg * p.hkv * P + hrow), 0,
                          smem_u32(&B.full[s_]));
          } else {
            int np = 0;
            for (int pi = 0; pi < ppt && pi * P < c_nk; ++pi) np += p.base_pages[c_bo + pi] >= 0;
            mbar_expect_tx(smem_u32(&B.full[s_]), (uint32_t)np * P * 256);
            for (int pi = 0; pi < ppt && pi * P < c_nk; ++pi) {
              const int pg = p.base_pages[c_bo + pi];
              if (pg < 0) continue;
              const int r0 = (int)(p.base_rows_layer + (int64_t)pg * p.hkv * P + hrow);
              tma_load_2d(dst + pi * P * 128, m2, 0, r0, smem_u32(&B.full[s_]));
              tma_load_2d(dst + 16384 + pi * P * 128, m2, 64, r0, smem_u32(&B.full[s_]));
            }
          }
          B.prog[9 + my_kind] = (int)u;
          ++kt;
          c_pg = n_pg; c_h = n_h; c_nk = n_nk; c_bo = n_bo;
          have = tn != -2;
        }, [&](int k) { ring_release(k); });
      }
    } else {
      // ====== residual pages: warp 6 R_k, warp 7 R_v; one bulk copy per (slot, page), lanes in parallel ======
      // lane s owns slot s (P = 128: one page per slot and tile; the next tile's record is read one step ahead)
      const int my_kind = wid == 6 ? 2 : 3;
      const int P = p.P;
      const int ppt = 128 / P;  // pages per slot and tile (<= 8)
      const uint8_t* rp = (const uint8_t*)(my_kind == 3 ? p.res_v : p.res_k) + (size_t)p.layer * p.res_layer_elems * 2;
      int c_pg = -1, c_nk = 0, c_ns = 0;
      bool have = false;
      int kt = 0;
      auto rec = [&](int ti, int& pg, int& nk, int& ns) {
        const RTile* T0 = p.tiles + ti;
        nk = __ldg(&T0->n_keys);
        ns = __ldg(&T0->n_slots);
        pg = (P == 128 && lane < ns) ? p.res_pages[__ldg(&T0->res_off[lane])] : -1;
      };
      walk([&](int kind, uint32_t u, int, int, int ti, int, int tn) {
        if (kind != my_kind) return;
        if (!have) rec(ti, c_pg, c_nk, c_ns);
        const int pg = c_pg, nk = c_nk, ns = c_ns;
        if (tn >= 0) rec(tn, c_pg, c_nk, c_ns);
        have = tn >= 0;  // -2: the next item is not known yet, -1: none
        const RTile* Tp = p.tiles + ti;
        const uint32_t s_ = u % kNU;
        if (lane == 0) B.prog[my_kind == 2 ? 7 : 8] = (int)u;
        slot_wait_free(u);
        if (lane == 0) stamp(p, my_kind == 2 ? 18 : 20, kt);
        const uint32_t dst = sb + OFF_RING + s_ * kUnit;
        if (P == 128 && (p.flags & 1)) {
          // 16-byte cp.async by all lanes (LSU path, per-lane addresses: no uniform-operand waterfall); completion
          // through cp.async.mbarrier.arrive (pending +1 per lane) and one plain arrive
          for (int sl = 0; sl < ns; ++sl) {
            const int pgs = __shfl_sync(0xffffffffu, pg, sl);
            if (pgs < 0) continue;
            const uint8_t* src = rp + (size_t)pgs * 4096;
#pragma unroll
            for (int c = 0; c < 8; ++c) cp_async16(dst + 4096u * sl + 16u * (lane + 32 * c), src + 16 * (lane + 32 * c));
          }
          cp_async_arrive_inc(smem_u32(&B.full[s_]));
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&B.full[s_]));
        } else if (P == 128) {
          const int mine = (pg >= 0 && !(p.flags & 64)) ? 4096 : 0;  // diagnostics: bit 6 skips the residual copies
          int tot = mine;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
          if (lane == 0) mbar_expect_tx(smem_u32(&B.full[s_]), (uint32_t)tot);
          __syncwarp();
          if (mine) bulk_g2s(dst + 4096u * lane, rp + (size_t)pg * 4096, 4096, smem_u32(&B.full[s_]));
        } else {
          // pages of 16..64 tokens: (slot, page) pieces over the lanes (tile fields re-read: not prefetched)
          const int np = ns * ppt;
          int mine = 0;
          for (int q = lane; q < np; q += 32) {
            const int sl = q / ppt, pi = q % ppt;
            if (pi * P < nk && p.res_pages[__ldg(&Tp->res_off[sl]) + pi] >= 0) mine += P * 32;
          }
          int tot = mine;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
          if (lane == 0) mbar_expect_tx(smem_u32(&B.full[s_]), (uint32_t)tot);
          __syncwarp();
          for (int q = lane; q < np; q += 32) {
            const int sl = q / ppt, pi = q % ppt;
            if (pi * P >= nk) continue;
            const int pgq = p.res_pages[__ldg(&Tp->res_off[sl]) + pi];
            if (pgq >= 0)
              bulk_g2s(dst + 4096u * sl + pi * P * 32, rp + (size_t)pgq * P * 32, P * 32, smem_u32(&B.full[s_]));
          }
        }
        if (lane == 0) B.prog[my_kind == 2 ? 11 : 12] = (int)u;
        ++kt;
      }, [&](int k) {
        if (lane == 0) ring_release(k);
      });
    }
  } else {
    // ======================= aux warpgroup: q~, Q image, epilogue (thread = row = TMEM lane) =======================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 176;\n" ::: "memory");
    release_dependents();
    const int row = tid - 256;
    const uint32_t lane_base = (uint32_t)(32 * (wid - 8)) << 16;
    const __nv_bfloat16* Qg = (const __nv_bfloat16*)p.Q;
    // the queue's producer (one thread): take the next item from the global queue and publish it as ring entry k
    auto push = [&](int k) {
      if (row == 0) {
        const int q = atomicAdd(p.ctr, 1);
        const int id = q < p.n_items ? __ldg(&p.sched_items[q]) : -1;
        wait_bar(smem_u32(&B.ring_empty[k & 3]), ((k >> 2) & 1) ^ 1);
        *reinterpret_cast<volatile int*>(&B.ring_id[k & 3]) = id;
        mbar_arrive(smem_u32(&B.ring_full[k & 3]));  // release: the id store is visible to the waiters
      }
    };
    // q~ = Q B_k^h^T (bf16, fp32 accumulate) of item `io` into q~ image io & 1 with warp-level MMA
    // (m16n8k16): the 16 rows of an m16 tile are computed once per distinct (adapter, kv head) among them
    auto qtilde = [&](int io, int id) {
      const RItem it = p.items[id];
      const uint32_t qtb = sb + OFF_QT + 4096u * (io & 1);
      const int gq = lane >> 2, tq = lane & 3;
      for (int mt = 0; mt < 2; ++mt) {
        const int r0 = 32 * (wid - 8) + 16 * mt;
        const RRow ra = p.rows[it.row0 + r0 + gq], rb = p.rows[it.row0 + r0 + gq + 8];
        // A fragments: rows r0 + gq, r0 + gq + 8; k = 16 ks + 2 tq (+1, +8, +9)
        uint32_t af[8][4];
        {
          const uint32_t* qa = (const uint32_t*)(Qg + (size_t)max(ra.q_row, 0) * 128);
          const uint32_t* qb = (const uint32_t*)(Qg + (size_t)max(rb.q_row, 0) * 128);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            af[ks][0] = ra.q_row >= 0 ? __ldg(qa + 8 * ks + tq) : 0u;
            af[ks][1] = rb.q_row >= 0 ? __ldg(qb + 8 * ks + tq) : 0u;
            af[ks][2] = ra.q_row >= 0 ? __ldg(qa + 8 * ks + tq + 4) : 0u;
            af[ks][3] = rb.q_row >= 0 ? __ldg(qb + 8 * ks + tq + 4) : 0u;
          }
        }
        const int meta_a = ra.q_row >= 0 ? (ra.meta >> 8) : -1, meta_b = rb.q_row >= 0 ? (rb.meta >> 8) : -1;
        uint32_t done_a = meta_a < 0, done_b = meta_b < 0;
        while (__any_sync(0xffffffffu, !done_a || !done_b)) {
          // the next (adapter, head) still to compute: the first lane with an undone row
          const uint32_t ba = __ballot_sync(0xffffffffu, !done_a), bbm = __ballot_sync(0xffffffffu, !done_b);
          const int src = ba ? __ffs(ba) - 1 : __ffs(bbm) - 1;
          const int meta = __shfl_sync(0xffffffffu, ba ? meta_a : meta_b, src);
          const int h = meta & 0xff, ad = meta >> 8;
          const uint32_t* bk = (const uint32_t*)((const __nv_bfloat16*)p.adapters[2 * ad] +
                                                 (size_t)p.layer * p.adapter_layer_elems + (size_t)h * 16 * 128);
          float c[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            uint32_t bf[8][2];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              bf[ks][0] = __ldg(bk + (8 * nt + gq) * 64 + 8 * ks + tq);
              bf[ks][1] = __ldg(bk + (8 * nt + gq) * 64 + 8 * ks + tq + 4);
            }
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              asm volatile(
                  "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
                  "{%8, %9}, {%0, %1, %2, %3};\n"
                  : "+f"(c[nt][0]), "+f"(c[nt][1]), "+f"(c[nt][2]), "+f"(c[nt][3])
                  : "r"(af[ks][0]), "r"(af[ks][1]), "r"(af[ks][2]), "r"(af[ks][3]), "r"(bf[ks][0]), "r"(bf[ks][1]));
          }
          // rows of this (adapter, head): store q~[row][8 nt + 2 tq .. +1] into the SW32 K-major image
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const bool mine = half == 0 ? (!done_a && meta_a == meta) : (!done_b && meta_b == meta);
            if (mine) {
              const int r = r0 + gq + 8 * half;
#pragma unroll
              for (int nt = 0; nt < 2; ++nt) {
                const uint32_t v = pack_bf16x2(c[nt][2 * half], c[nt][2 * half + 1]);
                const int j = 8 * nt + 2 * tq;
                const uint32_t addr = qtb + 32u * r + 16u * ((uint32_t)(j >> 3) ^ (uint32_t)((r >> 2) & 1)) + 2u * (j & 7);
                asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
              }
            }
          }
          if (!done_a && meta_a == meta) done_a = 1;
          if (!done_b && meta_b == meta) done_b = 1;
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&B.qt_full[io & 1]));
      if (row == 0) stamp(p, 10, io);
    };
    // Q rows of item `io` into the (single) Q image, SW128 K-major [d-half][row][128 B]
    // Q rows of an item: each aux thread loads its row (TMEM lane) into registers early, and writes it into the Q
    // columns of TMEM (bf16 pairs: the A operand layout of the S MMAs) once the previous item's last S has run
    uint32_t qv[64];
    auto qload = [&](int id) {
      const RItem it = p.items[id];
      const int qr = p.rows[it.row0 + row].q_row;
      const uint4* src = reinterpret_cast<const uint4*>(Qg + (size_t)max(qr, 0) * 128);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const uint4 v = qr >= 0 ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
        qv[4 * c] = v.x; qv[4 * c + 1] = v.y; qv[4 * c + 2] = v.z; qv[4 * c + 3] = v.w;
      }
    };
    auto qstore = [&]() {
      FKV_TMEM_ST16(tm + lane_base + T_Q + 0, (qv + 0));
      FKV_TMEM_ST16(tm + lane_base + T_Q + 16, (qv + 16));
      FKV_TMEM_ST16(tm + lane_base + T_Q + 32, (qv + 32));
      FKV_TMEM_ST16(tm + lane_base + T_Q + 48, (qv + 48));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&B.q_full));
    };
    push(0);
    int id = ring_get(0);
    int n_done = 0;
    if (id >= 0) {
      qload(id);
      qstore();
      qtilde(0, id);
    }
    for (int io = 0; id >= 0; ++io) {
      push(io + 1);
      const int nid = ring_get(io + 1);
      if (nid >= 0) {
        qtilde(io + 1, nid);  // its image buffer was freed by the last S of item io - 1 (waited in the last iteration)
        qload(nid);
        wait_bar(smem_u32(&B.q_empty), io & 1);
        tc_fence_after();
        qstore();
      }
      // epilogue of item io
      if (row == 0) B.prog[13] = io;
      const RItem it = p.items[id];
      const RRow rr = p.rows[it.row0 + row];
      wait_bar(smem_u32(&B.ml_full[io & 1]), (io >> 1) & 1);
      wait_bar(smem_u32(&B.o_final), io & 1);
      if (row == 0) stamp(p, 11, io);
      tc_fence_after();
      float* e = rr.entry >= 0 ? p.ws + (size_t)rr.entry * p.entry_stride : nullptr;
      const float2 ml = B.ml[io & 1][row];
      // O and the row's slot of A_r into registers (all loads in flight together), hand the accumulators back
      // to the next item's PV (o_free) and only then store the partial entry: the stores no longer delay it
      uint32_t o[128], ar[16];
      FKV_TMEM_LD32(tm + lane_base + T_O + 0, (o + 0));
      FKV_TMEM_LD32(tm + lane_base + T_O + 32, (o + 32));
      FKV_TMEM_LD32(tm + lane_base + T_O + 64, (o + 64));
      FKV_TMEM_LD32(tm + lane_base + T_O + 96, (o + 96));
      const int slot = rr.meta & 0xff;
      for (int s = 0; s < kRowsMaxSlots; ++s) {
        if (!__any_sync(0xffffffffu, rr.q_row >= 0 && slot == s)) continue;
        uint32_t t16[16];
        FKV_TMEM_LD16(tm + lane_base + T_AR + 16 * (s & 3), t16);
        tmem_ld_wait();
        if (slot == s) {
#pragma unroll
          for (int j = 0; j < 16; ++j) ar[j] = t16[j];
        }
      }
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&B.o_free));
      // entry = [m, l, pad x 6, acc[128], acc_r[16]] (kEntAcc = 8): staged 8 rows at a time, then each row is
      // written by the whole warp (5 x 128-byte coalesced stores)
      float* stg = reinterpret_cast<float*>(smem + OFF_EPI) + (wid - 8) * kEpiRows * kEpiStride;
      for (int r0 = 0; r0 < 32; r0 += kEpiRows) {
        if (lane >= r0 && lane < r0 + kEpiRows) {
          float* d = stg + (lane - r0) * kEpiStride;
          d[0] = ml.x;
          d[1] = ml.y;
#pragma unroll
          for (int j = 0; j < 6; ++j) d[2 + j] = 0.f;
#pragma unroll
          for (int j = 0; j < 128; ++j) d[kEntAcc + j] = __uint_as_float(o[j]);
#pragma unroll
          for (int j = 0; j < 16; ++j) d[kEntAcc + 128 + j] = __uint_as_float(ar[j]);
        }
        __syncwarp();
#pragma unroll 1
        for (int q = 0; q < kEpiRows; ++q) {
          const int ent = __shfl_sync(0xffffffffu, rr.entry, r0 + q);
          if (ent >= 0) {
            float* g = p.ws + (size_t)ent * p.entry_stride;
            const float* sr = stg + q * kEpiStride;
#pragma unroll
            for (int c = 0; c < 5; ++c)
              if (lane + 32 * c < kEntAcc + 128 + 16) g[lane + 32 * c] = sr[lane + 32 * c];
          }
        }
        __syncwarp();
      }
      (void)e;
      if (row == 0) stamp(p, 12, io);
      ++n_done;
      id = nid;
    }
    if (row == 0) B.prog[15] = n_done;
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (wid == 4) tmem_dealloc(tm, 512);
  if (tid == 0) {
    // the last CTA to finish resets the queue counters for the next launch over the same workspace
    __threadfence();
    if (atomicAdd(p.ctr + 1, 1) == (int)gridDim.x - 1) {
      p.ctr[0] = 0;
      p.ctr[1] = 0;
      __threadfence();
    }
  }
  if (kDbg && tid == 0 && blockIdx.x < 512) {
    p.dbg[30 * 512 + blockIdx.x] = clock64() - t_start;
    p.dbg[31 * 512 + blockIdx.x] = B.prog[15];
  }
}

}  // namespace

long long* hang_slot() {
  static long long* host = nullptr;
  static long long* devp = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    if (std::getenv("FKV_HANG_DIAG") &&
        cudaHostAlloc((void**)&host, 32 * sizeof(long long), cudaHostAllocMapped) == cudaSuccess) {
      for (int i = 0; i < 32; ++i) host[i] = 0;
      if (cudaHostGetDevicePointer((void**)&devp, host, 0) != cudaSuccess) devp = nullptr;
    }
  }
  return devp;
}

// the report (host side of hang_slot): "" if no deadlock was recorded
std::string hang_report() {
  hang_slot();
  static long long* h = nullptr;
  if (!h) {
    long long* d = hang_slot();
    if (!d) return "";
    cudaHostGetDevicePointer((void**)&h, d, 0);  // unused: the mapped host pointer equals the device one on UVA
    h = d;
  }
  if (h[0] == 0) return "";
  char buf[512];
  int n = std::snprintf(buf, sizeof(buf),
                        "rows kernel deadlock: block %lld thread %lld barrier@smem+%lld parity %lld (ra_rows.cu:%lld); "
                        "progress softmax g %lld %lld %lld %lld | mma u %lld | K wait %lld issued %lld | res wait %lld "
                        "issued %lld | V wait %lld issued %lld | aux io %lld",
                        h[1], h[2], h[3], h[4], h[5], h[8], h[9], h[10], h[11], h[12], h[13], h[17], h[14], h[18], h[15],
                        h[19], h[16]);
  (void)n;
  return buf;
}

cudaError_t launch_attention_rows(const RowsParams& p, const RowsMaps& maps, cudaStream_t s) {
  // the max-dynamic-shared-memory opt-in is per device
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(ra_rows_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(ra_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  if (p.n_ctas <= 0) return cudaSuccess;
  // plain stream-ordered launch: as a programmatic dependent launch (either trigger placement) back-to-back
  // instances or an early-scheduled combine grid hung / failed on B200; FKV_ROWS_FLAGS bit 1
  // selects the PDL launch for experiments
  if (p.flags & 2) {
    if (p.dbg != nullptr) return launch_pdl(ra_rows_kernel<true>, dim3(p.n_ctas), dim3(kThreads), kSmemBytes, s, p, maps);
    return launch_pdl(ra_rows_kernel<false>, dim3(p.n_ctas), dim3(kThreads), kSmemBytes, s, p, maps);
  }
  if (p.dbg != nullptr) ra_rows_kernel<true><<<p.n_ctas, kThreads, kSmemBytes, s>>>(p, maps);
  else ra_rows_kernel<false><<<p.n_ctas, kThreads, kSmemBytes, s>>>(p, maps);
  return cudaGetLastError();
}

}  // namespace k
}  // namespace fkv
