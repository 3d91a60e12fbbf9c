// Grouped ResidualAttention, bf16 in / fp32 accumulate, d = 128, r = 16.
// Tensor-core path v1 (warp-level mma.sync.m16n8k16; the tcgen05 kernel in
// ra_tc.cu replaces it on the hot shared-prefix items).
//
// One CTA = one plan item: a kv head h, a key range [k0, k1) of a base-page
// segment shared by all the CTA's rows, and up to 8 warps. Each warp owns 16
// query rows of ONE residual owner (same adapter, same residual pages).
// Per 64-key tile (cp.async double buffered, pages gathered through the
// block tables):
//   Stage 1 (Alg1.332-336):  S  = Q K_base^T                     (shared tile)
//            DEFERRED:       S += Q RoPE_t(R_k B_k^h)^T          (K_lora rebuilt
//                            per 16-key m-tile in registers: the fp32 mma
//                            accumulator fragment of R_k B_k IS the B-operand
//                            fragment of Q K^T after rotation + bf16 packing)
//            NONE:           S += (Q B_k^T) R_k^T                (north-star split)
//   Stage 2 (Alg1.338-346):  one online softmax (m, l) per row,
//                            acc += P V_base, acc_r += P R_v
//   Stage 3 (Alg1.348-350) is applied once per row in the combine kernel.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace fkv {
namespace k {
namespace {

constexpr int kD = 128;
constexpr int kR = 16;
constexpr int kTile = 64;
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kKVStride = kD + 8;                      // padded row (elements) -> conflict-free ldmatrix
constexpr int kKVBytes = kTile * kKVStride * 2;         // 17408
constexpr int kRBytes = kTile * kR * 2;                 // 2048 per warp per tensor
constexpr int kStageBytes = 2 * kKVBytes + 2 * kWarps * kRBytes;  // K, V, Rk[8], Rv[8]
constexpr int kBkBytes = kR * kD * 2;                   // 4096 per warp
constexpr int kSmemBytes = 2 * kStageBytes + kWarps * kBkBytes;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr));
}

// D += A(16x16, row) * B(16x8, col), bf16 inputs, fp32 accumulate
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// R tiles: [64 keys][2 x 16B chunks], chunk swizzled by bit 2 of the key.
__device__ __forceinline__ uint32_t r_off(int key, int chunk) {
  return key * 32 + ((chunk ^ ((key >> 2) & 1)) << 4);
}
// B_k tile: [16 rows][16 x 16B chunks], chunk swizzled by row & 7.
__device__ __forceinline__ uint32_t bk_off(int row, int chunk) { return row * 256 + ((chunk ^ (row & 7)) << 4); }

__global__ void __launch_bounds__(kThreads, 1) ra_mma_kernel(AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const DevItem it = p.items[blockIdx.x];
  const bool active = wid < it.n_warps;
  const int h = it.kv_head;
  const int P = p.P;
  const __nv_bfloat16* Kb = (const __nv_bfloat16*)p.base_k + (int64_t)p.layer * p.base_layer_stride;
  const __nv_bfloat16* Vb = (const __nv_bfloat16*)p.base_v + (int64_t)p.layer * p.base_layer_stride;
  const __nv_bfloat16* Rk = (const __nv_bfloat16*)p.res_k + (int64_t)p.layer * p.res_layer_stride;
  const __nv_bfloat16* Rv = (const __nv_bfloat16*)p.res_v + (int64_t)p.layer * p.res_layer_stride;
  DevWarp w{};
  if (active) w = p.warps[it.warp_off + wid];
  uint8_t* bk_s = smem + 2 * kStageBytes + wid * kBkBytes;
  // ---- B_k^h of this warp's adapter -> smem (swizzled) ----
  if (active) {
    const __nv_bfloat16* Bk = (const __nv_bfloat16*)p.adapters[2 * w.adapter_slot] +
                              (int64_t)p.layer * p.adapter_layer_stride + (int64_t)h * kR * kD;
    for (int c = lane; c < kR * 16; c += 32) {
      const int row = c >> 4, ch = c & 15;
      cp_async16(smem_u32(bk_s + bk_off(row, ch)), Bk + row * kD + ch * 8, true);
    }
  }
  const int n_tiles = (it.key_end - it.key_begin + kTile - 1) / kTile;

  auto issue_tile = [&](int tile, int stage) {
    uint8_t* st = smem + stage * kStageBytes;
    const int t0 = it.key_begin + tile * kTile;
    // K and V base tiles: 64 rows x 16 chunks each, all threads
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = tid + q * kThreads;  // 0..1023
      const int row = c >> 4, ch = c & 15;
      const int t = t0 + row;
      const bool valid = t < it.key_end;
      const int tt = valid ? t : it.key_begin;
      const int pg = p.base_pages[it.base_off + tt / P];
      const int64_t off = (((int64_t)pg * p.hkv + h) * P + (tt % P)) * kD + ch * 8;
      const uint32_t so = (row * kKVStride + ch * 8) * 2;
      cp_async16(smem_u32(st + so), Kb + off, valid);
      cp_async16(smem_u32(st + kKVBytes + so), Vb + off, valid);
    }
    if (active) {
      uint8_t* rk_s = st + 2 * kKVBytes + wid * kRBytes;
      uint8_t* rv_s = st + 2 * kKVBytes + kWarps * kRBytes + wid * kRBytes;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = lane + q * 32;  // 0..127
        const int row = c >> 1, ch = c & 1;
        const int t = t0 + row;
        const bool valid = t < it.key_end;
        const int tt = valid ? t : it.key_begin;
        const int pg = p.res_pages[w.res_off + tt / P];
        const int64_t off = ((int64_t)pg * P + (tt % P)) * kR + res_col(tt % P, ch * 8, p.res_swz);
        cp_async16(smem_u32(rk_s + r_off(row, ch)), Rk + off, valid);
        cp_async16(smem_u32(rv_s + r_off(row, ch)), Rv + off, valid);
      }
    }
  };

  issue_tile(0, 0);
  cp_commit();
  if (n_tiles > 1) issue_tile(1, 1);
  cp_commit();

  // ---- per-warp state ----
  const int r0 = lane >> 2, cq = (lane & 3) * 2;
  int pos0 = -1, pos1 = -1;
  uint32_t qf[8][4];
  if (active) {
    const DevRow ra = p.rows[w.row_off + r0], rb = p.rows[w.row_off + r0 + 8];
    pos0 = ra.seq >= 0 ? ra.pos : -1;
    pos1 = rb.seq >= 0 ? rb.pos : -1;
    const uint32_t* qa = ra.seq >= 0 ? (const uint32_t*)((const __nv_bfloat16*)p.Q +
                                                         ((int64_t)(p.seqs[ra.seq].q_row0 + ra.qi) * p.hq + ra.qh) * kD)
                                     : nullptr;
    const uint32_t* qb = rb.seq >= 0 ? (const uint32_t*)((const __nv_bfloat16*)p.Q +
                                                         ((int64_t)(p.seqs[rb.seq].q_row0 + rb.qi) * p.hq + rb.qh) * kD)
                                     : nullptr;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int c0 = (ks * 16 + cq) / 2, c1 = (ks * 16 + 8 + cq) / 2;
      qf[ks][0] = qa ? qa[c0] : 0u;
      qf[ks][1] = qb ? qb[c0] : 0u;
      qf[ks][2] = qa ? qa[c1] : 0u;
      qf[ks][3] = qb ? qb[c1] : 0u;
    }
  }
  const bool deferred = p.rope_mode == FKV_ROPE_DEFERRED;
  float o_acc[16][4];
  float r_acc[2][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o_acc[i][0] = o_acc[i][1] = o_acc[i][2] = o_acc[i][3] = 0.f;
#pragma unroll
  for (int i = 0; i < 2; ++i) r_acc[i][0] = r_acc[i][1] = r_acc[i][2] = r_acc[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qt[4] = {0u, 0u, 0u, 0u};  // NONE mode: (Q B_k^T) as an A fragment

  for (int tile = 0; tile < n_tiles; ++tile) {
    cp_wait<1>();
    __syncthreads();
    const int stage = tile & 1;
    const uint8_t* st = smem + stage * kStageBytes;
    const uint32_t k_s = smem_u32(st), v_s = smem_u32(st + kKVBytes);
    const uint32_t rk_s = smem_u32(st + 2 * kKVBytes + wid * kRBytes);
    const uint32_t rv_s = smem_u32(st + 2 * kKVBytes + kWarps * kRBytes + wid * kRBytes);
    const uint32_t bk_a = smem_u32(bk_s);
    const int t0 = it.key_begin + tile * kTile;
    if (active) {
      if (!deferred && tile == 0) {
        // q~ = Q B_k^T : [16 rows x 16 r]
        float c2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t b00, b01, b10, b11;
          // matrices: (r0-7, chunk 2ks), (r0-7, 2ks+1), (r8-15, 2ks), (r8-15, 2ks+1)
          const int mi = lane >> 3, rr = (lane & 7) + ((mi >> 1) << 3), ch = 2 * ks + (mi & 1);
          ldsm_x4(bk_a + bk_off(rr, ch), b00, b01, b10, b11);
          mma16816(c2[0], qf[ks], b00, b01);
          mma16816(c2[1], qf[ks], b10, b11);
        }
        qt[0] = pack_bf16(c2[0][0], c2[0][1]);
        qt[1] = pack_bf16(c2[0][2], c2[0][3]);
        qt[2] = pack_bf16(c2[1][0], c2[1][1]);
        qt[3] = pack_bf16(c2[1][2], c2[1][3]);
      }
      float s[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
      // ---- S = Q K_base^T ----
#pragma unroll
      for (int kp = 0; kp < 4; ++kp) {  // 16-key groups
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t b0, b1, b2, b3;
          const int mi = lane >> 3;
          const int key = kp * 16 + (lane & 7) + ((mi >> 1) << 3);
          const int col = ks * 16 + ((mi & 1) << 3);
          ldsm_x4(k_s + (key * kKVStride + col) * 2, b0, b1, b2, b3);
          mma16816(s[2 * kp], qf[ks], b0, b1);
          mma16816(s[2 * kp + 1], qf[ks], b2, b3);
        }
      }
      if (deferred) {
        // ---- S += Q RoPE_t(R_k B_k^h)^T, per 16-key m-tile ----
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          uint32_t ra[4];
          {
            const int mi = lane >> 3;
            const int key = mt * 16 + (lane & 7) + ((mi & 1) << 3);
            ldsm_x4(rk_s + r_off(key, mi >> 1), ra[0], ra[1], ra[2], ra[3]);
          }
          const int keyA = t0 + mt * 16 + r0, keyB = keyA + 8;
          const float2* cosA = (const float2*)(p.rope_cos + (int64_t)min(keyA, it.key_end - 1) * (kD / 2));
          const float2* sinA = (const float2*)(p.rope_sin + (int64_t)min(keyA, it.key_end - 1) * (kD / 2));
          const float2* cosB = (const float2*)(p.rope_cos + (int64_t)min(keyB, it.key_end - 1) * (kD / 2));
          const float2* sinB = (const float2*)(p.rope_sin + (int64_t)min(keyB, it.key_end - 1) * (kD / 2));
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            // K_lora n-tiles 2ks, 2ks+1 (d < 64) and their RoPE partners 2ks+8, 2ks+9
            float c[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a) c[a][0] = c[a][1] = c[a][2] = c[a][3] = 0.f;
            {
              uint32_t b0, b1, b2, b3;
              const int mi = lane >> 3;
              const int rr = (lane & 7) + ((mi & 1) << 3);
              ldsm_x4_t(bk_a + bk_off(rr, 2 * ks + (mi >> 1)), b0, b1, b2, b3);
              mma16816(c[0], ra, b0, b1);
              mma16816(c[1], ra, b2, b3);
              ldsm_x4_t(bk_a + bk_off(rr, 2 * ks + 8 + (mi >> 1)), b0, b1, b2, b3);
              mma16816(c[2], ra, b0, b1);
              mma16816(c[3], ra, b2, b3);
            }
            // rotate pairs (i, i+64): c[a] holds d = 16ks + 8a + cq + {0,1}, c[a+2] the partner
            uint32_t kb_lo[2][2], kb_hi[2][2];  // [n-tile a][key half]
#pragma unroll
            for (int a = 0; a < 2; ++a) {
              const int fi = (16 * ks + 8 * a + cq) >> 1;
              const float2 ca = __ldg(cosA + fi), sa = __ldg(sinA + fi);
              const float2 cb = __ldg(cosB + fi), sb = __ldg(sinB + fi);
              const float x0a = c[a][0], x1a = c[a][1], y0a = c[a + 2][0], y1a = c[a + 2][1];
              const float x0b = c[a][2], x1b = c[a][3], y0b = c[a + 2][2], y1b = c[a + 2][3];
              kb_lo[a][0] = pack_bf16(x0a * ca.x - y0a * sa.x, x1a * ca.y - y1a * sa.y);
              kb_hi[a][0] = pack_bf16(x0a * sa.x + y0a * ca.x, x1a * sa.y + y1a * ca.y);
              kb_lo[a][1] = pack_bf16(x0b * cb.x - y0b * sb.x, x1b * cb.y - y1b * sb.y);
              kb_hi[a][1] = pack_bf16(x0b * sb.x + y0b * cb.x, x1b * sb.y + y1b * cb.y);
            }
            // k-step ks (d 16ks..16ks+15) and ks+4 (d 64+16ks..): keys r0 -> S n-tile 2mt, keys r0+8 -> 2mt+1
            mma16816(s[2 * mt], qf[ks], kb_lo[0][0], kb_lo[1][0]);
            mma16816(s[2 * mt + 1], qf[ks], kb_lo[0][1], kb_lo[1][1]);
            mma16816(s[2 * mt], qf[ks + 4], kb_hi[0][0], kb_hi[1][0]);
            mma16816(s[2 * mt + 1], qf[ks + 4], kb_hi[0][1], kb_hi[1][1]);
          }
        }
      } else {
        // ---- S += q~ R_k^T ----
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {
          uint32_t b0, b1, b2, b3;
          const int mi = lane >> 3;
          const int key = kp * 16 + (lane & 7) + ((mi >> 1) << 3);
          ldsm_x4(rk_s + r_off(key, mi & 1), b0, b1, b2, b3);
          mma16816(s[2 * kp], qt, b0, b1);
          mma16816(s[2 * kp + 1], qt, b2, b3);
        }
      }
      // ---- online softmax (one m, l per row; Alg1.339-341) ----
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int key = t0 + nt * 8 + cq;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int kk = key + e;
          const bool ok0 = kk < it.key_end && kk <= pos0;
          const bool ok1 = kk < it.key_end && kk <= pos1;
          s[nt][e] = ok0 ? s[nt][e] * p.scale_log2 : -INFINITY;
          s[nt][2 + e] = ok1 ? s[nt][2 + e] * p.scale_log2 : -INFINITY;
          mx0 = fmaxf(mx0, s[nt][e]);
          mx1 = fmaxf(mx1, s[nt][2 + e]);
        }
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float ms0 = mn0 == -INFINITY ? 0.f : mn0, ms1 = mn1 == -INFINITY ? 0.f : mn1;
      const float al0 = exp2f(m0 - ms0), al1 = exp2f(m1 - ms1);
      m0 = mn0; m1 = mn1;
      float ls0 = 0.f, ls1 = 0.f;
      uint32_t pa[4][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float p0 = exp2f(s[nt][0] - ms0), p1 = exp2f(s[nt][1] - ms0);
        const float p2 = exp2f(s[nt][2] - ms1), p3 = exp2f(s[nt][3] - ms1);
        ls0 += p0 + p1;
        ls1 += p2 + p3;
        // A fragment of P for k-step nt/2: regs 0,1 from even n-tile, 2,3 from odd
        pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
        pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
      }
      l0 = l0 * al0 + ls0;
      l1 = l1 * al1 + ls1;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        o_acc[i][0] *= al0; o_acc[i][1] *= al0; o_acc[i][2] *= al1; o_acc[i][3] *= al1;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        r_acc[i][0] *= al0; r_acc[i][1] *= al0; r_acc[i][2] *= al1; r_acc[i][3] *= al1;
      }
      // ---- acc += P V_base ; acc_r += P R_v (Alg1.343-344) ----
#pragma unroll
      for (int kp = 0; kp < 4; ++kp) {
        const int mi = lane >> 3;
        const int key = kp * 16 + (lane & 7) + ((mi & 1) << 3);
#pragma unroll
        for (int np = 0; np < 8; ++np) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(v_s + (key * kKVStride + np * 16 + ((mi >> 1) << 3)) * 2, b0, b1, b2, b3);
          mma16816(o_acc[2 * np], pa[kp], b0, b1);
          mma16816(o_acc[2 * np + 1], pa[kp], b2, b3);
        }
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(rv_s + r_off(key, mi >> 1), b0, b1, b2, b3);
        mma16816(r_acc[0], pa[kp], b0, b1);
        mma16816(r_acc[1], pa[kp], b2, b3);
      }
    }
    __syncthreads();
    if (tile + 2 < n_tiles) issue_tile(tile + 2, stage);
    cp_commit();
  }
  cp_wait<0>();
  if (!active) return;
  // ---- partial entry: [m, l, acc[128], acc_r[16]] ----
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int row = r0 + half * 8;
    if (row >= w.n_rows) continue;
    float* ent = p.ws + (int64_t)(w.entry_off + row) * p.entry_stride;
    if ((lane & 3) == 0) {
      ent[0] = half ? m1 : m0;
      ent[1] = half ? l1 : l0;
    }
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      ent[kEntAcc + nt * 8 + cq] = o_acc[nt][half * 2];
      ent[kEntAcc + nt * 8 + cq + 1] = o_acc[nt][half * 2 + 1];
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      ent[kEntAcc + kD + nt * 8 + cq] = r_acc[nt][half * 2];
      ent[kEntAcc + kD + nt * 8 + cq + 1] = r_acc[nt][half * 2 + 1];
    }
  }
}

}  // namespace

cudaError_t launch_attention_mma(const AttnParams& p, cudaStream_t s) {
  if (p.n_items == 0) return cudaSuccess;
  if (p.d != kD || p.r != kR || p.dtype != FKV_DTYPE_BF16) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ra_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  ra_mma_kernel<<<p.n_items, kThreads, kSmemBytes, s>>>(p);
  return cudaGetLastError();
}

}  // namespace k
}  // namespace fkv
