// sm_100a kernels: KV-row scatter (§8(a) a3), CoW page copy (a2/a3),
// split-KV combine + late V fusion (a6, Alg1.348-350 / Eq.4), the plain SIMT
// ResidualAttention (fp32 parity path and fallback), and the device copy of
// the synthetic input generator.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace fkv {
namespace k {

namespace {

template <int N>
struct Runs {
  WriteRun r[N];
};
template <int N>
struct Copies {
  CopyOp c[N];
};

// Copy `n` elements of size `es` bytes; uses 16-byte vectors when aligned.
__device__ __forceinline__ void copy_elems(void* dst, const void* src, int64_t n, int es, int tid, int nt) {
  const int64_t bytes = n * es;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0 && (bytes & 15) == 0) {
    const uint4* s = (const uint4*)src;
    uint4* d = (uint4*)dst;
    for (int64_t i = tid; i < bytes / 16; i += nt) d[i] = s[i];
  } else if ((((uintptr_t)dst | (uintptr_t)src) & 3) == 0 && (bytes & 3) == 0) {
    const uint32_t* s = (const uint32_t*)src;
    uint32_t* d = (uint32_t*)dst;
    for (int64_t i = tid; i < bytes / 4; i += nt) d[i] = s[i];
  } else {
    const uint16_t* s = (const uint16_t*)src;
    uint16_t* d = (uint16_t*)dst;
    for (int64_t i = tid; i < bytes / 2; i += nt) d[i] = s[i];
  }
}

// One CTA per run (blockIdx.y strides over its rows). Every 16-byte chunk of a row (K_base and V_base of all the
// rank's kv heads, R_k, R_v) is one independent load + store by one thread, so a row costs one memory latency
// (a per-head copy loop serialises its loads behind the previous head's stores: the pointers may alias).
// Residual rows of the swizzled format (res_col) land with their two 16-byte halves swapped on rows 4..7 of each
// 8-row group. Unaligned shapes (tiny d or r) take the element-wise path.
template <int N>
__global__ void __launch_bounds__(256) kv_write_kernel(PoolView pv, int32_t layer, Runs<N> runs, int32_t n_runs,
                                                       const uint8_t* kb, const uint8_t* vb, const uint8_t* rk,
                                                       const uint8_t* rv, uint32_t mask) {
  pdl_wait();
  pdl_trigger();
  const int run = blockIdx.x;
  if (run >= n_runs) return;
  const WriteRun w = runs.r[run];
  const int es = pv.dtype == FKV_DTYPE_BF16 ? 2 : 4;
  const int64_t hb = (int64_t)pv.d * es;         // bytes of one head row
  const int64_t bb = (int64_t)pv.hkv * hb;       // bytes of one source base row (all local heads)
  const int64_t rb = (int64_t)pv.r * es;         // bytes of one residual row
  const bool vec = (hb % 16) == 0 && (rb % 16) == 0 &&
                   (((uintptr_t)kb | (uintptr_t)vb | (uintptr_t)rk | (uintptr_t)rv) & 15) == 0;
  for (int j = blockIdx.y; j < w.n; j += gridDim.y) {
    const int64_t src = w.src_row + j;
    const int row = w.row0 + j;
    const int64_t bdst0 = (((int64_t)layer * pv.nb + w.base_page) * pv.hkv * pv.P + row) * hb;  // head 0
    const int64_t rdst = (((int64_t)layer * pv.nr + w.res_page) * pv.P + row) * rb;
    if (vec) {
      const int nbc = (int)(bb / 16), nrc = (int)(rb / 16);
      const int swz = pv.res_swz && ((row >> 2) & 1);  // 2 chunks per residual row in the swizzled format
      for (int i = threadIdx.x; i < 2 * nbc + 2 * nrc; i += blockDim.x) {
        const uint8_t* sp;
        uint8_t* dp;
        if (i < 2 * nbc) {
          const int v = i >= nbc, c = i - v * nbc;
          if (!(mask & (v ? FKV_WRITE_VBASE : FKV_WRITE_KBASE))) continue;
          const int64_t off = (int64_t)c * 16, h = off / hb;
          sp = (v ? vb : kb) + src * bb + off;
          dp = (uint8_t*)(v ? pv.base_v : pv.base_k) + bdst0 + h * pv.P * hb + (off - h * hb);
        } else {
          const int v = i - 2 * nbc >= nrc, c = i - 2 * nbc - v * nrc;
          if (!(mask & (v ? FKV_WRITE_RV : FKV_WRITE_RK))) continue;
          sp = (v ? rv : rk) + src * rb + c * 16;
          dp = (uint8_t*)(v ? pv.res_v : pv.res_k) + rdst + (swz ? (c ^ 1) : c) * 16;
        }
        *(uint4*)dp = __ldg((const uint4*)sp);
      }
      continue;
    }
    for (int h = 0; h < pv.hkv; ++h) {
      const int64_t dst = bdst0 + (int64_t)h * pv.P * hb;
      if (mask & FKV_WRITE_KBASE)
        copy_elems((uint8_t*)pv.base_k + dst, kb + src * bb + h * hb, pv.d, es, threadIdx.x, blockDim.x);
      if (mask & FKV_WRITE_VBASE)
        copy_elems((uint8_t*)pv.base_v + dst, vb + src * bb + h * hb, pv.d, es, threadIdx.x, blockDim.x);
    }
    if (pv.res_swz && (row >> 2) & 1) {  // swizzled row: swap the two 8-element halves
      const int hr = pv.r / 2;
      for (int hh = 0; hh < 2; ++hh) {
        if (mask & FKV_WRITE_RK)
          copy_elems((uint8_t*)pv.res_k + rdst + hh * hr * es, rk + (src * pv.r + (1 - hh) * hr) * es, hr, es,
                     threadIdx.x, blockDim.x);
        if (mask & FKV_WRITE_RV)
          copy_elems((uint8_t*)pv.res_v + rdst + hh * hr * es, rv + (src * pv.r + (1 - hh) * hr) * es, hr, es,
                     threadIdx.x, blockDim.x);
      }
    } else {
      if (mask & FKV_WRITE_RK) copy_elems((uint8_t*)pv.res_k + rdst, rk + src * rb, pv.r, es, threadIdx.x, blockDim.x);
      if (mask & FKV_WRITE_RV) copy_elems((uint8_t*)pv.res_v + rdst, rv + src * rb, pv.r, es, threadIdx.x, blockDim.x);
    }
  }
}

// CoW: copy rows [0, rows) of page src -> dst for every layer (and head).
__global__ void cow_copy_kernel(PoolView pv, Copies<kMaxCopies> ops, int32_t n_ops) {
  const int op = blockIdx.x;
  if (op >= n_ops) return;
  const CopyOp c = ops.c[op];
  const int layer = blockIdx.y;
  const int es = pv.dtype == FKV_DTYPE_BF16 ? 2 : 4;
  if (c.kind == FKV_KIND_BASE) {
    for (int h = 0; h < pv.hkv; ++h) {
      const int64_t s = ((((int64_t)layer * pv.nb + c.src) * pv.hkv + h) * pv.P) * (int64_t)pv.d;
      const int64_t d = ((((int64_t)layer * pv.nb + c.dst) * pv.hkv + h) * pv.P) * (int64_t)pv.d;
      copy_elems((uint8_t*)pv.base_k + d * es, (const uint8_t*)pv.base_k + s * es, (int64_t)c.rows * pv.d, es,
                 threadIdx.x, blockDim.x);
      copy_elems((uint8_t*)pv.base_v + d * es, (const uint8_t*)pv.base_v + s * es, (int64_t)c.rows * pv.d, es,
                 threadIdx.x, blockDim.x);
    }
  } else {
    const int64_t s = (((int64_t)layer * pv.nr + c.src) * pv.P) * (int64_t)pv.r;
    const int64_t d = (((int64_t)layer * pv.nr + c.dst) * pv.P) * (int64_t)pv.r;
    copy_elems((uint8_t*)pv.res_k + d * es, (const uint8_t*)pv.res_k + s * es, (int64_t)c.rows * pv.r, es,
               threadIdx.x, blockDim.x);
    copy_elems((uint8_t*)pv.res_v + d * es, (const uint8_t*)pv.res_v + s * es, (int64_t)c.rows * pv.r, es,
               threadIdx.x, blockDim.x);
  }
}

// ---- synthetic generator (bit-identical to workloads/synth.py) ------------
__device__ __forceinline__ uint64_t dsplitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void synth_kernel(void* dst, int32_t dtype, uint64_t stream, int32_t layer, int64_t pos0, int32_t n_pos,
                             int32_t head0, int32_t n_head, int32_t n_col, float scale) {
  const int64_t total = (int64_t)n_pos * n_head * n_col;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i % n_col;
    const int64_t h = (i / n_col) % n_head;
    const int64_t p = i / ((int64_t)n_col * n_head);
    const uint64_t idx = ((uint64_t)layer << 44) | ((uint64_t)(pos0 + p) << 16) | ((uint64_t)(head0 + h) << 8) |
                         (uint64_t)col;
    const uint64_t z = dsplitmix64(stream + idx);
    const int64_t u = (int64_t)(z >> 40);
    const float unit = (float)(2 * u + 1 - (1 << 24)) * (1.0f / 16777216.0f);
    const float v = __fmul_rn(unit, scale);
    if (dtype == FKV_DTYPE_BF16)
      ((__nv_bfloat16*)dst)[i] = __float2bfloat16_rn(v);
    else
      ((float*)dst)[i] = v;
  }
}

// ---- combine: merge split partials, late V fusion (Eq.4), write O ----------
template <typename T>
__device__ __forceinline__ float ldf(const T* p, int64_t i);
template <>
__device__ __forceinline__ float ldf<float>(const float* p, int64_t i) {
  return p[i];
}
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

template <typename T>
__global__ void combine_kernel(AttnParams p) {
  // one warp per output row: merge the split partials (m, l, acc, acc_r) and apply the late V fusion (Eq.4)
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= p.n_out_rows) return;
  const int qrow = warp / p.hq, qh = warp % p.hq;
  const int h = qh / p.group;
  const int seq = p.qrow_seq[qrow];
  const int slot = p.seqs[seq].adapter_slot;
  const int e0 = p.out_ptr[warp], e1 = p.out_ptr[warp + 1];
  const int d = p.d, r = p.r;
  constexpr int kMaxD = 256 / 32;
  float acc[kMaxD];
#pragma unroll
  for (int c = 0; c < kMaxD; ++c) acc[c] = 0.f;
  float accr0 = 0.f, accr1 = 0.f, l = 0.f;
  float Mrun = -INFINITY;
  for (int eb = e0; eb < e1; eb += 32) {
    // up to 32 entries at once: lane i reads entry eb + i's (m, l); weights 2^(m_i - M) (entries with l > 0 only)
    const int ne = min(32, e1 - eb);
    const float* my = lane < ne ? p.ws + (int64_t)p.out_entries[eb + lane] * p.entry_stride : nullptr;
    const float mi = my ? my[0] : -INFINITY, li = my ? my[1] : 0.f;
    const bool ok = li > 0.f;
    float M = ok ? mi : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    M = fmaxf(M, Mrun);
    if (Mrun != -INFINITY && M != Mrun) {  // more than 32 entries: rescale the earlier batches
      const float sc = exp2f(Mrun - M);
      l *= sc; accr0 *= sc; accr1 *= sc;
#pragma unroll
      for (int c = 0; c < kMaxD; ++c) acc[c] *= sc;
    }
    Mrun = M;
    const float wi = ok ? exp2f(mi - M) : 0.f;
    float lsum = wi * li;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    l += lsum;
#pragma unroll 4
    for (int i = 0; i < ne; ++i) {
      const float w = __shfl_sync(0xffffffffu, wi, i);
      const float* ent = p.ws + (int64_t)p.out_entries[eb + i] * p.entry_stride;
      if (w != 0.f) {
#pragma unroll
        for (int c = 0; c < kMaxD; ++c)
          if (lane + 32 * c < d) acc[c] += w * ent[kEntAcc + lane + 32 * c];
        if (lane < r) accr0 += w * ent[kEntAcc + d + lane];
        if (lane + 32 < r) accr1 += w * ent[kEntAcc + d + lane + 32];
      }
    }
  }
  // late fusion: O = (acc + acc_r . B_v^h) / l   (Alg1.349-350)
  const T* bv = (const T*)p.adapters[2 * slot + 1] + (int64_t)p.layer * p.adapter_layer_stride + (int64_t)h * r * d;
#pragma unroll 8
  for (int j = 0; j < r; ++j) {
    const float a = __shfl_sync(0xffffffffu, j < 32 ? accr0 : accr1, j & 31);
#pragma unroll
    for (int c = 0; c < kMaxD; ++c)
      if (lane + 32 * c < d) acc[c] += a * ldf<T>(bv, (int64_t)j * d + lane + 32 * c);
  }
  // a row with no keys in this plan's key range (range plans, §8(f) f4): O = 0, lse = -inf
  const float inv = l > 0.f ? 1.f / l : 0.f;
  if (p.lse && lane == 0) p.lse[warp] = l > 0.f ? (Mrun + log2f(l)) * 0.69314718055994531f : -INFINITY;
  T* o = (T*)p.O + (int64_t)warp * d;
#pragma unroll
  for (int c = 0; c < kMaxD; ++c) {
    const int e = lane + 32 * c;
    if (e < d) {
      if constexpr (sizeof(T) == 2)
        o[e] = __float2bfloat16_rn(acc[c] * inv);
      else
        o[e] = acc[c] * inv;
    }
  }
}

// ---- SIMT ResidualAttention (Alg.1, one key at a time per warp) -----------
// Each warp owns up to 16 query rows of one residual owner (same adapter and
// residual pages) and one kv head. Lane `l` holds head-dim elements
// e = l + 32c. Per key t: rebuild K[t] = Kb[t] + rho_t(Rk[t] B_K^h) (Stage 1,
// Alg1.335-336), scores for the 16 rows, one online-softmax state (m, l) per
// row, acc += p Vb[t], acc_r += p Rv[t] (Stage 2, Alg1.343-344). Stage 3 (the
// B_v fusion) happens in combine_kernel.
template <typename T, int D>
__global__ void __launch_bounds__(256) attention_simt_kernel(AttnParams p) {
  constexpr int NC = D / 32;
  const int item_id = blockIdx.x;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const DevItem it = p.items[item_id];
  if (wid >= it.n_warps) return;
  const DevWarp w = p.warps[it.warp_off + wid];
  const int h = it.kv_head;
  const int r = p.r;
  const T* Kb = (const T*)p.base_k + (int64_t)p.layer * p.base_layer_stride;
  const T* Vb = (const T*)p.base_v + (int64_t)p.layer * p.base_layer_stride;
  const T* Rk = (const T*)p.res_k + (int64_t)p.layer * p.res_layer_stride;
  const T* Rv = (const T*)p.res_v + (int64_t)p.layer * p.res_layer_stride;
  const T* Bk = (const T*)p.adapters[2 * w.adapter_slot] + (int64_t)p.layer * p.adapter_layer_stride +
                (int64_t)h * r * D;
  // query rows
  float q[16][NC];
  int pos[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const DevRow rw = p.rows[w.row_off + i];
    pos[i] = rw.seq >= 0 ? rw.pos : -1;
    const T* qp = (const T*)p.Q;
    const int64_t qoff = rw.seq >= 0 ? ((int64_t)(p.seqs[rw.seq].q_row0 + rw.qi) * p.hq + rw.qh) * D : 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) q[i][c] = rw.seq >= 0 ? ldf<T>(qp, qoff + lane + 32 * c) : 0.f;
  }
  float acc[16][NC];
  float accr[16][2];
  float m = -INFINITY, l = 0.f;  // lane i (< 16) owns row i; lanes 16..31 mirror
#pragma unroll
  for (int i = 0; i < 16; ++i) {
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[i][c] = 0.f;
    accr[i][0] = accr[i][1] = 0.f;
  }
  const int P = p.P;
  for (int t = it.key_begin; t < it.key_end; ++t) {
    const int bp = p.base_pages[it.base_off + t / P];
    const int rp = p.res_pages[w.res_off + t / P];
    const int row = t % P;
    const int64_t boff = (((int64_t)bp * p.hkv + h) * P + row) * D;
    const int64_t roff = ((int64_t)rp * P + row) * r;
    float u[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) u[c] = 0.f;
    for (int j = 0; j < r; ++j) {
      const float rk = ldf<T>(Rk, roff + res_col(row, j, p.res_swz));
#pragma unroll
      for (int c = 0; c < NC; ++c) u[c] += rk * ldf<T>(Bk, (int64_t)j * D + lane + 32 * c);
    }
    float kf[NC];
    if (p.rope_mode == FKV_ROPE_DEFERRED) {
      // pairs (e, e + D/2) live in the same lane: c and c + NC/2
#pragma unroll
      for (int c = 0; c < NC / 2; ++c) {
        const int i = lane + 32 * c;
        const float cs = p.rope_cos[(int64_t)t * (D / 2) + i], sn = p.rope_sin[(int64_t)t * (D / 2) + i];
        const float x0 = u[c], x1 = u[c + NC / 2];
        kf[c] = ldf<T>(Kb, boff + i) + (x0 * cs - x1 * sn);
        kf[c + NC / 2] = ldf<T>(Kb, boff + i + D / 2) + (x0 * sn + x1 * cs);
      }
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) kf[c] = ldf<T>(Kb, boff + lane + 32 * c) + u[c];
    }
    // scores: partial dot products, then a transposed butterfly so that lane
    // i (and i + 16) ends up with the full score of row i.
    float s[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float a = 0.f;
#pragma unroll
      for (int c = 0; c < NC; ++c) a += q[i][c] * kf[c];
      s[i] = a;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
    }
    float mine = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if ((lane & 15) == i) mine = s[i];
    const int ri = lane & 15;
    float myp = 0.f, alpha = 1.f;
    {
      int mypos = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (ri == i) mypos = pos[i];
      const float sv = (t <= mypos) ? mine * p.scale_log2 : -INFINITY;
      const float mn = fmaxf(m, sv);
      if (mn == -INFINITY) {
        alpha = 1.f; myp = 0.f;
      } else {
        alpha = exp2f(m - mn);
        myp = exp2f(sv - mn);
      }
      l = l * alpha + myp;
      m = mn;
    }
    float vf[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) vf[c] = ldf<T>(Vb, boff + lane + 32 * c);
    const float rv0 = lane < r ? ldf<T>(Rv, roff + res_col(row, lane, p.res_swz)) : 0.f;
    const float rv1 = lane + 32 < r ? ldf<T>(Rv, roff + res_col(row, lane + 32, p.res_swz)) : 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float a = __shfl_sync(0xffffffffu, alpha, i);
      const float pp = __shfl_sync(0xffffffffu, myp, i);
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[i][c] = acc[i][c] * a + pp * vf[c];
      accr[i][0] = accr[i][0] * a + pp * rv0;
      accr[i][1] = accr[i][1] * a + pp * rv1;
    }
  }
  // write partial entries: [m, l, acc[D], acc_r[r]] (m in log2 units)
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i >= w.n_rows) break;
    float* ent = p.ws + (int64_t)(w.entry_off + i) * p.entry_stride;
    const float mi = __shfl_sync(0xffffffffu, m, i), li = __shfl_sync(0xffffffffu, l, i);
    if (lane == 0) { ent[0] = mi; ent[1] = li; }
#pragma unroll
    for (int c = 0; c < NC; ++c) ent[kEntAcc + lane + 32 * c] = acc[i][c];
    if (lane < r) ent[kEntAcc + D + lane] = accr[i][0];
    if (lane + 32 < r) ent[kEntAcc + D + lane + 32] = accr[i][1];
  }
}

}  // namespace

cudaError_t launch_kv_write(const PoolView& pv, int32_t layer, const WriteRun* runs, int32_t n_runs, const void* kb,
                            const void* vb, const void* rk, const void* rv, uint32_t mask, cudaStream_t s) {
  int maxn = 1;
  for (int i = 0; i < n_runs; ++i) maxn = max(maxn, runs[i].n);
  dim3 grid(n_runs, min(maxn, 16));
  if (n_runs <= 64) {  // a decode step's runs: a 2-KB parameter block instead of 16 KB (launch cost)
    Runs<64> rr;
    for (int i = 0; i < n_runs; ++i) rr.r[i] = runs[i];
    return launch_pdl(kv_write_kernel<64>, grid, dim3(256), 0, s, pv, layer, rr, n_runs, (const uint8_t*)kb,
                      (const uint8_t*)vb, (const uint8_t*)rk, (const uint8_t*)rv, mask);
  }
  Runs<kMaxRuns> rr;
  for (int i = 0; i < n_runs; ++i) rr.r[i] = runs[i];
  return launch_pdl(kv_write_kernel<kMaxRuns>, grid, dim3(256), 0, s, pv, layer, rr, n_runs, (const uint8_t*)kb,
                    (const uint8_t*)vb, (const uint8_t*)rk, (const uint8_t*)rv, mask);
}

cudaError_t launch_cow_copy(const PoolView& pv, const CopyOp* ops, int32_t n_ops, cudaStream_t s) {
  Copies<kMaxCopies> cc;
  for (int i = 0; i < n_ops; ++i) cc.c[i] = ops[i];
  cow_copy_kernel<<<dim3(n_ops, pv.L), 256, 0, s>>>(pv, cc, n_ops);
  return cudaGetLastError();
}

cudaError_t launch_synth_fill(void* dst, int32_t dtype, uint64_t seed, int32_t kind, uint64_t owner, int32_t layer,
                              int64_t pos0, int32_t n_pos, int32_t head0, int32_t n_head, int32_t n_col, float scale,
                              cudaStream_t s) {
  const uint64_t st = fkv::splitmix64(fkv::splitmix64(seed * 256ull + (uint64_t)kind) ^ owner);
  const int64_t total = (int64_t)n_pos * n_head * n_col;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
  synth_kernel<<<blocks, 256, 0, s>>>(dst, dtype, st, layer, pos0, n_pos, head0, n_head, n_col, scale);
  return cudaGetLastError();
}

// d = 128, r = 16: lane l owns head-dim elements 4l..4l+3 (16-byte partial-entry loads, a batch of entries in
// flight at once) and, for l < 16, acc_r[l]; the late V fusion reads B_v rows as 4-element vectors. <= 128
// registers: all 2048-row C2 warps resident in one wave
template <typename T>
__global__ void __launch_bounds__(256, 2) combine128_kernel(AttnParams p) {
  // the plan's records (row -> entry range, entry ids, B_v address) are read before griddepcontrol.wait: the
  // main kernel does not write them, so two of the dependent load round trips overlap its tail; the partial
  // entries are read after the wait
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const bool live = warp < p.n_out_rows;
  longlong2 cr = make_longlong2(0, 0);
  if (live) cr = p.comb_rows[warp];
  const int e0 = (int)(cr.x & 0xffffffffll), e1 = (int)(cr.x >> 32);
  const int my_e0 = live && lane < e1 - e0 ? p.out_entries[e0 + lane] : 0;
  // B_v^h rows (16 x 128) for the late fusion: prefetched into L1 now (one 128-byte line per lane), read at the end
  const T* bv = (const T*)cr.y + (int64_t)p.layer * p.adapter_layer_stride;
  if (live) asm volatile("prefetch.global.L1 [%0];" ::"l"((const char*)bv + 128 * lane * (int)sizeof(T) / 2));
  pdl_wait();
  pdl_trigger();
  if (!live) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float accr = 0.f, l = 0.f, Mrun = -INFINITY;
  for (int eb = e0; eb < e1; eb += 32) {
    const int ne = min(32, e1 - eb);
    const int my_e = eb == e0 ? my_e0 : (lane < ne ? p.out_entries[eb + lane] : 0);
    const float* my = p.ws + (int64_t)my_e * p.entry_stride;
    const float2 ml = lane < ne ? *(const float2*)my : make_float2(-INFINITY, 0.f);
    for (int i0 = 0; i0 < ne; i0 += 16) {
      float4 v[16];
      float vr[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {  // the batch's loads first (they do not depend on the weights)
        const int e = __shfl_sync(0xffffffffu, my_e, i0 + k < ne ? i0 + k : ne - 1);
        const float* ent = p.ws + (int64_t)e * p.entry_stride + kEntAcc;
        v[k] = *(const float4*)(ent + 4 * lane);
        vr[k] = lane < 16 ? ent[128 + lane] : 0.f;
      }
      if (i0 == 0) {  // weights of this batch of <= 32 entries: 2^(m_i - M), entries with l > 0 only
        const bool ok = ml.y > 0.f;
        float M = ok ? ml.x : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        M = fmaxf(M, Mrun);
        if (Mrun != -INFINITY && M != Mrun) {  // more than 32 entries: rescale the earlier batches
          const float sc = exp2f(Mrun - M);
          l *= sc; accr *= sc;
          acc.x *= sc; acc.y *= sc; acc.z *= sc; acc.w *= sc;
        }
        Mrun = M;
      }
      const float wi = ml.y > 0.f ? exp2f(ml.x - Mrun) : 0.f;
      if (i0 == 0) {
        float lsum = wi * ml.y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        l += lsum;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float w = i0 + k < ne ? __shfl_sync(0xffffffffu, wi, i0 + k) : 0.f;
        if (w != 0.f) {  // an entry with l = 0 may hold non-finite accumulators
          acc.x += w * v[k].x; acc.y += w * v[k].y; acc.z += w * v[k].z; acc.w += w * v[k].w;
          accr += w * vr[k];
        }
      }
    }
  }
  // late fusion: O = (acc + acc_r . B_v^h) / l   (Alg1.349-350)
  uint2 bvu[16];  // bf16: 4 elements; f32: elements 4l, 4l+1 (the other two below)
#pragma unroll
  for (int j = 0; j < 16; ++j) bvu[j] = __ldg((const uint2*)(bv + j * 128 + 4 * lane));
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float a = __shfl_sync(0xffffffffu, accr, j);
    float4 b;
    if constexpr (sizeof(T) == 2) {
      b = make_float4(__uint_as_float(bvu[j].x << 16), __uint_as_float(bvu[j].x & 0xffff0000u),
                      __uint_as_float(bvu[j].y << 16), __uint_as_float(bvu[j].y & 0xffff0000u));
    } else {
      const float2 hi = __ldg((const float2*)(bv + j * 128 + 4 * lane + 2));
      b = make_float4(__uint_as_float(bvu[j].x), __uint_as_float(bvu[j].y), hi.x, hi.y);
    }
    acc.x += a * b.x; acc.y += a * b.y; acc.z += a * b.z; acc.w += a * b.w;
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;   // no keys in a range plan's key range: O = 0, lse = -inf
  if (p.lse && lane == 0) p.lse[warp] = l > 0.f ? (Mrun + log2f(l)) * 0.69314718055994531f : -INFINITY;
  T* o = (T*)p.O + (int64_t)warp * 128 + 4 * lane;
  if constexpr (sizeof(T) == 2) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv), hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    uint2 u;
    u.x = *(uint32_t*)&lo;
    u.y = *(uint32_t*)&hi;
    *(uint2*)o = u;
  } else {
    *(float4*)o = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  }
}

cudaError_t launch_combine(const AttnParams& p, cudaStream_t s) {
  if (p.d > 256 || p.r > 64) return cudaErrorInvalidValue;
  const int threads = 256;
  const int blocks = (p.n_out_rows * 32 + threads - 1) / threads;
  if (p.d == 128 && p.r == 16 && ((uintptr_t)p.O & 15) == 0 && (p.entry_stride & 3) == 0) {
    if (p.dtype == FKV_DTYPE_BF16) return launch_pdl(combine128_kernel<__nv_bfloat16>, dim3(blocks), dim3(threads), 0, s, p);
    return launch_pdl(combine128_kernel<float>, dim3(blocks), dim3(threads), 0, s, p);
  }
  if (p.dtype == FKV_DTYPE_BF16)
    combine_kernel<__nv_bfloat16><<<blocks, threads, 0, s>>>(p);
  else
    combine_kernel<float><<<blocks, threads, 0, s>>>(p);
  return cudaGetLastError();
}

// LSE merge of G partial attention outputs of the same rows over disjoint key ranges (blocking invariance of
// softmax; the late V fusion is linear so each part's fused O merges exactly): warp per row, lanes over d
template <typename T>
__global__ void merge_lse_kernel(int32_t G, int64_t n_rows, int32_t d, const T* __restrict__ Op,
                                 const float* __restrict__ lp, T* __restrict__ O, float* __restrict__ lse_out) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  float M = -INFINITY;
  for (int g = 0; g < G; ++g) M = fmaxf(M, lp[(int64_t)g * n_rows + row]);
  float den = 0.f;
  for (int g = 0; g < G; ++g) {
    const float v = lp[(int64_t)g * n_rows + row];
    den += v == -INFINITY ? 0.f : __expf(v - M);
  }
  for (int e = lane; e < d; e += 32) {
    float acc = 0.f;
    for (int g = 0; g < G; ++g) {
      const float v = lp[(int64_t)g * n_rows + row];
      if (v != -INFINITY) acc += __expf(v - M) * ldf<T>(Op, ((int64_t)g * n_rows + row) * d + e);
    }
    const float o = den > 0.f ? acc / den : 0.f;
    if constexpr (sizeof(T) == 2) O[row * d + e] = __float2bfloat16_rn(o);
    else O[row * d + e] = o;
  }
  if (lse_out && lane == 0) lse_out[row] = den > 0.f ? M + __logf(den) : -INFINITY;
}

cudaError_t launch_merge_lse(int32_t n_parts, int64_t n_rows, int32_t d, const void* O_parts, const float* lse_parts,
                             void* O, float* lse_out, int32_t dtype, cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  const int64_t blocks = (n_rows * 32 + 255) / 256;
  if (dtype == FKV_DTYPE_BF16)
    merge_lse_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, s>>>(n_parts, n_rows, d, (const __nv_bfloat16*)O_parts,
                                                                     lse_parts, (__nv_bfloat16*)O, lse_out);
  else
    merge_lse_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(n_parts, n_rows, d, (const float*)O_parts, lse_parts,
                                                             (float*)O, lse_out);
  return cudaGetLastError();
}

cudaError_t launch_attention_simt(const AttnParams& p, cudaStream_t s) {
  if (p.n_items == 0) return cudaSuccess;
  if (p.r > 64 || (p.d != 64 && p.d != 128)) return cudaErrorInvalidValue;
  dim3 grid(p.n_items);
  if (p.dtype == FKV_DTYPE_BF16) {
    if (p.d == 128) attention_simt_kernel<__nv_bfloat16, 128><<<grid, 256, 0, s>>>(p);
    else attention_simt_kernel<__nv_bfloat16, 64><<<grid, 256, 0, s>>>(p);
  } else {
    if (p.d == 128) attention_simt_kernel<float, 128><<<grid, 256, 0, s>>>(p);
    else attention_simt_kernel<float, 64><<<grid, 256, 0, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace k
}  // namespace fkv
