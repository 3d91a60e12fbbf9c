// Launch interface between the host library and the sm_100a kernels.
#pragma once
#include <cstdlib>
#include <string>
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.hpp"
#include "rows.hpp"

namespace fkv {
namespace k {

struct PoolView {
  void* base_k;
  void* base_v;
  void* res_k;
  void* res_v;
  int64_t nb, nr;  // pages per pool
  int32_t hkv, P, d, r, L, dtype;
  int32_t res_swz;  // residual rows stored in SW32 order (see res_col)
};

// A contiguous run of rows written into one (base page, residual page) slot.
struct WriteRun {
  int32_t base_page, res_page, row0, n, src_row;
  int32_t pad_[3];
};
constexpr int kMaxRuns = 512;

struct CopyOp {
  int32_t kind, src, dst, rows;
};
constexpr int kMaxCopies = 512;

cudaError_t launch_kv_write(const PoolView& pv, int32_t layer, const WriteRun* runs, int32_t n_runs,
                            const void* kb, const void* vb, const void* rk, const void* rv, uint32_t mask,
                            cudaStream_t s);
cudaError_t launch_cow_copy(const PoolView& pv, const CopyOp* ops, int32_t n_ops, cudaStream_t s);

// Per-item header of the persistent tcgen05 kernel, staged into shared memory with the item's Q rows.
// S = slots (16 query rows each): 4 (64-row CTAs, 176 B) or 8 (128-row CTAs, 336 B).
template <int S>
struct ItemRecT {
  // n_tiles: bits 0..15 tiles, bit 16 + g: 32-column chunk g has a causally masked query column;
  // meta = n_slots | n_groups << 4 | group-first slot mask << 8 | kv head << 16
  int32_t k0, k1, n_tiles, meta;
  int32_t n_rows[S];              // query rows of each slot
  int32_t entry_off[S];           // first partial entry of each slot
  uint16_t pos1[16 * S];          // per query column: position - k0 + 1 (key t visible iff t - k0 < pos1), 0 = none
};
static_assert(sizeof(ItemRecT<4>) == 176 && sizeof(ItemRecT<8>) == 336, "ItemRec");
constexpr int kTileRecInts = 16;  // tile record: t0, k1, meta, base page, residual page of slots 0..7, pad

struct AttnParams {
  float* lse;              // optional per output row log-sum-exp of the scaled logits (natural log; -inf = no keys)
  const void* base_k;
  const void* base_v;
  const void* res_k;
  const void* res_v;
  const float* rope_cos;
  const float* rope_sin;
  const void* Q;
  void* O;
  float* ws;
  const DevSeq* seqs;
  const int32_t* base_pages;
  const int32_t* res_pages;
  const DevItem* items;
  const DevWarp* warps;
  const DevRow* rows;
  const int32_t* out_ptr;
  const int32_t* out_entries;
  const longlong2* comb_rows;  // per output row: (e0 | e1 << 32, B_v^h address of layer 0)
  const int64_t* adapters;  // [slot][2]: B_K, B_V device pointers
  const int32_t* qrow_seq;  // query row -> plan seq
  int64_t base_layer_stride;  // elements per layer of base pool
  int64_t res_layer_stride;   // elements per layer of residual pool
  int64_t adapter_layer_stride;  // elements per layer of B_K / B_V (= Hkv_local * r * d)
  int64_t nb, nr;                // pages per pool
  int32_t layer, hkv, hq, group, P, d, r, rope_mode, dtype;
  int32_t n_items, n_out_rows, entry_stride;
  float scale_log2;  // sm_scale * log2(e)
  long long* dbg;    // diagnostics: per-event clock64 stamps of CTA dbg_block (nullptr = off)
  int32_t dbg_block;
  // persistent tcgen05 kernel: CTA c runs items sched_items[sched_ptr[c] .. sched_ptr[c+1])
  const int32_t* sched_ptr;
  const int32_t* sched_items;
  int32_t n_ctas;
  // per-CTA tile records, CTA c owns records [tile_ptr[c], tile_ptr[c+1]) in its processing order:
  // {t0, k1, meta (as ItemRecT::meta), base page, residual page of slots 0..7, pad} (kTileRecInts ints; pages are
  // only meaningful when P == 128: one page per tile)
  const int32_t* tile_ptr;
  const int4* tile_recs;
  const void* item_recs;  // per plan item: ItemRecT<tc_rows / 16>
  int32_t tc_rows;        // query rows per CTA of the tcgen05 kernel (64 | 128)
  int32_t tc_pp;          // kernel 2, NONE, 64 rows: ping-pong key warpgroups (two partial entries per row and item)
  int32_t l2_evict_first; // base K / V tiles read by few row blocks: stream them through L2 evict-first
  const int32_t* stage_src;  // staged image i is built from warp slot stage_src[i]; DevItem::pad_[0] = first image
  const int4* stage_desc;    // per image, 5 x int4: {B_k^h address (layer 0) lo, hi, n_rows, kv head}, Q rows [16]
  int32_t max_pos;
  int32_t tc_prefetch;  // L2 prefetch distance in tiles (tcgen05 producer; 0 = off)
  uint8_t* stage;  // per-warp-slot staged operand images (ws region, kStageBytes each)
  int32_t res_swz;  // residual rows stored in SW32 order (see res_col)
};
// partial entry: [m, l, pad x 6, acc[D], acc_r[r]] (acc 32-byte aligned: 256-bit stores, vector loads)
constexpr int kEntAcc = 8;
constexpr int kStageBytes = 8192;

// Residual page format (bf16, r = 16): row i of a page holds R[i][j] at column j ^ (8 * ((i >> 2) & 1)), i.e.
// the two 16-byte halves of rows 4..7 of every 8-row group are swapped. This is exactly the 32-byte-swizzled
// K-major operand layout of tcgen05 (SW32), so a residual page streams into shared memory with one plain
// 128-byte-row TMA box and is an MMA operand as is (tcgen05 kernel, ra_tc.cu).
__host__ __device__ __forceinline__ int res_col(int row, int j, int swz) { return swz ? (j ^ (((row >> 2) & 1) << 3)) : j; }  // per warp slot: Q image 4 KB + (q~ 512 B | packed B_k 4 KB)

// Programmatic dependent launch (stream-ordered kernels of one layer): the kernel may be scheduled while its
// predecessor drains; it runs griddepcontrol.wait (full completion + memory of the predecessor) before touching
// anything the predecessor writes, then lets its own dependent launch (pdl_trigger).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  static const bool no_pdl = std::getenv("FKV_NO_PDL") != nullptr;  // diagnostics: plain stream-ordered launches
  cfg.numAttrs = no_pdl ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

cudaError_t launch_attention_mma(const AttnParams& p, cudaStream_t s);
cudaError_t launch_attention_simt(const AttnParams& p, cudaStream_t s);
cudaError_t launch_attention_tc(const AttnParams& p, const void* maps, cudaStream_t s);
cudaError_t launch_stage(const AttnParams& p, int32_t n_warps, cudaStream_t s);
size_t tc_maps_bytes();
cudaError_t launch_combine(const AttnParams& p, cudaStream_t s);
// O = sum_p exp(lse_p - L) O_p, L = log sum_p exp(lse_p): merge of attention outputs over disjoint key ranges
cudaError_t launch_merge_lse(int32_t n_parts, int64_t n_rows, int32_t d, const void* O_parts, const float* lse_parts,
                             void* O, float* lse_out, int32_t dtype, cudaStream_t s);
cudaError_t launch_attention_rows(const RowsParams& p, const RowsMaps& maps, cudaStream_t s);
// host-mapped deadlock report of the rows kernel (allocated on first use when FKV_HANG_DIAG is set, else nullptr)
long long* hang_slot();
// project.cu: the projection producer (§8(f) f2 / f3)
cudaError_t gemm_rowmajor_f32out(int64_t T, int64_t N, int64_t K, const void* X, const void* W, float* Y, int32_t dtype,
                                 cudaStream_t s, std::string* err);
cudaError_t launch_adapter_proj(const void* x, const int64_t* aptr, int32_t n_rows, int32_t hidden, int32_t r,
                                int32_t dtype, float* out, cudaStream_t s);
cudaError_t launch_project_stage(const float* yk, const float* yv, const float* yr, const int32_t* pos,
                                 const float* rope_cos, const float* rope_sin, int32_t n_rows, int32_t hkv, int32_t d,
                                 int32_t r, int32_t rope, int32_t dtype, void* kb, void* vb, void* rk, void* rv,
                                 cudaStream_t s);
std::string hang_report();

cudaError_t launch_synth_fill(void* dst, int32_t dtype, uint64_t seed, int32_t kind, uint64_t owner, int32_t layer,
                              int64_t pos0, int32_t n_pos, int32_t head0, int32_t n_head, int32_t n_col, float scale,
                              cudaStream_t s);

}  // namespace k
}  // namespace fkv
