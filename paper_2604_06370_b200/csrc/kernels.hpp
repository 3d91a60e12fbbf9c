// Launch interface between the host library and the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.hpp"

namespace fkv {
namespace k {

struct PoolView {
  void* base_k;
  void* base_v;
  void* res_k;
  void* res_v;
  int64_t nb, nr;  // pages per pool
  int32_t hkv, P, d, r, L, dtype;
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

struct AttnParams {
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
  int32_t tc_prefetch;  // tiles of L2 prefetch lookahead in the tcgen05 producer (0 = off)
};

cudaError_t launch_attention_mma(const AttnParams& p, cudaStream_t s);
cudaError_t launch_attention_simt(const AttnParams& p, cudaStream_t s);
cudaError_t launch_attention_tc(const AttnParams& p, const void* maps, cudaStream_t s);
size_t tc_maps_bytes();
cudaError_t launch_combine(const AttnParams& p, cudaStream_t s);

cudaError_t launch_synth_fill(void* dst, int32_t dtype, uint64_t seed, int32_t kind, uint64_t owner, int32_t layer,
                              int64_t pos0, int32_t n_pos, int32_t head0, int32_t n_head, int32_t n_col, float scale,
                              cudaStream_t s);

}  // namespace k
}  // namespace fkv
