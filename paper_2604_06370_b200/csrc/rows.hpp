// Plan records of the rows-on-lanes tcgen05 ResidualAttention kernel (ra_rows.cu), shared by the planner
// (plan_rows.cpp) and the kernel. All records are read-only device data uploaded with the plan blob.
//
// Work decomposition:
//   item  = up to 128 query rows (one per TMEM lane) processed by one CTA with one Q image;
//   WU    = a work unit of an item: a set of lanes + up to 8 residual slots (owners) sharing one ordered list of
//           128-key tiles of one kv head (the rows of one agent group over one shared-page segment piece, or the
//           rows of one sequence over its private pages); an item is a sequence of WUs, each WU's tiles in order;
//   tile  = 128 (or fewer) keys of one kv head: base pages + per-slot residual pages.
#pragma once
#include <cuda.h>

#include <cstdint>

namespace fkv {
namespace k {

constexpr int kRowsLanes = 128;
constexpr int kRowsMaxSlots = 8;

struct RRow {          // one lane of an item (16 bytes)
  int32_t q_row;       // row of Q / O viewed as [rows][d] (= (seq q_row0 + qi) * hq_local + qh); -1 = empty lane
  int32_t pos;         // absolute position of the query (causal: key t visible iff t <= pos)
  int32_t entry;       // partial entry index (-1 = none)
  int32_t meta;        // slot | kv head << 8 | adapter slot << 16
};
struct RWu {           // 192 bytes
  uint32_t lanes[4];          // active lanes of the WU
  uint32_t slot_lanes[8][4];  // lanes of each residual slot (owner) of the WU
  uint32_t lanes_lo[4];       // lanes of slots 0-3 (their A_r columns 16 s), and of slots 4-7 (16 (s - 4))
  uint32_t lanes_hi[4];
  int32_t n_slots;            // residual slots 0..n_slots-1
  int32_t pad_[3];
};
static_assert(sizeof(RWu) == 192, "RWu");
struct RTile {         // 64 bytes
  int32_t key0;        // absolute position of the tile's first key
  int32_t n_keys;      // 1..128
  int32_t flags;       // kTileFirst: first tile of its WU (PV overwrites O / A_r of the WU's lanes);
                       // kTileCausal: some lane has keys it must not see (pos < key0 + n_keys - 1)
  int32_t wu;          // WU record index
  int32_t base_off;    // base_pages[base_off + i], i < 128 / P (page ids, -1 = none)
  int32_t kv_head;     // local kv head
  int32_t res_off[8];  // res_pages[res_off[s] + i] for slot s
  int32_t n_slots;     // residual slots of the tile's WU (copy of RWu::n_slots: one dependent load less)
  int32_t base_page;   // base_pages[base_off] (the tile's only page when P = 128), -1 = none
};
static_assert(sizeof(RTile) == 64, "RTile");
constexpr int32_t kTileFirst = 1, kTileCausal = 2;
struct RItem {         // 32 bytes
  int32_t tile0, n_tiles;  // tiles [tile0, tile0 + n_tiles) (all WUs of the item, WU by WU)
  int32_t row0;            // RRow index of lane 0 (128 rows per item)
  int32_t n_rows;          // lanes 0..n_rows-1 may be used
  int32_t pad_[4];
};
static_assert(sizeof(RItem) == 32, "RItem");

struct RowsParams {
  const void* base_k;
  const void* base_v;
  const void* res_k;
  const void* res_v;
  const void* Q;
  float* ws;                   // partial entries [m, l, pad x 6, acc[128], acc_r[16]]
  const RItem* items;
  const RWu* wus;
  const RTile* tiles;
  const RRow* rows;
  const int32_t* base_pages;
  const int32_t* res_pages;
  const int64_t* adapters;     // [adapter slot][2]: B_K, B_V device pointers (layer 0)
  const int32_t* sched_ptr;    // (unused by the dynamic schedule)
  const int32_t* sched_items;  // the item queue in the planner's order (cost-descending, locality)
  int32_t* ctr;                // workspace: [0] next queue position, [1] finished CTAs (zero between launches)
  int32_t n_items;
  int64_t base_rows_layer;     // TMA row index of (layer, page 0, head 0, key 0) = layer * nb * hkv * P
  int64_t res_layer_elems;     // elements per layer of a residual pool (= nr * P * r)
  int64_t adapter_layer_elems; // elements per layer of B_K / B_V (= hkv_local * r * d)
  int32_t layer, hkv, P, n_ctas;
  int32_t entry_stride;        // floats per partial entry
  float scale_log2;            // sm_scale * log2(e)
  long long* dbg;              // diagnostics timeline (nullptr = off)
  int32_t dbg_block;
  int32_t flags;               // diagnostics switches (FKV_ROWS_FLAGS): bit 0 = residual pages by cp.async instead of bulk copies
  long long* hang;             // host-mapped deadlock report (FKV_HANG_DIAG; nullptr = off)
  int32_t prefetch;            // L2 prefetch distance of the loaders in tiles (0 = off; FKV_ROWS_PREFETCH)
};

// TMA maps of the rows kernel over the base K / V pools: whole 128-key tiles {64 d, 128 keys, 2 d-halves} (3D,
// SW128; P = 128) or per-page d-half boxes {64, P} (2D, SW128; P < 128). Both land as [d-half][key][128 B].
struct RowsMaps {
  CUtensorMap k3d, v3d, k2d, v2d;
};

}  // namespace k
}  // namespace fkv
