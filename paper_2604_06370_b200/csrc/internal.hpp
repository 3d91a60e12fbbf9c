// Internal structures of the forkkv library (not part of the ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <algorithm>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/forkkv.h"

namespace fkv {

struct Error : std::runtime_error {
  fkv_status code;
  Error(fkv_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// R1: one page pool. Free set ordered by (rank, id).
struct PagePool {
  int64_t n = 0;
  uint64_t seed = 0;
  int32_t layers = 0;
  std::vector<int32_t> rc;
  std::vector<uint8_t> in_tree;
  std::set<std::pair<uint64_t, int32_t>> free_set;
  std::vector<uint64_t> written;  // [page][layer][2] row bitmask (rows < 128)

  void init(int64_t n_pages, uint64_t s, int32_t n_layers) {
    n = n_pages; seed = s; layers = n_layers;
    rc.assign(n, 0); in_tree.assign(n, 0);
    written.assign((size_t)n * n_layers * 2, 0);
    free_set.clear();
    for (int64_t i = 0; i < n; ++i) free_set.insert({rank(i), (int32_t)i});
  }
  uint64_t rank(int64_t id) const { return seed == 0 ? (uint64_t)id : splitmix64(seed ^ (uint64_t)id); }
  int64_t n_free() const { return (int64_t)free_set.size(); }
  int32_t alloc() {
    auto it = free_set.begin();
    int32_t id = it->second;
    free_set.erase(it);
    rc[id] = 1; in_tree[id] = 0;
    for (int32_t l = 0; l < 2 * layers; ++l) written[(size_t)id * layers * 2 + l] = 0;
    return id;
  }
  void retain(int32_t id) { rc[id] += 1; }
  void release(int32_t id) {
    rc[id] -= 1;
    if (rc[id] == 0) { in_tree[id] = 0; free_set.insert({rank(id), id}); }
  }
  bool writable(int32_t id) const { return rc[id] - (in_tree[id] ? 1 : 0) == 1; }
  uint64_t* wmask(int32_t id, int32_t layer) { return &written[((size_t)id * layers + layer) * 2]; }
  static uint64_t lowbits(int n) { return n <= 0 ? 0ull : (n >= 64 ? ~0ull : ((1ull << n) - 1)); }
  void wclear_bit(int32_t id, int32_t layer, int off) { wmask(id, layer)[off >> 6] &= ~(1ull << (off & 63)); }
  void wset_range(int32_t id, int32_t layer, int row0, int n) {
    uint64_t* w = wmask(id, layer);
    for (int k = 0; k < 2; ++k) {
      const int lo = std::max(row0, 64 * k), hi = std::min(row0 + n, 64 * k + 64);
      if (hi > lo) w[k] |= lowbits(hi - lo) << (lo - 64 * k);
    }
  }
  void wcopy_prefix(int32_t dst, int32_t src, int32_t layer, int rows) {
    uint64_t *d = wmask(dst, layer), *s = wmask(src, layer);
    d[0] = s[0] & lowbits(rows);
    d[1] = s[1] & lowbits(rows - 64);
  }
  bool wtest_prefix(int32_t id, int32_t layer, int rows) {
    uint64_t* w = wmask(id, layer);
    return (w[0] & lowbits(rows)) == lowbits(rows) && (w[1] & lowbits(rows - 64)) == lowbits(rows - 64);
  }
};

struct Agent {
  int64_t id = 0;
  int32_t adapter = 0;
  int64_t owner = 0;   // residual tree key
  int64_t seqlen = 0;
  std::vector<int32_t> base, res;
  std::vector<int32_t> tokens;
};

struct TreeNode {
  int32_t page = -1;
  int64_t last = 0;   // the tree's LRU clock at the last access (R10)
  int64_t seq = -1;   // insertion number in the tree (LRU tie-break)
  std::map<std::vector<int32_t>, std::unique_ptr<TreeNode>> children;
};

struct AdapterSlot {
  int32_t id;
  const void* bk;
  const void* bv;
  const void* ak = nullptr;  // down projections A_k, A_v [L][hidden][r] (projection producer; optional)
  const void* av = nullptr;
  int32_t hidden = 0;
};

struct Ctx {
  fkv_config cfg{};
  fkv_buffers buf{};
  int32_t hkv_local = 0, hq_local = 0, group = 0;
  bool device = false;
  PagePool pools[2];
  std::unordered_map<int64_t, Agent> agents;
  TreeNode base_root;
  std::map<int64_t, std::unique_ptr<TreeNode>> res_roots;
  std::map<int64_t, int32_t> res_adapter;  // residual lineage -> adapter whose xA_i rows it holds (R11)
  int64_t clock[2] = {0, 0};               // independent LRU clocks of the base tree and residual forest (R10)
  int64_t nseq[2] = {0, 0};                // insertion counters
  std::vector<int32_t> copy_log;  // quads (kind, src, dst, rows)
  std::vector<AdapterSlot> adapters;
  std::unordered_map<int32_t, int32_t> adapter_slot;
  uint64_t generation = 1;
  bool has_tc_maps = false;
  bool has_rows_maps = false;
  std::vector<uint8_t> rows_maps;  // k::RowsMaps (ra_rows.cu)
  std::vector<uint8_t> tc_maps;  // 5 CUtensorMap (base K, base V, R_k, R_v, K d-halves) for the tcgen05 kernel
  std::string last_error;
  size_t elem = 2;
  uint64_t upload_seq = 0;                      // plan uploads so far
  std::map<const void*, uint64_t> buffer_owner;  // device plan buffer -> upload id of the plan it holds
  void* dbg = nullptr;  // diagnostics buffer (fkv_debug_timeline)
  int32_t dbg_block = 0;

  Agent& agent(int64_t a) {
    auto it = agents.find(a);
    if (it == agents.end()) throw Error(FKV_E_UNKNOWN_AGENT, "unknown agent " + std::to_string(a));
    return it->second;
  }
};

// ---- plan -------------------------------------------------------------------
// Device-side plan records (uploaded as one blob).
struct DevSeq {         // per sequence
  int32_t q_row0;       // first query row in Q/O
  int32_t q_len;
  int32_t seqlen;
  int32_t adapter_slot;
};
struct DevWarp {        // one warp = up to 16 rows of one residual owner
  int32_t row_off;      // index into rows[] (16 entries, padded with -1)
  int32_t n_rows;
  int32_t res_off;      // offset in res_pages[] of the owner's table (slot 0)
  int32_t adapter_slot;
  int32_t entry_off;    // first partial entry
  int32_t pad_[3];
};
struct DevItem {        // one CTA
  int32_t kv_head;      // local kv head
  int32_t key_begin;    // token range [key_begin, key_end)
  int32_t key_end;
  int32_t base_off;     // offset in base_pages[] of the leader seq's table (slot 0)
  int32_t warp_off;
  int32_t n_warps;
  int32_t pad_[2];
};
struct DevRow {         // query row: (seq, query index, local q head)
  int32_t seq;
  int32_t qi;
  int32_t qh;
  int32_t pos;          // absolute position of the query (causal limit)
};

// a maximal run of page slots [slot0, slot1) over which the member sequences hold the same base pages
struct PlanSeg {
  int64_t slot0, slot1;
  std::vector<int32_t> members;  // plan seq indices
};

struct Plan {
  uint64_t generation = 0;
  int32_t n_seqs = 0;
  int64_t n_rows_q = 0;  // total query rows (sum q_len)
  int32_t kernel = 0;    // 0 mma grouped, 1 simt, 2 tcgen05 (keys on lanes, round 1), 3 tcgen05 rows on lanes
  int32_t tc_rows = 64;  // tcgen05: query rows per CTA
  int32_t tc_pp = 0;     // tcgen05 NONE 64-row: ping-pong key warpgroups (entries per slot doubled)
  std::vector<DevSeq> seqs;
  std::vector<int32_t> base_pages, res_pages;
  std::vector<DevItem> items;
  std::vector<DevWarp> warps;
  std::vector<DevRow> rows;        // warp rows (16 per warp)
  std::vector<int32_t> out_ptr;    // CSR over output rows (n_rows_q * hq_local + 1)
  std::vector<int64_t> comb_rows;  // per output row: e0 | e1 << 32, B_v^h address of layer 0 (combine kernel)
  std::vector<int32_t> out_entries;
  std::vector<int64_t> adapter_ptrs;  // [slot][2] device pointers
  std::vector<int32_t> qrow_seq;      // query row -> plan seq index
  std::vector<int32_t> sched_ptr, sched_items;  // persistent tcgen05 kernel: per-CTA item lists
  std::vector<int32_t> tile_ptr, tile_recs;      // per-CTA tile records (8 ints each, see kernels.hpp)
  std::vector<uint8_t> item_recs;                // per-item k::ItemRecT
  std::vector<int32_t> stage_src;                // staged image -> source warp slot
  bool l2_evict_first = false;                   // see AttnParams::l2_evict_first
  std::vector<int32_t> stage_desc;               // per image: B_k^h address (2 ints), n_rows, h, Q row index [16]
  int32_t n_ctas = 0;
  bool key_range = false;
  size_t ws_ctr_off = 0;             // kernel 3: workspace offset of the item-queue counters
  mutable const void* ws_zeroed = nullptr;  // the workspace whose counters were last zeroed for this plan  // range plan (§8(f) f4): output rows may see no key of [key_begin, key_end)
  size_t stage_off = 0;  // workspace offset of the staged operand images (tcgen05 kernel)
  int64_t n_segments = 0, n_entries = 0, key_tiles = 0, alg_bytes = 0, alg_rank_bytes = 0;
  // rows-on-lanes tcgen05 kernel (kernel 3): k::RItem / RWu / RTile / RRow records (rows.hpp)
  std::vector<uint8_t> r_items, r_wus, r_tiles, r_rows;
  size_t off_ritems = 0, off_rwus = 0, off_rtiles = 0, off_rrows = 0;
  // device layout (offsets into the uploaded blob)
  std::vector<uint8_t> blob;
  size_t off_seqs = 0, off_base = 0, off_res = 0, off_items = 0, off_warps = 0, off_rows = 0, off_outptr = 0,
         off_outent = 0, off_adapters = 0, off_qrow = 0, off_comb = 0,
         off_sptr = 0, off_sitems = 0, off_tptr = 0, off_trecs = 0, off_irecs = 0, off_ssrc = 0, off_sdesc = 0;
  void* dev = nullptr;
  uint64_t upload_id = 0;  // Ctx::upload_seq at the upload into `dev`
  size_t ws_bytes = 0;
};

// Makes the ctx's device current for the scope of a library call that launches work (and restores the caller's).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const Ctx& c) {
    if (c.device && cudaGetDevice(&prev) == cudaSuccess && prev != c.cfg.device) cudaSetDevice(c.cfg.device);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// control.cpp
void ctx_create(Ctx& c, const fkv_config& cfg, const fkv_buffers* buf);
void create_root(Ctx& c, int64_t a, int32_t adapter);
void fork(Ctx& c, int64_t parent, int64_t L, int64_t child, int32_t adapter, uint32_t flags, void* stream);
int64_t fork_tokens(Ctx& c, int64_t child, int32_t adapter, const int32_t* tokens, int64_t n);
void fork_resume(Ctx& c, int64_t child, int32_t adapter, int64_t owner, const int32_t* tokens, int64_t n,
                 int64_t* base_hit, int64_t* res_hit, int64_t* mapped);
int64_t evict(Ctx& c, int32_t kind, int64_t n_pages);
int64_t evictable_pages(const Ctx& c, int32_t kind);
void append(Ctx& c, int32_t n, const int64_t* agents, const int32_t* n_new, const int32_t* tokens, void* stream);
void write_kv(Ctx& c, int32_t layer, int32_t n, const int64_t* agents, const int64_t* start, const int32_t* count,
              const void* kb, const void* vb, const void* rk, const void* rv, uint32_t mask, void* stream);
void release(Ctx& c, int64_t a);
std::string dump(const Ctx& c);
size_t project_workspace_bytes(const Ctx& c, int64_t n_rows);
void project_kv(Ctx& c, int32_t layer, int32_t n, const int64_t* agents, const int64_t* start, const int32_t* count,
                const void* x, int32_t hidden, const void* W_k, const void* W_v, uint32_t mask, void* ws,
                size_t ws_bytes, void* stream);

// plan_rows.cpp: items / WUs / tiles / rows, partial entries, combine CSR and schedule of kernel 3
void build_rows_plan(Ctx& c, Plan& pl, const std::vector<PlanSeg>& segs, const std::vector<const Agent*>& ags,
                     const std::vector<int64_t>& base_off, const std::vector<int64_t>& res_off, int sms);

// plan.cpp
Plan* make_plan(Ctx& c, int32_t n, const fkv_seq* seqs, uint32_t flags, int64_t key_begin = 0,
                int64_t key_end = INT64_MAX);
void upload_plan(Ctx& c, Plan& p, void* dev, size_t bytes, void* stream);
void run_attention(Ctx& c, const Plan& p, int32_t layer, const void* Q, void* O, float scale, void* ws,
                   size_t ws_bytes, void* stream, uint32_t phases = 3u, float* lse = nullptr);

}  // namespace fkv
