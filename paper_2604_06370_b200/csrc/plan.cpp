// Agent-grouping planner (§8(a) row a4) and the attention launch (a5, a6).
//
// Agents forked from the same prefix hold the same physical base pages
// (§5.2 "mapping the globally shared bCache"); the planner finds these
// shared page runs (an LCP over the batch's base block tables), so that one
// CTA streams each shared base tile once and applies it to the query rows of
// every agent holding it.  Inside a segment, rows are grouped by residual
// owner (same adapter and same residual pages), 16 rows per warp: the warp
// rebuilds its owner's K_lora = RoPE(K_res B_k) tile once (Alg1.335) and uses
// it for all its rows.  Long segments are split along the keys (split-KV) to
// fill the 148 SMs; partial (m, l, acc, acc_r) are merged by the combine
// kernel, which also applies the late V fusion acc + acc_r B_v (Eq.4).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <array>
#include <map>
#include <tuple>
#include <set>
#include <string>
#include <unordered_map>

#include "internal.hpp"
#include "kernels.hpp"

namespace fkv {

namespace {
constexpr int kRowsPerWarp = 16;

using Seg = PlanSeg;

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

template <class T>
size_t put(std::vector<uint8_t>& blob, const std::vector<T>& v) {
  size_t off = align256(blob.size());
  blob.resize(off + std::max<size_t>(v.size() * sizeof(T), 16));
  if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
  return off;
}
}  // namespace

Plan* make_plan(Ctx& c, int32_t n, const fkv_seq* seqs, uint32_t flags, int64_t key_begin, int64_t key_end) {
  if (n < 1 || !seqs) throw Error(FKV_E_INVALID, "plan: empty batch");
  const int P = c.cfg.page_size;
  const int g = c.group;
  auto plan = std::make_unique<Plan>();
  Plan& pl = *plan;
  // kernel choice: tcgen05 (2) > mma.sync (0) > SIMT (1)
  const int32_t d_ = c.cfg.head_dim, r_ = c.cfg.rank;
  // diagnostics: FKV_PLAN_TIMING prints the planner's section times; FKV_PLAN_ASSUME_TC plans for kernel 2 on a
  // host-only ctx (planner profiling without a GPU; such a plan cannot run)
  const bool timing = getenv("FKV_PLAN_TIMING") != nullptr;
  const bool assume_tc = getenv("FKV_PLAN_ASSUME_TC") != nullptr;
  auto tic = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "plan %-12s %8.1f us\n", what, std::chrono::duration<double, std::micro>(now - tic).count());
    tic = now;
  };
  const bool tc_ok = c.cfg.dtype == FKV_DTYPE_BF16 && d_ == 128 && r_ == 16 && (c.has_tc_maps || (assume_tc && !c.device)) && (128 % P) == 0 &&
                     P >= 8 && !(flags & (FKV_PLAN_FORCE_SIMT | FKV_PLAN_FORCE_MMA));
  const bool mma_ok = c.cfg.dtype == FKV_DTYPE_BF16 && d_ == 128 && r_ == 16 && !(flags & FKV_PLAN_FORCE_SIMT);
  // rows-on-lanes tcgen05 kernel (kernel 3, ra_rows.cu): NONE residual-RoPE mode, pages of 16..128 tokens
  const bool rows_ok = c.cfg.dtype == FKV_DTYPE_BF16 && d_ == 128 && r_ == 16 && c.has_rows_maps && (128 % P) == 0 &&
                       P >= 16 && c.cfg.rope_mode == FKV_ROPE_NONE && !(flags & (FKV_PLAN_FORCE_SIMT | FKV_PLAN_FORCE_MMA));
  // the mma.sync kernel (warp-level, pre-Blackwell instruction set) is kept only as a comparison baseline: it runs
  // when FKV_PLAN_FORCE_MMA asks for it, never by automatic selection (shapes the tcgen05 kernels do not take run
  // on the SIMT kernel)
  // default: the keys-on-lanes tcgen05 kernel (kernel 2, both RoPE modes: 108 us per C2 layer in NONE mode). The
  // rows-on-lanes kernel (kernel 3) is selected by FKV_PLAN_ROWS_KERNEL / FKV_KERNEL=3: its load pipeline does not
  // beat kernel 2 yet
  pl.kernel = tc_ok ? 2 : ((mma_ok && (flags & FKV_PLAN_FORCE_MMA)) ? 0 : 1);
  bool want_rows = flags & FKV_PLAN_ROWS_KERNEL;
  if (const char* kenv = getenv("FKV_KERNEL")) {
    const int kk = atoi(kenv);
    if (kk == 2 && tc_ok) pl.kernel = 2;
    if (kk == 3) want_rows = true;
  }
  if (want_rows && rows_ok) pl.kernel = 3;
  // tcgen05: 64 query rows per CTA. NONE also has a 128-row variant (FKV_TC_ROWS=128): every MMA instruction then
  // covers N = 128 rows (a tcgen05.mma costs ~120 cycles for any N <= 128, tools/ubench_mma.cu), but its key warps
  // (64 columns each, SIMT row sums, single P^T buffer) are the bottleneck today, so it is not the default;
  // DEFERRED is 64-row only (its K_lora buffers need the TMEM)
  if (pl.kernel == 2) {
    const char* renv = getenv("FKV_TC_ROWS");
    pl.tc_rows = renv ? atoi(renv) : 64;
    if (pl.tc_rows != 64 && pl.tc_rows != 128) pl.tc_rows = 64;
    if (c.cfg.rope_mode != FKV_ROPE_NONE) pl.tc_rows = 64;
    const char* penv = getenv("FKV_TC_PINGPONG");
    pl.tc_pp = (penv ? atoi(penv) : 0) != 0 && pl.tc_rows == 64 && c.cfg.rope_mode == FKV_ROPE_NONE;
  }
  const int kWarpsPerCta = pl.kernel == 2 ? pl.tc_rows / kRowsPerWarp : 8;
  const int kTileKeys = pl.kernel == 2 ? 128 : 64;
  pl.generation = c.generation;
  pl.n_seqs = n;
  std::vector<int64_t> nslots(n), base_off(n), res_off(n);
  std::vector<const Agent*> ags(n);
  int64_t qrow = 0;
  for (int32_t b = 0; b < n; ++b) {
    const Agent& ag = c.agent(seqs[b].agent);
    if (seqs[b].q_len < 1) throw Error(FKV_E_INVALID, "plan: q_len must be >= 1");
    if (seqs[b].q_len > ag.seqlen) throw Error(FKV_E_NO_KEYS, "plan: a query row has no keys");
    // DEFERRED rotates every key at its absolute position (Alg1.335): the RoPE table must cover the sequence
    if (c.device && c.cfg.rope_mode == FKV_ROPE_DEFERRED && ag.seqlen > c.cfg.max_pos)
      throw Error(FKV_E_INVALID, "plan: agent " + std::to_string(ag.id) + " seqlen " + std::to_string(ag.seqlen) +
                                     " exceeds the RoPE table (max_pos " + std::to_string(c.cfg.max_pos) + ")");
    auto it = c.adapter_slot.find(ag.adapter);
    if (it == c.adapter_slot.end()) throw Error(FKV_E_INVALID, "plan: adapter not registered");
    ags[b] = &ag;
    nslots[b] = (ag.seqlen + P - 1) / P;
    base_off[b] = (int64_t)pl.base_pages.size();
    res_off[b] = (int64_t)pl.res_pages.size();
    pl.base_pages.insert(pl.base_pages.end(), ag.base.begin(), ag.base.begin() + nslots[b]);
    pl.res_pages.insert(pl.res_pages.end(), ag.res.begin(), ag.res.begin() + nslots[b]);
    pl.seqs.push_back({(int32_t)qrow, seqs[b].q_len, (int32_t)ag.seqlen, it->second});
    for (int32_t i = 0; i < seqs[b].q_len; ++i) pl.qrow_seq.push_back(b);
    qrow += seqs[b].q_len;
    if (flags & FKV_PLAN_CHECK_WRITTEN) {
      for (int64_t s = 0; s < nslots[b]; ++s) {
        const int rows = (int)std::min<int64_t>(P, ag.seqlen - s * P);
        for (int32_t l = 0; l < c.cfg.n_layers; ++l)
          if (!c.pools[0].wtest_prefix(ag.base[s], l, rows) || !c.pools[1].wtest_prefix(ag.res[s], l, rows))
            throw Error(FKV_E_UNWRITTEN, "plan: agent " + std::to_string(ag.id) + " slot " + std::to_string(s) +
                                             " layer " + std::to_string(l) + " not written");
      }
    }
  }
  if (qrow > INT32_MAX / 64) throw Error(FKV_E_INVALID, "plan: too many query rows");
  pl.n_rows_q = qrow;

  lap("seqs");
  // ---- segments: maximal slot runs over which the member set shares pages --
  std::vector<Seg> segs;
  {
    std::vector<std::pair<std::vector<int32_t>, int64_t>> stack;
    std::vector<int32_t> all(n);
    for (int32_t b = 0; b < n; ++b) all[b] = b;
    stack.push_back({all, 0});
    while (!stack.empty()) {
      auto [mem, slot] = std::move(stack.back());
      stack.pop_back();
      int64_t s = slot;
      for (;;) {
        bool ok = true;
        for (int32_t b : mem)
          if (nslots[b] <= s || ags[b]->base[s] != ags[mem[0]]->base[s]) { ok = false; break; }
        if (!ok) break;
        ++s;
      }
      if (s > slot) segs.push_back({slot, s, mem});
      std::map<int32_t, std::vector<int32_t>> groups;  // page id -> members (deterministic order)
      for (int32_t b : mem)
        if (nslots[b] > s) groups[ags[b]->base[s]].push_back(b);
      // push in reverse so segments come out in ascending page-id order
      for (auto it = groups.rbegin(); it != groups.rend(); ++it) stack.push_back({it->second, s});
    }
  }
  lap("segments");
  // range plan (§8(f) f4, sequence split across GPUs): only the keys of [key_begin, key_end), page-aligned
  if (key_begin != 0 || key_end != INT64_MAX) {
    const int P_ = c.cfg.page_size;
    if (key_begin < 0 || key_end <= key_begin || key_begin % P_ || (key_end != INT64_MAX && key_end % P_))
      throw Error(FKV_E_INVALID, "plan: key range must be page-aligned and non-empty");
    pl.key_range = true;
    const int64_t s0 = key_begin / P_, s1 = key_end == INT64_MAX ? INT64_MAX : key_end / P_;
    std::vector<Seg> kept;
    for (Seg sg : segs) {
      sg.slot0 = std::max<int64_t>(sg.slot0, s0);
      sg.slot1 = std::min<int64_t>(sg.slot1, s1);
      if (sg.slot1 > sg.slot0) kept.push_back(std::move(sg));
    }
    segs.swap(kept);
  }
  pl.n_segments = (int64_t)segs.size();
  int sms = 148;
  if (c.device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, c.cfg.device) == cudaSuccess && v > 0) sms = v;
  }
  if (pl.kernel == 3) {
    build_rows_plan(c, pl, segs, ags, base_off, res_off, sms);
    return plan.release();
  }

  // ---- rows -> owner groups -> warps -> CTAs -> key splits ------------------
  struct Cta {
    int32_t kv_head;
    int64_t k0, k1;
    int32_t base_off;
    std::vector<int32_t> warp_ids;
  };
  std::vector<Cta> ctas;
  std::vector<std::vector<int32_t>> warp_rows;  // row indices into pl.rows per warp (before splitting)
  std::vector<DevWarp> proto_warps;
  std::vector<DevRow> proto_rows;
  int64_t res_bytes = 0, base_bytes = 0;
  const size_t el = c.elem;
  const int32_t hkv = c.hkv_local, d = c.cfg.head_dim, r = c.cfg.rank;
  for (const Seg& sg : segs) {
    int64_t maxlen = 0;
    for (int32_t b : sg.members) maxlen = std::max<int64_t>(maxlen, ags[b]->seqlen);
    const int64_t k0 = sg.slot0 * P, k1 = std::min<int64_t>(sg.slot1 * P, maxlen);
    if (k1 <= k0) continue;
    base_bytes += (k1 - k0) * hkv * d * 2 * (int64_t)el;
    // owner key: adapter slot + residual pages over the segment. Members sorted by that key in place (no key
    // copies), equal runs are one owner; the order matches the former map over (adapter, page list)
    std::vector<std::pair<std::pair<int32_t, int32_t>, std::vector<int32_t>>> owners;  // ((adapter, -), members)
    {
      std::vector<int32_t> mem(sg.members);
      auto rb = [&](int32_t b) { return ags[b]->res.begin() + sg.slot0; };
      auto re = [&](int32_t b) { return ags[b]->res.begin() + sg.slot1; };
      auto less = [&](int32_t a, int32_t b) {
        const int32_t sa = pl.seqs[a].adapter_slot, sb = pl.seqs[b].adapter_slot;
        if (sa != sb) return sa < sb;
        return std::lexicographical_compare(rb(a), re(a), rb(b), re(b));
      };
      std::stable_sort(mem.begin(), mem.end(), less);
      for (size_t i = 0; i < mem.size(); ++i) {
        if (i == 0 || less(mem[i - 1], mem[i]))
          owners.push_back({{pl.seqs[mem[i]].adapter_slot, 0}, {}});
        owners.back().second.push_back(mem[i]);
      }
    }
    for (const auto& ow : owners) {
      int64_t okeys = 0;
      for (int32_t b : ow.second) okeys = std::max<int64_t>(okeys, std::min<int64_t>(k1, ags[b]->seqlen) - k0);
      res_bytes += okeys * r * 2 * (int64_t)el;
    }
    for (int32_t h = 0; h < hkv; ++h) {
      std::vector<int32_t> cta_warps;
      for (const auto& ow : owners) {
        std::vector<DevRow> rows;
        for (int32_t b : ow.second) {
          const int32_t L = pl.seqs[b].seqlen, C = pl.seqs[b].q_len;
          for (int32_t i = 0; i < C; ++i) {
            const int32_t pos = L - C + i;
            if (pos < k0) continue;  // no key of this segment is visible to the row
            for (int32_t kk = h * g; kk < (h + 1) * g; ++kk) rows.push_back({b, i, kk, pos});
          }
        }
        for (size_t o = 0; o < rows.size(); o += kRowsPerWarp) {
          DevWarp w{};
          w.row_off = (int32_t)proto_rows.size();
          w.n_rows = (int32_t)std::min<size_t>(kRowsPerWarp, rows.size() - o);
          w.res_off = (int32_t)res_off[ow.second[0]];
          w.adapter_slot = ow.first.first;
          for (int j = 0; j < kRowsPerWarp; ++j)
            proto_rows.push_back(j < w.n_rows ? rows[o + j] : DevRow{-1, 0, 0, -1});
          cta_warps.push_back((int32_t)proto_warps.size());
          proto_warps.push_back(w);
          if ((int)cta_warps.size() == kWarpsPerCta) {
            ctas.push_back({h, k0, k1, (int32_t)base_off[sg.members[0]], cta_warps});
            cta_warps.clear();
          }
        }
      }
      if (!cta_warps.empty()) ctas.push_back({h, k0, k1, (int32_t)base_off[sg.members[0]], cta_warps});
    }
  }
  lap("ctas");
  // L2 policy of the base tiles: evict-first when each (segment, kv head) tile is read by <= 4 row blocks (decode
  // batches), normal when many row blocks reuse it (prefill chunks, large agent counts); FKV_L2_EVICT=0/1 forces
  {
    std::map<std::tuple<int64_t, int32_t, int32_t>, int32_t> readers;  // (segment start, base pages, kv head)
    int32_t most = 0;
    for (const Cta& ct : ctas) most = std::max(most, ++readers[std::make_tuple(ct.k0, ct.base_off, ct.kv_head)]);
    const char* eenv = getenv("FKV_L2_EVICT");
    pl.l2_evict_first = eenv ? atoi(eenv) != 0 : most <= 4;
  }
  // key split. mma.sync / SIMT: ~2 waves of CTAs over the SMs. tcgen05 (persistent, one CTA per SM):
  // pieces of about half the average per-CTA load, so the greedy schedule below balances.
  int64_t total_tiles = 0;
  for (const Cta& ct : ctas) total_tiles += (ct.k1 - ct.k0 + kTileKeys - 1) / kTileKeys;
  int64_t split_tiles;
  if (pl.kernel == 2) {
    const char* penv = getenv("FKV_PIECE_TILES");
    // pieces of ~0.55 of the average per-CTA load (C2: 8 pieces of 32 tiles per 256-tile segment; measured on B200:
    // 29-tile pieces -2%, 43-tile pieces -13%)
    split_tiles = penv ? std::max<int64_t>(1, atoll(penv)) : std::max<int64_t>(4, (int64_t)(total_tiles / (1.8 * sms)));
    split_tiles = std::min<int64_t>(split_tiles, 511);  // ItemRecT::pos1 is 16-bit relative to the item start
  } else {
    const char* wenv = getenv("FKV_SPLIT_WAVES");
    const double waves = wenv ? atof(wenv) : 2.0;
    const int64_t target = std::max<int64_t>(1, (int64_t)(waves * sms));
    split_tiles = std::max<int64_t>(2, (total_tiles + target - 1) / std::max<int64_t>(1, target));
  }
  int64_t entries = 0;
  std::vector<std::array<int64_t, 3>> order_key;  // (segment start, piece, cta) per item
  std::vector<int64_t> item_cost;
  {
    size_t n_it = 0, n_w = 0;
    for (const Cta& ct : ctas) {
      const int64_t tiles = (ct.k1 - ct.k0 + kTileKeys - 1) / kTileKeys;
      const int64_t pieces = (tiles + split_tiles - 1) / split_tiles;
      n_it += pieces;
      n_w += pieces * ct.warp_ids.size();
    }
    pl.items.reserve(n_it);
    order_key.reserve(n_it);
    item_cost.reserve(n_it);
    pl.warps.reserve(n_w);
    pl.rows.reserve(n_w * kRowsPerWarp);
  }
  for (size_t ci = 0; ci < ctas.size(); ++ci) {
    const Cta& ct = ctas[ci];
    const int64_t tiles = (ct.k1 - ct.k0 + kTileKeys - 1) / kTileKeys;
    const int64_t n_pieces = (tiles + split_tiles - 1) / split_tiles;
    const int64_t piece = (tiles + n_pieces - 1) / n_pieces;
    for (int64_t t = 0, pi = 0; t < tiles; t += piece, ++pi) {
      const int64_t kb = ct.k0 + t * kTileKeys;
      const int64_t ke = std::min<int64_t>(ct.k1, ct.k0 + (t + piece) * kTileKeys);
      // rows that see no key of this split get no entry
      DevItem it{};
      it.kv_head = ct.kv_head;
      it.key_begin = (int32_t)kb;
      it.key_end = (int32_t)ke;
      it.base_off = ct.base_off;
      it.warp_off = (int32_t)pl.warps.size();
      for (int32_t wi : ct.warp_ids) {
        DevWarp w = proto_warps[wi];
        w.row_off = (int32_t)pl.rows.size();
        int32_t nr = 0;
        DevRow keep[kRowsPerWarp];
        for (int j = 0; j < proto_warps[wi].n_rows; ++j) {
          const DevRow& rw = proto_rows[proto_warps[wi].row_off + j];
          if (rw.pos >= kb) keep[nr++] = rw;
        }
        if (nr == 0) continue;
        w.n_rows = nr;
        w.entry_off = (int32_t)entries;
        // entries are per warp slot (padded) for simple indexing; ping-pong: one block of 16 per key warpgroup
        entries += (pl.tc_pp ? 2 : 1) * kRowsPerWarp;
        for (int j = 0; j < kRowsPerWarp; ++j) pl.rows.push_back(j < nr ? keep[j] : DevRow{-1, 0, 0, -1});
        pl.warps.push_back(w);
      }
      it.n_warps = (int32_t)pl.warps.size() - it.warp_off;
      if (it.n_warps > 0) {
        pl.items.push_back(it);
        const int64_t nt = (ke - kb + kTileKeys - 1) / kTileKeys;
        pl.key_tiles += nt;
        order_key.push_back({ct.k0, pi, (int64_t)ci});
        if (pl.kernel == 2) {
          // tcgen05: a tile costs its MMA instructions (S 8 + one per residual group, PV 8; ~115 cycles each, the
          // binding resource), an item ~22 more (header, first-tile softmax setup, epilogue; B200 timeline)
          int32_t ng = 0;
          for (int o = 0; o < it.n_warps; ++o) {
            const DevWarp& w = pl.warps[it.warp_off + o];
            ng += o == 0 || w.res_off != pl.warps[it.warp_off + o - 1].res_off ||
                  w.adapter_slot != pl.warps[it.warp_off + o - 1].adapter_slot;
          }
          static const int64_t ovh = getenv("FKV_ITEM_OVERHEAD") ? atoll(getenv("FKV_ITEM_OVERHEAD")) : 22;
          item_cost.push_back(nt * (16 + ng) + ovh);
        } else {
          // cost in KB of shared-memory ingest: base K + V tiles, R_k + R_v per slot, + ~5 tiles per item
          item_cost.push_back((nt + 5) * (64 + 8 * it.n_warps));
        }
      }
    }
  }
  lap("items");
  if (pl.kernel == 2) {
    // staged operand images (Q rows, q~ / packed B_k) per item slot; the key-range pieces of one row block carry
    // identical slots, so they share one contiguous block of images (DevItem::pad_[0] = first image)
    // items of one CTA row block (order_key[i][2]) carry the same slots unless a causal split dropped rows: an
    // item reuses the images of an earlier item of its row block whose slots match exactly
    std::unordered_map<int64_t, std::vector<int32_t>> img_of;  // row block -> items that own an image block
    auto same_slots = [&](const DevItem& a, const DevItem& b) {
      if (a.n_warps != b.n_warps) return false;
      for (int o = 0; o < a.n_warps; ++o) {
        const DevWarp& wa = pl.warps[a.warp_off + o];
        const DevWarp& wb = pl.warps[b.warp_off + o];
        if (wa.adapter_slot != wb.adapter_slot || wa.n_rows != wb.n_rows ||
            std::memcmp(&pl.rows[wa.row_off], &pl.rows[wb.row_off], sizeof(DevRow) * kRowsPerWarp) != 0)
          return false;
      }
      return true;
    };
    for (size_t i = 0; i < pl.items.size(); ++i) {
      DevItem& it = pl.items[i];
      auto& cand = img_of[order_key[i][2]];
      int32_t found = -1;
      for (int32_t j : cand)
        if (same_slots(pl.items[j], it)) { found = pl.items[j].pad_[0]; break; }
      if (found < 0) {
        found = (int32_t)pl.stage_src.size();
        for (int o = 0; o < it.n_warps; ++o) pl.stage_src.push_back(it.warp_off + o);
        cand.push_back((int32_t)i);
      }
      it.pad_[0] = found;
    }
    // persistent schedule: items in (segment, piece, row block) order, each to the least-loaded CTA, so the
    // row blocks and kv heads that stream the same base / residual pages run at the same time (L2 reuse)
    const int32_t n_items = (int32_t)pl.items.size();
    std::vector<int32_t> idx(n_items);
    for (int32_t i = 0; i < n_items; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return order_key[a] < order_key[b]; });
    pl.n_ctas = std::max<int32_t>(1, std::min<int32_t>(sms, n_items));
    std::vector<std::vector<int32_t>> per(pl.n_ctas);
    std::set<std::pair<int64_t, int32_t>> load;
    for (int32_t cc = 0; cc < pl.n_ctas; ++cc) load.insert({0, cc});
    for (int32_t i : idx) {
      auto lo = *load.begin();
      load.erase(load.begin());
      per[lo.second].push_back(i);
      load.insert({lo.first + item_cost[i], lo.second});
    }
    pl.sched_ptr.assign(1, 0);
    for (auto& v : per) {
      pl.sched_items.insert(pl.sched_items.end(), v.begin(), v.end());
      pl.sched_ptr.push_back((int32_t)pl.sched_items.size());
    }
  lap("schedule");
    // item records (k::ItemRecT<slots>)
    auto build_recs = [&](auto tag) {
      using Rec = decltype(tag);
      constexpr int S = (int)(sizeof(Rec::n_rows) / sizeof(int32_t));
      pl.item_recs.assign(pl.items.size() * sizeof(Rec), 0);
      for (size_t i = 0; i < pl.items.size(); ++i) {
        const DevItem& it = pl.items[i];
        if (it.n_warps > S) throw Error(FKV_E_INVALID, "plan: item has too many slots");
        Rec r{};
        r.k0 = it.key_begin;
        r.k1 = it.key_end;
        r.n_tiles = (it.key_end - it.key_begin + kTileKeys - 1) / kTileKeys;
        int32_t ng = 0, gmask = 0;
        for (int o = 0; o < it.n_warps; ++o) {
          const DevWarp& w = pl.warps[it.warp_off + o];
          const bool first = o == 0 || w.res_off != pl.warps[it.warp_off + o - 1].res_off ||
                             w.adapter_slot != pl.warps[it.warp_off + o - 1].adapter_slot;
          if (first) { ++ng; gmask |= 1 << o; }
          r.n_rows[o] = w.n_rows;
          r.entry_off[o] = w.entry_off;
          for (int j = 0; j < w.n_rows; ++j) {
            const int64_t v = (int64_t)pl.rows[w.row_off + j].pos - it.key_begin + 1;
            r.pos1[16 * o + j] = (uint16_t)std::min<int64_t>(65535, std::max<int64_t>(0, v));
          }
        }
        r.meta = it.n_warps | (ng << 4) | (gmask << 8) | (it.kv_head << 16);
        // bits 16..: per 32-column chunk, some real query column does not see every key of the item (causal masking;
        // the kernel masks unused columns from n_rows)
        for (int o = 0; o < it.n_warps; ++o)
          for (int j = 0; j < r.n_rows[o]; ++j)
            if ((int64_t)r.pos1[16 * o + j] < (int64_t)it.key_end - it.key_begin) r.n_tiles |= 1 << (16 + (16 * o + j) / 32);
        std::memcpy(pl.item_recs.data() + i * sizeof(Rec), &r, sizeof(r));
      }
    };
    if (pl.tc_rows == 128) build_recs(k::ItemRecT<8>{}); else build_recs(k::ItemRecT<4>{});
  lap("itemrecs");
    // tile records (the residual loader and the TMA producer stream them instead of chasing page tables)
    pl.tile_ptr.assign(1, 0);
    pl.tile_recs.clear();
    pl.tile_recs.reserve((size_t)pl.key_tiles * k::kTileRecInts);
    for (auto& v : per) {
      for (int32_t i : v) {
        const DevItem& it = pl.items[i];
        int32_t meta = it.n_warps, ng = 0, gmask = 0;
        for (int o = 0; o < it.n_warps; ++o) {
          const DevWarp& w = pl.warps[it.warp_off + o];
          const bool first = o == 0 || w.res_off != pl.warps[it.warp_off + o - 1].res_off ||
                             w.adapter_slot != pl.warps[it.warp_off + o - 1].adapter_slot;
          if (first) { ++ng; gmask |= 1 << o; }
        }
        meta |= (ng << 4) | (gmask << 8) | (it.kv_head << 16);
        for (int32_t t0 = it.key_begin; t0 < it.key_end; t0 += kTileKeys) {
          const int32_t sl = t0 / P;
          const size_t at = pl.tile_recs.size();
          pl.tile_recs.resize(at + k::kTileRecInts, 0);
          int32_t* rec = pl.tile_recs.data() + at;
          rec[0] = t0; rec[1] = it.key_end; rec[2] = meta; rec[3] = pl.base_pages[it.base_off + sl];
          for (int o = 0; o < 8; ++o) rec[4 + o] = -1;
          for (int o = 0; o < it.n_warps; ++o) rec[4 + o] = pl.res_pages[pl.warps[it.warp_off + o].res_off + sl];
        }
      }
      pl.tile_ptr.push_back((int32_t)(pl.tile_recs.size() / k::kTileRecInts));
    }
  }
  lap("tilerecs");
  if (entries > INT32_MAX) throw Error(FKV_E_INVALID, "plan: too many partial entries");
  pl.n_entries = entries;
  // CSR: output row -> entries
  const int64_t n_out = pl.n_rows_q * c.hq_local;
  std::vector<int32_t> cnt(n_out + 1, 0);
  const int n_halves = pl.tc_pp ? 2 : 1;  // ping-pong: each row has one partial entry per key warpgroup and item
  for (const DevWarp& w : pl.warps)
    for (int j = 0; j < w.n_rows; ++j) {
      const DevRow& rw = pl.rows[w.row_off + j];
      cnt[(int64_t)(pl.seqs[rw.seq].q_row0 + rw.qi) * c.hq_local + rw.qh + 1] += n_halves;
    }
  for (int64_t i = 0; i < n_out; ++i) cnt[i + 1] += cnt[i];
  pl.out_ptr = cnt;
  pl.out_entries.assign(cnt[n_out], 0);
  std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
  for (const DevWarp& w : pl.warps)
    for (int j = 0; j < w.n_rows; ++j) {
      const DevRow& rw = pl.rows[w.row_off + j];
      const int64_t o = (int64_t)(pl.seqs[rw.seq].q_row0 + rw.qi) * c.hq_local + rw.qh;
      for (int hv = 0; hv < n_halves; ++hv) pl.out_entries[fill[o]++] = w.entry_off + kRowsPerWarp * hv + j;
    }
  for (int64_t o = 0; o < n_out; ++o)
    if (!pl.key_range && pl.out_ptr[o + 1] == pl.out_ptr[o]) throw Error(FKV_E_NO_KEYS, "plan: an output row has no keys");
  lap("csr");
  // adapters
  pl.adapter_ptrs.resize(c.adapters.size() * 2);
  for (size_t s = 0; s < c.adapters.size(); ++s) {
    pl.adapter_ptrs[2 * s] = (int64_t)(intptr_t)c.adapters[s].bk;
    pl.adapter_ptrs[2 * s + 1] = (int64_t)(intptr_t)c.adapters[s].bv;
  }
  // algorithmic bytes per layer: shared base once per segment,
  // stager descriptors: one 80-byte record per image (no pointer chasing in the stage kernel)
  pl.stage_desc.assign(pl.stage_src.size() * 20, 0);
  for (size_t i = 0; i < pl.stage_src.size(); ++i) {
    const DevWarp& w = pl.warps[pl.stage_src[i]];
    const int32_t h = pl.rows[w.row_off].qh / c.group;
    const int64_t bk = pl.adapter_ptrs[2 * w.adapter_slot] + (int64_t)h * r * d * el;
    int32_t* dsc = pl.stage_desc.data() + 20 * i;
    dsc[0] = (int32_t)(bk & 0xffffffffll);
    dsc[1] = (int32_t)(bk >> 32);
    dsc[2] = w.n_rows;
    dsc[3] = h;
    for (int j = 0; j < 16; ++j) {
      if (j < w.n_rows) {
        const DevRow& rw = pl.rows[w.row_off + j];
        dsc[4 + j] = (pl.seqs[rw.seq].q_row0 + rw.qi) * c.hq_local + rw.qh;
      } else {
        dsc[4 + j] = -1;
      }
    }
  }
  // combine rows: entry range and the row's B_v^h (one 16-byte load per output row)
  pl.comb_rows.assign(2 * n_out, 0);
  for (int64_t o = 0; o < n_out; ++o) {
    const int32_t qrow = (int32_t)(o / c.hq_local), qh = (int32_t)(o % c.hq_local), h = qh / c.group;
    const int32_t slot = pl.seqs[pl.qrow_seq[qrow]].adapter_slot;
    pl.comb_rows[2 * o] = (int64_t)(uint32_t)pl.out_ptr[o] | ((int64_t)pl.out_ptr[o + 1] << 32);
    pl.comb_rows[2 * o + 1] = pl.adapter_ptrs[2 * slot + 1] + (int64_t)h * r * d * el;
  }
  // residual once per (segment, owner), adapters once, Q in + O out.
  std::set<int32_t> used_adapters;
  for (const DevSeq& s : pl.seqs) used_adapters.insert(s.adapter_slot);
  pl.alg_rank_bytes = res_bytes + (int64_t)used_adapters.size() * 2 * r * d * hkv * (int64_t)el;
  pl.alg_bytes = base_bytes + res_bytes + (int64_t)used_adapters.size() * 2 * r * d * hkv * (int64_t)el +
                 pl.n_rows_q * c.hq_local * d * 2 * (int64_t)el;
  lap("desc");
  // blob
  // one allocation: offsets first, then the copies (resizing per array re-copied the growing blob)
  {
    size_t total = 0;
    auto at = [&](const auto& v) {
      const size_t off = align256(total);
      total = off + std::max<size_t>(v.size() * sizeof(v[0]), 16);
      return off;
    };
    pl.off_seqs = at(pl.seqs);
    pl.off_base = at(pl.base_pages);
    pl.off_res = at(pl.res_pages);
    pl.off_items = at(pl.items);
    pl.off_warps = at(pl.warps);
    pl.off_rows = at(pl.rows);
    pl.off_outptr = at(pl.out_ptr);
    pl.off_outent = at(pl.out_entries);
    pl.off_adapters = at(pl.adapter_ptrs);
    pl.off_qrow = at(pl.qrow_seq);
    pl.off_comb = at(pl.comb_rows);
    pl.off_sptr = at(pl.sched_ptr);
    pl.off_sitems = at(pl.sched_items);
    pl.off_tptr = at(pl.tile_ptr);
    pl.off_trecs = at(pl.tile_recs);
    pl.off_irecs = at(pl.item_recs);
    pl.off_ssrc = at(pl.stage_src);
    pl.off_sdesc = at(pl.stage_desc);
    pl.blob.assign(align256(total), 0);
    auto cp = [&](size_t off, const auto& v) {
      if (!v.empty()) std::memcpy(pl.blob.data() + off, v.data(), v.size() * sizeof(v[0]));
    };
    cp(pl.off_seqs, pl.seqs);
    cp(pl.off_base, pl.base_pages);
    cp(pl.off_res, pl.res_pages);
    cp(pl.off_items, pl.items);
    cp(pl.off_warps, pl.warps);
    cp(pl.off_rows, pl.rows);
    cp(pl.off_outptr, pl.out_ptr);
    cp(pl.off_outent, pl.out_entries);
    cp(pl.off_adapters, pl.adapter_ptrs);
    cp(pl.off_qrow, pl.qrow_seq);
    cp(pl.off_comb, pl.comb_rows);
    cp(pl.off_sptr, pl.sched_ptr);
    cp(pl.off_sitems, pl.sched_items);
    cp(pl.off_tptr, pl.tile_ptr);
    cp(pl.off_trecs, pl.tile_recs);
    cp(pl.off_irecs, pl.item_recs);
    cp(pl.off_ssrc, pl.stage_src);
    cp(pl.off_sdesc, pl.stage_desc);
  }
  pl.blob.resize(align256(pl.blob.size()));
  lap("blob");
  pl.ws_bytes = align256((size_t)pl.n_entries * (size_t)(k::kEntAcc + d + r) * sizeof(float));
  if (pl.kernel == 2) {
    pl.stage_off = pl.ws_bytes;
    pl.ws_bytes += align256(pl.stage_src.size() * (size_t)k::kStageBytes);
  }
  return plan.release();
}

void upload_plan(Ctx& c, Plan& p, void* dev, size_t bytes, void* stream) {
  if (!c.device) throw Error(FKV_E_INVALID, "plan_upload: host-only ctx");
  if (!dev || bytes < p.blob.size() || ((uintptr_t)dev & 255)) throw Error(FKV_E_INVALID, "plan_upload: bad buffer");
  DeviceGuard dg(c);
  cudaError_t e = cudaMemcpyAsync(dev, p.blob.data(), p.blob.size(), cudaMemcpyHostToDevice, (cudaStream_t)stream);
  if (e != cudaSuccess) throw Error(FKV_E_CUDA, std::string("plan_upload: ") + cudaGetErrorString(e));
  p.dev = dev;
  p.upload_id = ++c.upload_seq;
  c.buffer_owner[dev] = p.upload_id;  // a buffer belongs to the plan uploaded into it last
}

void run_attention(Ctx& c, const Plan& p, int32_t layer, const void* Q, void* O, float scale, void* ws,
                   size_t ws_bytes, void* stream, uint32_t phases, float* lse) {
  if (phases == 0 || (phases & ~15u) || ((phases & FKV_PHASE_STAGE) && (phases & (FKV_PHASE_NOSTAGE | FKV_PHASE_MAIN))) ||
      ((phases & FKV_PHASE_NOSTAGE) && !(phases & FKV_PHASE_MAIN)))
    throw Error(FKV_E_INVALID, "attention: bad phases");
  if (!c.device) throw Error(FKV_E_INVALID, "attention: host-only ctx");
  if (p.generation != c.generation) throw Error(FKV_E_STALE, "attention: plan is stale");
  if (!p.dev) throw Error(FKV_E_INVALID, "attention: plan not uploaded");
  {
    auto it = c.buffer_owner.find(p.dev);
    if (it == c.buffer_owner.end() || it->second != p.upload_id)
      throw Error(FKV_E_STALE, "attention: another plan was uploaded into this plan's device buffer since");
  }
  DeviceGuard dg(c);
  if (layer < 0 || layer >= c.cfg.n_layers || !Q || !O) throw Error(FKV_E_INVALID, "attention: bad layer/Q/O");
  if (!ws || ws_bytes < p.ws_bytes || ((uintptr_t)ws & 255)) throw Error(FKV_E_INVALID, "attention: workspace too small or not 256-byte aligned");
  const uint8_t* base = (const uint8_t*)p.dev;
  k::AttnParams a{};
  a.lse = lse;
  a.base_k = c.buf.base_k; a.base_v = c.buf.base_v; a.res_k = c.buf.res_k; a.res_v = c.buf.res_v;
  a.rope_cos = c.buf.rope_cos; a.rope_sin = c.buf.rope_sin;
  a.Q = Q; a.O = O; a.ws = (float*)ws;
  a.seqs = (const DevSeq*)(base + p.off_seqs);
  a.base_pages = (const int32_t*)(base + p.off_base);
  a.res_pages = (const int32_t*)(base + p.off_res);
  a.items = (const DevItem*)(base + p.off_items);
  a.warps = (const DevWarp*)(base + p.off_warps);
  a.rows = (const DevRow*)(base + p.off_rows);
  a.out_ptr = (const int32_t*)(base + p.off_outptr);
  a.out_entries = (const int32_t*)(base + p.off_outent);
  a.adapters = (const int64_t*)(base + p.off_adapters);
  a.qrow_seq = (const int32_t*)(base + p.off_qrow);
  a.comb_rows = (const longlong2*)(base + p.off_comb);
  const int64_t P = c.cfg.page_size, d = c.cfg.head_dim, r = c.cfg.rank;
  a.base_layer_stride = c.cfg.n_base_pages * c.hkv_local * P * d;
  a.res_layer_stride = c.cfg.n_res_pages * P * r;
  a.adapter_layer_stride = (int64_t)c.hkv_local * r * d;
  a.nb = c.cfg.n_base_pages;
  a.nr = c.cfg.n_res_pages;
  a.layer = layer; a.hkv = c.hkv_local; a.hq = c.hq_local; a.group = c.group; a.P = (int32_t)P;
  a.d = (int32_t)d; a.r = (int32_t)r; a.rope_mode = c.cfg.rope_mode; a.dtype = c.cfg.dtype;
  a.n_items = (int32_t)p.items.size();
  a.n_out_rows = (int32_t)(p.n_rows_q * c.hq_local);
  a.entry_stride = (int32_t)(k::kEntAcc + d + r);
  if (scale <= 0.f) scale = 1.0f / std::sqrt((float)d);
  a.scale_log2 = scale * 1.4426950408889634f;
  a.dbg = (long long*)c.dbg;
  a.dbg_block = c.dbg_block;
  a.max_pos = c.cfg.max_pos;
  { const char* e = getenv("FKV_TC_PREFETCH"); a.tc_prefetch = e ? atoi(e) : 3; }
  a.res_swz = c.cfg.dtype == FKV_DTYPE_BF16 && c.cfg.rank == 16;
  a.sched_ptr = (const int32_t*)(base + p.off_sptr);
  a.sched_items = (const int32_t*)(base + p.off_sitems);
  a.tile_ptr = (const int32_t*)(base + p.off_tptr);
  a.tile_recs = (const int4*)(base + p.off_trecs);
  a.item_recs = base + p.off_irecs;
  a.tc_rows = p.tc_rows;
  a.tc_pp = p.tc_pp;
  a.l2_evict_first = p.l2_evict_first ? 1 : 0;
  a.stage_src = (const int32_t*)(base + p.off_ssrc);
  a.stage_desc = (const int4*)(base + p.off_sdesc);
  a.n_ctas = p.n_ctas;
  a.stage = p.kernel == 2 ? (uint8_t*)ws + p.stage_off : nullptr;
  cudaError_t e = cudaSuccess;
  if (p.kernel == 3) {
    if (phases & FKV_PHASE_MAIN) {
      k::RowsParams rp{};
      rp.base_k = c.buf.base_k; rp.base_v = c.buf.base_v; rp.res_k = c.buf.res_k; rp.res_v = c.buf.res_v;
      rp.Q = Q; rp.ws = (float*)ws;
      rp.items = (const k::RItem*)(base + p.off_ritems);
      rp.wus = (const k::RWu*)(base + p.off_rwus);
      rp.tiles = (const k::RTile*)(base + p.off_rtiles);
      rp.rows = (const k::RRow*)(base + p.off_rrows);
      rp.base_pages = a.base_pages;
      rp.res_pages = a.res_pages;
      rp.adapters = a.adapters;
      rp.sched_ptr = a.sched_ptr;
      rp.sched_items = a.sched_items;
      rp.n_items = (int32_t)(p.r_items.size() / sizeof(k::RItem));
      rp.ctr = (int32_t*)((uint8_t*)ws + p.ws_ctr_off);
      if (p.ws_zeroed != ws) {  // the kernel leaves the counters zero; a fresh workspace needs them zeroed once
        e = cudaMemsetAsync(rp.ctr, 0, 8, (cudaStream_t)stream);
        if (e != cudaSuccess) throw Error(FKV_E_CUDA, std::string("attention: ") + cudaGetErrorString(e));
        p.ws_zeroed = ws;
      }
      rp.base_rows_layer = (int64_t)layer * c.cfg.n_base_pages * c.hkv_local * P;
      rp.res_layer_elems = a.res_layer_stride;
      rp.adapter_layer_elems = a.adapter_layer_stride;
      rp.layer = layer; rp.hkv = c.hkv_local; rp.P = (int32_t)P; rp.n_ctas = p.n_ctas;
      rp.entry_stride = a.entry_stride;
      rp.scale_log2 = a.scale_log2;
      rp.dbg = a.dbg; rp.dbg_block = a.dbg_block;
      rp.flags = getenv("FKV_ROWS_FLAGS") ? atoi(getenv("FKV_ROWS_FLAGS")) : 0;
      rp.hang = k::hang_slot();
      rp.prefetch = getenv("FKV_ROWS_PREFETCH") ? atoi(getenv("FKV_ROWS_PREFETCH")) : 3;
      e = k::launch_attention_rows(rp, *(const k::RowsMaps*)c.rows_maps.data(), (cudaStream_t)stream);
    }
    if (e == cudaSuccess && (phases & FKV_PHASE_COMBINE)) e = k::launch_combine(a, (cudaStream_t)stream);
    if (e != cudaSuccess) throw Error(FKV_E_CUDA, std::string("attention: ") + cudaGetErrorString(e));
    return;
  }
  // FKV_DIAG_NOSTAGE (diagnostics only: the main kernel reads whatever images the last stager left) times the
  // stager's share of the step
  static const bool no_stage = getenv("FKV_DIAG_NOSTAGE") != nullptr;
  static int stage_calls = 0;  // the first calls stage real images (finite scores in the skipped ones)
  if (((phases & FKV_PHASE_MAIN) && !(phases & FKV_PHASE_NOSTAGE) || (phases & FKV_PHASE_STAGE)) && p.kernel == 2 &&
      !(no_stage && ++stage_calls > 64))
    e = k::launch_stage(a, (int32_t)p.stage_src.size(), (cudaStream_t)stream);
  if (e == cudaSuccess && (phases & FKV_PHASE_MAIN))
    e = p.kernel == 2   ? k::launch_attention_tc(a, c.tc_maps.data(), (cudaStream_t)stream)
        : p.kernel == 0 ? k::launch_attention_mma(a, (cudaStream_t)stream)
                        : k::launch_attention_simt(a, (cudaStream_t)stream);
  const bool no_combine = getenv("FKV_DIAG_NOCOMBINE") != nullptr;  // diagnostics: timing only (read per call)
  if (e == cudaSuccess && (phases & FKV_PHASE_COMBINE) && !no_combine) e = k::launch_combine(a, (cudaStream_t)stream);
  if (e != cudaSuccess) throw Error(FKV_E_CUDA, std::string("attention: ") + cudaGetErrorString(e));
}

}  // namespace fkv
