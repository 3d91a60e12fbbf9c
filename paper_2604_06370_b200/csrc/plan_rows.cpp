// Planner of the rows-on-lanes tcgen05 kernel (§8(a) row a4, kernel 3 = ra_rows.cu).
//
// Agents forked from the same prefix hold the same physical base pages (§5.2); make_plan finds these
// shared page runs (segments). Here every (segment, kv head) becomes row blocks of <= 128 query rows (the
// TMEM lanes of one CTA) grouped by residual owner (same adapter and residual pages, <= 8 owners = residual
// slots per block), so one CTA streams each shared base tile once for all the rows that read it and adds
// each owner's rank-r term to its own rows only (Eq.4 split). Long key ranges are cut into
// pieces (split-KV) so that the static greedy schedule balances the 148 SMs; small work units (one sequence's
// private pages) are packed several per item. The combine kernel merges every row's partials (CSR below).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <queue>
#include <set>
#include <string>
#include <vector>

#include "internal.hpp"
#include "kernels.hpp"

namespace fkv {

namespace {

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

template <class T>
size_t put(std::vector<uint8_t>& blob, const std::vector<T>& v) {
  size_t off = align256(blob.size());
  blob.resize(off + std::max<size_t>(v.size() * sizeof(T), 16));
  if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
  return off;
}

struct RowC {
  int32_t q_row, pos, slot, adapter;
};
struct WuC {                   // work-unit candidate: rows of one kv head over one key range
  int32_t h = 0;
  int64_t kb = 0, ke = 0;      // keys [kb, ke)
  int64_t base_off = 0;        // flat base_pages index of page slot 0 of the sequence holding the keys
  std::vector<RowC> rows;
  std::vector<int64_t> slot_res_off;  // per slot: flat res_pages index of page slot 0 of the owner
  int64_t cost = 0;
  std::array<int64_t, 4> loc{};       // locality key (segment start, piece, block, head)
};

// estimated cycles of one tile: the tensor pipe (tcgen05.mma M=128: max(44, N/2) cycles per K=16 step,
// tools/ub_mix.cu), the softmax (MUFU ex2 of 128 rows x keys on one warpgroup) and the ring fill (whole K and V
// pages plus 8 KB per residual slot at the ~26 B/cycle a CTA sustains in the kernel: a 1-key tile costs a page
// load like a full one), whichever binds
int64_t tile_cost(int n_keys, int n_slots) {
  auto c = [](int n) { return std::max<int64_t>(44, n / 2); };
  const int ns = (n_keys + 15) & ~15, nk = (n_keys + 15) / 16;
  const int64_t tensor = (8 + n_slots) * c(ns) + nk * (c(128) + c(16 * n_slots));
  const int64_t soft = 1100 * ns / 128;
  const int64_t fill = (65536 + 8192 * (int64_t)n_slots) / 26;
  return std::max(std::max(tensor, soft), fill) + 150;
}

}  // namespace

void build_rows_plan(Ctx& c, Plan& pl, const std::vector<PlanSeg>& segs, const std::vector<const Agent*>& ags,
                     const std::vector<int64_t>& base_off, const std::vector<int64_t>& res_off, int sms) {
  const int P = c.cfg.page_size, g = c.group, hkv = c.hkv_local, hq = c.hq_local;
  const int64_t d = c.cfg.head_dim, r = c.cfg.rank;
  const size_t el = c.elem;
  const int n = pl.n_seqs;
  constexpr int kTile = 128, kLanes = k::kRowsLanes, kSlots = k::kRowsMaxSlots;

  // ---- work-unit candidates (unsplit) -------------------------------------------------------------------
  std::vector<WuC> big;    // row blocks that get their own items (split along the keys)
  std::vector<WuC> small;  // packed several per item
  int64_t base_bytes = 0, res_bytes = 0;
  for (size_t si = 0; si < segs.size(); ++si) {
    const PlanSeg& sg = segs[si];
    int64_t maxlen = 0;
    for (int32_t b : sg.members) maxlen = std::max<int64_t>(maxlen, ags[b]->seqlen);
    const int64_t k0 = sg.slot0 * P, k1 = std::min<int64_t>(sg.slot1 * P, maxlen);
    if (k1 <= k0) continue;
    base_bytes += (k1 - k0) * hkv * d * 2 * (int64_t)el;
    // owners: same adapter slot and the same residual pages over the segment
    std::map<std::pair<int32_t, std::vector<int32_t>>, std::vector<int32_t>> owners;
    for (int32_t b : sg.members) {
      std::vector<int32_t> rp(ags[b]->res.begin() + sg.slot0, ags[b]->res.begin() + sg.slot1);
      owners[{pl.seqs[b].adapter_slot, std::move(rp)}].push_back(b);
    }
    for (const auto& ow : owners) {
      int64_t okeys = 0;
      for (int32_t b : ow.second) okeys = std::max<int64_t>(okeys, std::min<int64_t>(k1, ags[b]->seqlen) - k0);
      res_bytes += okeys * r * 2 * (int64_t)el;
    }
    for (int32_t h = 0; h < hkv; ++h) {
      // rows of each owner (every query of every member that sees a key of the segment, q heads of group h)
      struct OwnerRows {
        int64_t res;
        int32_t adapter;
        std::vector<RowC> rows;
      };
      std::vector<OwnerRows> orows;
      for (const auto& ow : owners) {
        OwnerRows o{res_off[ow.second[0]], ow.first.first, {}};
        for (int32_t b : ow.second) {
          const int32_t L = pl.seqs[b].seqlen, C = pl.seqs[b].q_len;
          for (int32_t i = 0; i < C; ++i) {
            const int32_t pos = L - C + i;
            if (pos < k0) continue;
            for (int32_t qh = h * g; qh < (h + 1) * g; ++qh)
              o.rows.push_back({(pl.seqs[b].q_row0 + i) * hq + qh, pos, 0, ow.first.first});
          }
        }
        if (!o.rows.empty()) orows.push_back(std::move(o));
      }
      // row blocks: owners with > 128 rows alone in 128-row chunks; the rest packed (<= 128 rows, <= 8 slots)
      std::vector<WuC> blocks;
      WuC cur;
      auto flush = [&]() {
        if (!cur.rows.empty()) blocks.push_back(std::move(cur));
        cur = WuC();
      };
      for (const OwnerRows& o : orows) {
        if ((int)o.rows.size() > kLanes) {
          for (size_t i0 = 0; i0 < o.rows.size(); i0 += kLanes) {
            WuC w;
            w.slot_res_off.push_back(o.res);
            for (size_t i = i0; i < std::min(o.rows.size(), i0 + kLanes); ++i) w.rows.push_back(o.rows[i]);
            blocks.push_back(std::move(w));
          }
          continue;
        }
        if ((int)(cur.rows.size() + o.rows.size()) > kLanes || (int)cur.slot_res_off.size() == kSlots) flush();
        const int32_t slot = (int32_t)cur.slot_res_off.size();
        cur.slot_res_off.push_back(o.res);
        for (RowC rw : o.rows) {
          rw.slot = slot;
          cur.rows.push_back(rw);
        }
      }
      flush();
      for (size_t bi = 0; bi < blocks.size(); ++bi) {
        WuC& w = blocks[bi];
        w.h = h;
        w.kb = k0;
        w.ke = k1;
        w.base_off = base_off[sg.members[0]];
        const int64_t tiles = (k1 - k0 + kTile - 1) / kTile;
        w.cost = 0;
        for (int64_t t = 0; t < tiles; ++t)
          w.cost += tile_cost((int)std::min<int64_t>(kTile, k1 - k0 - t * kTile), (int)w.slot_res_off.size());
        w.loc = {k0, 0, (int64_t)bi, h};
        // a row block that fills at least half the lanes gets its own items; small ones are packed
        if ((int)w.rows.size() * 2 >= kLanes || tiles > 8) big.push_back(std::move(w));
        else if (getenv("FKV_DIAG_SKIP_SMALL")) continue;  // diagnostics only: drops the small WUs (wrong output)
        else small.push_back(std::move(w));
      }
    }
  }

  // ---- key pieces for balance ----------------------------------------------------------------------------
  int64_t total = 0;
  for (const WuC& w : big) total += w.cost + 3000;
  for (const WuC& w : small) total += w.cost + 500;
  const double frac = getenv("FKV_PIECE_FRAC") ? atof(getenv("FKV_PIECE_FRAC")) : 0.15;
  const int64_t target = std::max<int64_t>(1, (int64_t)(frac * (double)total / sms));
  std::vector<WuC> wus;  // final work units, each with its key range
  auto split = [&](const WuC& w, bool allow) {
    const int64_t tiles = (w.ke - w.kb + kTile - 1) / kTile;
    const int64_t force_tiles = getenv("FKV_PIECE_TILES") ? atoll(getenv("FKV_PIECE_TILES")) : 0;
    int64_t pieces = allow ? std::max<int64_t>(1, (w.cost + target - 1) / target) : 1;
    if (allow && force_tiles > 0) pieces = (tiles + force_tiles - 1) / force_tiles;
    pieces = std::min(pieces, tiles);
    const int64_t per = (tiles + pieces - 1) / pieces;
    for (int64_t t0 = 0, pi = 0; t0 < tiles; t0 += per, ++pi) {
      WuC x;
      x.h = w.h;
      x.kb = w.kb + t0 * kTile;
      x.ke = std::min<int64_t>(w.ke, w.kb + (t0 + per) * kTile);
      x.base_off = w.base_off;
      x.slot_res_off = w.slot_res_off;
      for (const RowC& rw : w.rows)
        if (rw.pos >= x.kb) x.rows.push_back(rw);
      if (x.rows.empty()) continue;
      x.cost = 0;
      for (int64_t k = x.kb; k < x.ke; k += kTile)
        x.cost += tile_cost((int)std::min<int64_t>(kTile, x.ke - k), (int)x.slot_res_off.size());
      x.loc = {w.loc[0], pi, w.loc[2], w.loc[3]};
      wus.push_back(std::move(x));
    }
  };
  for (const WuC& w : big) split(w, true);
  const size_t n_big = wus.size();
  for (const WuC& w : small) split(w, false);

  // ---- items: one big WU each; small WUs packed (<= 128 lanes, bounded cost) ------------------------------
  const int64_t small_cap = std::max<int64_t>(1, total / sms / 4);
  struct ItemC {
    std::vector<int32_t> wu;
    int64_t cost = 0;
    std::array<int64_t, 4> loc{};
  };
  std::vector<ItemC> items;
  for (size_t i = 0; i < n_big; ++i) items.push_back({{(int32_t)i}, wus[i].cost + 3000, wus[i].loc});
  {
    ItemC cur;
    int lanes = 0;
    for (size_t i = n_big; i < wus.size(); ++i) {
      const int nr = (int)wus[i].rows.size();
      // small items stay short (they fill the tail of the dynamic queue): at most 1/4 of a CTA's even share
      if (!cur.wu.empty() && (lanes + nr > kLanes || cur.cost + wus[i].cost > std::min(target, small_cap))) {
        items.push_back(std::move(cur));
        cur = ItemC();
        lanes = 0;
      }
      if (cur.wu.empty()) {
        cur.cost = 3000;
        cur.loc = {INT64_MAX, (int64_t)items.size(), 0, 0};
      }
      cur.wu.push_back((int32_t)i);
      cur.cost += wus[i].cost + 500;
      lanes += nr;
    }
    if (!cur.wu.empty()) items.push_back(std::move(cur));
  }

  // ---- records ----------------------------------------------------------------------------------------------
  std::vector<k::RItem> ritems;
  std::vector<k::RWu> rwus;
  std::vector<k::RTile> rtiles;
  std::vector<k::RRow> rrows;
  std::vector<int32_t> entry_qrow;  // entry -> output row
  for (const ItemC& ic : items) {
    k::RItem ri{};
    ri.tile0 = (int32_t)rtiles.size();
    ri.row0 = (int32_t)rrows.size();
    rrows.resize(rrows.size() + kLanes, k::RRow{-1, -1, -1, 0});
    int lane = 0;
    for (int32_t wi : ic.wu) {
      const WuC& w = wus[wi];
      k::RWu rw{};
      rw.n_slots = (int32_t)w.slot_res_off.size();
      int64_t min_pos = INT64_MAX;
      for (const RowC& rc : w.rows) {
        if (lane >= kLanes) throw Error(FKV_E_INVALID, "plan: item lanes overflow");
        k::RRow& rr = rrows[ri.row0 + lane];
        rr.q_row = rc.q_row;
        rr.pos = rc.pos;
        rr.entry = (int32_t)entry_qrow.size();
        rr.meta = rc.slot | (w.h << 8) | (rc.adapter << 16);
        entry_qrow.push_back(rc.q_row);
        rw.lanes[lane >> 5] |= 1u << (lane & 31);
        rw.slot_lanes[rc.slot][lane >> 5] |= 1u << (lane & 31);
        (rc.slot < 4 ? rw.lanes_lo : rw.lanes_hi)[lane >> 5] |= 1u << (lane & 31);
        min_pos = std::min<int64_t>(min_pos, rc.pos);
        ++lane;
      }
      const int32_t wu_idx = (int32_t)rwus.size();
      rwus.push_back(rw);
      for (int64_t k = w.kb; k < w.ke; k += kTile) {
        k::RTile t{};
        t.key0 = (int32_t)k;
        t.n_keys = (int32_t)std::min<int64_t>(kTile, w.ke - k);
        t.flags = (k == w.kb ? k::kTileFirst : 0) | (min_pos < k + t.n_keys - 1 ? k::kTileCausal : 0);
        t.wu = wu_idx;
        t.base_off = (int32_t)(w.base_off + k / P);
        t.base_page = pl.base_pages[t.base_off];
        t.n_slots = rw.n_slots;
        t.kv_head = w.h;
        for (int s = 0; s < kSlots; ++s)
          t.res_off[s] = s < (int)w.slot_res_off.size() ? (int32_t)(w.slot_res_off[s] + k / P) : 0;
        rtiles.push_back(t);
        pl.key_tiles += 1;
      }
    }
    ri.n_tiles = (int32_t)rtiles.size() - ri.tile0;
    ri.n_rows = lane;
    ritems.push_back(ri);
  }
  if (entry_qrow.size() > (size_t)INT32_MAX) throw Error(FKV_E_INVALID, "plan: too many partial entries");
  pl.n_entries = (int64_t)entry_qrow.size();

  // ---- schedule: longest first onto the least-loaded CTA; ties in locality order so that the items reading
  // the same base / residual tiles (same piece, both row blocks, all kv heads) run at the same time ------------
  const int32_t n_items = (int32_t)items.size();
  std::vector<int32_t> idx(n_items);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
    const int64_t ca = items[a].cost / 4096, cb = items[b].cost / 4096;  // cost buckets of ~2 tiles
    if (ca != cb) return ca > cb;
    return items[a].loc < items[b].loc;
  });
  // dynamic schedule: the persistent CTAs take items from this queue in order (longest first, so the tail is made
  // of short items; ties in locality order so that the items reading the same base / residual tiles run at the
  // same time)
  pl.n_ctas = std::max<int32_t>(1, std::min<int32_t>(sms, n_items));
  pl.sched_items = idx;
  pl.sched_ptr = {0, n_items};

  // ---- combine CSR: output row -> its entries ---------------------------------------------------------------
  const int64_t n_out = pl.n_rows_q * hq;
  std::vector<int32_t> cnt(n_out + 1, 0);
  for (int32_t q : entry_qrow) cnt[q + 1]++;
  for (int64_t o = 0; o < n_out; ++o) cnt[o + 1] += cnt[o];
  pl.out_ptr = cnt;
  pl.out_entries.assign(cnt[n_out], 0);
  {
    std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
    for (size_t e = 0; e < entry_qrow.size(); ++e) pl.out_entries[fill[entry_qrow[e]]++] = (int32_t)e;
  }
  for (int64_t o = 0; o < n_out; ++o)
    if (!pl.key_range && pl.out_ptr[o + 1] == pl.out_ptr[o])
      throw Error(FKV_E_NO_KEYS, "plan: an output row has no keys");
  pl.adapter_ptrs.resize(c.adapters.size() * 2);
  for (size_t s = 0; s < c.adapters.size(); ++s) {
    pl.adapter_ptrs[2 * s] = (int64_t)(intptr_t)c.adapters[s].bk;
    pl.adapter_ptrs[2 * s + 1] = (int64_t)(intptr_t)c.adapters[s].bv;
  }
  pl.comb_rows.assign(2 * n_out, 0);
  for (int64_t o = 0; o < n_out; ++o) {
    const int32_t qrow = (int32_t)(o / hq), qh = (int32_t)(o % hq), h = qh / g;
    const int32_t slot = pl.seqs[pl.qrow_seq[qrow]].adapter_slot;
    pl.comb_rows[2 * o] = (int64_t)(uint32_t)pl.out_ptr[o] | ((int64_t)pl.out_ptr[o + 1] << 32);
    pl.comb_rows[2 * o + 1] = pl.adapter_ptrs[2 * slot + 1] + (int64_t)h * r * d * (int64_t)el;
  }
  // algorithmic bytes per layer: shared base once per segment, residual once per (segment,
  // owner), adapters once, Q in + O out
  std::set<int32_t> used_adapters;
  for (const DevSeq& s : pl.seqs) used_adapters.insert(s.adapter_slot);
  pl.alg_rank_bytes = res_bytes + (int64_t)used_adapters.size() * 2 * r * d * hkv * (int64_t)el;
  pl.alg_bytes = base_bytes + res_bytes + (int64_t)used_adapters.size() * 2 * r * d * hkv * (int64_t)el +
                 pl.n_rows_q * hq * d * 2 * (int64_t)el;
  pl.n_segments = (int64_t)segs.size();
  (void)n;

  auto bytes_of = [](const auto& v) {
    std::vector<uint8_t> out(v.size() * sizeof(v[0]));
    if (!v.empty()) std::memcpy(out.data(), v.data(), out.size());
    return out;
  };
  pl.r_items = bytes_of(ritems);
  pl.r_wus = bytes_of(rwus);
  pl.r_tiles = bytes_of(rtiles);
  pl.r_rows = bytes_of(rrows);
  pl.items.assign(ritems.size(), DevItem{});  // counted by fkv_plan_get_info
  pl.blob.clear();
  pl.off_seqs = put(pl.blob, pl.seqs);
  pl.off_base = put(pl.blob, pl.base_pages);
  pl.off_res = put(pl.blob, pl.res_pages);
  pl.off_outptr = put(pl.blob, pl.out_ptr);
  pl.off_outent = put(pl.blob, pl.out_entries);
  pl.off_adapters = put(pl.blob, pl.adapter_ptrs);
  pl.off_qrow = put(pl.blob, pl.qrow_seq);
  pl.off_comb = put(pl.blob, pl.comb_rows);
  pl.off_sptr = put(pl.blob, pl.sched_ptr);
  pl.off_sitems = put(pl.blob, pl.sched_items);
  pl.off_ritems = put(pl.blob, pl.r_items);
  pl.off_rwus = put(pl.blob, pl.r_wus);
  pl.off_rtiles = put(pl.blob, pl.r_tiles);
  pl.off_rrows = put(pl.blob, pl.r_rows);
  pl.blob.resize(align256(pl.blob.size()));
  pl.ws_ctr_off = align256((size_t)pl.n_entries * (size_t)(k::kEntAcc + d + r) * sizeof(float));
  pl.ws_bytes = pl.ws_ctr_off + 256;  // + the queue counters
}

}  // namespace fkv
