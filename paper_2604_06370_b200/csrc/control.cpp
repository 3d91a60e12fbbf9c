// Control plane: page pools, per-agent block tables, fork with copy-on-write,
// DualRadixTree.  Rules R1-R9 of DESIGN.md ("Control-plane rules"), from
// PAPER.md §5.1 (P:269 separate bCache/rCache pools), §5.2 (P:291
// DualRadixTree keys, P:300 two-step fork: prefix match then CoW residual
// allocation) and P:87/P:219 (no in-place update of shared cache).
#include <algorithm>
#include <cstring>
#include <sstream>

#include "internal.hpp"
#include "kernels.hpp"
#include "tma_host.hpp"

namespace fkv {

namespace {

k::PoolView pool_view(const Ctx& c) {
  k::PoolView pv{};
  pv.base_k = c.buf.base_k; pv.base_v = c.buf.base_v; pv.res_k = c.buf.res_k; pv.res_v = c.buf.res_v;
  pv.nb = c.cfg.n_base_pages; pv.nr = c.cfg.n_res_pages;
  pv.hkv = c.hkv_local; pv.P = c.cfg.page_size; pv.d = c.cfg.head_dim; pv.r = c.cfg.rank;
  pv.L = c.cfg.n_layers; pv.dtype = c.cfg.dtype;
  pv.res_swz = c.cfg.dtype == FKV_DTYPE_BF16 && c.cfg.rank == 16;
  return pv;
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(FKV_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// R7: page `slot` of `ag` became full: walk/insert its chunks 0..slot in the
// base tree and in the residual tree under ag.owner (a missing chunk, e.g. an
// evicted one, is (re)inserted with the agent's page). New nodes take one ref.
// The walk is one access of each tree: one tick of its own clock (R10).
void tree_insert(Ctx& c, Agent& ag, int64_t slot) {
  const int P = c.cfg.page_size;
  for (int kind = 0; kind < 2; ++kind) {
    TreeNode* node;
    if (kind == FKV_KIND_BASE) {
      node = &c.base_root;
    } else {
      auto& root = c.res_roots[ag.owner];
      if (!root) {
        root = std::make_unique<TreeNode>();
        c.res_adapter[ag.owner] = ag.adapter;
      }
      node = root.get();
    }
    const int64_t tick = ++c.clock[kind];
    const auto& table = kind == FKV_KIND_BASE ? ag.base : ag.res;
    for (int64_t k = 0; k <= slot; ++k) {
      std::vector<int32_t> chunk(ag.tokens.begin() + k * P, ag.tokens.begin() + (k + 1) * P);
      auto it = node->children.find(chunk);
      if (it == node->children.end()) {
        auto nd = std::make_unique<TreeNode>();
        nd->page = table[k];
        nd->seq = c.nseq[kind]++;
        c.pools[kind].retain(table[k]);
        c.pools[kind].in_tree[table[k]] = 1;
        TreeNode* raw = nd.get();
        node->children.emplace(std::move(chunk), std::move(nd));
        node = raw;
      } else {
        node = it->second.get();
      }
      node->last = tick;
    }
  }
}

// longest full-page prefix of tokens[0, n) stored under `root` (no touch)
std::vector<TreeNode*> match_path(const TreeNode* root, const int32_t* tokens, int64_t n, int P) {
  std::vector<TreeNode*> path;
  const TreeNode* node = root;
  if (!node) return path;
  for (int64_t s = 0; s < n / P; ++s) {
    std::vector<int32_t> chunk(tokens + s * P, tokens + (s + 1) * P);
    auto it = node->children.find(chunk);
    if (it == node->children.end()) break;
    path.push_back(it->second.get());
    node = it->second.get();
  }
  return path;
}

// R11: a residual lineage (tree key) holds the xA_i rows of ONE adapter: its surviving tree and every live view of
// it must use `adapter`
bool lineage_ok(const Ctx& c, int64_t owner, int32_t adapter) {
  auto it = c.res_adapter.find(owner);
  if (it != c.res_adapter.end() && it->second != adapter) return false;
  for (const auto& kv : c.agents)
    if (kv.second.owner == owner && kv.second.adapter != adapter) return false;
  return true;
}

}  // namespace

void ctx_create(Ctx& c, const fkv_config& cfg, const fkv_buffers* buf) {
  const int P = cfg.page_size;
  if (cfg.n_layers < 1 || cfg.n_kv_heads < 1 || cfg.n_q_heads < cfg.n_kv_heads ||
      cfg.n_q_heads % cfg.n_kv_heads != 0 || cfg.head_dim < 2 || (cfg.head_dim & 1) || cfg.head_dim > 256 ||
      cfg.rank < 1 || cfg.rank > 64 || P < 1 || P > 128 || (128 % P) != 0 || cfg.n_base_pages < 1 ||
      cfg.n_res_pages < 1 || cfg.n_base_pages > INT32_MAX || cfg.n_res_pages > INT32_MAX || cfg.max_pos < 0 ||
      (cfg.dtype != FKV_DTYPE_BF16 && cfg.dtype != FKV_DTYPE_F32) ||
      (cfg.rope_mode != FKV_ROPE_NONE && cfg.rope_mode != FKV_ROPE_DEFERRED))
    throw Error(FKV_E_INVALID, "invalid fkv_config");
  c.cfg = cfg;
  int32_t h0 = cfg.kv_head_begin, h1 = cfg.kv_head_end;
  if (h0 == 0 && h1 == 0) h1 = cfg.n_kv_heads;
  if (h0 < 0 || h1 > cfg.n_kv_heads || h0 >= h1) throw Error(FKV_E_INVALID, "invalid kv head shard");
  c.cfg.kv_head_begin = h0; c.cfg.kv_head_end = h1;
  c.hkv_local = h1 - h0;
  c.group = cfg.n_q_heads / cfg.n_kv_heads;
  c.hq_local = c.hkv_local * c.group;
  c.device = cfg.device >= 0;
  c.elem = cfg.dtype == FKV_DTYPE_BF16 ? 2 : 4;
  if (buf) c.buf = *buf;
  if (c.device) {
    if (!buf || !buf->base_k || !buf->base_v || !buf->res_k || !buf->res_v)
      throw Error(FKV_E_INVALID, "device ctx needs pool buffers");
    if (cfg.rope_mode == FKV_ROPE_DEFERRED && (!buf->rope_cos || !buf->rope_sin || cfg.max_pos < 1))
      throw Error(FKV_E_INVALID, "DEFERRED rope needs rope_cos/rope_sin tables");
    check_cuda(cudaSetDevice(cfg.device), "cudaSetDevice");
    // TMA tensor maps over the pools for the tcgen05 kernel (2D views, one page per box)
    if (cfg.dtype == FKV_DTYPE_BF16 && cfg.head_dim == 128 && cfg.rank == 16 && (128 % P) == 0 && P >= 8) {
      const uint64_t brows = (uint64_t)cfg.n_layers * cfg.n_base_pages * c.hkv_local * P;
      const uint64_t rrows = (uint64_t)cfg.n_layers * cfg.n_res_pages * P;
      if (brows < (1ull << 31) && rrows < (1ull << 31)) {
        // see TcMaps in ra_tc.cu: K_base whole tiles (3D, both d-halves) when P = 128, V_base 64-key halves,
        // residual pages as 128-byte rows (the page format is already the SW32 operand layout, res_col)
        const uint32_t Pm = P < 64 ? (uint32_t)P : 64u;
        CUtensorMap m[5];
        m[0] = P == 128 ? make_tmap_3d_bf16_halves(buf->base_k, brows, 128)
                        : make_tmap_2d_bf16(buf->base_k, brows, 128, 256, 64, P, 128);
        m[1] = P >= 64 ? make_tmap_3d_bf16_halves(buf->base_v, brows, 64)
                       : make_tmap_2d_bf16(buf->base_v, brows, 128, 256, 64, P, 128);
        m[2] = make_tmap_2d_bf16(buf->res_k, rrows / 4, 64, 128, 64, P / 4, 0);
        m[3] = make_tmap_2d_bf16(buf->res_v, rrows / 4, 64, 128, 64, Pm / 4, 0);
        m[4] = make_tmap_2d_bf16(buf->base_k, brows, 128, 256, 64, P, 128);  // K_base d-half boxes
        c.tc_maps.assign((const uint8_t*)m, (const uint8_t*)m + sizeof(m));
        c.has_tc_maps = true;
        if (P >= 16) {
          // rows-on-lanes kernel (ra_rows.cu): whole-tile boxes {64, 128, 2} (P = 128) or per-page d-half boxes
          k::RowsMaps rm;
          std::memset(&rm, 0, sizeof(rm));
          rm.k2d = make_tmap_2d_bf16(buf->base_k, brows, 128, 256, 64, P, 128);
          rm.v2d = make_tmap_2d_bf16(buf->base_v, brows, 128, 256, 64, P, 128);
          if (P == 128) {
            rm.k3d = make_tmap_3d_bf16_halves(buf->base_k, brows, 128);
            rm.v3d = make_tmap_3d_bf16_halves(buf->base_v, brows, 128);
          }
          c.rows_maps.assign((const uint8_t*)&rm, (const uint8_t*)&rm + sizeof(rm));
          c.has_rows_maps = true;
        }
      }
    }
  }
  c.pools[0].init(cfg.n_base_pages, cfg.alloc_order_seed, cfg.n_layers);
  c.pools[1].init(cfg.n_res_pages, cfg.alloc_order_seed, cfg.n_layers);
}

void create_root(Ctx& c, int64_t a, int32_t adapter) {
  if (c.agents.count(a) || a < 0 || adapter < 0 || !lineage_ok(c, a, adapter)) throw Error(FKV_E_INVALID, "create_root: bad agent/adapter");
  Agent ag;
  ag.id = a; ag.adapter = adapter; ag.owner = a;
  c.agents.emplace(a, std::move(ag));
  ++c.generation;
}

void fork(Ctx& c, int64_t parent, int64_t L, int64_t child, int32_t adapter, uint32_t flags, void*) {
  Agent& p = c.agent(parent);
  if (c.agents.count(child) || child < 0 || adapter < 0 || L < 0 || L > p.seqlen)
    throw Error(FKV_E_INVALID, "fork: bad child/adapter/prefix_len");
  const bool share = flags & FKV_FORK_SHARE_RESIDUAL;
  if (share && adapter != p.adapter) throw Error(FKV_E_INVALID, "fork: SHARE_RESIDUAL needs the parent's adapter");
  if (!share && !lineage_ok(c, child, adapter))
    throw Error(FKV_E_INVALID, "fork: the child's residual lineage holds another adapter's rows");
  const int P = c.cfg.page_size;
  const int64_t k = (L + P - 1) / P;
  if (!share && c.pools[FKV_KIND_RES].n_free() < k) throw Error(FKV_E_NEEDS_EVICTION, "fork: residual pool exhausted");
  Agent ch;
  ch.id = child; ch.adapter = adapter; ch.owner = share ? p.owner : child; ch.seqlen = L;
  ch.base.assign(p.base.begin(), p.base.begin() + k);
  for (int32_t pg : ch.base) c.pools[FKV_KIND_BASE].retain(pg);
  if (share) {
    ch.res.assign(p.res.begin(), p.res.begin() + k);
    for (int32_t pg : ch.res) c.pools[FKV_KIND_RES].retain(pg);
  } else {
    for (int64_t i = 0; i < k; ++i) ch.res.push_back(c.pools[FKV_KIND_RES].alloc());
  }
  ch.tokens.assign(p.tokens.begin(), p.tokens.begin() + L);
  c.agents.emplace(child, std::move(ch));
  ++c.generation;
}

int64_t fork_tokens(Ctx& c, int64_t child, int32_t adapter, const int32_t* tokens, int64_t n) {
  if (c.agents.count(child) || child < 0 || adapter < 0 || n < 0 || (n > 0 && !tokens) ||
      !lineage_ok(c, child, adapter))
    throw Error(FKV_E_INVALID, "fork_tokens: bad child/adapter/tokens");
  const int P = c.cfg.page_size;
  const std::vector<TreeNode*> path = match_path(&c.base_root, tokens, n, P);
  std::vector<int32_t> pages;
  for (const TreeNode* nd : path) pages.push_back(nd->page);
  const int64_t k = (int64_t)pages.size();
  if (c.pools[FKV_KIND_RES].n_free() < k) throw Error(FKV_E_NEEDS_EVICTION, "fork_tokens: residual pool exhausted");
  if (!path.empty()) {  // the match is one access of the base tree (R10)
    const int64_t tick = ++c.clock[FKV_KIND_BASE];
    for (TreeNode* nd : path) nd->last = tick;
  }
  Agent ch;
  ch.id = child; ch.adapter = adapter; ch.owner = child; ch.seqlen = k * P;
  ch.base = pages;
  for (int32_t pg : pages) c.pools[FKV_KIND_BASE].retain(pg);
  for (int64_t i = 0; i < k; ++i) ch.res.push_back(c.pools[FKV_KIND_RES].alloc());
  ch.tokens.assign(tokens, tokens + k * P);
  c.agents.emplace(child, std::move(ch));
  ++c.generation;
  return k * P;
}

// R11 (P:300 Step 1 + Step 2, P:304 partial hit): map the surviving base pages AND the surviving residual pages of
// lineage `owner`; the rows of whichever part is missing are fresh pages the engine recomputes (xW only, or xA_i
// only). All mapped pages are full and are inserted into both trees at once.
void fork_resume(Ctx& c, int64_t child, int32_t adapter, int64_t owner, const int32_t* tokens, int64_t n,
                 int64_t* base_hit, int64_t* res_hit, int64_t* mapped) {
  if (c.agents.count(child) || child < 0 || adapter < 0 || owner < 0 || n < 0 || (n > 0 && !tokens))
    throw Error(FKV_E_INVALID, "fork_resume: bad child/adapter/owner/tokens");
  if (!lineage_ok(c, owner, adapter))
    throw Error(FKV_E_INVALID, "fork_resume: the residual lineage holds another adapter's rows");
  const int P = c.cfg.page_size;
  auto rt = c.res_roots.find(owner);
  const std::vector<TreeNode*> bpath = match_path(&c.base_root, tokens, n, P);
  const std::vector<TreeNode*> rpath = match_path(rt == c.res_roots.end() ? nullptr : rt->second.get(), tokens, n, P);
  const int64_t bm = (int64_t)bpath.size(), rm = (int64_t)rpath.size(), k = std::max(bm, rm);
  if (c.pools[FKV_KIND_BASE].n_free() < k - bm || c.pools[FKV_KIND_RES].n_free() < k - rm)
    throw Error(FKV_E_NEEDS_EVICTION, "fork_resume: pool exhausted");
  Agent ch;
  ch.id = child; ch.adapter = adapter; ch.owner = owner; ch.seqlen = k * P;
  for (const TreeNode* nd : bpath) { ch.base.push_back(nd->page); c.pools[FKV_KIND_BASE].retain(nd->page); }
  for (const TreeNode* nd : rpath) { ch.res.push_back(nd->page); c.pools[FKV_KIND_RES].retain(nd->page); }
  for (int64_t i = bm; i < k; ++i) ch.base.push_back(c.pools[FKV_KIND_BASE].alloc());
  for (int64_t i = rm; i < k; ++i) ch.res.push_back(c.pools[FKV_KIND_RES].alloc());
  ch.tokens.assign(tokens, tokens + k * P);
  Agent& ref = c.agents.emplace(child, std::move(ch)).first->second;
  if (k > 0) tree_insert(c, ref, k - 1);
  ++c.generation;
  *base_hit = bm * P; *res_hit = rm * P; *mapped = k * P;
}

namespace {
// pages of the subtree of `nd` that evict() could free, and whether every page in it is tree-only (refcount 1)
std::pair<int64_t, bool> evictable_walk(const TreeNode& nd, const PagePool& pool) {
  int64_t tot = 0;
  bool clean = true;
  for (const auto& kv : nd.children) {
    auto r = evictable_walk(*kv.second, pool);
    tot += r.first;
    clean = clean && r.second;
  }
  if (nd.page >= 0) {
    clean = clean && pool.rc[nd.page] == 1;
    tot += clean ? 1 : 0;
  }
  return {tot, clean};
}
std::vector<TreeNode*> roots_of(Ctx& c, int32_t kind) {
  std::vector<TreeNode*> r;
  if (kind == FKV_KIND_BASE) r.push_back(&c.base_root);
  else for (auto& kv : c.res_roots) r.push_back(kv.second.get());
  return r;
}
}  // namespace

int64_t evictable_pages(const Ctx& c, int32_t kind) {
  if (kind == FKV_KIND_BASE) return evictable_walk(c.base_root, c.pools[0]).first;
  int64_t t = 0;
  for (const auto& kv : c.res_roots) t += evictable_walk(*kv.second, c.pools[1]).first;
  return t;
}

// R12 decoupled eviction (§5.2): free n_pages pages of ONE tree by repeatedly dropping its least
// recently used leaf (smallest (last, seq)) whose page no live view holds. The other tree, its clock and every
// agent table are untouched. Atomic: fewer evictable pages than asked -> E_NEEDS_EVICTION, nothing evicted.
int64_t evict(Ctx& c, int32_t kind, int64_t n_pages) {
  if ((kind != FKV_KIND_BASE && kind != FKV_KIND_RES) || n_pages < 1) throw Error(FKV_E_INVALID, "evict: bad kind/count");
  const int64_t avail = evictable_pages(c, kind);
  if (avail < n_pages)
    throw Error(FKV_E_NEEDS_EVICTION, "evict: only " + std::to_string(avail) + " evictable pages, " +
                                          std::to_string(n_pages) + " asked");
  PagePool& pool = c.pools[kind];
  int64_t freed = 0;
  while (freed < n_pages) {
    TreeNode* best = nullptr;
    TreeNode* best_parent = nullptr;
    const std::vector<int32_t>* best_key = nullptr;
    std::vector<TreeNode*> stack = roots_of(c, kind);
    while (!stack.empty()) {
      TreeNode* nd = stack.back();
      stack.pop_back();
      for (auto& kv : nd->children) {
        TreeNode* ch = kv.second.get();
        if (ch->children.empty() && pool.rc[ch->page] == 1 &&
            (!best || ch->last < best->last || (ch->last == best->last && ch->seq < best->seq))) {
          best = ch; best_parent = nd; best_key = &kv.first;
        }
        stack.push_back(ch);
      }
    }
    const int32_t pg = best->page;
    best_parent->children.erase(*best_key);
    pool.release(pg);
    ++freed;
    if (kind == FKV_KIND_RES) {
      for (auto it = c.res_roots.begin(); it != c.res_roots.end();) {
        if (it->second->children.empty()) {
          c.res_adapter.erase(it->first);
          it = c.res_roots.erase(it);
        } else {
          ++it;
        }
      }
    }
  }
  return freed;
}

void append(Ctx& c, int32_t n, const int64_t* agents, const int32_t* n_new, const int32_t* tokens, void* stream) {
  if (n < 0 || (n > 0 && (!agents || !n_new))) throw Error(FKV_E_INVALID, "append: bad arrays");
  {
    std::vector<int64_t> ids(agents, agents + n);
    std::sort(ids.begin(), ids.end());
    if (std::adjacent_find(ids.begin(), ids.end()) != ids.end()) throw Error(FKV_E_INVALID, "append: duplicate agent");
  }
  int64_t total = 0;
  for (int32_t i = 0; i < n; ++i) {
    c.agent(agents[i]);
    if (n_new[i] < 0) throw Error(FKV_E_INVALID, "append: negative count");
    total += n_new[i];
  }
  if (total > 0 && !tokens) throw Error(FKV_E_INVALID, "append: token ids required");
  const int P = c.cfg.page_size;
  // Dry run: pages needed, simulating refcount drops of earlier CoWs (atomicity).
  int64_t need[2] = {0, 0};
  std::map<std::pair<int, int32_t>, int32_t> delta;
  for (int32_t i = 0; i < n; ++i) {
    const Agent& ag = c.agents.at(agents[i]);
    const int64_t t0 = ag.seqlen, cnt = n_new[i];
    if (cnt == 0) continue;
    if (t0 % P != 0) {
      const int64_t slot = t0 / P;
      for (int kind = 0; kind < 2; ++kind) {
        const int32_t pg = (kind == 0 ? ag.base : ag.res)[slot];
        const int32_t rc = c.pools[kind].rc[pg] + delta[{kind, pg}];
        if (rc > 1) { need[kind] += 1; delta[{kind, pg}] -= 1; }
      }
    }
    const int64_t first_new = (t0 + P - 1) / P, last = t0 + cnt - 1;
    const int64_t pages = last >= first_new * P ? last / P - first_new + 1 : 0;
    need[0] += pages; need[1] += pages;
  }
  if (need[0] > c.pools[0].n_free() || need[1] > c.pools[1].n_free())
    throw Error(FKV_E_NEEDS_EVICTION, "append: pool exhausted");
  std::vector<k::CopyOp> copies;
  int64_t tok = 0;
  for (int32_t i = 0; i < n; ++i) {
    Agent& ag = c.agents.at(agents[i]);
    for (int32_t j = 0; j < n_new[i]; ++j) {
      const int64_t t = ag.seqlen + j, slot = t / P;
      const int off = (int)(t % P);
      if (off == 0) {
        ag.base.push_back(c.pools[0].alloc());
        ag.res.push_back(c.pools[1].alloc());
      } else if (j == 0) {
        for (int kind = 0; kind < 2; ++kind) {
          auto& table = kind == 0 ? ag.base : ag.res;
          const int32_t pg = table[slot];
          if (c.pools[kind].rc[pg] > 1) {  // copy-on-write (C-10)
            const int32_t nw = c.pools[kind].alloc();
            copies.push_back({kind, pg, nw, off});
            c.copy_log.insert(c.copy_log.end(), {kind, pg, nw, off});
            for (int32_t l = 0; l < c.cfg.n_layers; ++l) c.pools[kind].wcopy_prefix(nw, pg, l, off);
            c.pools[kind].release(pg);
            table[slot] = nw;
          }
        }
      }
      for (int kind = 0; kind < 2; ++kind) {
        const int32_t pg = (kind == 0 ? ag.base : ag.res)[slot];
        for (int32_t l = 0; l < c.cfg.n_layers; ++l) c.pools[kind].wclear_bit(pg, l, off);
      }
      ag.tokens.push_back(tokens[tok + j]);
      if (off == P - 1) tree_insert(c, ag, slot);
    }
    ag.seqlen += n_new[i];
    tok += n_new[i];
  }
  ++c.generation;
  if (c.device && !copies.empty()) {
    DeviceGuard dg(c);
    const auto pv = pool_view(c);
    for (size_t o = 0; o < copies.size(); o += k::kMaxCopies) {
      const int32_t m = (int32_t)std::min<size_t>(k::kMaxCopies, copies.size() - o);
      check_cuda(k::launch_cow_copy(pv, copies.data() + o, m, (cudaStream_t)stream), "cow_copy");
    }
  }
}

void write_kv(Ctx& c, int32_t layer, int32_t n, const int64_t* agents, const int64_t* start, const int32_t* count,
              const void* kb, const void* vb, const void* rk, const void* rv, uint32_t mask, void* stream) {
  if (layer < 0 || layer >= c.cfg.n_layers || (mask & ~15u) || n < 0 || (n > 0 && (!agents || !start || !count)))
    throw Error(FKV_E_INVALID, "write_kv: bad layer/mask/arrays");
  for (int32_t i = 0; i < n; ++i) {
    const Agent& ag = c.agent(agents[i]);
    if (start[i] < 0 || count[i] < 0 || start[i] + count[i] > ag.seqlen)
      throw Error(FKV_E_INVALID, "write_kv: rows not reserved");
  }
  const int P = c.cfg.page_size;
  for (int32_t i = 0; i < n; ++i) {
    const Agent& ag = c.agents.at(agents[i]);
    if (count[i] == 0) continue;
    for (int64_t s = start[i] / P; s <= (start[i] + count[i] - 1) / P; ++s) {
      if ((mask & 3u) && !c.pools[0].writable(ag.base[s])) throw Error(FKV_E_READONLY, "write_kv: shared base page");
      if ((mask & 12u) && !c.pools[1].writable(ag.res[s])) throw Error(FKV_E_READONLY, "write_kv: shared residual page");
    }
  }
  if (c.device) {
    if (((mask & FKV_WRITE_KBASE) && !kb) || ((mask & FKV_WRITE_VBASE) && !vb) || ((mask & FKV_WRITE_RK) && !rk) ||
        ((mask & FKV_WRITE_RV) && !rv))
      throw Error(FKV_E_INVALID, "write_kv: missing source");
  }
  std::vector<k::WriteRun> runs;
  int64_t src = 0;
  for (int32_t i = 0; i < n; ++i) {
    const Agent& ag = c.agents.at(agents[i]);
    int64_t t = start[i];
    const int64_t end = start[i] + count[i];
    while (t < end) {
      const int64_t s = t / P;
      const int32_t row0 = (int32_t)(t % P);
      const int32_t m = (int32_t)std::min<int64_t>(P - row0, end - t);
      runs.push_back({ag.base[s], ag.res[s], row0, m, (int32_t)src, {0, 0, 0}});
      if ((mask & 3u) == 3u) c.pools[0].wset_range(ag.base[s], layer, row0, m);
      if ((mask & 12u) == 12u) c.pools[1].wset_range(ag.res[s], layer, row0, m);
      t += m; src += m;
    }
  }
  if (c.device && !runs.empty()) {
    DeviceGuard dg(c);
    const auto pv = pool_view(c);
    for (size_t o = 0; o < runs.size(); o += k::kMaxRuns) {
      const int32_t m = (int32_t)std::min<size_t>(k::kMaxRuns, runs.size() - o);
      const bool no_write = getenv("FKV_DIAG_NOKVWRITE") != nullptr;  // diagnostics: timing only (read per call)
      if (!no_write)
      check_cuda(k::launch_kv_write(pv, layer, runs.data() + o, m, kb, vb, rk, rv, mask, (cudaStream_t)stream),
                 "kv_write");
    }
  }
}

// ---- projection producer (§8(f) f2 / f3; Eq.2) -----------------------------------------
namespace {
size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

size_t project_workspace_bytes(const Ctx& c, int64_t T) {
  const int64_t n = (int64_t)c.hkv_local * c.cfg.head_dim, r = c.cfg.rank;
  return al256(T * 4) + al256(T * 16) + 2 * al256(T * n * 4) + al256(T * 2 * r * 4) + 2 * al256(T * n * c.elem) +
         2 * al256(T * r * c.elem);
}

void project_kv(Ctx& c, int32_t layer, int32_t n, const int64_t* agents, const int64_t* start, const int32_t* count,
                const void* x, int32_t hidden, const void* W_k, const void* W_v, uint32_t mask, void* ws,
                size_t ws_bytes, void* stream) {
  if (!c.device) throw Error(FKV_E_INVALID, "project_kv: host-only ctx");
  if (layer < 0 || layer >= c.cfg.n_layers || hidden < 1 || (mask & ~15u) || mask == 0 || !x || n < 0 ||
      (n > 0 && (!agents || !start || !count)))
    throw Error(FKV_E_INVALID, "project_kv: bad layer/hidden/mask/arrays");
  const bool base = mask & 3u, res = mask & 12u;
  if ((mask & 3u) && (mask & 3u) != 3u) throw Error(FKV_E_INVALID, "project_kv: base planes are written together");
  if ((mask & 12u) && (mask & 12u) != 12u) throw Error(FKV_E_INVALID, "project_kv: residual planes are written together");
  if (base && (!W_k || !W_v)) throw Error(FKV_E_INVALID, "project_kv: W_k / W_v required for the base planes");
  if (base && (!c.buf.rope_cos || !c.buf.rope_sin))
    throw Error(FKV_E_INVALID, "project_kv: the RoPE table is required (K_base is cached post-RoPE, P:269)");
  const int r = c.cfg.rank;
  if (res && r != 8 && r != 16 && r != 32 && r != 64) throw Error(FKV_E_INVALID, "project_kv: rank must be 8/16/32/64");
  int64_t T = 0;
  std::vector<int32_t> pos;
  std::vector<int64_t> aptr;
  for (int32_t i = 0; i < n; ++i) {
    const Agent& ag = c.agent(agents[i]);
    if (start[i] < 0 || count[i] < 0 || start[i] + count[i] > ag.seqlen)
      throw Error(FKV_E_INVALID, "project_kv: rows not reserved");
    if (base && start[i] + count[i] > c.cfg.max_pos) throw Error(FKV_E_INVALID, "project_kv: position beyond RoPE table");
    const AdapterSlot* as = nullptr;
    if (res) {
      auto it = c.adapter_slot.find(ag.adapter);
      if (it == c.adapter_slot.end() || !c.adapters[it->second].ak)
        throw Error(FKV_E_INVALID, "project_kv: agent's adapter has no registered down projection (A_k, A_v)");
      as = &c.adapters[it->second];
      if (as->hidden != hidden) throw Error(FKV_E_INVALID, "project_kv: hidden size differs from the adapter's A");
    }
    for (int32_t j = 0; j < count[i]; ++j) {
      pos.push_back((int32_t)(start[i] + j));
      const int64_t off = (int64_t)layer * hidden * r * (int64_t)c.elem;
      aptr.push_back(as ? (int64_t)(intptr_t)as->ak + off : 0);
      aptr.push_back(as ? (int64_t)(intptr_t)as->av + off : 0);
    }
    T += count[i];
  }
  if (T == 0) return;
  if (!ws || ws_bytes < project_workspace_bytes(c, T) || ((uintptr_t)ws & 255))
    throw Error(FKV_E_INVALID, "project_kv: workspace too small or not 256-byte aligned");
  DeviceGuard dg(c);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nn = (int64_t)c.hkv_local * c.cfg.head_dim;
  uint8_t* w = (uint8_t*)ws;
  int32_t* dpos = (int32_t*)w;                      w += al256(T * 4);
  int64_t* daptr = (int64_t*)w;                     w += al256(T * 16);
  float* yk = (float*)w;                            w += al256(T * nn * 4);
  float* yv = (float*)w;                            w += al256(T * nn * 4);
  float* yr = (float*)w;                            w += al256(T * 2 * r * 4);
  void* skb = w;                                    w += al256(T * nn * c.elem);
  void* svb = w;                                    w += al256(T * nn * c.elem);
  void* srk = w;                                    w += al256(T * r * c.elem);
  void* srv = w;
  check_cuda(cudaMemcpyAsync(dpos, pos.data(), T * 4, cudaMemcpyHostToDevice, s), "project_kv: upload");
  check_cuda(cudaMemcpyAsync(daptr, aptr.data(), T * 16, cudaMemcpyHostToDevice, s), "project_kv: upload");
  std::string err;
  if (base) {
    cudaError_t e = k::gemm_rowmajor_f32out(T, nn, hidden, x, W_k, yk, c.cfg.dtype, s, &err);
    if (e == cudaSuccess) e = k::gemm_rowmajor_f32out(T, nn, hidden, x, W_v, yv, c.cfg.dtype, s, &err);
    if (e != cudaSuccess) throw Error(FKV_E_CUDA, "project_kv: base GEMM: " + (err.empty() ? std::string(cudaGetErrorString(e)) : err));
  }
  if (res) check_cuda(k::launch_adapter_proj(x, daptr, (int32_t)T, hidden, r, c.cfg.dtype, yr, s), "project_kv: adapters");
  check_cuda(k::launch_project_stage(base ? yk : nullptr, yv, res ? yr : nullptr, dpos, (const float*)c.buf.rope_cos,
                                     (const float*)c.buf.rope_sin, (int32_t)T, c.hkv_local, c.cfg.head_dim, r, 1,
                                     c.cfg.dtype, skb, svb, srk, srv, s),
             "project_kv: stage");
  // the staged rows go through the ordinary row write (permission checks, written bits, page scatter)
  write_kv(c, layer, n, agents, start, count, skb, svb, srk, srv, mask, stream);
}

void release(Ctx& c, int64_t a) {
  Agent& ag = c.agent(a);
  for (int32_t pg : ag.base) c.pools[0].release(pg);
  for (int32_t pg : ag.res) c.pools[1].release(pg);
  c.agents.erase(a);
  ++c.generation;
}

namespace {
void join(std::ostringstream& o, const std::vector<int32_t>& v) {
  for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
}
void walk(std::ostringstream& o, const TreeNode& nd, int depth, const PagePool& pool) {
  for (const auto& kv : nd.children) {
    o << " " << depth << " page=" << kv.second->page << " rc=" << pool.rc[kv.second->page]
      << " last=" << kv.second->last << " seq=" << kv.second->seq << " tok=";
    join(o, kv.first);
    o << "\n";
    walk(o, *kv.second, depth + 1, pool);
  }
}
}  // namespace

std::string dump(const Ctx& c) {
  std::ostringstream o;
  o << "P=" << c.cfg.page_size << "\n";
  std::vector<int64_t> ids;
  for (const auto& kv : c.agents) ids.push_back(kv.first);
  std::sort(ids.begin(), ids.end());
  for (int64_t a : ids) {
    const Agent& ag = c.agents.at(a);
    o << "agent " << ag.id << " adapter=" << ag.adapter << " owner=" << ag.owner << " seqlen=" << ag.seqlen
      << " base=";
    join(o, ag.base);
    o << " res=";
    join(o, ag.res);
    o << "\n";
  }
  const char* names[2] = {"base", "res"};
  for (int kind = 0; kind < 2; ++kind) {
    const PagePool& p = c.pools[kind];
    o << names[kind] << "_free " << p.free_set.size() << " order=";
    bool first = true;
    for (const auto& e : p.free_set) { o << (first ? "" : ",") << e.second; first = false; }
    o << "\n" << names[kind] << "_rc ";
    first = true;
    for (int64_t i = 0; i < p.n; ++i)
      if (p.rc[i] > 0) { o << (first ? "" : " ") << i << ":" << p.rc[i]; first = false; }
    o << "\n";
  }
  o << "base_tree clock=" << c.clock[0] << " seq=" << c.nseq[0] << "\n";
  walk(o, c.base_root, 0, c.pools[0]);
  o << "res_forest clock=" << c.clock[1] << " seq=" << c.nseq[1] << "\n";
  for (const auto& kv : c.res_roots) {
    o << "res_tree owner=" << kv.first << " adapter=" << c.res_adapter.at(kv.first) << "\n";
    walk(o, *kv.second, 0, c.pools[1]);
  }
  return o.str();
}

}  // namespace fkv
