#include <cstdio>
// extern "C" boundary: argument checks, exception -> status translation.
#include <cmath>
#include <cstring>

#include "internal.hpp"
#include "kernels.hpp"

using fkv::Ctx;
using fkv::Error;

struct fkv_ctx {
  Ctx c;
};
struct fkv_plan {
  fkv::Plan* p;
};

namespace {
thread_local std::string g_err;

template <class F>
fkv_status guard(fkv_ctx* ctx, F&& f) {
  try {
    f();
    return FKV_OK;
  } catch (const Error& e) {
    if (ctx) ctx->c.last_error = e.what();
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->c.last_error = e.what();
    g_err = e.what();
    return FKV_E_INVALID;
  } catch (...) {
    if (ctx) ctx->c.last_error = "unknown error";
    g_err = "unknown error";
    return FKV_E_INVALID;
  }
}
}  // namespace

extern "C" {

const char* fkv_version(void) { return "forkkv-b200 0.1 (sm_100a)"; }

fkv_status fkv_create(const fkv_config* cfg, const fkv_buffers* buf, fkv_ctx** out) {
  if (!cfg || !out) return FKV_E_INVALID;
  *out = nullptr;
  auto* ctx = new fkv_ctx();
  fkv_status st = guard(ctx, [&] { fkv::ctx_create(ctx->c, *cfg, buf); });
  if (st != FKV_OK) {
    delete ctx;
    return st;
  }
  *out = ctx;
  return FKV_OK;
}

fkv_status fkv_destroy(fkv_ctx* ctx) {
  delete ctx;
  return FKV_OK;
}

const char* fkv_last_error(const fkv_ctx* ctx) { return ctx ? ctx->c.last_error.c_str() : g_err.c_str(); }

fkv_status fkv_register_adapter(fkv_ctx* ctx, int32_t adapter_id, const void* B_K, const void* B_V) {
  if (!ctx) return FKV_E_INVALID;
  return guard(ctx, [&] {
    if (adapter_id < 0) throw Error(FKV_E_INVALID, "register_adapter: negative id");
    if (ctx->c.device && (!B_K || !B_V)) throw Error(FKV_E_INVALID, "register_adapter: null B_K/B_V");
    if (ctx->c.device && (((uintptr_t)B_K | (uintptr_t)B_V) & 15))
      throw Error(FKV_E_INVALID, "register_adapter: B_K/B_V must be 16-byte aligned");
    auto it = ctx->c.adapter_slot.find(adapter_id);
    if (it == ctx->c.adapter_slot.end()) {
      ctx->c.adapter_slot[adapter_id] = (int32_t)ctx->c.adapters.size();
      ctx->c.adapters.push_back({adapter_id, B_K, B_V});
    } else {
      ctx->c.adapters[it->second] = {adapter_id, B_K, B_V};
    }
    ++ctx->c.generation;
  });
}

fkv_status fkv_create_root(fkv_ctx* ctx, int64_t agent, int32_t adapter_id) {
  if (!ctx) return FKV_E_INVALID;
  return guard(ctx, [&] { fkv::create_root(ctx->c, agent, adapter_id); });
}

fkv_status fkv_fork(fkv_ctx* ctx, int64_t parent, int64_t prefix_len, int64_t child, int32_t adapter_id,
                    uint32_t flags) {
  if (!ctx) return FKV_E_INVALID;
  return guard(ctx, [&] { fkv::fork(ctx->c, parent, prefix_len, child, adapter_id, flags, nullptr); });
}

fkv_status fkv_fork_tokens(fkv_ctx* ctx, int64_t child, int32_t adapter_id, const int32_t* tokens, int64_t n,
                           int64_t* matched) {
  if (!ctx) return FKV_E_INVALID;
  return guard(ctx, [&] {
    int64_t m = fkv::fork_tokens(ctx->c, child, adapter_id, tokens, n);
    if (matched) *matched = m;
  });
}

fkv_status fkv_register_adapter_down(fkv_ctx* ctx, int32_t adapter_id, const void* A_K, const void* A_V,
                                     int32_t hidden) {
  if (!ctx) return FKV_E_INVALID;
  return guard(ctx, [&] {
    auto it = ctx->c.adapter_slot.find(adapter_id);
    if (it == ctx->c.adapter_slot.end())
      throw Error(FKV_E_INVALID, "register_adapter_down: register the adapter's B first (fkv_register_adapter)");
    if (hidden < 1 || (ctx->c.device && (!A_K || !A_V)))
      throw Error(FKV_E_INVALID, "register_adapter_down: null A_K/A_V or hidden < 1");
    auto& a = ctx->c.adapters[it->second];
    a.ak = A_K; a.av = A_V; a.hidden = hidden;
  });
}

fkv_status fkv_project_workspace_bytes(fkv_ctx* ctx, int64_t n_rows, size_t* bytes) {
  if (!ctx || !bytes || n_rows < 0) return FKV_E_INVALID;
  *bytes = fkv::project_workspace_bytes(ctx->c, n_rows);
  return FKV_OK;
}

fkv_status fkv_project_kv(fkv_ctx* ctx, int32_t layer, int32_t n, const int64_t* agents, const int64_t* start,
                          const int32_t* count, const void* x, int32_t hidden, const void* W_k, const void* W_v,
                          uint32_t which_mask, void* workspace, size_t ws_bytes, void* stream) {
  if (!ctx) return FKV_E_INVALID;
  return guard(ctx, [&] {
    fkv::project_kv(ctx->c, layer, n, agents, start, count, x, hidden, W_k, W_v, which_mask, workspace, ws_bytes,
                    stream);
  });
}

fkv_status fkv_fork_resume(fkv_ctx* ctx, int64_t child, int32_t adapter_id, int64_t owner, const int32_t* tokens,
                           int64_t n, int64_t* base_hit, int64_t* res_hit, int64_t* mapped) {
  if (!ctx || !base_hit || !res_hit || !mapped) return FKV_E_INVALID;
  return guard(ctx, [&] { fkv::fork_resume(ctx->c, child, adapter_id, owner, tokens, n, base_hit, res_hit, mapped); });
}

fkv_status fkv_evict(fkv_ctx* ctx, int32_t kind, int64_t n_pages, int64_t* freed) {
  if (!ctx) return FKV_E_INVALID;
  return guard(ctx, [&] {
    const int64_t f = fkv::evict(ctx->c, kind, n_pages);
    if (freed) *freed = f;
  });
}

fkv_status fkv_evictable_pages(fkv_ctx* ctx, int32_t kind, int64_t* n_pages) {
  if (!ctx || !n_pages || (kind != FKV_KIND_BASE && kind != FKV_KIND_RES)) return FKV_E_INVALID;
  return guard(ctx, [&] { *n_pages = fkv::evictable_pages(ctx->c, kind); });
}

fkv_status fkv_append(fkv_ctx* ctx, int32_t n, const int64_t* agents, const int32_t* n_new,
                      const int32_t* token_ids, void* stream) {
  if (!ctx) return FKV_E_INVALID;
  return guard(ctx, [&] { fkv::append(ctx->c, n, agents, n_new, token_ids, stream); });
}

fkv_status fkv_write_kv(fkv_ctx* ctx, int32_t layer, int32_t n, const int64_t* agents, const int64_t* start,
                        const int32_t* count, const void* k_base, const void* v_base, const void* r_k,
                        const void* r_v, uint32_t which_mask, void* stream) {
  if (!ctx) return FKV_E_INVALID;
  return guard(ctx, [&] {
    fkv::write_kv(ctx->c, layer, n, agents, start, count, k_base, v_base, r_k, r_v, which_mask, stream);
  });
}

fkv_status fkv_release(fkv_ctx* ctx, int64_t agent) {
  if (!ctx) return FKV_E_INVALID;
  return guard(ctx, [&] { fkv::release(ctx->c, agent); });
}

fkv_status fkv_get_table(const fkv_ctx* ctx, int64_t agent, int64_t cap, int32_t* base_pages, int32_t* res_pages,
                         int64_t* n_pages, int64_t* seqlen) {
  if (!ctx) return FKV_E_INVALID;
  auto it = ctx->c.agents.find(agent);
  if (it == ctx->c.agents.end()) return FKV_E_UNKNOWN_AGENT;
  const auto& ag = it->second;
  const int64_t np = (int64_t)ag.base.size();
  if (n_pages) *n_pages = np;
  if (seqlen) *seqlen = ag.seqlen;
  if (cap < np) return (base_pages || res_pages) ? FKV_E_INVALID : FKV_OK;
  if (base_pages) std::memcpy(base_pages, ag.base.data(), np * sizeof(int32_t));
  if (res_pages) std::memcpy(res_pages, ag.res.data(), np * sizeof(int32_t));
  return FKV_OK;
}

fkv_status fkv_get_agent(const fkv_ctx* ctx, int64_t agent, int32_t* adapter_id, int64_t* residual_owner) {
  if (!ctx) return FKV_E_INVALID;
  auto it = ctx->c.agents.find(agent);
  if (it == ctx->c.agents.end()) return FKV_E_UNKNOWN_AGENT;
  if (adapter_id) *adapter_id = it->second.adapter;
  if (residual_owner) *residual_owner = it->second.owner;
  return FKV_OK;
}

fkv_status fkv_page_refcount(const fkv_ctx* ctx, int32_t kind, int64_t page, int32_t* rc) {
  if (!ctx || kind < 0 || kind > 1 || !rc) return FKV_E_INVALID;
  const auto& pool = ctx->c.pools[kind];
  if (page < 0 || page >= pool.n) return FKV_E_INVALID;
  *rc = pool.rc[page];
  return FKV_OK;
}

fkv_status fkv_free_pages(const fkv_ctx* ctx, int32_t kind, int64_t* n_free) {
  if (!ctx || kind < 0 || kind > 1 || !n_free) return FKV_E_INVALID;
  *n_free = ctx->c.pools[kind].n_free();
  return FKV_OK;
}

fkv_status fkv_dump(const fkv_ctx* ctx, char* buf, size_t cap, size_t* needed) {
  if (!ctx) return FKV_E_INVALID;
  std::string s = fkv::dump(ctx->c);
  if (needed) *needed = s.size() + 1;
  if (!buf) return FKV_OK;
  if (cap < s.size() + 1) return FKV_E_INVALID;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return FKV_OK;
}

fkv_status fkv_take_copy_log(fkv_ctx* ctx, int32_t* buf, int64_t cap_quads, int64_t* n_quads) {
  if (!ctx) return FKV_E_INVALID;
  const int64_t nq = (int64_t)ctx->c.copy_log.size() / 4;
  if (n_quads) *n_quads = nq;
  if (!buf) return FKV_OK;
  if (cap_quads < nq) return FKV_E_INVALID;
  std::memcpy(buf, ctx->c.copy_log.data(), ctx->c.copy_log.size() * sizeof(int32_t));
  ctx->c.copy_log.clear();
  return FKV_OK;
}

fkv_status fkv_plan_create(fkv_ctx* ctx, int32_t n, const fkv_seq* seqs, uint32_t flags, fkv_plan** out) {
  if (!ctx || !out) return FKV_E_INVALID;
  *out = nullptr;
  fkv::Plan* p = nullptr;
  fkv_status st = guard(ctx, [&] { p = fkv::make_plan(ctx->c, n, seqs, flags); });
  if (st != FKV_OK) return st;
  *out = new fkv_plan{p};
  return FKV_OK;
}

fkv_status fkv_plan_create_range(fkv_ctx* ctx, int32_t n, const fkv_seq* seqs, uint32_t flags, int64_t key_begin,
                                 int64_t key_end, fkv_plan** out) {
  if (!ctx || !out) return FKV_E_INVALID;
  *out = nullptr;
  fkv::Plan* p = nullptr;
  fkv_status st = guard(ctx, [&] { p = fkv::make_plan(ctx->c, n, seqs, flags, key_begin, key_end); });
  if (st != FKV_OK) return st;
  *out = new fkv_plan{p};
  return FKV_OK;
}

fkv_status fkv_residual_attention_lse(fkv_ctx* ctx, const fkv_plan* plan, int32_t layer, const void* Q, void* O,
                                      float* lse, float sm_scale, void* workspace, size_t ws_bytes, void* stream) {
  if (!ctx || !plan || !lse) return FKV_E_INVALID;
  return guard(ctx, [&] {
    fkv::run_attention(ctx->c, *plan->p, layer, Q, O, sm_scale, workspace, ws_bytes, stream, 3u, lse);
  });
}

fkv_status fkv_merge_lse(int32_t n_parts, int64_t n_rows, int32_t head_dim, int32_t dtype, const void* O_parts,
                         const float* lse_parts, void* O, float* lse_out, void* stream) {
  if (n_parts < 1 || n_rows < 0 || head_dim < 1 || !O_parts || !lse_parts || !O ||
      (dtype != FKV_DTYPE_BF16 && dtype != FKV_DTYPE_F32))
    return FKV_E_INVALID;
  const cudaError_t e = fkv::k::launch_merge_lse(n_parts, n_rows, head_dim, O_parts, lse_parts, O, lse_out, dtype,
                                                 (cudaStream_t)stream);
  return e == cudaSuccess ? FKV_OK : FKV_E_CUDA;
}

fkv_status fkv_partition_keys(int64_t max_seqlen, int32_t G, int32_t page_size, int32_t rank, int64_t* key_begin,
                              int64_t* key_end) {
  if (G < 1 || rank < 0 || rank >= G || page_size < 1 || max_seqlen < 0 || !key_begin || !key_end)
    return FKV_E_INVALID;
  // G page-aligned ranges of ~equal page count over [0, max_seqlen); the last one open-ended
  const int64_t pages = (max_seqlen + page_size - 1) / page_size;
  const int64_t lo = pages * rank / G, hi = pages * (rank + 1) / G;
  *key_begin = lo * page_size;
  *key_end = rank == G - 1 ? INT64_MAX : hi * page_size;
  return FKV_OK;
}

fkv_status fkv_plan_get_info(const fkv_plan* plan, fkv_plan_info* info) {
  if (!plan || !info) return FKV_E_INVALID;
  const fkv::Plan& p = *plan->p;
  info->n_seqs = p.n_seqs;
  info->n_rows = p.n_rows_q;
  info->n_segments = p.n_segments;
  info->n_items = (int64_t)p.items.size();
  info->n_ctas = p.kernel >= 2 ? (int64_t)p.n_ctas : (int64_t)p.items.size();  // persistent kernels: p.n_ctas
  info->n_warps = (int64_t)p.warps.size();
  info->n_entries = p.n_entries;
  info->key_tiles = p.key_tiles;
  info->alg_bytes = p.alg_bytes;
  info->kernel = p.kernel;
  info->device_bytes = (int64_t)p.blob.size();
  info->workspace_bytes = (int64_t)p.ws_bytes;
  info->alg_rank_bytes = p.alg_rank_bytes;
  return FKV_OK;
}

fkv_status fkv_plan_upload(fkv_ctx* ctx, fkv_plan* plan, void* dev, size_t bytes, void* stream) {
  if (!ctx || !plan) return FKV_E_INVALID;
  return guard(ctx, [&] { fkv::upload_plan(ctx->c, *plan->p, dev, bytes, stream); });
}

fkv_status fkv_residual_attention(fkv_ctx* ctx, const fkv_plan* plan, int32_t layer, const void* Q, void* O,
                                  float sm_scale, void* workspace, size_t ws_bytes, void* stream) {
  if (!ctx || !plan) return FKV_E_INVALID;
  return guard(ctx, [&] { fkv::run_attention(ctx->c, *plan->p, layer, Q, O, sm_scale, workspace, ws_bytes, stream); });
}

fkv_status fkv_residual_attention_phases(fkv_ctx* ctx, const fkv_plan* plan, int32_t layer, const void* Q, void* O,
                                         float sm_scale, void* workspace, size_t ws_bytes, void* stream,
                                         uint32_t phases) {
  if (!ctx || !plan) return FKV_E_INVALID;
  return guard(ctx, [&] {
    fkv::run_attention(ctx->c, *plan->p, layer, Q, O, sm_scale, workspace, ws_bytes, stream, phases);
  });
}

fkv_status fkv_residual_attention_host(fkv_ctx* ctx, const fkv_plan* plan, int32_t layer, const void* Q_host,
                                       void* O_host, void* dQ, void* dO, float sm_scale, void* workspace,
                                       size_t ws_bytes, void* stream) {
  if (!ctx || !plan || !Q_host || !O_host || !dQ || !dO) return FKV_E_INVALID;
  return guard(ctx, [&] {
    const size_t bytes = (size_t)plan->p->n_rows_q * ctx->c.hq_local * ctx->c.cfg.head_dim * ctx->c.elem;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(dQ, Q_host, bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) throw Error(FKV_E_CUDA, std::string("H2D: ") + cudaGetErrorString(e));
    fkv::run_attention(ctx->c, *plan->p, layer, dQ, dO, sm_scale, workspace, ws_bytes, stream);
    e = cudaMemcpyAsync(O_host, dO, bytes, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) throw Error(FKV_E_CUDA, std::string("D2H: ") + cudaGetErrorString(e));
  });
}

fkv_status fkv_plan_free(fkv_plan* plan) {
  if (plan) {
    delete plan->p;
    delete plan;
  }
  return FKV_OK;
}

fkv_status fkv_build_rope_table(int32_t max_pos, int32_t d, double theta, int32_t llama3, double factor,
                                double low_freq_factor, double high_freq_factor, double orig_max_pos,
                                float* cos_out, float* sin_out) {
  if (max_pos < 1 || d < 2 || (d & 1) || theta <= 0 || !cos_out || !sin_out) return FKV_E_INVALID;
  const int h = d / 2;
  std::vector<double> f(h);
  for (int i = 0; i < h; ++i) {
    double fr = std::pow(theta, -2.0 * i / d);
    if (llama3) {
      // Llama-3.1 rope_scaling (public model config; C-2)
      const double wavelen = 2.0 * M_PI / fr;
      const double lo = orig_max_pos / low_freq_factor, hi = orig_max_pos / high_freq_factor;
      if (wavelen > lo) {
        fr = fr / factor;
      } else if (wavelen >= hi) {
        const double sm = (orig_max_pos / wavelen - low_freq_factor) / (high_freq_factor - low_freq_factor);
        fr = (1.0 - sm) * fr / factor + sm * fr;
      }
    }
    f[i] = fr;
  }
  for (int64_t p = 0; p < max_pos; ++p)
    for (int i = 0; i < h; ++i) {
      const double a = (double)p * f[i];
      cos_out[p * h + i] = (float)std::cos(a);
      sin_out[p * h + i] = (float)std::sin(a);
    }
  return FKV_OK;
}

fkv_status fkv_synth_fill(void* dst, int32_t dtype, uint64_t seed, int32_t kind, uint64_t owner, int32_t layer,
                          int64_t pos0, int32_t n_pos, int32_t head0, int32_t n_head, int32_t n_col, float scale,
                          void* stream) {
  if (!dst || n_pos < 0 || n_head < 1 || n_col < 1 || n_col > 256 || head0 < 0 || head0 + n_head > 256 ||
      (dtype != FKV_DTYPE_BF16 && dtype != FKV_DTYPE_F32))
    return FKV_E_INVALID;
  if (n_pos == 0) return FKV_OK;
  cudaError_t e = fkv::k::launch_synth_fill(dst, dtype, seed, kind, owner, layer, pos0, n_pos, head0, n_head, n_col,
                                            scale, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return FKV_E_CUDA;
  }
  return FKV_OK;
}

fkv_status fkv_partition(int32_t G, int32_t n_kv_heads, int64_t base_bytes, int64_t res_bytes, int32_t* H,
                         int32_t* D) {
  if (G < 1 || n_kv_heads < 1 || base_bytes < 0 || res_bytes < 0 || !H || !D) return FKV_E_INVALID;
  // Splitting by kv head divides base pages and B slices but replicates the
  // head-shared residual; splitting by agent batch divides residual/private
  // pages but replicates the shared base.
  double best = 1e300;
  int32_t bh = -1, bd = -1;
  for (int32_t h = 1; h <= G; ++h) {
    if (G % h || n_kv_heads % h) continue;
    const int32_t dd = G / h;
    const double cost = (double)base_bytes / h + (double)res_bytes / dd;
    if (cost < best - 1e-9) { best = cost; bh = h; bd = dd; }
  }
  if (bh < 0) return FKV_E_INVALID;
  *H = bh;
  *D = bd;
  return FKV_OK;
}

fkv_status fkv_partition_shard(int32_t rank, int32_t H, int32_t D, int32_t n_kv_heads, int64_t n_agents, int32_t* h0,
                               int32_t* h1, int64_t* a0, int64_t* a1) {
  if (H < 1 || D < 1 || rank < 0 || rank >= H * D || n_kv_heads % H || n_agents < 0 || !h0 || !h1 || !a0 || !a1)
    return FKV_E_INVALID;
  const int32_t hi = rank % H, di = rank / H;
  const int32_t per = n_kv_heads / H;
  *h0 = hi * per;
  *h1 = (hi + 1) * per;
  *a0 = n_agents * di / D;
  *a1 = n_agents * (di + 1) / D;
  return FKV_OK;
}

}  // extern "C"

extern "C" fkv_status fkv_debug_hang_report(char* buf, int64_t cap) {
  if (!buf || cap < 1) return FKV_E_INVALID;
  const std::string r = fkv::k::hang_report();
  std::snprintf(buf, (size_t)cap, "%s", r.c_str());
  return FKV_OK;
}

extern "C" fkv_status fkv_debug_timeline(fkv_ctx* ctx, void* dbg, int32_t block) {
  if (!ctx || block < 0) return FKV_E_INVALID;
  ctx->c.dbg = dbg;
  ctx->c.dbg_block = block;
  return FKV_OK;
}
