/*
 * forkkv.h — C ABI of the B200-native ForkKV ResidualAttention hot path.
 *
 * ForkKV (arxiv 2604.06370, /root/reference/PAPER.md) serves many LoRA agents
 * forked from a shared context by disaggregating each agent's KV cache into
 *   bCache = xW   (K stored post-RoPE; shared zero-copy by every agent that
 *                  holds the same tokens)                  P:269 §5.1, Eq.2
 *   rCache = xA_i (rank r, per agent, stored without RoPE)  P:130-134 §2.2
 * tracked by a DualRadixTree (base tree keyed by token ids, residual tree
 * keyed by agent id + token ids, §5.2) with OS-style fork + copy-on-write
 * (§5.2), and by ResidualAttention (Alg.1, Eq.4)
 * which rebuilds K = K_base + RoPE(K_res B_k) and V = V_base + V_res B_v on
 * chip so a full per-agent K/V never reaches HBM.
 *
 * Ownership
 *   - Device memory (pools, RoPE table, adapters, Q, O, plan buffers,
 *     workspace) is CALLER-owned and passed as raw pointers; the library only
 *     borrows it. The caller keeps it alive until fkv_destroy / plan free.
 *   - The library owns all host metadata (pools, tables, trees, plans).
 *   - Streams are caller-supplied (cudaStream_t passed as void*; NULL = the
 *     legacy default stream). Nothing synchronises internally except where a
 *     function says so.
 * Errors
 *   Every call returns fkv_status (int32). Nothing throws or aborts across
 *   the ABI. fkv_last_error(ctx) returns a message for the last failure on
 *   that ctx. Mutating calls are atomic: on failure tables, refcounts and
 *   trees are unchanged ("never silently evicts").
 * Concurrency
 *   One mutation gate: a ctx is not thread-safe; the caller serialises calls
 *   on a ctx. Kernels enqueued on streams may run concurrently.
 * Host-only mode
 *   fkv_config.device = -1 creates a control-plane-only ctx (no CUDA calls;
 *   kernels are skipped, data pointers may be NULL). Used by CPU tests.
 */
#ifndef FORKKV_H_
#define FORKKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t fkv_status;
enum {
  FKV_OK = 0,
  FKV_E_INVALID = 1,          /* dimension/shape/argument mismatch */
  FKV_E_NEEDS_EVICTION = 2,   /* a pool is exhausted; nothing evicted */
  FKV_E_UNKNOWN_AGENT = 3,    /* no such agent */
  FKV_E_STALE = 4,            /* plan built against an older table generation */
  FKV_E_READONLY = 5,         /* write to a page with more than one holder */
  FKV_E_NO_KEYS = 6,          /* a causal query row has no keys */
  FKV_E_UNWRITTEN = 7,        /* attention would read rows never written */
  FKV_E_CUDA = 8              /* CUDA error; message from cudaGetErrorString */
};

enum { FKV_DTYPE_BF16 = 0, FKV_DTYPE_F32 = 1 };
/* Residual-key RoPE (reading C-1). DEFERRED = the paper's
 * K_lora = RoPE(K_res B_k) at the key's absolute position (Alg1.335).
 * NONE = no rotation of the residual term, i.e. the north-star split
 * q.(K_base + R_K B_K)^T = q K_base^T + (q B_K^T) R_K^T (exact only then). */
enum { FKV_ROPE_NONE = 0, FKV_ROPE_DEFERRED = 1 };
enum { FKV_KIND_BASE = 0, FKV_KIND_RES = 1 };

#define FKV_FORK_SHARE_RESIDUAL 1u  /* same-agent branch: share residual pages CoW (C-12) */

#define FKV_WRITE_KBASE 1u
#define FKV_WRITE_VBASE 2u
#define FKV_WRITE_RK 4u
#define FKV_WRITE_RV 8u

#define FKV_PLAN_CHECK_WRITTEN 1u   /* verify every key row of every layer was written */
#define FKV_PLAN_FORCE_SIMT 2u      /* use the plain SIMT kernel (fp32 path is always SIMT) */
#define FKV_PLAN_FORCE_MMA 4u       /* use the warp-level mma.sync kernel instead of tcgen05 */
#define FKV_PLAN_ROWS_KERNEL 8u     /* NONE mode, bf16, d 128, r 16: the rows-on-lanes tcgen05 kernel (kernel 3) */

typedef struct fkv_config {
  int32_t n_layers;       /* L */
  int32_t n_q_heads;      /* Hq (whole model; the shard holds heads of [kv_head_begin, kv_head_end)) */
  int32_t n_kv_heads;     /* Hkv (whole model) */
  int32_t head_dim;       /* d: 64 or 128 (bf16 tensor-core path needs 128; SIMT path: even, <=256) */
  int32_t rank;           /* r: LoRA rank of the residual pool; adapters of smaller rank are zero-padded (C-8) */
  int32_t page_size;      /* P: tokens per page, any divisor of 128 (C-9); the tcgen05 kernels take 16..128,
                             128 = one key tile per page (bench default) */
  int64_t n_base_pages;   /* pages in the bCache pool */
  int64_t n_res_pages;    /* pages in the rCache pool */
  int32_t max_pos;        /* rows of the RoPE table; DEFERRED plans refuse sequences longer than it (E_INVALID) */
  int32_t dtype;          /* FKV_DTYPE_*: element type of pools, adapters, Q and O */
  int32_t rope_mode;      /* FKV_ROPE_* */
  int32_t device;         /* CUDA device ordinal, or -1 for a host-only control plane */
  uint64_t alloc_order_seed; /* 0: ascending page ids; else seeded rank order (C-11) */
  int32_t kv_head_begin;  /* KV-head shard [begin, end) held by this ctx (§8(e)); 0,0 = all */
  int32_t kv_head_end;
} fkv_config;

/* Device pools (caller-owned), element type = config.dtype.
 *   base_k, base_v : [L][n_base_pages][Hkv_local][P][d]   (K post-RoPE)
 *   res_k,  res_v  : [L][n_res_pages][P][r]                (no RoPE)
 *                    bf16 with r = 16: row i of a page stores element j at column
 *                    j ^ (8 * ((i >> 2) & 1)) (the tcgen05 32-byte-swizzled operand
 *                    order). The pools are written only through
 *                    fkv_write_kv and are otherwise opaque to the caller.
 *   Pools must hold finite values (e.g. zero-initialised): tiles are read whole and
 *   rows beyond a sequence's length are masked after the products, not skipped.
 *   rope_cos, rope_sin : fp32 [max_pos][d/2], built host-side in fp64
 *                        (fkv_build_rope_table) — reading C-2, SURVEY H7. */
typedef struct fkv_buffers {
  void* base_k;
  void* base_v;
  void* res_k;
  void* res_v;
  const float* rope_cos;
  const float* rope_sin;
} fkv_buffers;

typedef struct fkv_ctx fkv_ctx;
typedef struct fkv_plan fkv_plan;

/* One sequence of a batch: the agent's block table and length define the
 * keys; its query rows are the LAST q_len positions (decode: q_len = 1;
 * chunked prefill: q_len = chunk). Causal: the query at position p sees keys
 * t <= p (C-6). */
typedef struct fkv_seq {
  int64_t agent;
  int32_t q_len;
  int32_t pad_;
} fkv_seq;

typedef struct fkv_plan_info {
  int64_t n_seqs, n_rows, n_segments, n_items, n_ctas, n_warps, n_entries;
  int64_t key_tiles;        /* 64-key tiles summed over CTAs (one layer) */
  int64_t alg_bytes;        /* algorithmic HBM bytes per layer (SURVEY §8(d) formula) */
  int64_t kernel;           /* 0 = mma.sync (forced only), 1 = SIMT, 2 = tcgen05 keys-on-lanes, 3 = tcgen05 rows-on-lanes */
  int64_t device_bytes;     /* bytes fkv_plan_upload needs */
  int64_t workspace_bytes;  /* bytes fkv_residual_attention needs */
  int64_t alg_rank_bytes;   /* the part of alg_bytes proportional to the rank r (residual pages + adapters):
                               an adapter of rank r' < r zero-padded into the pool (C-8) needs r'/r of it */
} fkv_plan_info;

/* ---- lifetime ------------------------------------------------------- */
fkv_status fkv_create(const fkv_config* cfg, const fkv_buffers* buf, fkv_ctx** out);
fkv_status fkv_destroy(fkv_ctx* ctx);
const char* fkv_last_error(const fkv_ctx* ctx);
const char* fkv_version(void);

/* Register adapter `adapter_id` (>= 0): B_K, B_V device arrays
 * [L][Hkv_local][r][d] (the kv-head column slices of B), LoRA alpha/r
 * folded in (C-7). Borrowed; device contexts need 16-byte aligned arrays
 * (E_INVALID otherwise: vector loads). Re-registering an id replaces the
 * pointers and invalidates existing plans (E_STALE). */
fkv_status fkv_register_adapter(fkv_ctx* ctx, int32_t adapter_id, const void* B_K, const void* B_V);

/* ---- control plane (R1-R9) ----------------------------------- */
/* New agent with empty tables; its residual tree key is itself (R3). */
fkv_status fkv_create_root(fkv_ctx* ctx, int64_t agent, int32_t adapter_id);
/* Fork `child` from `parent`'s first prefix_len tokens: base pages
 * [0, ceil(L/P)) are shared read-only (+1 ref each, a partial tail page is
 * copied on first write, C-10); residual pages are fresh and exclusive
 * (CoW footprint; the caller writes the child's residual rows), or shared CoW
 * with FKV_FORK_SHARE_RESIDUAL (same adapter required). Atomic. */
fkv_status fkv_fork(fkv_ctx* ctx, int64_t parent, int64_t prefix_len, int64_t child, int32_t adapter_id,
                    uint32_t flags);
/* Step 1 of P:300 by token ids: longest full-page prefix match in the base
 * radix tree; matched pages are mapped (+1 each), fresh residual pages are
 * allocated for them, seqlen = *matched. The caller appends the rest. */
fkv_status fkv_fork_tokens(fkv_ctx* ctx, int64_t child, int32_t adapter_id, const int32_t* tokens, int64_t n,
                           int64_t* matched);
/* Fork with a partial hit (P:300 Step 1 + Step 2; "recomputes only the
 * missing base projection xW ... directly reuses the surviving xA_i", §5.2).
 * `owner` names the residual lineage (residual radix tree key) whose
 * surviving xA_i rows the child may reuse; it must hold rows of `adapter_id`
 * (else E_INVALID). The child maps
 *   base pages   of the longest full-page prefix of tokens in the base tree,
 *   residual pages of the longest full-page prefix in the lineage's tree,
 * each +1, and gets FRESH (unwritten) pages for the rest of
 * [0, *mapped = max of both): base rows [*base_hit, *mapped) must be
 * recomputed (xW only: fkv_write_kv with FKV_WRITE_KBASE|FKV_WRITE_VBASE),
 * residual rows [*res_hit, *mapped) likewise (xA_i only). Tokens
 * [*mapped, n) are a cold miss: the caller appends them. All mapped pages are
 * full and are inserted into both trees (one access of each tree's LRU
 * clock). seqlen = *mapped; the child's residual lineage is `owner`.
 * Errors: E_INVALID (ids, lineage adapter), E_NEEDS_EVICTION (pools; nothing
 * changed). Outputs are token counts, multiples of page_size. */
fkv_status fkv_fork_resume(fkv_ctx* ctx, int64_t child, int32_t adapter_id, int64_t owner, const int32_t* tokens,
                           int64_t n, int64_t* base_hit, int64_t* res_hit, int64_t* mapped);
/* ---- sequence split across GPUs (§8(f) row f4) ------------------------------
 * A very long shared prefix with few agents does not partition by agent or
 * head; its keys do. Softmax is invariant to blocking (P-6): each GPU
 * attends over its own key range and the partial outputs are merged by their
 * log-sum-exp; the late V fusion (Eq.4) is linear, so the merge is exact.
 * fkv_plan_create_range: as fkv_plan_create, restricted to the keys
 *   [key_begin, key_end) (page-aligned; key_end = INT64_MAX for "to the end");
 *   rows that see no key of the range produce O = 0 and lse = -inf.
 * fkv_residual_attention_lse: fkv_residual_attention that also writes
 *   lse [sum q_len][Hq_local] (fp32, natural log of sum_t exp(scale q.k_t)).
 * fkv_merge_lse: O = sum_p exp(lse_p - L) O_p, L = log sum_p exp(lse_p), for
 *   O_parts [n_parts][n_rows][head_dim] (dtype) and lse_parts [n_parts][n_rows]
 *   (device; e.g. gathered over NCCL); lse_out (nullable) receives L. Rows
 *   with every lse_p = -inf give O = 0. No ctx: a pure device routine. */
/* Key range [*key_begin, *key_end) of `rank` among G: page-aligned, ~equal page counts over [0, max_seqlen), the
 * last range open-ended (INT64_MAX). */
fkv_status fkv_partition_keys(int64_t max_seqlen, int32_t G, int32_t page_size, int32_t rank, int64_t* key_begin,
                              int64_t* key_end);
fkv_status fkv_plan_create_range(fkv_ctx* ctx, int32_t n, const fkv_seq* seqs, uint32_t flags, int64_t key_begin,
                                 int64_t key_end, fkv_plan** plan);
fkv_status fkv_residual_attention_lse(fkv_ctx* ctx, const fkv_plan* plan, int32_t layer, const void* Q, void* O,
                                      float* lse, float sm_scale, void* workspace, size_t ws_bytes, void* stream);
fkv_status fkv_merge_lse(int32_t n_parts, int64_t n_rows, int32_t head_dim, int32_t dtype, const void* O_parts,
                         const float* lse_parts, void* O, float* lse_out, void* stream);
/* ---- projection producer (§8(f) rows f2, f3) -------------------------------
 * The step in front of the hot path: it fills the disaggregated pools from a
 * layer's input activations (Eq.2: bCache = xW, rCache = xA_i;
 * P:269 §5.1: base K is cached post-RoPE, the residual without RoPE;
 * P:370 §6 the "LoRA replacement module"; a forked child
 * recomputes its own residual over the inherited prefix, a partial hit only
 * the base rows).
 *
 * fkv_register_adapter_down: the adapter's down projections A_K, A_V
 *   [L][hidden][rank] (dtype, row-major, device, borrowed; LoRA alpha/r folded
 *   into B, C-7). The adapter's B must be registered first (E_INVALID).
 * fkv_project_kv: for rows [start[i], start[i]+count[i]) of agents[i] (rows
 *   reserved by fkv_append / a fork), with x [sum count][hidden] (dtype,
 *   device, rows concatenated in the same order) computes
 *     K_base = RoPE_t(x W_k), V_base = x W_v     (W [hidden][Hkv_local][d]:
 *                                                  this ctx's kv-head columns)
 *     R_k = x A_k, R_v = x A_v                    (the agent's adapter, `layer`)
 *   (fp32 accumulate; t = the row's absolute position, rotated with the ctx's
 *   RoPE table, NeoX pairs, C-2) and writes the planes of which_mask
 *   (FKV_WRITE_KBASE|FKV_WRITE_VBASE and/or FKV_WRITE_RK|FKV_WRITE_RV, each
 *   pair together) exactly as fkv_write_kv (same permission rules and errors).
 *   The base GEMM runs on cuBLAS (loaded at run time; E_CUDA if unavailable),
 *   the rank-r products and the rotation in the library's kernels. workspace:
 *   device, 256-byte aligned, >= fkv_project_workspace_bytes(n_rows). */
fkv_status fkv_register_adapter_down(fkv_ctx* ctx, int32_t adapter_id, const void* A_K, const void* A_V,
                                     int32_t hidden);
fkv_status fkv_project_workspace_bytes(fkv_ctx* ctx, int64_t n_rows, size_t* bytes);
fkv_status fkv_project_kv(fkv_ctx* ctx, int32_t layer, int32_t n, const int64_t* agents, const int64_t* start,
                          const int32_t* count, const void* x, int32_t hidden, const void* W_k, const void* W_v,
                          uint32_t which_mask, void* workspace, size_t ws_bytes, void* stream);
/* Decoupled eviction (§5.2: "independent Least Recently Used (LRU)
 * states to each radix tree"). Frees n_pages pages of ONE tree
 * (kind FKV_KIND_BASE = the base tree, FKV_KIND_RES = the residual forest) by
 * repeatedly removing its least recently used leaf, ties to the older
 * insertion, among leaves whose page no live agent view holds (a view acts
 * as the lock). Never touches the other tree, its clock or any agent table.
 * Atomic: if fewer than n_pages pages are evictable, nothing is evicted and
 * E_NEEDS_EVICTION is returned (fkv_evictable_pages tells how many are).
 * *freed (may be NULL) = pages returned to the pool's free set. */
fkv_status fkv_evict(fkv_ctx* ctx, int32_t kind, int64_t n_pages, int64_t* freed);
/* Pages fkv_evict(kind, .) could free right now. */
fkv_status fkv_evictable_pages(fkv_ctx* ctx, int32_t kind, int64_t* n_pages);
/* Reserve n_new[i] slots for agents[i] (token ids concatenated in
 * token_ids). A first write into a page shared by >1 holder copies it
 * (CoW kernel enqueued on `stream`). Pages that become full are inserted into
 * both radix trees. Atomic over the whole call (E_NEEDS_EVICTION leaves no
 * change). */
fkv_status fkv_append(fkv_ctx* ctx, int32_t n, const int64_t* agents, const int32_t* n_new,
                      const int32_t* token_ids, void* stream);
/* Scatter rows [start[i], start[i]+count[i]) of agents[i] for `layer` into
 * the pools. Device sources, rows concatenated over i:
 *   k_base, v_base [sum count][Hkv_local][d];  r_k, r_v [sum count][r].
 * which_mask selects the planes (FKV_WRITE_*). Rows must be reserved; a page
 * with more than one holder is never written (E_READONLY). A row counts as
 * written for a pool when one call stores both its K and V. */
fkv_status fkv_write_kv(fkv_ctx* ctx, int32_t layer, int32_t n, const int64_t* agents, const int64_t* start,
                        const int32_t* count, const void* k_base, const void* v_base, const void* r_k,
                        const void* r_v, uint32_t which_mask, void* stream);
/* Drop the agent's tables; pages reaching refcount 0 return to the free set. */
fkv_status fkv_release(fkv_ctx* ctx, int64_t agent);

/* ---- introspection (parity tests) -------------------------------------- */
fkv_status fkv_get_table(const fkv_ctx* ctx, int64_t agent, int64_t cap, int32_t* base_pages,
                         int32_t* res_pages, int64_t* n_pages, int64_t* seqlen);
fkv_status fkv_get_agent(const fkv_ctx* ctx, int64_t agent, int32_t* adapter_id, int64_t* residual_owner);
fkv_status fkv_page_refcount(const fkv_ctx* ctx, int32_t kind, int64_t page, int32_t* rc);
fkv_status fkv_free_pages(const fkv_ctx* ctx, int32_t kind, int64_t* n_free);
/* Deterministic text dump of agents, pools and both trees (R8). */
fkv_status fkv_dump(const fkv_ctx* ctx, char* buf, size_t cap, size_t* needed);
/* CoW copy log since the last call: quadruples (kind, src, dst, rows). */
fkv_status fkv_take_copy_log(fkv_ctx* ctx, int32_t* buf, int64_t cap_quads, int64_t* n_quads);

/* ---- the hot path ------------------------------------------------------- */
/* Build a plan for one batch: groups sequences by shared base-page runs
 * (agents forked from the same prefix read each shared base tile once),
 * groups rows by residual owner, picks the KV split. Host only. */
fkv_status fkv_plan_create(fkv_ctx* ctx, int32_t n, const fkv_seq* seqs, uint32_t flags, fkv_plan** out);
fkv_status fkv_plan_get_info(const fkv_plan* plan, fkv_plan_info* info);
/* Copy the plan's device arrays into a caller buffer (>= info.device_bytes,
 * 256-byte aligned) on `stream`. Must precede fkv_residual_attention. */
fkv_status fkv_plan_upload(fkv_ctx* ctx, fkv_plan* plan, void* dev, size_t bytes, void* stream);
/* ResidualAttention for one layer (Alg.1 + Eq.4):
 *   Q [n_rows_q][Hq_local][d], O same (rows = seqs in plan order, each its
 *   q_len rows), workspace >= info.workspace_bytes (fp32 partials),
 *   256-byte aligned (E_INVALID otherwise); O 16-byte aligned.
 * sm_scale <= 0 selects 1/sqrt(d) (C-4). Enqueued on `stream`. The kernels
 * use programmatic dependent launch: the first one may start, and read Q,
 * the adapters and the uploaded plan, while the preceding kernel on `stream`
 * finishes, so that kernel must not trigger its dependents
 * (griddepcontrol.launch_dependents) before its writes to Q are done (plain
 * launches, memcpys and this library's own kernels satisfy this). */
fkv_status fkv_residual_attention(fkv_ctx* ctx, const fkv_plan* plan, int32_t layer, const void* Q, void* O,
                                  float sm_scale, void* workspace, size_t ws_bytes, void* stream);
/* The kernels of fkv_residual_attention separately (for per-kernel timing):
 * phases = FKV_PHASE_MAIN (split partials, Stages 1-2: the tcgen05 kernel's
 * operand stager + the main kernel) and/or FKV_PHASE_COMBINE (merge + late V
 * fusion, Stage 3). FKV_PHASE_STAGE alone launches only the stager and
 * FKV_PHASE_NOSTAGE | FKV_PHASE_MAIN only the main kernel, so the main kernel
 * can be timed by itself; STAGE must then precede it (kernel 2; other kernels
 * have no stager and ignore both bits). MAIN must precede COMBINE on the same
 * stream with the same workspace. */
#define FKV_PHASE_MAIN 1u
#define FKV_PHASE_COMBINE 2u
#define FKV_PHASE_STAGE 4u
#define FKV_PHASE_NOSTAGE 8u
fkv_status fkv_residual_attention_phases(fkv_ctx* ctx, const fkv_plan* plan, int32_t layer, const void* Q, void* O,
                                         float sm_scale, void* workspace, size_t ws_bytes, void* stream,
                                         uint32_t phases);
/* Same as fkv_residual_attention with HOST Q/O (pinned for async copies):
 * H2D of Q_host into dQ, attention into dO, D2H of dO into O_host, all
 * enqueued on `stream`; O_host is valid once the stream has synchronised. */
fkv_status fkv_residual_attention_host(fkv_ctx* ctx, const fkv_plan* plan, int32_t layer, const void* Q_host,
                                       void* O_host, void* dQ, void* dO, float sm_scale, void* workspace,
                                       size_t ws_bytes, void* stream);
fkv_status fkv_plan_free(fkv_plan* plan);

/* ---- helpers -------------------------------------------------------------- */
/* RoPE table in fp64, stored fp32: angle = p * inv_freq[i], inv_freq plain
 * theta^(-2i/d) or Llama-3.1 scaled (llama3 != 0). Host arrays [max_pos][d/2]. */
fkv_status fkv_build_rope_table(int32_t max_pos, int32_t d, double theta, int32_t llama3, double factor,
                                double low_freq_factor, double high_freq_factor, double orig_max_pos,
                                float* cos_out, float* sin_out);
/* Device fill with the counter-based synthetic generator of workloads/synth.py
 * (bit-identical): dst[n_pos][n_head][n_col] = value(seed, kind, owner, layer,
 * pos0 + i, head0 + h, col) * scale, stored as dtype. */
fkv_status fkv_synth_fill(void* dst, int32_t dtype, uint64_t seed, int32_t kind, uint64_t owner, int32_t layer,
                          int64_t pos0, int32_t n_pos, int32_t head0, int32_t n_head, int32_t n_col, float scale,
                          void* stream);
/* Head x agent-batch partitioner (§8(e)): choose H kv-head shards and D
 * agent shards with H*D = G, H | n_kv_heads, minimising the per-GPU bytes
 * base_bytes/H + res_bytes/D: a GPU holds the shared base of its H-th of the
 * kv heads (replicated over the D agent shards) and the head-shared residual
 * of its D-th of the agents (replicated over the H head shards). */
fkv_status fkv_partition(int32_t G, int32_t n_kv_heads, int64_t base_bytes, int64_t res_bytes, int32_t* H,
                         int32_t* D);
/* Shard of `rank` under (H, D): kv heads [*h0, *h1), agents [*a0, *a1) of n_agents. */
fkv_status fkv_partition_shard(int32_t rank, int32_t H, int32_t D, int32_t n_kv_heads, int64_t n_agents,
                               int32_t* h0, int32_t* h1, int64_t* a0, int64_t* a1);

/* ---- diagnostics ---------------------------------------------------------- */
/* Self-test of the tcgen05 operand layouts used by the tensor-core kernel:
 * D[M][N] (fp32) = A[M][K] . B[N][K]^T with A, B bf16 row-major device
 * arrays staged into shared memory in layout `test` (0: K-major SW128 x2,
 * 1: MN-major SW128 x2, 2: K-major SW32 A x MN-major SW128 B, 3: MN-major
 * SW32 A x MN-major SW128 B, 4: A in TMEM x K-major SW128 B) and multiplied
 * by tcgen05.mma; test 5 checks a TMA SW128 box load (D[0] = mismatches). */
fkv_status fkv_selftest_umma(int32_t test, const void* A, const void* B, float* D, int32_t M, int32_t N, int32_t K,
                             void* stream);
/* Pipeline timeline of one CTA of the tcgen05 kernel: when `dbg` (device,
 * int64 [32 events][256 tiles], zeroed by the caller) is non-NULL, CTA
 * `block` stores clock64() stamps of its pipeline events. NULL disables. */
fkv_status fkv_debug_timeline(fkv_ctx* ctx, void* dbg, int32_t block);
/* Diagnostics: with the environment variable FKV_HANG_DIAG set, a pipeline wait of the rows kernel that spins
 * far beyond any legitimate latency records where it waited (in host-mapped memory) and traps; this copies the
 * report ("" if none) into buf (cap bytes, NUL-terminated). Readable after the resulting launch failure. */
fkv_status fkv_debug_hang_report(char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* FORKKV_H_ */
