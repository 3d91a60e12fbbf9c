"""Thin Python binding over the C ABI (include/forkkv.h).

Argument marshalling only: every step of the path runs in libforkkv.so
(C++ control plane + sm_100a kernels). PyTorch provides device memory and
streams. Names follow the C calls without the ``fkv_`` prefix.
"""
from __future__ import annotations

import ctypes
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from ._lib import FkvError


def _check(lib, ctx, st):
    if st != L.OK:
        msg = lib.fkv_last_error(ctx).decode(errors="replace") if ctx is not None else ""
        raise FkvError(st, msg)


def _arr(a, ct):
    a = np.ascontiguousarray(a, dtype={ctypes.c_int32: np.int32, ctypes.c_int64: np.int64}[ct])
    return a, a.ctypes.data_as(ctypes.POINTER(ct))


def _stream_handle(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def build_rope_table(max_pos: int, d: int, theta: float = 10000.0, llama3: bool = False, factor: float = 8.0,
                     low: float = 1.0, high: float = 4.0, orig: float = 8192.0):
    """fp32 cos/sin [max_pos][d/2] computed in fp64 on the host (C-2, H7)."""
    lib = L.load()
    cos = np.zeros((max_pos, d // 2), dtype=np.float32)
    sin = np.zeros((max_pos, d // 2), dtype=np.float32)
    _check(lib, None, lib.fkv_build_rope_table(max_pos, d, theta, int(llama3), factor, low, high, orig,
                                               cos.ctypes.data_as(ctypes.c_void_p),
                                               sin.ctypes.data_as(ctypes.c_void_p)))
    return cos, sin


def synth_fill(dst, seed: int, kind: int, owner: int, layer: int, pos0: int, head0: int = 0, scale: float = 1.0,
               stream=None):
    """Fill a device tensor [n_pos][n_head][n_col] (or [n_pos][n_col]) with the
    counter-based generator of workloads/synth.py, bit-identically."""
    import torch
    lib = L.load()
    shape = dst.shape
    if len(shape) == 2:
        n_pos, n_head, n_col = shape[0], 1, shape[1]
    else:
        n_pos, n_head, n_col = shape
    dt = L.DTYPE_BF16 if dst.dtype == torch.bfloat16 else L.DTYPE_F32
    _check(lib, None, lib.fkv_synth_fill(_ptr(dst), dt, seed, kind, owner, layer, pos0, n_pos, head0, n_head, n_col,
                                         scale, _stream_handle(stream)))


def merge_lse(O_parts, lse_parts, O=None, lse_out=None, stream=None):
    """fkv_merge_lse: O_parts [G][rows...][d], lse_parts [G][rows...] (device) -> merged O (and lse)."""
    import torch
    G = O_parts.shape[0]
    d = O_parts.shape[-1]
    n_rows = lse_parts[0].numel()
    if O is None:
        O = torch.empty(O_parts.shape[1:], dtype=O_parts.dtype, device=O_parts.device)
    lib = L.load()
    dt = L.DTYPE_BF16 if O_parts.dtype == torch.bfloat16 else L.DTYPE_F32
    _check(lib, None, lib.fkv_merge_lse(G, n_rows, d, dt, _ptr(O_parts), _ptr(lse_parts), _ptr(O), _ptr(lse_out),
                                         _stream_handle(stream)))
    return O


def partition_keys(max_seqlen: int, G: int, page_size: int, rank: int) -> Tuple[int, Optional[int]]:
    """Key range (begin, end) of `rank` for the cross-GPU sequence split (end None = open-ended)."""
    lib = L.load()
    kb, ke = ctypes.c_int64(), ctypes.c_int64()
    _check(lib, None, lib.fkv_partition_keys(max_seqlen, G, page_size, rank, ctypes.byref(kb), ctypes.byref(ke)))
    return kb.value, (None if ke.value == (1 << 63) - 1 else ke.value)


def partition(G: int, n_kv_heads: int, base_bytes: int, res_bytes: int) -> Tuple[int, int]:
    lib = L.load()
    H, D = ctypes.c_int32(), ctypes.c_int32()
    _check(lib, None, lib.fkv_partition(G, n_kv_heads, base_bytes, res_bytes, ctypes.byref(H), ctypes.byref(D)))
    return H.value, D.value


def partition_shard(rank: int, H: int, D: int, n_kv_heads: int, n_agents: int):
    lib = L.load()
    h0, h1, a0, a1 = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib, None, lib.fkv_partition_shard(rank, H, D, n_kv_heads, n_agents, ctypes.byref(h0), ctypes.byref(h1),
                                              ctypes.byref(a0), ctypes.byref(a1)))
    return (h0.value, h1.value), (a0.value, a1.value)


class Plan:
    """A batch plan (host) plus its uploaded device copy and workspace."""

    def __init__(self, owner: "ForkKV", handle, info):
        self.owner = owner
        self.handle = handle
        self.info = info
        self.dev = None
        self.ws = None

    def __del__(self):
        try:
            if self.handle:
                L.load().fkv_plan_free(self.handle)
                self.handle = None
        except Exception:
            pass


class ForkKV:
    """One ForkKV context: pools (torch-owned device memory), RoPE table,
    adapters, control plane. ``device=None`` -> host-only control plane."""

    def __init__(self, n_layers: int, n_q_heads: int, n_kv_heads: int, head_dim: int, rank: int, page_size: int,
                 n_base_pages: int, n_res_pages: int, dtype: str = "bf16", rope_mode: str = "deferred",
                 device: Optional[int] = 0, max_pos: int = 0, alloc_order_seed: int = 0,
                 kv_heads: Optional[Tuple[int, int]] = None, rope_theta: float = 10000.0, llama3: bool = False):
        self.lib = L.load()
        h0, h1 = kv_heads if kv_heads is not None else (0, n_kv_heads)
        self.hkv = h1 - h0
        self.group = n_q_heads // n_kv_heads
        self.hq = self.hkv * self.group
        self.L, self.d, self.r, self.P = n_layers, head_dim, rank, page_size
        self.nb, self.nr = n_base_pages, n_res_pages
        self.dtype_name = dtype
        self.dtype_code = L.DTYPE_BF16 if dtype == "bf16" else L.DTYPE_F32
        self.rope_mode = L.ROPE_DEFERRED if rope_mode == "deferred" else L.ROPE_NONE
        self.device = device
        cfg = L.fkv_config(n_layers, n_q_heads, n_kv_heads, head_dim, rank, page_size, n_base_pages, n_res_pages,
                           max_pos, self.dtype_code, self.rope_mode, -1 if device is None else device,
                           alloc_order_seed, h0, h1)
        buf = L.fkv_buffers()
        self.tensors = {}
        if device is not None:
            import torch
            tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
            dev = torch.device("cuda", device)
            mk = lambda *s: torch.zeros(*s, dtype=tdt, device=dev)
            self.base_k = mk(n_layers, n_base_pages, self.hkv, page_size, head_dim)
            self.base_v = mk(n_layers, n_base_pages, self.hkv, page_size, head_dim)
            self.res_k = mk(n_layers, n_res_pages, page_size, rank)
            self.res_v = mk(n_layers, n_res_pages, page_size, rank)
            if max_pos > 0:
                c, s = build_rope_table(max_pos, head_dim, rope_theta, llama3)
                self.rope_cos = torch.from_numpy(c).to(dev)
                self.rope_sin = torch.from_numpy(s).to(dev)
            else:
                self.rope_cos = self.rope_sin = None
            buf.base_k, buf.base_v = self.base_k.data_ptr(), self.base_v.data_ptr()
            buf.res_k, buf.res_v = self.res_k.data_ptr(), self.res_v.data_ptr()
            buf.rope_cos = self.rope_cos.data_ptr() if self.rope_cos is not None else None
            buf.rope_sin = self.rope_sin.data_ptr() if self.rope_sin is not None else None
        self.ctx = ctypes.c_void_p()
        st = self.lib.fkv_create(ctypes.byref(cfg), ctypes.byref(buf), ctypes.byref(self.ctx))
        if st != L.OK:
            raise FkvError(st, self.lib.fkv_last_error(None).decode())
        self.adapters = {}

    def __del__(self):
        try:
            if self.ctx:
                self.lib.fkv_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    def _c(self, st):
        _check(self.lib, self.ctx, st)

    # ---- adapters ---------------------------------------------------------
    def register_adapter(self, adapter_id: int, B_K=None, B_V=None):
        """B_K, B_V: [L][Hkv_local][r][d] device tensors (kept alive here)."""
        self.adapters[adapter_id] = (B_K, B_V)
        self._c(self.lib.fkv_register_adapter(self.ctx, adapter_id, _ptr(B_K), _ptr(B_V)))

    # ---- control plane -------------------------------------------------------
    def create_root(self, agent: int, adapter_id: int):
        self._c(self.lib.fkv_create_root(self.ctx, agent, adapter_id))

    def fork(self, parent: int, prefix_len: int, child: int, adapter_id: int, flags: int = 0):
        self._c(self.lib.fkv_fork(self.ctx, parent, prefix_len, child, adapter_id, flags))

    def fork_tokens(self, child: int, adapter_id: int, tokens: Sequence[int]) -> int:
        a, p = _arr(tokens if len(tokens) else [0], ctypes.c_int32)
        m = ctypes.c_int64()
        self._c(self.lib.fkv_fork_tokens(self.ctx, child, adapter_id, p, len(tokens), ctypes.byref(m)))
        return m.value

    def register_adapter_down(self, adapter_id: int, A_K, A_V):
        """Down projections A_K, A_V [L][hidden][r] of a registered adapter (projection producer, §8(f) f2)."""
        self.adapters[("A", adapter_id)] = (A_K, A_V)
        self._c(self.lib.fkv_register_adapter_down(self.ctx, adapter_id, _ptr(A_K), _ptr(A_V), A_K.shape[-2]))

    def project_kv(self, layer: int, agents, start, count, x, W_k=None, W_v=None, mask: int = L.WRITE_ALL,
                   stream=None, ws=None):
        """fkv_project_kv: fill rows [start, start+count) of each agent from the layer input x [sum count][hidden]
        (K_base = RoPE(x W_k), V_base = x W_v, R = x A of the agent's adapter)."""
        import torch
        T = int(np.sum(count)) if len(count) else 0
        need = ctypes.c_size_t()
        self._c(self.lib.fkv_project_workspace_bytes(self.ctx, T, ctypes.byref(need)))
        if ws is None or ws.numel() * ws.element_size() < need.value:
            ws = torch.empty(max(256, need.value), dtype=torch.uint8, device=x.device)
        aa, pa = _arr(agents, ctypes.c_int64)
        ss, ps = _arr(start, ctypes.c_int64)
        cc, pc = _arr(count, ctypes.c_int32)
        self._c(self.lib.fkv_project_kv(self.ctx, layer, len(agents), pa, ps, pc, _ptr(x), x.shape[-1], _ptr(W_k),
                                        _ptr(W_v), mask, _ptr(ws), ws.numel() * ws.element_size(),
                                        _stream_handle(stream)))
        return ws

    def fork_resume(self, child: int, adapter_id: int, owner: int, tokens: Sequence[int]):
        """Partial-hit fork: returns (base_hit, res_hit, mapped) in tokens."""
        a, p = _arr(tokens if len(tokens) else [0], ctypes.c_int32)
        bh, rh, mp = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self._c(self.lib.fkv_fork_resume(self.ctx, child, adapter_id, owner, p, len(tokens), ctypes.byref(bh),
                                         ctypes.byref(rh), ctypes.byref(mp)))
        return bh.value, rh.value, mp.value

    def evict(self, kind: int, n_pages: int) -> int:
        """Decoupled eviction of one tree; returns the pages freed."""
        f = ctypes.c_int64()
        self._c(self.lib.fkv_evict(self.ctx, kind, n_pages, ctypes.byref(f)))
        return f.value

    def evictable_pages(self, kind: int) -> int:
        n = ctypes.c_int64()
        self._c(self.lib.fkv_evictable_pages(self.ctx, kind, ctypes.byref(n)))
        return n.value

    def append(self, agents: Sequence[int], n_new: Sequence[int], token_ids: Sequence[int], stream=None):
        expected = int(np.sum(n_new)) if len(n_new) else 0
        if len(token_ids) != expected:
            raise FkvError(L.E_INVALID, "token_ids length != sum(n_new)")
        aa, pa = _arr(agents, ctypes.c_int64)
        nn, pn = _arr(n_new, ctypes.c_int32)
        tt, pt = _arr(token_ids if len(token_ids) else [0], ctypes.c_int32)
        self._c(self.lib.fkv_append(self.ctx, len(agents), pa, pn, pt, _stream_handle(stream)))

    def write_kv(self, layer: int, agents: Sequence[int], start: Sequence[int], count: Sequence[int], k_base=None,
                 v_base=None, r_k=None, r_v=None, mask: int = L.WRITE_ALL, stream=None):
        aa, pa = _arr(agents, ctypes.c_int64)
        ss, ps = _arr(start, ctypes.c_int64)
        cc, pc = _arr(count, ctypes.c_int32)
        self._c(self.lib.fkv_write_kv(self.ctx, layer, len(agents), pa, ps, pc, _ptr(k_base), _ptr(v_base),
                                      _ptr(r_k), _ptr(r_v), mask, _stream_handle(stream)))

    def release(self, agent: int):
        self._c(self.lib.fkv_release(self.ctx, agent))

    # ---- introspection ------------------------------------------------------
    def get_table(self, agent: int):
        n, sl = ctypes.c_int64(), ctypes.c_int64()
        self._c(self.lib.fkv_get_table(self.ctx, agent, 0, None, None, ctypes.byref(n), ctypes.byref(sl)))
        b = np.zeros(max(n.value, 1), np.int32)
        r = np.zeros(max(n.value, 1), np.int32)
        self._c(self.lib.fkv_get_table(self.ctx, agent, n.value, b.ctypes.data_as(L._pi32),
                                       r.ctypes.data_as(L._pi32), ctypes.byref(n), ctypes.byref(sl)))
        return b[:n.value].tolist(), r[:n.value].tolist(), sl.value

    def get_agent(self, agent: int):
        a, o = ctypes.c_int32(), ctypes.c_int64()
        self._c(self.lib.fkv_get_agent(self.ctx, agent, ctypes.byref(a), ctypes.byref(o)))
        return a.value, o.value

    def page_refcount(self, kind: int, page: int) -> int:
        rc = ctypes.c_int32()
        self._c(self.lib.fkv_page_refcount(self.ctx, kind, page, ctypes.byref(rc)))
        return rc.value

    def free_pages(self, kind: int) -> int:
        n = ctypes.c_int64()
        self._c(self.lib.fkv_free_pages(self.ctx, kind, ctypes.byref(n)))
        return n.value

    def dump(self) -> str:
        need = ctypes.c_size_t()
        self._c(self.lib.fkv_dump(self.ctx, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        self._c(self.lib.fkv_dump(self.ctx, buf, need.value, ctypes.byref(need)))
        return buf.value.decode()

    def take_copy_log(self) -> List[Tuple[int, int, int, int]]:
        n = ctypes.c_int64()
        self._c(self.lib.fkv_take_copy_log(self.ctx, None, 0, ctypes.byref(n)))
        buf = np.zeros(max(1, 4 * n.value), np.int32)
        self._c(self.lib.fkv_take_copy_log(self.ctx, buf.ctypes.data_as(L._pi32), n.value, ctypes.byref(n)))
        return [tuple(buf[4 * i:4 * i + 4].tolist()) for i in range(n.value)]

    # ---- hot path -------------------------------------------------------------
    def plan(self, seqs: Iterable[Tuple[int, int]], flags: int = 0, upload: bool = True, stream=None,
             key_range: Optional[Tuple[int, int]] = None) -> Plan:
        """fkv_plan_create, or fkv_plan_create_range when key_range = (begin, end) (end None = to the end)."""
        seqs = list(seqs)
        arr = (L.fkv_seq * len(seqs))(*[L.fkv_seq(a, q, 0) for a, q in seqs])
        h = ctypes.c_void_p()
        if key_range is None:
            self._c(self.lib.fkv_plan_create(self.ctx, len(seqs), arr, flags, ctypes.byref(h)))
        else:
            kb, ke = key_range
            self._c(self.lib.fkv_plan_create_range(self.ctx, len(seqs), arr, flags, kb,
                                                   (1 << 63) - 1 if ke is None else ke, ctypes.byref(h)))
        info = L.fkv_plan_info()
        self._c(self.lib.fkv_plan_get_info(h, ctypes.byref(info)))
        pl = Plan(self, h, info)
        if upload and self.device is not None:
            self.plan_upload(pl, stream=stream)
        return pl

    def plan_upload(self, pl: Plan, dev=None, ws=None, stream=None):
        import torch
        d = torch.device("cuda", self.device)
        if dev is None or dev.numel() < pl.info.device_bytes:
            dev = torch.empty(max(256, pl.info.device_bytes), dtype=torch.uint8, device=d)
        if ws is None or ws.numel() * 4 < pl.info.workspace_bytes:
            ws = torch.empty(max(64, pl.info.workspace_bytes // 4), dtype=torch.float32, device=d)
        pl.dev, pl.ws = dev, ws
        self._c(self.lib.fkv_plan_upload(self.ctx, pl.handle, _ptr(dev), dev.numel(), _stream_handle(stream)))

    def residual_attention(self, pl: Plan, layer: int, Q, O=None, sm_scale: float = 0.0, stream=None):
        import torch
        if O is None:
            O = torch.empty_like(Q)
        self._c(self.lib.fkv_residual_attention(self.ctx, pl.handle, layer, _ptr(Q), _ptr(O), sm_scale,
                                                _ptr(pl.ws), pl.ws.numel() * 4, _stream_handle(stream)))
        return O

    def residual_attention_lse(self, pl: Plan, layer: int, Q, O=None, lse=None, sm_scale: float = 0.0, stream=None):
        """Attention plus the per-row log-sum-exp [rows][Hq_local] (fp32), for the cross-GPU LSE merge (§8(f) f4)."""
        import torch
        if O is None:
            O = torch.empty_like(Q)
        if lse is None:
            lse = torch.empty(Q.shape[0], Q.shape[1], dtype=torch.float32, device=Q.device)
        self._c(self.lib.fkv_residual_attention_lse(self.ctx, pl.handle, layer, _ptr(Q), _ptr(O), _ptr(lse), sm_scale,
                                                    _ptr(pl.ws), pl.ws.numel() * 4, _stream_handle(stream)))
        return O, lse

    def residual_attention_phases(self, pl: Plan, layer: int, Q, O, phases: int, sm_scale: float = 0.0,
                                  stream=None):
        self._c(self.lib.fkv_residual_attention_phases(self.ctx, pl.handle, layer, _ptr(Q), _ptr(O), sm_scale,
                                                       _ptr(pl.ws), pl.ws.numel() * 4, _stream_handle(stream),
                                                       phases))
        return O

    def residual_attention_host(self, pl: Plan, layer: int, Q_host, O_host, dQ, dO, sm_scale: float = 0.0,
                                stream=None):
        self._c(self.lib.fkv_residual_attention_host(self.ctx, pl.handle, layer, _ptr(Q_host), _ptr(O_host),
                                                     _ptr(dQ), _ptr(dO), sm_scale, _ptr(pl.ws), pl.ws.numel() * 4,
                                                     _stream_handle(stream)))
        return O_host
