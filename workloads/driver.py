"""Drive a Scenario through the product API (fork / append / write_kv) with
device-side synthetic rows (fkv_synth_fill, bit-identical to synth.py)."""
from __future__ import annotations

from typing import Iterable, Optional

import numpy as np

from . import synth
from .recipes import Scenario

_CHUNK = 65536       # rows per staged write (base rows: 65536 x Hkv x d x 2 B = 128 MiB at 8 heads)
_CHUNK_RES = 1 << 20  # residual-only writes are r-wide: stage up to 1M rows


def make_adapter(fkv, seed: int, adapter_id: int, h0: int, r_eff: Optional[int] = None):
    import torch
    from paper_2604_06370_b200.api import synth_fill
    tdt = torch.bfloat16 if fkv.dtype_name == "bf16" else torch.float32
    dev = torch.device("cuda", fkv.device)
    bk = torch.empty(fkv.L, fkv.hkv, fkv.r, fkv.d, dtype=tdt, device=dev)
    bv = torch.empty_like(bk)
    for layer in range(fkv.L):
        for hl in range(fkv.hkv):
            synth_fill(bk[layer, hl], seed, synth.KIND_BK, adapter_id, layer, 0, head0=h0 + hl,
                       scale=synth.SCALE[synth.KIND_BK])
            synth_fill(bv[layer, hl], seed, synth.KIND_BV, adapter_id, layer, 0, head0=h0 + hl,
                       scale=synth.SCALE[synth.KIND_BV])
    if r_eff is not None and r_eff < fkv.r:   # an adapter of rank r_eff zero-padded into the pool rank (C-8)
        bk[:, :, r_eff:] = 0
        bv[:, :, r_eff:] = 0
    return bk, bv


def write_rows(fkv, seed: int, agent: int, writer: int, pos0: int, n: int, mask: int, h0: int,
               layers: Optional[Iterable[int]] = None, stage=None, r_eff: Optional[int] = None):
    import torch
    from paper_2604_06370_b200.api import synth_fill
    if n <= 0:
        return
    tdt = torch.bfloat16 if fkv.dtype_name == "bf16" else torch.float32
    dev = torch.device("cuda", fkv.device)
    chunk = _CHUNK if mask & 3 else _CHUNK_RES
    m = min(n, chunk)
    if stage is None:
        stage = {}
    if (mask & 3) and stage.get("nb", 0) < m:
        stage.update(nb=m, kb=torch.empty(m, fkv.hkv, fkv.d, dtype=tdt, device=dev),
                     vb=torch.empty(m, fkv.hkv, fkv.d, dtype=tdt, device=dev))
    if stage.get("nr", 0) < m:
        stage.update(nr=m, rk=torch.empty(m, fkv.r, dtype=tdt, device=dev),
                     rv=torch.empty(m, fkv.r, dtype=tdt, device=dev))
    for layer in (range(fkv.L) if layers is None else layers):
        for o in range(0, n, chunk):
            c = min(chunk, n - o)
            kb = stage["kb"][:c] if mask & 3 else None
            vb = stage["vb"][:c] if mask & 3 else None
            rk, rv = stage["rk"][:c], stage["rv"][:c]
            if mask & 3:
                synth_fill(kb, seed, synth.KIND_KBASE, writer, layer, pos0 + o, head0=h0)
                synth_fill(vb, seed, synth.KIND_VBASE, writer, layer, pos0 + o, head0=h0)
            if mask & 12:
                synth_fill(rk, seed, synth.KIND_RK, writer, layer, pos0 + o)
                synth_fill(rv, seed, synth.KIND_RV, writer, layer, pos0 + o)
                if r_eff is not None and r_eff < fkv.r:   # xA_i of a rank-r_eff adapter, zero-padded (C-8)
                    rk[:, r_eff:] = 0
                    rv[:, r_eff:] = 0
            fkv.write_kv(layer, [agent], [pos0 + o], [c], kb, vb, rk, rv, mask)


def build(fkv, scen: Scenario, seed: int, h0: int = 0, layers=None, r_eff: Optional[int] = None):
    """Create every agent of the scenario through the API and write its rows (r_eff: adapters and residual rows
    of rank r_eff < fkv.r, zero-padded into the pool, C-8)."""
    from paper_2604_06370_b200 import _lib as L
    stage = {}
    adapters = sorted({s.adapter for s in scen.agents})
    for ad in adapters:
        bk, bv = make_adapter(fkv, seed, ad, h0, r_eff)
        fkv.register_adapter(ad, bk, bv)
    for s in scen.agents:
        if s.parent is None:
            fkv.create_root(s.id, s.adapter)
        else:
            fkv.fork(s.parent, s.fork_len, s.id, s.adapter, L.FORK_SHARE_RESIDUAL if s.share_res else 0)
            if not s.share_res:
                write_rows(fkv, seed, s.id, s.id, 0, s.fork_len, L.WRITE_RK | L.WRITE_RV, h0, layers, stage, r_eff)
        if s.n_private:
            toks = synth.tokens(seed, s.id, s.fork_len, s.n_private).tolist()
            fkv.append([s.id], [s.n_private], toks)
            write_rows(fkv, seed, s.id, s.id, s.fork_len, s.n_private, L.WRITE_ALL, h0, layers, stage, r_eff)


def make_queries(fkv, scen: Scenario, seed: int, layer: int, step: int = 0, h0: int = 0, out=None):
    import torch
    from paper_2604_06370_b200.api import synth_fill
    batch = scen.batch()
    C = scen.q_len
    tdt = torch.bfloat16 if fkv.dtype_name == "bf16" else torch.float32
    if out is None:
        out = torch.empty(len(batch) * C, fkv.hq, fkv.d, dtype=tdt, device=torch.device("cuda", fkv.device))
    for i, a in enumerate(batch):
        synth_fill(out[i * C:(i + 1) * C], seed, synth.KIND_Q, a, layer, step * 4096, head0=h0 * fkv.group,
                   scale=synth.SCALE[synth.KIND_Q])
    return out
