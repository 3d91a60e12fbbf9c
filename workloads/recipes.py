"""Synthetic workloads shaped like the paper's (§7.1).

A scenario is a fork tree of agents over a shared root prefix. ``build``
drives the product API (fork / append / write_kv) and fills rows with the
counter-based generator on the device; ``oracle_inputs`` regenerates the same
logical rows on the host for the oracle. Logical content of an agent's row t
is labelled by its writer: rows before a fork point are the parent's, a
non-shared child writes its own residual rows over the inherited prefix
(its x A_i, "exclusively allocating the rCache"), and every agent
writes its own appended rows.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import synth

LLAMA8B = dict(n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128)
LLAMA70B = dict(n_layers=80, n_q_heads=64, n_kv_heads=8, head_dim=128)


@dataclass
class AgentSpec:
    id: int
    adapter: int
    parent: Optional[int] = None      # None -> root
    fork_len: int = 0                 # tokens inherited from parent
    share_res: bool = False           # same-agent branch (FKV_FORK_SHARE_RESIDUAL)
    n_private: int = 0                # tokens appended after the fork (or by the root)
    decode: bool = True               # appears in the decode batch


@dataclass
class Scenario:
    name: str
    agents: List[AgentSpec]
    q_len: int = 1                    # query rows per batch sequence (1 = decode)
    extra: Dict = field(default_factory=dict)

    def spec(self, a: int) -> AgentSpec:
        for s in self.agents:
            if s.id == a:
                return s
        raise KeyError(a)

    def seqlen(self, a: int) -> int:
        s = self.spec(a)
        return s.fork_len + s.n_private

    def batch(self) -> List[int]:
        return [s.id for s in self.agents if s.decode]

    def writers(self, a: int, t: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
        """(base writer, residual writer) labels of agent a's rows t."""
        s = self.spec(a)
        bw = np.full(len(t), a, dtype=np.int64)
        rw = np.full(len(t), a, dtype=np.int64)
        if s.parent is not None:
            inh = t < s.fork_len
            if inh.any():
                pb, pr = self.writers(s.parent, t[inh])
                bw[inh] = pb
                if s.share_res:
                    rw[inh] = pr
        return bw, rw

    def pages_needed(self, P: int, slack: int = 2) -> Tuple[int, int]:
        """Upper bound on (base, residual) pages the build allocates: own
        appended pages (+1 for a CoW'd partial tail), a non-shared child's
        residual over the whole inherited prefix."""
        nb = nr = 0
        for s in self.agents:
            L = s.fork_len + s.n_private
            tot = -(-L // P)
            own = tot - (s.fork_len // P if s.parent is not None else 0)
            nb += own + 1
            nr += (own + 1) if (s.share_res or s.parent is None) else tot + 1
        return nb + slack, nr + slack


# ---- the BASELINE.json configs -------------------------------------------------

def c1(prefix=2048, n_agents=4, private=128) -> Scenario:
    """configs[0]: 1 layer, 4 agents (adapters 0-3) forked from a 2K root,
    128-token private suffix, one decode step (+1 token)."""
    ag = [AgentSpec(1000, 1000, None, 0, False, prefix, decode=False)]
    for i in range(n_agents):
        ag.append(AgentSpec(i, i, 1000, prefix, False, private + 1))
    return Scenario("C1", ag)


def c2(prefix=32768, n_agents=16, branches=4, private=128) -> Scenario:
    """configs[1] (primary reading): 16 agents / 16 adapters
    forked from a 32K root with their own residual over the prefix, 4
    same-agent branches each (residual prefix pages shared CoW) -> decode
    batch 64, 128-token private suffix + 1 decode token."""
    ag = [AgentSpec(100000, 100000, None, 0, False, prefix, decode=False)]
    for i in range(n_agents):
        ag.append(AgentSpec(1000 + i, i, 100000, prefix, False, 0, decode=False))
        for b in range(branches):
            ag.append(AgentSpec(i * branches + b, i, 1000 + i, prefix, True, private + 1))
    return Scenario("C2", ag)


def c3(prefix=32768, n_agents=8, private=4096, chunk=1024) -> Scenario:
    """configs[2]: chunked prefill of 4K-token agent-private contexts over a
    32K shared prefix, 8 agents with distinct r=16 adapters (8 workflows,
    P:401). The batch is one 1024-token chunk per agent (the last chunk)."""
    ag = [AgentSpec(100000, 100000, None, 0, False, prefix, decode=False)]
    for i in range(n_agents):
        ag.append(AgentSpec(i, i, 100000, prefix, False, private))
    return Scenario("C3", ag, q_len=chunk)


def c5(prefix=32768, n_agents=64, private=128) -> Scenario:
    """configs[4] point: N independent agents (residual per sequence)."""
    ag = [AgentSpec(100000, 100000, None, 0, False, prefix, decode=False)]
    for i in range(n_agents):
        ag.append(AgentSpec(i, i, 100000, prefix, False, private + 1))
    return Scenario("C5", ag)


def fanout(n_agents, prefix=32768, private=128) -> Scenario:
    """configs[4] sweep point: fork fan-out N (4-256) agents with distinct adapters, each with its own residual
    over the shared prefix (the C5 shape at fan-out N)."""
    return c5(prefix=prefix, n_agents=n_agents, private=private)


# ---- host-side oracle inputs --------------------------------------------------

_RUN_CACHE: Dict = {}


def _run(seed, kind, writer, layer, t0, t1, heads, ncol, dtype):
    key = (seed, kind, writer, layer, t0, t1, heads, ncol, dtype)
    v = _RUN_CACHE.get(key)
    if v is None:
        if len(_RUN_CACHE) > 64:
            _RUN_CACHE.clear()
        v = synth.maybe_round(synth.values(seed, kind, writer, layer,
                                           np.arange(t0, t1, dtype=np.uint64)[:, None, None],
                                           np.asarray(heads, dtype=np.uint64)[None, :, None],
                                           np.arange(ncol, dtype=np.uint64)[None, None, :]), dtype)
        _RUN_CACHE[key] = v
    return v


def oracle_inputs(scen: Scenario, seed: int, a: int, layer: int, n_kv: int, d: int, r: int, n_q: int,
                  q_len: int, dtype: str, kv_heads: Tuple[int, int] = None, step: int = 0):
    """Logical per-sequence arrays for oracle.ra.residual_attention."""
    L = scen.seqlen(a)
    t = np.arange(L, dtype=np.int64)
    bw, rw = scen.writers(a, t)
    h0, h1 = kv_heads if kv_heads else (0, n_kv)
    g = n_q // n_kv
    heads = np.arange(h0, h1, dtype=np.uint64)

    def rows(kind, writers, ncol, heads_):
        out = np.empty((L, len(heads_), ncol), dtype=np.float32)
        # runs of a constant writer are generated once and memoised (shared
        # prefixes are identical for every agent of a fork tree)
        edges = np.nonzero(np.diff(writers))[0] + 1
        starts = np.concatenate([[0], edges]).astype(int)
        ends = np.concatenate([edges, [L]]).astype(int)
        for s0, s1 in zip(starts, ends):
            if s1 > s0:
                out[s0:s1] = _run(seed, kind, int(writers[s0]), layer, s0, s1, tuple(int(x) for x in heads_), ncol,
                                  dtype)
        return out

    Kb = rows(synth.KIND_KBASE, bw, d, heads)
    Vb = rows(synth.KIND_VBASE, bw, d, heads)
    Rk = rows(synth.KIND_RK, rw, r, np.zeros(1, np.uint64))[:, 0, :]
    Rv = rows(synth.KIND_RV, rw, r, np.zeros(1, np.uint64))[:, 0, :]
    ad = scen.spec(a).adapter
    Bk = np.stack([synth.maybe_round(synth.values(seed, synth.KIND_BK, ad, layer,
                                                  np.arange(r, dtype=np.uint64)[:, None], np.uint64(h),
                                                  np.arange(d, dtype=np.uint64)[None, :]), dtype) for h in heads])
    Bv = np.stack([synth.maybe_round(synth.values(seed, synth.KIND_BV, ad, layer,
                                                  np.arange(r, dtype=np.uint64)[:, None], np.uint64(h),
                                                  np.arange(d, dtype=np.uint64)[None, :]), dtype) for h in heads])
    qh = np.arange(h0 * g, h1 * g, dtype=np.uint64)
    Q = synth.maybe_round(synth.values(seed, synth.KIND_Q, a, layer,
                                       (np.uint64(step * 4096) + np.arange(q_len, dtype=np.uint64))[:, None, None],
                                       qh[None, :, None], np.arange(d, dtype=np.uint64)[None, None, :]), dtype)
    return dict(Kb=Kb, Vb=Vb, Rk=Rk, Rv=Rv, Bk=Bk, Bv=Bv, Q=Q)
