"""ORACLE (test infrastructure): the disaggregated K/V projection (§8(f) rows f2, f3).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module; it shares no code with the CUDA path.

What it follows:
  Eq.1 (§2.2)  a LoRA agent's K / V projection is  xW + xA_iB_i;
  Eq.2 (§2.2)  ForkKV stores the two parts separately: the shared
                          bCache xW and the agent's rank-r rCache xA_i;
  P:134 §2.2, §5.1  RoPE is applied to the base K before caching (K_base
                          = RoPE(xW_k)); the residual xA_k is cached WITHOUT
                          RoPE (its up-projection by B_k and the rotation are
                          deferred to attention, Alg1.335);
  P:300, §5.2       a forked child recomputes its own residual xA_i over
                          the inherited prefix (Step 2), and a partial hit
                          recomputes only the base xW.
Readings: NeoX half-split RoPE pairs (i, i + d/2) with the model's inv_freq
(C-2); positions are absolute token indices (C-3).  Plain fp64
matrix products, one rotation per row: no blocking or fusion.
"""
from __future__ import annotations

import numpy as np


def rope(v: np.ndarray, pos: np.ndarray, inv_freq: np.ndarray) -> np.ndarray:
    """Rotate v [T][H][d] at absolute positions pos [T]: for each pair (i, i + d/2),
    (a, b) -> (a cos(p w_i) - b sin(p w_i), b cos(p w_i) + a sin(p w_i))."""
    v = np.asarray(v, dtype=np.float64)
    d = v.shape[-1]
    ang = np.asarray(pos, dtype=np.float64)[:, None] * np.asarray(inv_freq, dtype=np.float64)[None, :]  # [T][d/2]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    a, b = v[..., : d // 2], v[..., d // 2:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)


def project(x, Wk, Wv, Ak, Av, pos, inv_freq, rope_k: bool = True):
    """The four cached planes of T token rows (Eq.2 split of Eq.1).

    x [T][hidden]; Wk, Wv [hidden][Hkv][d]; Ak, Av [hidden][r]; pos [T].
    Returns (K_base [T][Hkv][d] = RoPE_pos(x Wk), V_base = x Wv, R_k = x Ak, R_v = x Av), fp64.
    """
    x = np.asarray(x, dtype=np.float64)
    hidden, hkv, d = np.asarray(Wk).shape
    kb = (x @ np.asarray(Wk, dtype=np.float64).reshape(hidden, hkv * d)).reshape(-1, hkv, d)
    vb = (x @ np.asarray(Wv, dtype=np.float64).reshape(hidden, hkv * d)).reshape(-1, hkv, d)
    if rope_k:
        kb = rope(kb, pos, inv_freq)
    rk = x @ np.asarray(Ak, dtype=np.float64)
    rv = x @ np.asarray(Av, dtype=np.float64)
    return kb, vb, rk, rv


def lora_kv(x, Wk, Wv, Ak, Av, Bk, Bv, pos, inv_freq):
    """The unified (materialised) LoRA projection of Eq.1: K = RoPE(x (W_k + A_k B_k)), V = x (W_v + A_v B_v) per
    kv head (B [Hkv][r][d] = the head's column slice of the up-projection).  Used to pin `project` + the
    attention oracle's split against the plain definition."""
    x = np.asarray(x, dtype=np.float64)
    hidden, hkv, d = np.asarray(Wk).shape
    Wk_full = np.asarray(Wk, np.float64) + np.einsum("hr,krd->hkd", np.asarray(Ak, np.float64), np.asarray(Bk, np.float64))
    Wv_full = np.asarray(Wv, np.float64) + np.einsum("hr,krd->hkd", np.asarray(Av, np.float64), np.asarray(Bv, np.float64))
    k = (x @ Wk_full.reshape(hidden, hkv * d)).reshape(-1, hkv, d)
    v = (x @ Wv_full.reshape(hidden, hkv * d)).reshape(-1, hkv, d)
    return rope(k, pos, inv_freq), v
