"""ORACLE (test infrastructure): merge of attention outputs computed over disjoint key ranges (§8(f) f4).

Only tests/ and bench.py's cpu_baseline leg may use this module; it shares no code with the CUDA path.
Softmax over a row's keys is invariant to how the keys are blocked (P-6): with per-range outputs
O_p = sum_{t in range p} e^{s_t} V_t / l_p and lse_p = log l_p, the full output is
    O = sum_p e^{lse_p - L} O_p,   L = log sum_p e^{lse_p}
and the late V fusion (Eq.4) is linear in the probabilities, so it commutes with the merge.
A part with no keys has lse = -inf and weight 0.
"""
from __future__ import annotations

import numpy as np


def merge_lse(O_parts, lse_parts):
    """O_parts [G][...][d], lse_parts [G][...] -> (O [...][d], lse [...]) in fp64."""
    O_parts = np.asarray(O_parts, dtype=np.float64)
    lse_parts = np.asarray(lse_parts, dtype=np.float64)
    M = np.max(lse_parts, axis=0)
    Msafe = np.where(np.isfinite(M), M, 0.0)
    w = np.where(np.isfinite(lse_parts), np.exp(lse_parts - Msafe), 0.0)      # [G][...]
    den = w.sum(axis=0)
    O = np.einsum("g...,g...d->...d", w, O_parts) / np.where(den > 0, den, 1.0)[..., None]
    lse = np.where(den > 0, Msafe + np.log(np.where(den > 0, den, 1.0)), -np.inf)
    return O, lse
