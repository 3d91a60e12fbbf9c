"""ORACLE (test infrastructure): pure-Python scalar brute force, tiny inputs.

An independent second formulation of the same definition (Eq.2
P:130-132, deferred RoPE P:134/Alg.1): the rotation is
written with Python complex numbers (z_i = x_i + i x_{i+d/2}, rotated by
e^{i t f_i}) instead of the cos/sin pairs of ra_oracle.c, and the softmax is
the two-pass textbook form over Python floats.  Use only for <= a few keys.
"""
from __future__ import annotations

import cmath
import math


def rope_complex(x, t, inv_freq):
    """NeoX half-split RoPE of a list x at absolute position t (reading C-2)."""
    d = len(x)
    h = d // 2
    out = [0.0] * d
    for i in range(h):
        z = complex(x[i], x[i + h]) * cmath.exp(1j * t * inv_freq[i])
        out[i] = z.real
        out[i + h] = z.imag
    return out


def residual_attention(Kb, Vb, Rk, Rv, Bk, Bv, Q, inv_freq, deferred=True, scale=None):
    """Nested-list inputs: Kb/Vb [L][Hkv][d], Rk/Rv [L][r], Bk/Bv [Hkv][r][d],
    Q [C][Hq][d]. Returns O [C][Hq][d] as nested lists of floats."""
    L = len(Kb)
    Hkv = len(Kb[0])
    d = len(Kb[0][0])
    r = len(Rk[0]) if L else 0
    C = len(Q)
    Hq = len(Q[0])
    g = Hq // Hkv
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    O = [[[0.0] * d for _ in range(Hq)] for _ in range(C)]
    for k in range(Hq):
        h = k // g
        Ks, Vs = [], []
        for t in range(L):
            u = [sum(Rk[t][j] * Bk[h][j][e] for j in range(r)) for e in range(d)]
            if deferred:
                u = rope_complex(u, t, inv_freq)
            Ks.append([Kb[t][h][e] + u[e] for e in range(d)])
            w = [sum(Rv[t][j] * Bv[h][j][e] for j in range(r)) for e in range(d)]
            Vs.append([Vb[t][h][e] + w[e] for e in range(d)])
        for i in range(C):
            p = L - C + i
            s = [scale * sum(Q[i][k][e] * Ks[t][e] for e in range(d)) for t in range(p + 1)]
            m = max(s)
            w = [math.exp(x - m) for x in s]
            tot = sum(w)
            for e in range(d):
                O[i][k][e] = sum(w[t] * Vs[t][e] for t in range(p + 1)) / tot
    return O
