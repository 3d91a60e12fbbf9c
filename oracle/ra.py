"""ORACLE (test infrastructure): ctypes front-end of ``ra_oracle.c``.

``residual_attention`` is the plain materialising definition of
ResidualAttention (Alg.1 P:321-353 and Eq.4, reached
exactly up to rounding by the paper's kernel): per (sequence, kv head)
    K[t] = Kb[t] + rho_t(Rk[t] B_K^h),  V[t] = Vb[t] + Rv[t] B_V^h
then textbook softmax attention in fp64.  See ra_oracle.c for the readings.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ra_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

ROPE_NONE = 0
ROPE_DEFERRED = 1


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm", "-lpthread"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_residual_attention.argtypes = [ctypes.c_int] * 7 + [dp] * 8 + [ctypes.c_double, dp, dp, ctypes.c_int]
        lib.oracle_residual_attention.restype = ctypes.c_int
        lib.oracle_inv_freq.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double, dp]
        lib.oracle_inv_freq.restype = None
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def inv_freq(d: int, theta: float = 10000.0, llama3: bool = False, factor: float = 8.0,
             low: float = 1.0, high: float = 4.0, orig: float = 8192.0) -> np.ndarray:
    out = np.zeros(d // 2, dtype=np.float64)
    _load().oracle_inv_freq(d, theta, int(llama3), factor, low, high, orig, _p(out))
    return out


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


def residual_attention(Kb, Vb, Rk, Rv, Bk, Bv, Q, inv_freq_, rope_mode=ROPE_DEFERRED,
                       scale=None, threads=None, return_lse=False):
    """One sequence.

    Kb, Vb: [L][Hkv][d]; Rk, Rv: [L][r]; Bk, Bv: [Hkv][r][d]; Q: [C][Hq][d].
    Returns O [C][Hq][d] float64 (and lse [C][Hq] if return_lse).
    """
    c = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    Kb, Vb, Rk, Rv, Bk, Bv, Q = map(c, (Kb, Vb, Rk, Rv, Bk, Bv, Q))
    L, Hkv, d = Kb.shape
    C, Hq, _ = Q.shape
    r = Rk.shape[1] if Rk.ndim == 2 else 0
    if r == 0:
        Rk = np.zeros((L, 1)); Rv = np.zeros((L, 1))
        Bk = np.zeros((Hkv, 1, d)); Bv = np.zeros((Hkv, 1, d)); r = 1
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    fr = c(inv_freq_ if inv_freq_ is not None else np.zeros(d // 2))
    O = np.zeros((C, Hq, d), dtype=np.float64)
    lse = np.zeros((C, Hq), dtype=np.float64)
    if threads is None:
        threads = min(Hkv, os.cpu_count() or 1)
    st = _load().oracle_residual_attention(L, C, Hq, Hkv, d, r, int(rope_mode), _p(fr), _p(Kb), _p(Vb),
                                           _p(Rk), _p(Rv), _p(Bk), _p(Bv), _p(Q), float(scale), _p(O),
                                           _p(lse), int(threads))
    if st != 0:
        raise OracleError(st)
    return (O, lse) if return_lse else O
