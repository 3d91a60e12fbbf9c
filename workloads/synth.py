"""Seeded, counter-based synthetic input generator (input spec only).

This module is shared by the oracle side (tests, bench cpu_baseline) and the
product side (bench / tests feed its values through the C-ABI). It holds NONE
of the method's arithmetic: it only maps logical coordinates to pseudo-random
numbers. The product library carries a bit-identical CUDA implementation of
the same counter hash (``paper_2604_06370_b200/csrc/synth.cu``) so that
bench-scale pools can be filled on the device; a GPU test checks the two agree
bit for bit.

Definition
-------------------------------------
    splitmix64(x): x += 0x9E3779B97F4A7C15;
                   z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9;
                   z = (z ^ (z >> 27)) * 0x94D049BB133111EB;
                   return z ^ (z >> 31)            (all mod 2^64)
    stream(seed, kind, owner) = splitmix64(splitmix64(seed * 2^8 + kind) ^ owner)
    index(layer, pos, head, col) = (layer << 44) | (pos << 16) | (head << 8) | col
    z = splitmix64(stream + index)
    u = z >> 40                                      (24-bit integer)
    unit = (2u + 1 - 2^24) / 2^24                    (exact fp32, in (-1, 1))
    value = fp32(unit * scale)                       (scale is a power of two)

``kind`` selects the logical tensor (see KIND_*), ``owner`` is the writer of a
base row (the agent that produced the token), the residual owner of a residual
row, the adapter id of an adapter matrix, or the sequence id of a query.
"""
from __future__ import annotations

import numpy as np

KIND_KBASE = 1
KIND_VBASE = 2
KIND_RK = 3
KIND_RV = 4
KIND_BK = 5
KIND_BV = 6
KIND_Q = 7
KIND_TOKEN = 8
# projection producer inputs (§8(f) f2/f3): layer input x [T][hidden] (owner = writer agent, pos = token position,
# head = column >> 8, col = column & 255), the model's K / V projections W [hidden][Hkv][d] (owner 0, pos = hidden
# row) and the adapters' down projections A [hidden][r] (owner = adapter id, pos = hidden row)
KIND_X = 9
KIND_WK = 10
KIND_WV = 11
KIND_AK = 12
KIND_AV = 13

# Scales (powers of two so fp32 scaling is exact). Q is 4x so that logits
# have std ~1.3 at d=128; B is 1/8 so the residual K is ~25-30% of base K
# (SURVEY §8(d) "residual ≈25% of base magnitude").
SCALE = {
    KIND_KBASE: 1.0,
    KIND_VBASE: 1.0,
    KIND_RK: 1.0,
    KIND_RV: 1.0,
    KIND_BK: 0.125,
    KIND_BV: 0.125,
    KIND_Q: 4.0,
    KIND_X: 1.0,
    KIND_WK: 0.03125,   # x W has std ~0.67 at hidden 4096
    KIND_WV: 0.03125,
    KIND_AK: 0.03125,
    KIND_AV: 0.03125,
}

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_C0 = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    """Vectorised splitmix64 over uint64 numpy arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + _C0
        z = (x ^ (x >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def stream(seed: int, kind: int, owner: int) -> np.uint64:
    s = splitmix64(np.uint64((int(seed) * 256 + int(kind)) & 0xFFFFFFFFFFFFFFFF))
    return splitmix64(s ^ np.uint64(int(owner) & 0xFFFFFFFFFFFFFFFF))


def index(layer, pos, head, col):
    layer = np.asarray(layer, dtype=np.uint64)
    pos = np.asarray(pos, dtype=np.uint64)
    head = np.asarray(head, dtype=np.uint64)
    col = np.asarray(col, dtype=np.uint64)
    return (layer << np.uint64(44)) | (pos << np.uint64(16)) | (head << np.uint64(8)) | col


def unit(seed, kind, owner, layer, pos, head, col):
    """fp32 values in (-1, 1) for broadcastable logical coordinates."""
    st = stream(seed, kind, owner)
    with np.errstate(over="ignore"):
        z = splitmix64(st + index(layer, pos, head, col))
    u = (z >> np.uint64(40)).astype(np.int64)
    return ((2 * u + 1 - (1 << 24)).astype(np.float32)) / np.float32(1 << 24)


def values(seed, kind, owner, layer, pos, head, col, scale=None):
    s = SCALE[kind] if scale is None else scale
    return unit(seed, kind, owner, layer, pos, head, col) * np.float32(s)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (round to nearest even) and return as fp32."""
    x = np.asarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    b = (b + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 (already bf16-representable or not) -> uint16 bf16 bits (RNE)."""
    r = round_bf16(x)
    return (r.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def maybe_round(x: np.ndarray, dtype: str) -> np.ndarray:
    return round_bf16(x) if dtype == "bf16" else np.asarray(x, dtype=np.float32)


# ---------------------------------------------------------------------------
# Logical tensors (what an agent's rows contain, independent of paging)
# ---------------------------------------------------------------------------

def base_rows(seed, writer, layer, pos0, n, n_kv, d, kind=KIND_KBASE, dtype="bf16"):
    """[n][n_kv][d] base K (kind=KIND_KBASE, already 'roped' by definition of
    the synthetic workload: the generator emits the stored value) or V."""
    pos = np.arange(pos0, pos0 + n, dtype=np.uint64)[:, None, None]
    head = np.arange(n_kv, dtype=np.uint64)[None, :, None]
    col = np.arange(d, dtype=np.uint64)[None, None, :]
    return maybe_round(values(seed, kind, writer, layer, pos, head, col), dtype)


def base_rows_multi(seed, writers, layer, positions, n_kv, d, kind=KIND_KBASE, dtype="bf16"):
    """Rows for arbitrary (writer, position) pairs: [n][n_kv][d]."""
    writers = np.asarray(writers, dtype=np.uint64)
    positions = np.asarray(positions, dtype=np.uint64)
    out = np.empty((len(positions), n_kv, d), dtype=np.float32)
    for w in np.unique(writers):
        sel = writers == w
        pos = positions[sel][:, None, None]
        head = np.arange(n_kv, dtype=np.uint64)[None, :, None]
        col = np.arange(d, dtype=np.uint64)[None, None, :]
        out[sel] = values(seed, kind, int(w), layer, pos, head, col)
    return maybe_round(out, dtype)


def res_rows(seed, owner, layer, pos0, n, r, kind=KIND_RK, dtype="bf16"):
    """[n][r] residual rows (x A_i, stored without RoPE)."""
    pos = np.arange(pos0, pos0 + n, dtype=np.uint64)[:, None]
    col = np.arange(r, dtype=np.uint64)[None, :]
    return maybe_round(values(seed, kind, owner, layer, pos, 0, col), dtype)


def adapter(seed, adapter_id, layer, n_kv, r, d, kind=KIND_BK, dtype="bf16"):
    """[n_kv][r][d] up-projection slice per kv head (B_K^h or B_V^h)."""
    head = np.arange(n_kv, dtype=np.uint64)[:, None, None]
    j = np.arange(r, dtype=np.uint64)[None, :, None]
    col = np.arange(d, dtype=np.uint64)[None, None, :]
    # fold (head, j) into (head, pos) coordinates: pos = j
    return maybe_round(values(seed, kind, adapter_id, layer, j, head, col), dtype)


def queries(seed, seq, layer, step, n, n_q, d, dtype="bf16"):
    """[n][n_q][d] query rows for a sequence at a given step."""
    pos = (np.uint64(step) * np.uint64(4096) + np.arange(n, dtype=np.uint64))[:, None, None]
    head = np.arange(n_q, dtype=np.uint64)[None, :, None]
    col = np.arange(d, dtype=np.uint64)[None, None, :]
    return maybe_round(values(seed, KIND_Q, seq, layer, pos, head, col), dtype)


def tokens(seed, owner, pos0, n, vocab=128256):
    pos = np.arange(pos0, pos0 + n, dtype=np.uint64)
    st = stream(seed, KIND_TOKEN, owner)
    with np.errstate(over="ignore"):
        z = splitmix64(st + pos)
    return (z % np.uint64(vocab)).astype(np.int32)
