"""Pins for the projection oracle (oracle/project.py, §8(f) f2/f3): library routines and the plain LoRA definition
(Eq.1), not a retyping of its own formulas."""
import cmath

import numpy as np
import pytest
import torch

from oracle import project, ra


def _rng(seed):
    return np.random.default_rng(seed)


def test_rope_matches_hf_llama_rotary():
    """K_base = RoPE(x W_k): the rotation equals transformers' Llama apply_rotary_pos_emb (rotate_half
    convention, llama3-scaled inv_freq)."""
    from transformers.models.llama.modeling_llama import apply_rotary_pos_emb
    d, T, H = 128, 37, 3
    fr = ra.inv_freq(d, 500000.0, llama3=True)
    v = _rng(1).standard_normal((T, H, d))
    pos = np.array([0, 1, 2, 63, 64, 4095, 8191, 8192, 30000] + list(range(100, 128)), dtype=np.int64)
    emb = np.concatenate([pos[:, None] * fr[None, :]] * 2, axis=1)
    cos, sin = torch.tensor(np.cos(emb))[None], torch.tensor(np.sin(emb))[None]       # [1][T][d]
    t = torch.tensor(v)[None]                                                          # [1][T][H][d]
    ref, _ = apply_rotary_pos_emb(t, t, cos, sin, unsqueeze_dim=2)
    np.testing.assert_allclose(project.rope(v, pos, fr), ref[0].numpy(), rtol=0, atol=1e-12)


def test_rope_brute_force_complex():
    """Tiny case by complex numbers: the pair (a_i, b_i) is rotated by e^{i p w_i}."""
    d = 8
    fr = ra.inv_freq(d, 10000.0)
    v = _rng(2).standard_normal((3, 1, d))
    pos = np.array([0, 5, 1234])
    out = project.rope(v, pos, fr)
    for t in range(3):
        for i in range(d // 2):
            z = complex(v[t, 0, i], v[t, 0, i + d // 2]) * cmath.exp(1j * pos[t] * fr[i])
            assert abs(out[t, 0, i] - z.real) < 1e-12 and abs(out[t, 0, i + d // 2] - z.imag) < 1e-12


def test_identity_weights_and_zero_adapter():
    """Special cases: W = I (hidden = d, one kv head) gives K_base = RoPE(x), V_base = x; A = 0 gives zero
    residual planes (C-8 "no adapter")."""
    d = 16
    fr = ra.inv_freq(d, 10000.0)
    x = _rng(3).standard_normal((5, d))
    W = np.eye(d).reshape(d, 1, d)
    A = np.zeros((d, 4))
    pos = np.arange(5) * 7
    kb, vb, rk, rv = project.project(x, W, W, A, A, pos, fr)
    np.testing.assert_allclose(kb, project.rope(x[:, None, :], pos, fr), atol=1e-13)
    np.testing.assert_allclose(vb[:, 0], x, atol=1e-13)
    assert not rk.any() and not rv.any()


@pytest.mark.parametrize("seed", range(4))
def test_disaggregated_cache_attention_equals_unified_lora_attention(seed):
    """Eq.1 vs Eq.2 + deferred RoPE (Alg1.335): caching (RoPE(xW_k), xW_v, xA_k, xA_v) and
    running the attention oracle (DEFERRED) with the adapter's B equals textbook softmax attention over the unified
    LoRA projection K = RoPE(x (W_k + A_k B_k)), V = x (W_v + A_v B_v) (plain numpy, no split)."""
    rng = _rng(10 + seed)
    T, hidden, hkv, g, d, r = 23, 64, 2, 2, 16, 4
    fr = ra.inv_freq(d, 10000.0)
    x = rng.standard_normal((T, hidden))
    Wk, Wv = rng.standard_normal((2, hidden, hkv, d)) / 8
    Ak, Av = rng.standard_normal((2, hidden, r)) / 8
    Bk, Bv = rng.standard_normal((2, hkv, r, d)) / 4
    pos = np.arange(T)
    kb, vb, rk, rv = project.project(x, Wk, Wv, Ak, Av, pos, fr)
    C = 3
    Q = rng.standard_normal((C, hkv * g, d))
    O = ra.residual_attention(kb, vb, rk, rv, Bk, Bv, Q, fr, rope_mode=ra.ROPE_DEFERRED)
    K, V = project.lora_kv(x, Wk, Wv, Ak, Av, Bk, Bv, pos, fr)
    ref = np.zeros_like(O)
    for i in range(C):
        p = T - C + i
        for h in range(hkv * g):
            s = K[: p + 1, h // g] @ Q[i, h] / np.sqrt(d)
            w = np.exp(s - s.max())
            ref[i, h] = (w / w.sum()) @ V[: p + 1, h // g]
    np.testing.assert_allclose(O, ref, atol=1e-11)
