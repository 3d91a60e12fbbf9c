"""Pins for the data-plane oracle (oracle/ra.py), against things other than
itself: library routines (torch SDPA in fp64, transformers' Llama RoPE), a
hand-derived worked example (tests/golden), an independent pure-Python brute
force, and invariants the paper fixes.  Any plausible slip in the oracle (a
dropped residual term, wrong RoPE pairing/sign/position, transposed B, wrong
GQA head map, off-by-one causal mask) fails at least one of these."""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import brute, ra

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand_case(rng, L, C, Hq, Hkv, d, r):
    f = lambda *s: rng.standard_normal(s)
    return dict(Kb=f(L, Hkv, d), Vb=f(L, Hkv, d), Rk=f(L, r), Rv=f(L, r),
                Bk=0.3 * f(Hkv, r, d), Bv=0.3 * f(Hkv, r, d), Q=f(C, Hq, d))


def _sdpa(Q, K, V, scale):
    """torch fp64 SDPA with GQA (query head k -> kv head k // g) and the
    causal rule of reading C-6 (query i of C sits at position L - C + i)."""
    C, Hq, d = Q.shape
    L, Hkv, _ = K.shape
    g = Hq // Hkv
    q = torch.tensor(Q).permute(1, 0, 2)                     # [Hq][C][d]
    k = torch.tensor(K).permute(1, 0, 2).repeat_interleave(g, 0)
    v = torch.tensor(V).permute(1, 0, 2).repeat_interleave(g, 0)
    pos_q = torch.arange(L - C, L)[:, None]
    pos_k = torch.arange(L)[None, :]
    mask = pos_k <= pos_q
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, attn_mask=mask, scale=scale)
    return o.permute(1, 0, 2).numpy()


def _rope_hf(x, positions, inv_freq):
    """RoPE via transformers' Llama apply_rotary_pos_emb (rotate_half)."""
    from transformers.models.llama.modeling_llama import apply_rotary_pos_emb
    freqs = torch.tensor(positions, dtype=torch.float64)[:, None] * torch.tensor(inv_freq)[None, :]
    emb = torch.cat([freqs, freqs], -1)
    cos, sin = emb.cos()[None], emb.sin()[None]                          # [1][L][d]
    t = torch.tensor(x)[None]                                             # [1][L][H][d]
    out, _ = apply_rotary_pos_emb(t, t, cos, sin, unsqueeze_dim=2)
    return out[0].numpy()


@pytest.mark.parametrize("mode", [ra.ROPE_NONE, ra.ROPE_DEFERRED])
@pytest.mark.parametrize("zero", ["R", "B"])
def test_zero_residual_is_plain_prefix_attention(mode, zero):
    """P-1: R=0 or B=0 -> plain (paged-prefix) attention,
    checked against torch SDPA in fp64."""
    rng = np.random.default_rng(1)
    c = _rand_case(rng, L=37, C=5, Hq=8, Hkv=2, d=16, r=4)
    if zero == "R":
        c["Rk"][:] = 0; c["Rv"][:] = 0
    else:
        c["Bk"][:] = 0; c["Bv"][:] = 0
    fr = ra.inv_freq(16, 10000.0)
    O = ra.residual_attention(inv_freq_=fr, rope_mode=mode, **c)
    ref = _sdpa(c["Q"], c["Kb"], c["Vb"], 1 / 4.0)
    np.testing.assert_allclose(O, ref, atol=1e-12, rtol=0)


def test_none_mode_is_materialised_attention():
    """NONE mode == SDPA over K = Kb + Rk B_K^h, V = Vb + Rv B_V^h (Eq.2)."""
    rng = np.random.default_rng(2)
    c = _rand_case(rng, L=29, C=3, Hq=6, Hkv=3, d=8, r=3)
    O = ra.residual_attention(inv_freq_=None, rope_mode=ra.ROPE_NONE, **c)
    K = c["Kb"] + np.einsum("tj,hjd->thd", c["Rk"], c["Bk"])
    V = c["Vb"] + np.einsum("tj,hjd->thd", c["Rv"], c["Bv"])
    np.testing.assert_allclose(O, _sdpa(c["Q"], K, V, 1 / math.sqrt(8)), atol=1e-12, rtol=0)


def test_deferred_rope_equals_eager_merged_projection():
    """P-4: storing RoPE(xW) and xA and
    rebuilding RoPE(xA B) inside attention equals RoPE applied to the eagerly
    merged projection xW + xAB (Eq.1), with transformers' Llama RoPE
    (rotate_half pairing + llama3 frequency scaling) as the external rotary."""
    rng = np.random.default_rng(3)
    L, C, Hq, Hkv, d, r, m = 40, 4, 4, 2, 128, 8, 24
    x = rng.standard_normal((L, m))
    W = rng.standard_normal((m, Hkv * d)) / math.sqrt(m)
    Wv = rng.standard_normal((m, Hkv * d)) / math.sqrt(m)
    A = rng.standard_normal((m, r)) / math.sqrt(m)
    Av = rng.standard_normal((m, r)) / math.sqrt(m)
    B = 0.5 * rng.standard_normal((r, Hkv * d))
    Bv = 0.5 * rng.standard_normal((r, Hkv * d))
    Q = rng.standard_normal((C, Hq, d))
    # positions far enough that high-frequency rotations are non-trivial
    pos = np.arange(L) * 97
    fr = ra.inv_freq(d, 500000.0, llama3=True)
    from transformers import LlamaConfig
    from transformers.models.llama.modeling_llama import LlamaRotaryEmbedding
    cfg = LlamaConfig(hidden_size=Hq * d, num_attention_heads=Hq, num_key_value_heads=Hkv, head_dim=d,
                      rope_theta=500000.0, max_position_embeddings=131072,
                      rope_scaling={"rope_type": "llama3", "factor": 8.0, "low_freq_factor": 1.0,
                                    "high_freq_factor": 4.0, "original_max_position_embeddings": 8192})
    hf_inv = LlamaRotaryEmbedding(cfg).inv_freq.double().numpy()
    np.testing.assert_allclose(fr, hf_inv, rtol=1e-6)  # HF builds inv_freq in fp32
    # eager: K = RoPE(xW + xAB) at each token's absolute position
    Kfull = _rope_hf((x @ W + x @ A @ B).reshape(L, Hkv, d), pos, fr)
    Vfull = (x @ Wv + x @ Av @ Bv).reshape(L, Hkv, d)
    # disaggregated: bCache = RoPE(xW), rCache = xA (no RoPE)
    Kb = _rope_hf((x @ W).reshape(L, Hkv, d), pos, fr)
    Bk_h = B.reshape(r, Hkv, d).transpose(1, 0, 2)
    Bv_h = Bv.reshape(r, Hkv, d).transpose(1, 0, 2)
    # the oracle uses position index t; place token t at absolute position
    # pos[t] by expanding into a sparse sequence is not possible, so instead
    # scale inv_freq by 97 (angle = t * 97 * f) -- identical angles.
    O = ra.residual_attention(Kb, (x @ Wv).reshape(L, Hkv, d), x @ A, x @ Av, Bk_h, Bv_h, Q, fr * 97,
                              rope_mode=ra.ROPE_DEFERRED)
    ref = _sdpa(Q, Kfull, Vfull, 1 / math.sqrt(d))
    np.testing.assert_allclose(O, ref, atol=1e-11, rtol=0)
    # and the NONE reading is genuinely different here (C-1)
    On = ra.residual_attention(Kb, (x @ Wv).reshape(L, Hkv, d), x @ A, x @ Av, Bk_h, Bv_h, Q, fr * 97,
                               rope_mode=ra.ROPE_NONE)
    assert np.abs(On - ref).max() > 1e-3


def test_identity_rotation_reduces_deferred_to_none():
    """P-2: with all rotation angles zero, DEFERRED == NONE."""
    rng = np.random.default_rng(4)
    c = _rand_case(rng, L=20, C=2, Hq=4, Hkv=2, d=8, r=2)
    a = ra.residual_attention(inv_freq_=np.zeros(4), rope_mode=ra.ROPE_DEFERRED, **c)
    b = ra.residual_attention(inv_freq_=np.zeros(4), rope_mode=ra.ROPE_NONE, **c)
    np.testing.assert_array_equal(a, b)


def test_golden_hand_example():
    """Worked example in tests/golden/tiny_residual_attention.json."""
    g = json.load(open(os.path.join(GOLDEN, "tiny_residual_attention.json")))
    Q = np.array([[[math.log(3) / math.sqrt(2), 0.0]]])
    arr = {k: np.array(g[k], dtype=np.float64) for k in ("Kb", "Vb", "Rk", "Rv", "Bk", "Bv")}
    fr = np.array([math.pi / 2])
    Od = ra.residual_attention(Q=Q, inv_freq_=fr, rope_mode=ra.ROPE_DEFERRED, **arr)
    On = ra.residual_attention(Q=Q, inv_freq_=fr, rope_mode=ra.ROPE_NONE, **arr)
    np.testing.assert_allclose(Od[0, 0], g["expected_deferred"], atol=1e-14)
    np.testing.assert_allclose(On[0, 0], g["expected_none"], atol=1e-14)


def test_rope_frequency_spec_example():
    """head_dim=2, theta=10000, p=1 -> angle 1 rad."""
    g = json.load(open(os.path.join(GOLDEN, "rope_spec_example.json")))
    fr = ra.inv_freq(g["head_dim"], g["theta"])
    ang = g["p"] * fr[0]
    assert ang == g["angle"]
    assert abs(math.sin(ang) - g["sin"]) < 1e-6 and abs(math.cos(ang) - g["cos"]) < 1e-6


def test_single_key_and_two_key_softmax():
    """P-5: one key -> O is the rebuilt V row; two keys ->
    weights sigma(s0 - s1), sigma(s1 - s0) of the two logits."""
    rng = np.random.default_rng(5)
    c = _rand_case(rng, L=1, C=1, Hq=2, Hkv=1, d=4, r=2)
    O = ra.residual_attention(inv_freq_=ra.inv_freq(4), rope_mode=ra.ROPE_DEFERRED, **c)
    V0 = c["Vb"][0, 0] + c["Rv"][0] @ c["Bv"][0]
    np.testing.assert_allclose(O[0, 0], V0, atol=1e-14)
    np.testing.assert_allclose(O[0, 1], V0, atol=1e-14)
    # two keys: O must be a convex combination of the two rebuilt V rows and
    # equal (V0 + e^{s1-s0} V1)/(1 + e^{s1-s0}) for the lse-derived logits
    c = _rand_case(rng, L=2, C=1, Hq=1, Hkv=1, d=4, r=2)
    c["Bk"][:] = 0  # logits then come only from K_base: s_t = q.Kb_t / 2
    O, lse = ra.residual_attention(inv_freq_=ra.inv_freq(4), rope_mode=ra.ROPE_DEFERRED, return_lse=True, **c)
    s = [float(c["Q"][0, 0] @ c["Kb"][t, 0]) / 2 for t in range(2)]
    V = [c["Vb"][t, 0] + c["Rv"][t] @ c["Bv"][0] for t in range(2)]
    w1 = 1 / (1 + math.exp(s[0] - s[1]))
    np.testing.assert_allclose(O[0, 0], (1 - w1) * V[0] + w1 * V[1], atol=1e-14)
    assert abs(lse[0, 0] - (max(s) + math.log(math.exp(s[0] - max(s)) + math.exp(s[1] - max(s))))) < 1e-14


def test_causality():
    """P-7: output at position p is invariant to keys > p."""
    rng = np.random.default_rng(6)
    c = _rand_case(rng, L=30, C=6, Hq=4, Hkv=2, d=8, r=2)
    fr = ra.inv_freq(8)
    O1 = ra.residual_attention(inv_freq_=fr, **c)
    for k in ("Kb", "Vb"):
        c[k][27:] = rng.standard_normal(c[k][27:].shape) * 100
    for k in ("Rk", "Rv"):
        c[k][27:] = rng.standard_normal(c[k][27:].shape) * 100
    O2 = ra.residual_attention(inv_freq_=fr, **c)
    # query i sits at p = 24 + i; rows i <= 2 (p <= 26) only see keys <= 26
    np.testing.assert_array_equal(O1[:3], O2[:3])
    assert np.abs(O1[3:] - O2[3:]).max() > 1e-3


@pytest.mark.parametrize("seed", range(6))
def test_brute_force_tiny(seed):
    """P-8: pure-Python complex-number brute force on <=3 keys."""
    rng = np.random.default_rng(100 + seed)
    L = 1 + seed % 3
    C = 1 + (seed % L)
    c = _rand_case(rng, L=L, C=C, Hq=4, Hkv=2, d=4, r=2)
    fr = rng.uniform(0.1, 2.0, size=2)
    for mode in (ra.ROPE_NONE, ra.ROPE_DEFERRED):
        O = ra.residual_attention(inv_freq_=fr, rope_mode=mode, **c)
        B = brute.residual_attention(*[c[k].tolist() for k in ("Kb", "Vb", "Rk", "Rv", "Bk", "Bv", "Q")],
                                     inv_freq=fr.tolist(), deferred=(mode == ra.ROPE_DEFERRED))
        np.testing.assert_allclose(O, np.array(B), atol=1e-12)


def test_no_keys_is_an_error():
    """C-6 / S:410: a query row with no attendable keys is an error."""
    with pytest.raises(ra.OracleError) as e:
        ra.residual_attention(np.zeros((0, 1, 2)), np.zeros((0, 1, 2)), np.zeros((0, 1)), np.zeros((0, 1)),
                              np.zeros((1, 1, 2)), np.zeros((1, 1, 2)), np.zeros((1, 1, 2)), None)
    assert e.value.code in (1, 6)


def test_split_form_equals_materialised_form():
    """P-3 / Eq.4 on the value side and the NONE split on the key
    side: softmax(QK^T)(Vb + Rv Bv) = P Vb + (P Rv) Bv; q.(Kb + Rk Bk) =
    q.Kb + (q Bk^T).Rk.  Checked on the oracle's output against a split
    evaluation from its lse (fp64 difference <= 1e-12)."""
    rng = np.random.default_rng(7)
    c = _rand_case(rng, L=33, C=1, Hq=2, Hkv=1, d=8, r=3)
    O, lse = ra.residual_attention(inv_freq_=None, rope_mode=ra.ROPE_NONE, return_lse=True, **c)
    q = c["Q"][0]
    s = (q @ c["Kb"][:, 0].T + (q @ c["Bk"][0].T) @ c["Rk"].T) / math.sqrt(8)   # split K form
    P = np.exp(s - lse[0][:, None])
    O_split = P @ c["Vb"][:, 0] + (P @ c["Rv"]) @ c["Bv"][0]                     # late fusion
    np.testing.assert_allclose(O[0], O_split, atol=1e-12)
