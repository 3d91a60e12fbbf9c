"""GPU parity of the projection producer (§8(f) rows f2, f3) against oracle/project.py, and the end-to-end
chain x -> disaggregated pools -> ResidualAttention against the UNIFIED LoRA definition (Eq.1):
K = RoPE(x (W_k + A_k B_k)), V = x (W_v + A_v B_v), textbook softmax. Includes the second workload of P:300 /
P:304: a forked child recomputes its own residual over the inherited prefix (fresh CoW residual pages, base
rows shared), then runs its chunked prefill over that prefix (a7 at C = the prefix length)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import project, ra  # noqa: E402
from paper_2604_06370_b200 import _lib as L  # noqa: E402
from paper_2604_06370_b200.api import ForkKV, synth_fill  # noqa: E402
from workloads import synth  # noqa: E402

HID, HQ, HKV, D, R, P = 1024, 32, 8, 128, 16, 64
SEED = 17


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _x(owner, pos0, n):
    t = torch.empty(n, HID // 256, 256, dtype=torch.bfloat16, device="cuda")
    synth_fill(t, SEED, synth.KIND_X, owner, 0, pos0, scale=synth.SCALE[synth.KIND_X])
    return t.view(n, HID)


def _host(kind, owner, n_pos, n_head, n_col, pos0=0):
    v = synth.values(SEED, kind, owner, 0, np.arange(pos0, pos0 + n_pos, dtype=np.uint64)[:, None, None],
                     np.arange(n_head, dtype=np.uint64)[None, :, None], np.arange(n_col, dtype=np.uint64)[None, None, :])
    return synth.round_bf16(v)


def _x_host(owner, pos0, n):
    return _host(synth.KIND_X, owner, n, HID // 256, 256, pos0).reshape(n, HID)


def _setup(mode="deferred"):
    fkv = ForkKV(n_layers=1, n_q_heads=HQ, n_kv_heads=HKV, head_dim=D, rank=R, page_size=P, n_base_pages=64,
                 n_res_pages=64, dtype="bf16", rope_mode=mode, device=0, max_pos=1024, rope_theta=500000.0,
                 llama3=True)
    Wk = torch.empty(HID, HKV, D, dtype=torch.bfloat16, device="cuda")
    Wv = torch.empty_like(Wk)
    synth_fill(Wk, SEED, synth.KIND_WK, 0, 0, 0, scale=synth.SCALE[synth.KIND_WK])
    synth_fill(Wv, SEED, synth.KIND_WV, 0, 0, 0, scale=synth.SCALE[synth.KIND_WV])
    host = {"Wk": _host(synth.KIND_WK, 0, HID, HKV, D), "Wv": _host(synth.KIND_WV, 0, HID, HKV, D)}
    for ad in (0, 1):
        Bk = torch.empty(1, HKV, R, D, dtype=torch.bfloat16, device="cuda")
        Bv = torch.empty_like(Bk)
        for h in range(HKV):   # B rows r, head h, cols d (the oracle_inputs recipe)
            synth_fill(Bk[0, h], SEED, synth.KIND_BK, ad, 0, 0, head0=h, scale=synth.SCALE[synth.KIND_BK])
            synth_fill(Bv[0, h], SEED, synth.KIND_BV, ad, 0, 0, head0=h, scale=synth.SCALE[synth.KIND_BV])
        fkv.register_adapter(ad, Bk, Bv)
        Ak = torch.empty(1, HID, R, dtype=torch.bfloat16, device="cuda")
        Av = torch.empty_like(Ak)
        synth_fill(Ak[0], SEED, synth.KIND_AK, ad, 0, 0, scale=synth.SCALE[synth.KIND_AK])
        synth_fill(Av[0], SEED, synth.KIND_AV, ad, 0, 0, scale=synth.SCALE[synth.KIND_AV])
        fkv.register_adapter_down(ad, Ak, Av)
        host[("A", ad)] = (_host(synth.KIND_AK, ad, HID, 1, R)[:, 0], _host(synth.KIND_AV, ad, HID, 1, R)[:, 0])
        host[("B", ad)] = (synth.round_bf16(np.stack([synth.values(
            SEED, synth.KIND_BK, ad, 0, np.arange(R, dtype=np.uint64)[:, None], np.uint64(h),
            np.arange(D, dtype=np.uint64)[None, :]) for h in range(HKV)])), synth.round_bf16(np.stack([synth.values(
                SEED, synth.KIND_BV, ad, 0, np.arange(R, dtype=np.uint64)[:, None], np.uint64(h),
                np.arange(D, dtype=np.uint64)[None, :]) for h in range(HKV)])))
    return fkv, Wk, Wv, host


def _rows(fkv, agent, t0, t1):
    """Gather the cached planes of an agent's rows [t0, t1) from the pools (device -> host, fp32)."""
    b, rr, _ = fkv.get_table(agent)
    out = [[], [], [], []]
    for t in range(t0, t1):
        pg, pgr, o = b[t // P], rr[t // P], t % P
        out[0].append(fkv.base_k[0, pg, :, o].float().cpu().numpy())
        out[1].append(fkv.base_v[0, pg, :, o].float().cpu().numpy())
        out[2].append(fkv.res_k[0, pgr, o].float().cpu().numpy())
        out[3].append(fkv.res_v[0, pgr, o].float().cpu().numpy())
    out = [np.stack(v) for v in out]
    # residual pages are stored in the SW32 operand order (two 8-column halves swapped on rows 4..7 of each 8)
    for j in (2, 3):
        for i, t in enumerate(range(t0, t1)):
            if ((t % P) >> 2) & 1:
                out[j][i] = np.concatenate([out[j][i][8:], out[j][i][:8]])
    return out


def test_projection_producer_and_child_residual_recompute():
    fkv, Wk, Wv, host = _setup()
    fr = ra.inv_freq(D, 500000.0, llama3=True)
    prefix, priv = 300, 40
    # root (adapter 0): its prefix rows from x
    fkv.create_root(0, 0)
    fkv.append([0], [prefix], synth.tokens(SEED, 0, 0, prefix).tolist())
    fkv.project_kv(0, [0], [0], [prefix], _x(0, 0, prefix), Wk, Wv)
    # child (adapter 1) forked over the whole prefix: base pages shared, FRESH residual pages (P:300 Step 2) that
    # it recomputes from the prefix activations with its own adapter, then its private rows
    fkv.fork(0, prefix, 1, 1)
    fkv.project_kv(0, [1], [0], [prefix], _x(0, 0, prefix), mask=L.WRITE_RK | L.WRITE_RV)
    fkv.append([1], [priv], synth.tokens(SEED, 1, prefix, priv).tolist())
    fkv.project_kv(0, [1], [prefix], [priv], _x(1, prefix, priv), Wk, Wv)
    torch.cuda.synchronize()
    # (1) cached planes vs the oracle producer
    xr = _x_host(0, 0, prefix)
    xc = np.concatenate([xr, _x_host(1, prefix, priv)])
    pos_c = np.arange(prefix + priv)
    exp_root = project.project(xr, host["Wk"], host["Wv"], *host[("A", 0)], np.arange(prefix), fr)
    exp_child = project.project(xc, host["Wk"], host["Wv"], *host[("A", 1)], pos_c, fr)
    got_root = _rows(fkv, 0, 0, prefix)
    got_child = _rows(fkv, 1, 0, prefix + priv)
    for got, exp in ((got_root, exp_root), (got_child, exp_child)):
        for g, e in zip(got, exp):
            assert np.abs(g - e).max() <= 2e-2 * max(1.0, np.abs(e).max()), np.abs(g - e).max()
    # the child shares the root's base pages and owns fresh residual pages (CoW)
    b0, r0, _ = fkv.get_table(0)
    b1, r1, _ = fkv.get_table(1)
    assert b1[: prefix // P] == b0[: prefix // P] and not set(r1) & set(r0)
    # (2) attention over the produced pools == unified LoRA attention (Eq.1), for the child's decode row and for
    # its chunked prefill over the inherited prefix (C = 256 query rows of the prefix + its private rows)
    K, V = project.lora_kv(xc, host["Wk"], host["Wv"], *host[("A", 1)], *host[("B", 1)], pos_c, fr)
    for C in (1, 97):
        Q = torch.empty(C, HQ, D, dtype=torch.bfloat16, device="cuda")
        synth_fill(Q, SEED, synth.KIND_Q, 1, 0, 0, scale=synth.SCALE[synth.KIND_Q])
        pl = fkv.plan([(1, C)], flags=L.PLAN_CHECK_WRITTEN)
        O = fkv.residual_attention(pl, 0, Q).float().cpu().numpy()
        Qh = Q.float().cpu().numpy()
        Lq = prefix + priv
        ref = np.zeros((C, HQ, D))
        for i in range(C):
            p = Lq - C + i
            for h in range(HQ):
                s = K[: p + 1, h // (HQ // HKV)] @ Qh[i, h] / np.sqrt(D)
                w = np.exp(s - s.max())
                ref[i, h] = (w / w.sum()) @ V[: p + 1, h // (HQ // HKV)]
        assert np.abs(O - ref).max() <= 2e-2, (C, np.abs(O - ref).max())


def test_partial_hit_recomputes_only_base_rows():
    """P:304 partial hit through the producer: the root's residual survives in its lineage's tree while the base
    tail is evicted; a resumed fork maps the surviving residual, gets fresh base pages for the evicted range, the
    producer recomputes only x W there, and the attention equals the unified definition."""
    fkv, Wk, Wv, host = _setup()
    fr = ra.inv_freq(D, 500000.0, llama3=True)
    n = 256
    toks = synth.tokens(SEED, 0, 0, n).tolist()
    fkv.create_root(0, 0)
    fkv.append([0], [n], toks)
    fkv.project_kv(0, [0], [0], [n], _x(0, 0, n), Wk, Wv)
    torch.cuda.synchronize()
    fkv.release(0)
    assert fkv.evict(L.KIND_BASE, 2) == 2                      # the base tree's two LRU leaves: pages 2, 3
    bh, rh, mapped = fkv.fork_resume(5, 0, 0, toks)
    assert (bh, rh, mapped) == (2 * P, n, n)
    fkv.project_kv(0, [5], [bh], [mapped - bh], _x(0, bh, mapped - bh), Wk, Wv, mask=L.WRITE_KBASE | L.WRITE_VBASE)
    fkv.append([5], [1], [7])
    fkv.project_kv(0, [5], [n], [1], _x(5, n, 1), Wk, Wv)
    torch.cuda.synchronize()
    xs = np.concatenate([_x_host(0, 0, n), _x_host(5, n, 1)])
    K, V = project.lora_kv(xs, host["Wk"], host["Wv"], *host[("A", 0)], *host[("B", 0)], np.arange(n + 1), fr)
    Q = torch.empty(1, HQ, D, dtype=torch.bfloat16, device="cuda")
    synth_fill(Q, SEED, synth.KIND_Q, 5, 0, 0, scale=synth.SCALE[synth.KIND_Q])
    pl = fkv.plan([(5, 1)], flags=L.PLAN_CHECK_WRITTEN)
    O = fkv.residual_attention(pl, 0, Q).float().cpu().numpy()[0]
    Qh = Q.float().cpu().numpy()[0]
    ref = np.zeros((HQ, D))
    for h in range(HQ):
        s = K[:, h // (HQ // HKV)] @ Qh[h] / np.sqrt(D)
        w = np.exp(s - s.max())
        ref[h] = (w / w.sum()) @ V[:, h // (HQ // HKV)]
    assert np.abs(O - ref).max() <= 2e-2, np.abs(O - ref).max()
