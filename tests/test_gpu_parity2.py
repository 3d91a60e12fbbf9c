"""GPU parity, round 2 (VERDICT r1 "Make parity green"): the 70B head shape, C3 at size, needle / peaked inputs
that stress the lazy rescale and the split combine, the host-buffer entry point, a multi-step decode loop,
and the DEFERRED RoPE-table bound. CUDA path through the C-ABI vs the fp64 oracle on the same seeded inputs;
bf16 max-abs <= 2e-2 (north_star)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import ra  # noqa: E402
from paper_2604_06370_b200 import _lib as L  # noqa: E402
from paper_2604_06370_b200.api import ForkKV  # noqa: E402
from workloads import driver, recipes, synth  # noqa: E402

TOL = 2e-2
THETA, LLAMA3 = 500000.0, True


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ctx(scen, Hq, Hkv, P, mode, L_=1, kv_heads=None, extra_pos=8):
    nb, nr = scen.pages_needed(P)
    max_pos = max(scen.seqlen(s.id) for s in scen.agents) + extra_pos
    return ForkKV(n_layers=L_, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=128, rank=16, page_size=P,
                  n_base_pages=nb + 16, n_res_pages=nr + 16, dtype="bf16", rope_mode=mode, device=0,
                  max_pos=max_pos, rope_theta=THETA, llama3=LLAMA3, kv_heads=kv_heads)


def _oracle(inp, mode):
    fr = ra.inv_freq(128, THETA, llama3=LLAMA3)
    return ra.residual_attention(inv_freq_=fr, rope_mode=ra.ROPE_DEFERRED if mode == "deferred" else ra.ROPE_NONE,
                                 **inp)


def _check(fkv, scen, seed, layer, mode, seqs, Q=None, O=None, h0=0, patch=None, q_scale=1.0, step=0):
    batch = scen.batch()
    C = scen.q_len
    if O is None:
        pl = fkv.plan([(a, C) for a in batch], flags=L.PLAN_CHECK_WRITTEN)
        if Q is None:
            Q = driver.make_queries(fkv, scen, seed, layer, h0=h0, step=step)
        O = fkv.residual_attention(pl, layer, Q)
    torch.cuda.synchronize()
    O = O.float().cpu().numpy()
    worst = 0.0
    for i in seqs:
        a = batch[i]
        inp = recipes.oracle_inputs(scen, seed, a, layer, fkv.hkv, 128, 16, fkv.hq, C, "bf16",
                                    kv_heads=(h0, h0 + fkv.hkv), step=step)
        inp["Q"] = inp["Q"] * q_scale
        if patch:
            patch(a, inp)
        ref = _oracle(inp, mode)
        worst = max(worst, float(np.abs(O[i * C:(i + 1) * C] - ref).max()))
    return worst


# ---- (a) Llama-3.1-70B head shape (64 q / 8 kv heads, g = 8) ------------------------------------------------

@pytest.mark.parametrize("mode", ["none", "deferred"])
@pytest.mark.parametrize("shard", [None, (4, 8), (2, 3)])
def test_70b_shape_g8(mode, shard):
    """configs[3] head shape: g = 8 query heads per kv head, 16 independent agents (distinct adapters) plus a
    same-agent branch pair over a 1.5K shared prefix; whole model and kv-head shards (§8(e))."""
    ag = [recipes.AgentSpec(1000, 1000, None, 0, False, 1500, decode=False)]
    for i in range(16):
        ag.append(recipes.AgentSpec(i, i, 1000, 1500, False, 70 + 3 * i))
    ag.append(recipes.AgentSpec(500, 3, 3, 1500, True, 40))          # a branch sharing agent 3's residual
    scen = recipes.Scenario("70b", ag)
    h0 = shard[0] if shard else 0
    fkv = _ctx(scen, 64, 8, 128, mode, kv_heads=shard)
    driver.build(fkv, scen, seed=70, h0=h0)
    err = _check(fkv, scen, 70, 0, mode, seqs=range(len(scen.batch())), h0=h0)
    assert err <= TOL, err


# ---- (b) C3 at size: one 1024-row chunk per agent over 33-37K keys -------------------------------------------

@pytest.mark.parametrize("mode", ["none", "deferred"])
def test_c3_full_size_sampled_rows(mode):
    """configs[2] at the size bench.py times (8 agents, distinct adapters, 32K shared prefix, 4K private each,
    the last 1024-token chunk as the query rows): every agent, sampled rows of the chunk (first, middle, last)
    against the oracle of that row (a query at position p sees keys [0, p], C-6)."""
    scen = recipes.c3()
    fkv = _ctx(scen, 32, 8, 128, mode)
    driver.build(fkv, scen, seed=3)
    batch = scen.batch()
    C = scen.q_len
    pl = fkv.plan([(a, C) for a in batch], flags=L.PLAN_CHECK_WRITTEN)
    Q = driver.make_queries(fkv, scen, 3, 0)
    O = fkv.residual_attention(pl, 0, Q).float().cpu().numpy()
    worst = 0.0
    for i, a in enumerate(batch):
        Lq = scen.seqlen(a)
        inp = recipes.oracle_inputs(scen, 3, a, 0, 8, 128, 16, 32, C, "bf16")
        for qi in ((0, C // 2, C - 1) if i % 2 == 0 else (1, C - 2)):
            p = Lq - C + qi
            sub = dict(inp, Kb=inp["Kb"][:p + 1], Vb=inp["Vb"][:p + 1], Rk=inp["Rk"][:p + 1],
                       Rv=inp["Rv"][:p + 1], Q=inp["Q"][qi:qi + 1])
            ref = _oracle(sub, mode)
            worst = max(worst, float(np.abs(O[i * C + qi] - ref[0]).max()))
    assert err_ok(worst), worst


def err_ok(e):
    return e <= TOL


# ---- (c) needle / peaked inputs -----------------------------------------------------------------------------

@pytest.mark.parametrize("mode", ["none", "deferred"])
@pytest.mark.parametrize("pieces", [0, 1])
def test_needle_and_peaked_queries(mode, pieces, monkeypatch):
    """SURVEY §8(d) peaked variant: Q x 8 (logits std ~10, so the per-split maxima of different key pieces lie
    far more than 2^8 apart in exp2 units) plus a needle key in the shared prefix aligned with one agent's
    queries (it dominates that agent's softmax). With one-tile pieces (FKV_PIECE_TILES=1) every row merges
    ~20 split partials whose maxima differ wildly: the kernel's lazy rescale and the combine must agree with the
    exact softmax."""
    if pieces:
        monkeypatch.setenv("FKV_PIECE_TILES", "1")
    ag = [recipes.AgentSpec(1000, 1000, None, 0, False, 2500, decode=False)]
    for i in range(2):
        ag.append(recipes.AgentSpec(100 + i, i, 1000, 2500, False, 0, decode=False))
        for b in range(4):
            ag.append(recipes.AgentSpec(10 * i + b, i, 100 + i, 2500, True, 30 + 11 * b))
    ag.append(recipes.AgentSpec(50, 7, 1000, 2500, False, 90))
    scen = recipes.Scenario("needle", ag)
    P = 128
    fkv = _ctx(scen, 32, 8, P, mode)
    driver.build(fkv, scen, seed=9)
    batch = scen.batch()
    # the needle: base K row t* of the shared prefix (all 8 kv heads) = 2 x the mean direction of agent 50's
    # g = 4 query heads of that kv head (bf16-exact values written straight into the page)
    t_star = 1234
    a_n = 50
    Q = driver.make_queries(fkv, scen, 9, 0)
    Q *= 8.0                                              # peaked: exact in bf16 (power of two)
    qn = Q[batch.index(a_n)].float()                      # [32 heads][128]
    needle = torch.stack([qn[4 * h:4 * h + 4].mean(0) for h in range(8)])
    needle = (needle / needle.norm(dim=1, keepdim=True) * 24.0).to(torch.bfloat16)   # [8][128]
    b_tab, _, _ = fkv.get_table(a_n)
    pg = b_tab[t_star // P]
    fkv.base_k[0, pg, :, t_star % P, :] = needle
    torch.cuda.synchronize()
    needle_np = needle.float().cpu().numpy()

    def patch(a, inp):
        inp["Kb"][t_star] = needle_np                    # every agent inherits the root's page

    err = _check(fkv, scen, 9, 0, mode, seqs=range(len(batch)), Q=Q, patch=patch, q_scale=8.0)
    assert err <= TOL, err


# ---- (d) the host-buffer entry point (e2e leg of bench.py) ----------------------------------------------------

@pytest.mark.parametrize("mode", ["none", "deferred"])
def test_host_entry_point(mode):
    """fkv_residual_attention_host: Q from pinned host memory, O back to host memory, through the same plan."""
    scen = recipes.c1(prefix=900, private=50)
    fkv = _ctx(scen, 32, 8, 128, mode)
    driver.build(fkv, scen, seed=4)
    batch = scen.batch()
    pl = fkv.plan([(a, 1) for a in batch], flags=L.PLAN_CHECK_WRITTEN)
    Qd = driver.make_queries(fkv, scen, 4, 0)
    qh = Qd.cpu().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    dq, do = torch.empty_like(Qd), torch.empty_like(Qd)
    fkv.residual_attention_host(pl, 0, qh, oh, dq, do)
    torch.cuda.synchronize()
    err = _check(fkv, scen, 4, 0, mode, seqs=range(len(batch)), O=oh)
    assert err <= TOL, err


@pytest.mark.parametrize("mode", ["none", "deferred"])
def test_split_phases_stage_then_main(mode):
    """FKV_PHASE_STAGE then FKV_PHASE_MAIN | FKV_PHASE_NOSTAGE then FKV_PHASE_COMBINE (the bench's per-kernel
    timing path) gives the oracle's result, bit-identical to the one-call path; bad phase masks are refused."""
    scen = recipes.c1(prefix=900, private=50)
    fkv = _ctx(scen, 32, 8, 128, mode)
    driver.build(fkv, scen, seed=6)
    batch = scen.batch()
    pl = fkv.plan([(a, 1) for a in batch], flags=L.PLAN_CHECK_WRITTEN)
    Q = driver.make_queries(fkv, scen, 6, 0)
    O1 = fkv.residual_attention(pl, 0, Q)
    O2 = torch.empty_like(Q)
    fkv.residual_attention_phases(pl, 0, Q, O2, 4)
    fkv.residual_attention_phases(pl, 0, Q, O2, 1 | 8)
    fkv.residual_attention_phases(pl, 0, Q, O2, 2)
    torch.cuda.synchronize()
    assert torch.equal(O1, O2)
    err = _check(fkv, scen, 6, 0, mode, seqs=range(len(batch)), O=O2)
    assert err <= TOL, err
    for bad in (8, 4 | 1, 4 | 8, 16):
        with pytest.raises(Exception):
            fkv.residual_attention_phases(pl, 0, Q, O2, bad)


# ---- (e) a multi-step decode loop -----------------------------------------------------------------------------

@pytest.mark.parametrize("mode", ["none", "deferred"])
def test_decode_loop_three_steps(mode):
    """bench.py's step, three times: append one token per sequence (the first append of a same-agent branch
    hits a shared partial tail -> CoW), re-plan, write the new rows, attention; checked after every step."""
    ag = [recipes.AgentSpec(1000, 1000, None, 0, False, 700, decode=False)]
    for i in range(3):
        ag.append(recipes.AgentSpec(100 + i, i, 1000, 700, False, 5, decode=False))
        for b in range(3):
            ag.append(recipes.AgentSpec(10 * i + b, i, 100 + i, 705, True, 20 + b))
    scen = recipes.Scenario("loop", ag)
    fkv = _ctx(scen, 32, 8, 64, mode, extra_pos=16)
    driver.build(fkv, scen, seed=12)
    batch = scen.batch()
    for step in range(1, 4):
        pos = [scen.seqlen(a) for a in batch]
        fkv.append(batch, [1] * len(batch), synth.tokens(12, 0, step, len(batch)).tolist())
        for a, p in zip(batch, pos):
            driver.write_rows(fkv, 12, a, a, p, 1, L.WRITE_ALL, 0)
            scen.spec(a).n_private += 1
        err = _check(fkv, scen, 12, 0, mode, seqs=range(len(batch)), step=step)
        assert err <= TOL, (step, err)


# ---- RoPE-table bound ------------------------------------------------------------------------------

def test_deferred_plan_refuses_sequences_past_rope_table():
    scen = recipes.c1(prefix=100, private=20)
    fkv = _ctx(scen, 32, 8, 64, "deferred", extra_pos=0)
    driver.build(fkv, scen, seed=1)
    fkv.plan([(a, 1) for a in scen.batch()])                 # exactly covered: fine
    fkv.append([0], [1], [7])
    with pytest.raises(L.FkvError) as e:
        fkv.plan([(0, 1)])
    assert e.value.code == L.E_INVALID


# ---- §8(f) f4: key-range plans + LSE merge (the cross-GPU sequence split, on one GPU) -------------------------

@pytest.mark.parametrize("mode", ["none", "deferred"])
@pytest.mark.parametrize("G", [2, 3])
def test_sequence_split_range_plans_merge(mode, G):
    """G key-range plans (fkv_plan_create_range) of one batch, attention with lse (fkv_residual_attention_lse),
    fkv_merge_lse of the G partial outputs == the oracle over all keys; decode rows and a chunked-prefill chunk
    (rows whose causal window ends before a range see no key of it: O = 0, lse = -inf in that part)."""
    from paper_2604_06370_b200.api import merge_lse, partition_keys
    ag = [recipes.AgentSpec(1000, 1000, None, 0, False, 2000, decode=False)]
    for i in range(3):
        ag.append(recipes.AgentSpec(i, i, 1000, 2000, False, 60 + 30 * i))
    for C in (1, 90):
        scen = recipes.Scenario("split", ag, q_len=C)
        fkv = _ctx(scen, 32, 8, 64, mode)
        driver.build(fkv, scen, seed=31)
        batch = scen.batch()
        Q = driver.make_queries(fkv, scen, 31, 0)
        Ls = max(scen.seqlen(a) for a in batch)
        Os, ls = [], []
        for r in range(G):
            kb, ke = partition_keys(Ls, G, 64, r)
            pl = fkv.plan([(a, C) for a in batch], key_range=(kb, ke))
            O, lse = fkv.residual_attention_lse(pl, 0, Q)
            Os.append(O)
            ls.append(lse)
        Om = merge_lse(torch.stack(Os), torch.stack(ls))
        err = _check(fkv, scen, 31, 0, mode, seqs=range(len(batch)), O=Om)
        assert err <= TOL, (C, err)


# ---- opt-in ping-pong key warpgroups (FKV_TC_PINGPONG): same parity bar -----------------------

@pytest.mark.parametrize("pieces", [False, True])
def test_pingpong_variant_needle(pieces, monkeypatch):
    """The ping-pong variant (two partial entries per row and item, per-warpgroup running max) on the peaked /
    needle inputs, with one-tile pieces (1-tile items: one warpgroup has no tile and writes l = 0)."""
    monkeypatch.setenv("FKV_TC_PINGPONG", "1")
    test_needle_and_peaked_queries("none", pieces, monkeypatch)


def test_pingpong_variant_decode_loop(monkeypatch):
    monkeypatch.setenv("FKV_TC_PINGPONG", "1")
    test_decode_loop_three_steps("none")


@pytest.mark.parametrize("mode", ["none", "deferred"])
def test_newest_rows_visible_in_bench_order(mode):
    """bench.py's launch order: plan + upload first, then per step the new rows' write_kv and the attention back
    to back on one stream (kv_write -> stager -> main kernel chained by programmatic dependent launch). With a
    one-tile context the main kernel's first K / V loads read the page kv_write has just written: the stager
    must not let the main kernel launch before kv_write completed (a race fixed in session 3)."""
    scen = recipes.c1(prefix=96, private=4)
    fkv = _ctx(scen, 32, 8, 128, mode, extra_pos=24)
    driver.build(fkv, scen, seed=21)
    batch = scen.batch()
    stage = {}
    for step in range(1, 13):
        pos = [scen.seqlen(a) for a in batch]
        fkv.append(batch, [1] * len(batch), synth.tokens(21, 0, step, len(batch)).tolist())
        for a in batch:
            scen.spec(a).n_private += 1
        pl = fkv.plan([(a, 1) for a in batch])               # uploaded before the rows are written
        Q = driver.make_queries(fkv, scen, 21, 0, step=step)
        torch.cuda.synchronize()
        for a, p in zip(batch, pos):
            driver.write_rows(fkv, 21, a, a, p, 1, L.WRITE_ALL, 0, stage=stage)
        O = fkv.residual_attention(pl, 0, Q)
        err = _check(fkv, scen, 21, 0, mode, seqs=range(len(batch)), O=O, step=step)
        assert err <= TOL, (step, err)
