"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle on the
same seeded inputs. bf16 inputs / fp32 accumulate: max-abs <= 2e-2; fp32
path: max-abs <= 1e-5 (north_star tolerances)."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import ra  # noqa: E402
from paper_2604_06370_b200 import _lib as L  # noqa: E402
from paper_2604_06370_b200.api import ForkKV, synth_fill  # noqa: E402
from workloads import driver, recipes, synth  # noqa: E402

TOL = {"bf16": 2e-2, "f32": 1e-5}


def _tc_kernel(mode):
    """Default tcgen05 kernel id: 2 = keys on the TMEM lanes (ra_tc.cu, both modes); 3 = rows on the TMEM lanes
    (ra_rows.cu, NONE mode) when FKV_KERNEL=3 / FKV_PLAN_ROWS_KERNEL selects it."""
    import os
    return 3 if (mode == "none" and os.environ.get("FKV_KERNEL") == "3") else 2


@pytest.fixture(params=["default", "rows"])
def kernel_choice(request, monkeypatch):
    """Runs a NONE-mode test on both tcgen05 kernels (the default keys-on-lanes one and the rows-on-lanes one)."""
    if request.param == "rows":
        monkeypatch.setenv("FKV_KERNEL", "3")
    return request.param


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ctx(scen, L_, Hq, Hkv, d, r, P, dtype, mode, theta=10000.0, llama3=False, kv_heads=None):
    nb, nr = scen.pages_needed(P)
    max_pos = max(scen.seqlen(s.id) for s in scen.agents) + 1
    return ForkKV(n_layers=L_, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, rank=r, page_size=P, n_base_pages=nb,
                  n_res_pages=nr, dtype=dtype, rope_mode=mode, device=0, max_pos=max_pos, rope_theta=theta,
                  llama3=llama3, kv_heads=kv_heads)


def _run_and_check(fkv, scen, seed, layer, dtype, mode, flags=0, theta=10000.0, llama3=False, seqs=None, h0=0):
    batch = scen.batch()
    C = scen.q_len
    pl = fkv.plan([(a, C) for a in batch], flags=flags)
    Q = driver.make_queries(fkv, scen, seed, layer, h0=h0)
    O = fkv.residual_attention(pl, layer, Q)
    torch.cuda.synchronize()
    O = O.float().cpu().numpy()
    fr = ra.inv_freq(fkv.d, theta, llama3=llama3)
    worst = 0.0
    idx = range(len(batch)) if seqs is None else seqs
    for i in idx:
        a = batch[i]
        inp = recipes.oracle_inputs(scen, seed, a, layer, fkv.hkv, fkv.d, fkv.r, fkv.hq, C, dtype,
                                    kv_heads=(h0, h0 + fkv.hkv))
        ref = ra.residual_attention(inv_freq_=fr, rope_mode=ra.ROPE_DEFERRED if mode == "deferred" else ra.ROPE_NONE,
                                    **inp)
        err = np.abs(O[i * C:(i + 1) * C] - ref).max()
        worst = max(worst, err)
    return worst, pl


def test_device_synth_matches_host_generator():
    for dt, tdt in (("bf16", torch.bfloat16), ("f32", torch.float32)):
        t = torch.empty(37, 3, 40, dtype=tdt, device="cuda")
        synth_fill(t, 7, synth.KIND_KBASE, 123, 5, 1000, head0=2)
        host = synth.maybe_round(synth.values(7, synth.KIND_KBASE, 123, 5,
                                              np.arange(1000, 1037, dtype=np.uint64)[:, None, None],
                                              np.arange(2, 5, dtype=np.uint64)[None, :, None],
                                              np.arange(40, dtype=np.uint64)[None, None, :]), dt)
        np.testing.assert_array_equal(t.float().cpu().numpy(), host)


@pytest.mark.parametrize("mode", ["deferred", "none"])
@pytest.mark.parametrize("kernel", ["tc", "rows", "tc128", "mma", "simt"])
def test_c1_parity(mode, kernel, monkeypatch):
    """configs[0] (C1): 1 layer Llama-3.1-8B shape, r=16, 4 agents forked from a
    2K-token prefix + 128 private + 1 decode token; llama3 RoPE, theta 5e5."""
    expect = None
    if kernel == "rows":
        if mode == "deferred":
            pytest.skip("the rows-on-lanes kernel is NONE-mode only")
        monkeypatch.setenv("FKV_KERNEL", "3")
        kernel, expect = "tc", 3
    if kernel == "tc128":
        if mode == "deferred":
            pytest.skip("the 128-row variant is NONE-mode only")
        monkeypatch.setenv("FKV_TC_ROWS", "128")
        kernel, expect = "tc", 2
    scen = recipes.c1()
    fkv = _ctx(scen, 1, 32, 8, 128, 16, 64, "bf16", mode, theta=500000.0, llama3=True)
    driver.build(fkv, scen, seed=0)
    force = {"tc": 0, "mma": L.PLAN_FORCE_MMA, "simt": L.PLAN_FORCE_SIMT}[kernel]
    err, pl = _run_and_check(fkv, scen, 0, 0, "bf16", mode, flags=L.PLAN_CHECK_WRITTEN | force, theta=500000.0,
                             llama3=True)
    assert pl.info.kernel == (expect or {"tc": _tc_kernel(mode), "mma": 0, "simt": 1}[kernel])
    assert err <= TOL["bf16"], err


@pytest.mark.parametrize("mode,variant", [("deferred", 64), ("none", "rows"), ("none", 64), ("none", 128)])
@pytest.mark.parametrize("P", [16, 32, 64, 128])
def test_tc_kernel_page_sizes_and_groups(mode, variant, P, monkeypatch):
    """tcgen05 kernel: page sizes 16/32/64 (TMA box = one page), owner groups
    with several slots (same-agent branches: 4 branches x g=4 rows = one slot;
    a chunked-prefill owner spanning several slots), key ranges ending inside
    a page, and multi-tile split items; 64-row CTAs and (NONE) the 128-row
    variant (8 slots, row sums reduced on the CUDA cores)."""
    if variant != "rows":
        monkeypatch.setenv("FKV_TC_ROWS", str(variant))
    else:
        monkeypatch.setenv("FKV_KERNEL", "3")
    ag = [recipes.AgentSpec(100, 100, None, 0, False, 700, decode=False)]
    for i in range(3):
        ag.append(recipes.AgentSpec(1000 + i, i, 100, 700, False, 0, decode=False))
        for b in range(4):
            ag.append(recipes.AgentSpec(10 * i + b, i, 1000 + i, 700, True, 30 + 7 * b))
    scen = recipes.Scenario("tcgroups", ag, q_len=1)
    fkv = _ctx(scen, 1, 32, 8, 128, 16, P, "bf16", mode)
    driver.build(fkv, scen, seed=11)
    err, pl = _run_and_check(fkv, scen, 11, 0, "bf16", mode)
    assert pl.info.kernel == (3 if variant == "rows" else 2)
    assert err <= TOL["bf16"], err
    scen.q_len = 9   # multi-row chunk per sequence: slots of one owner span several warps
    err, pl = _run_and_check(fkv, scen, 11, 0, "bf16", mode)
    assert err <= TOL["bf16"], err


def _random_scenario(rnd, P, max_prefix=300):
    prefix = rnd.randint(1, max_prefix)
    ag = [recipes.AgentSpec(500, 50, None, 0, False, prefix, decode=rnd.random() < 0.5)]
    nxt = 0
    for _ in range(rnd.randint(1, 6)):
        par = rnd.choice(ag)
        Lp = par.fork_len + par.n_private
        fl = rnd.randint(1, Lp)
        share = rnd.random() < 0.35
        ad = par.adapter if share else rnd.randint(0, 4)
        ag.append(recipes.AgentSpec(nxt, ad, par.id, fl, share, rnd.randint(1, 80)))
        nxt += 1
    q = rnd.choice([1, 1, 1, 3, 17])
    q = min([q] + [a.fork_len + a.n_private for a in ag if a.decode])
    return recipes.Scenario("rand", ag, q_len=q)


@pytest.mark.parametrize("seed", range(1, 121))
def test_random_suite(seed, monkeypatch):
    """Random fork trees (unaligned forks -> CoW tail pages, same-agent
    branches sharing residual pages, chunked-prefill query rows), both RoPE
    modes, bf16 tensor-core path and fp32 SIMT path, page sizes 16/64/128,
    head shapes 8/2, 32/8 (8B) and 64/8 (70B, g = 8)."""
    rnd = random.Random(seed)
    P = rnd.choice([16, 64, 128])
    mode = rnd.choice(["deferred", "none"])
    dtype = "f32" if seed % 4 == 0 else "bf16"
    d = 64 if (dtype == "f32" and seed % 8 == 0) else 128
    hq, hkv = (8, 2) if dtype == "f32" else rnd.choice([(8, 2), (32, 8), (64, 8)])
    scen = _random_scenario(rnd, P)
    if seed % 2 == 1:
        monkeypatch.setenv("FKV_KERNEL", "3")   # NONE-mode seeds alternate between the two tcgen05 kernels
    fkv = _ctx(scen, 2, hq, hkv, d, 16, P, dtype, mode)
    driver.build(fkv, scen, seed=seed)
    for layer in (0, 1):
        err, pl = _run_and_check(fkv, scen, seed, layer, dtype, mode, flags=L.PLAN_CHECK_WRITTEN)
        assert err <= TOL[dtype], (layer, err, pl.info.kernel)


def test_cow_never_mutates_parent_pages():
    """P-11: after an unaligned fork, child appends/writes never change the
    bytes of any page the parent still maps."""
    scen = recipes.Scenario("cow", [recipes.AgentSpec(9, 9, None, 0, False, 150),
                                     recipes.AgentSpec(1, 9, 9, 100, True, 0, decode=False)])
    fkv = _ctx(scen, 2, 8, 2, 128, 16, 16, "bf16", "deferred")
    driver.build(fkv, scen, seed=3)
    b9, r9, _ = fkv.get_table(9)
    snap = [(fkv.base_k[:, b9].clone(), fkv.base_v[:, b9].clone(), fkv.res_k[:, r9].clone(), fkv.res_v[:, r9].clone())]
    toks = synth.tokens(3, 1, 100, 40).tolist()
    fkv.append([1], [40], toks)
    assert len(fkv.take_copy_log()) == 2          # base + residual tail page copied
    driver.write_rows(fkv, 3, 1, 1, 100, 40, L.WRITE_ALL, 0)
    torch.cuda.synchronize()
    now = (fkv.base_k[:, b9], fkv.base_v[:, b9], fkv.res_k[:, r9], fkv.res_v[:, r9])
    for a, b in zip(snap[0], now):
        assert torch.equal(a, b)
    # the child's copied rows [96, 100) equal the parent's rows in that page
    b1, r1, _ = fkv.get_table(1)
    assert torch.equal(fkv.base_k[:, b1[6], :, :4], fkv.base_k[:, b9[6], :, :4])
    # and its attention output matches the oracle
    scen.agents[1].n_private = 40
    scen.agents[1].decode = True
    scen.agents[0].decode = False
    err, _ = _run_and_check(fkv, scen, 3, 1, "bf16", "deferred")
    assert err <= TOL["bf16"]


def test_stale_plan_rejected():
    scen = recipes.c1(prefix=64, private=10)
    fkv = _ctx(scen, 1, 8, 2, 128, 16, 16, "bf16", "deferred")
    driver.build(fkv, scen, seed=1)
    pl = fkv.plan([(a, 1) for a in scen.batch()])
    fkv.append([0], [1], [5])
    Q = driver.make_queries(fkv, scen, 1, 0)
    with pytest.raises(L.FkvError) as e:
        fkv.residual_attention(pl, 0, Q)
    assert e.value.code == L.E_STALE


def test_prefill_chunk_parity():
    """Chunked prefill (a7): 3 agents with distinct adapters over a shared
    prefix, the last 200-token chunk of each private context."""
    ag = [recipes.AgentSpec(100, 100, None, 0, False, 700, decode=False)]
    for i in range(3):
        ag.append(recipes.AgentSpec(i, i, 100, 700, False, 300))
    scen = recipes.Scenario("prefill", ag, q_len=200)
    for mode in ("deferred", "none"):
        fkv = _ctx(scen, 1, 32, 8, 128, 16, 64, "bf16", mode)
        driver.build(fkv, scen, seed=5)
        err, pl = _run_and_check(fkv, scen, 5, 0, "bf16", mode)
        assert err <= TOL["bf16"], err


@pytest.mark.parametrize("mode", ["deferred", "none"])
def test_kv_head_shard_parity(mode):
    """§8(e) head sharding: a ctx holding kv heads [4, 8) only (pools, adapters
    and Q/O restricted to its heads) matches the oracle for those heads."""
    scen = recipes.c1(prefix=300, private=40)
    fkv = _ctx(scen, 1, 32, 8, 128, 16, 128, "bf16", mode, kv_heads=(4, 8))
    driver.build(fkv, scen, seed=21, h0=4)
    err, pl = _run_and_check(fkv, scen, 21, 0, "bf16", mode, h0=4)
    assert pl.info.kernel == _tc_kernel(mode)
    assert err <= TOL["bf16"], err


@pytest.mark.parametrize("mode", ["none", "deferred"])
def test_many_splits_combine(mode, monkeypatch, kernel_choice):
    """One-tile key-range pieces (FKV_PIECE_TILES=1) over a ~5K-key shared prefix: every output row merges
    ~40 split partials, which exercises the combine kernel's multi-batch (> 32 entries) path and items that
    share their staged Q / q~ images."""
    monkeypatch.setenv("FKV_PIECE_TILES", "1")
    ag = [recipes.AgentSpec(100, 100, None, 0, False, 5000, decode=False)]
    for i in range(2):
        ag.append(recipes.AgentSpec(1000 + i, i, 100, 5000, False, 0, decode=False))
        for b in range(2):
            ag.append(recipes.AgentSpec(10 * i + b, i, 1000 + i, 5000, True, 40 + 9 * b))
    scen = recipes.Scenario("manysplits", ag, q_len=1)
    fkv = _ctx(scen, 1, 32, 8, 128, 16, 128, "bf16", mode)
    driver.build(fkv, scen, seed=5)
    err, pl = _run_and_check(fkv, scen, 5, 0, "bf16", mode)
    assert pl.info.kernel == _tc_kernel(mode)
    assert pl.info.n_items > 8 * 39, pl.info.n_items
    assert err <= TOL["bf16"], err


@pytest.mark.parametrize("mode", ["none", "deferred"])
def test_c2_full_size_sampled(mode, kernel_choice):
    """Both tcgen05 kernels in NONE mode (kernel_choice). configs[1] at full size (32K shared prefix, 16 agents x 4 branches = 64 decode sequences, 32 q / 8 kv
    heads, d 128, r 16, page 128): one layer of exactly the launch configuration bench.py times (same plan,
    schedule and kernel variant), sampled sequences of every agent group against the fp64 oracle."""
    scen = recipes.c2()
    fkv = _ctx(scen, 1, 32, 8, 128, 16, 128, "bf16", mode, theta=500000.0, llama3=True)
    driver.build(fkv, scen, seed=0)
    err, pl = _run_and_check(fkv, scen, 0, 0, "bf16", mode, theta=500000.0, llama3=True, seqs=[0, 21, 42, 63])
    assert pl.info.kernel == _tc_kernel(mode) and pl.info.n_items > 148
    assert err <= TOL["bf16"], err
