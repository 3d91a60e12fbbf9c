"""Control-plane parity: the C-ABI library (host-only ctx) against the
control-plane oracle, bit-exact (block tables, refcounts, free-set order,
radix-tree dumps, CoW copy log, status codes) over random API sequences.
Runs on CPU (no GPU needed: fkv_config.device = -1)."""
import random

import pytest

from oracle import control as cp
from paper_2604_06370_b200 import _lib as L
from paper_2604_06370_b200.api import FkvError, ForkKV


def _lib_ctx(P, nb, nr, seed=0, L_=2):
    return ForkKV(n_layers=L_, n_q_heads=4, n_kv_heads=2, head_dim=8, rank=4, page_size=P, n_base_pages=nb,
                  n_res_pages=nr, dtype="f32", device=None, alloc_order_seed=seed)


def _sections(dump):
    """(agent tables, base pool + tree, residual pool + forest) of a dump."""
    lines = dump.splitlines()
    return ("\n".join(l for l in lines if l.startswith("agent ")),
            "\n".join(l for l in lines if l.startswith("base_")) + dump.split("base_tree")[1].split("res_forest")[0],
            "\n".join(l for l in lines if l.startswith("res_")) + dump.split("res_forest")[1])


def _st(fn, *a):
    try:
        r = fn(*a)
        return 0, r
    except FkvError as e:
        return e.code, None


def test_abi_exports_every_declared_symbol():
    """Every function declared in include/forkkv.h is exported by the .so."""
    import re, os
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "forkkv.h")).read()
    names = set(re.findall(r"^\s*(?:fkv_status|const char\*)\s+(fkv_\w+)\s*\(", hdr, re.M))
    lib = L.load()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
        assert n in L.SIGNATURES, n
    assert lib.fkv_version().startswith(b"forkkv-b200")


def test_dump_matches_oracle_simple():
    o = cp.ControlPlane(4, 32, 32)
    m = _lib_ctx(4, 32, 32)
    for obj in (o,):
        obj.create_root(0, 3)
        obj.append([0], [10], list(range(10)))
        obj.fork(0, 6, 1, 5)
        obj.fork(0, 10, 2, 3, cp.FORK_SHARE_RESIDUAL)
        obj.append([1, 2], [3, 2], [7, 8, 9, 1, 2])
    m.create_root(0, 3)
    m.append([0], [10], list(range(10)))
    m.fork(0, 6, 1, 5)
    m.fork(0, 10, 2, 3, L.FORK_SHARE_RESIDUAL)
    m.append([1, 2], [3, 2], [7, 8, 9, 1, 2])
    assert m.dump() == o.dump()
    assert m.take_copy_log() == o.copies


@pytest.mark.parametrize("seed", range(40))
def test_random_sequences_bit_exact(seed):
    rnd = random.Random(1000 + seed)
    P = rnd.choice([2, 4, 8, 16])
    nb, nr = rnd.randint(8, 48), rnd.randint(8, 64)
    aseed = rnd.choice([0, 0, 12345])
    o = cp.ControlPlane(P, nb, nr, alloc_order_seed=aseed)
    m = _lib_ctx(P, nb, nr, seed=aseed)
    nxt = 0
    for step in range(150):
        live = sorted(o.agents)
        x = rnd.random()
        if x < 0.12 or not live:
            a, ad = (nxt if rnd.random() < 0.95 else (live[0] if live else -1)), rnd.randrange(3)
            so = o.create_root(a, ad)
            sm, _ = _st(m.create_root, a, ad)
            nxt += 1
        elif x < 0.32:
            p = rnd.choice(live + [9999])
            Lp = o.agents[p].seqlen if p in o.agents else 3
            pl = rnd.randint(0, Lp + (1 if rnd.random() < 0.1 else 0))
            share = rnd.random() < 0.4
            ad = o.agents[p].adapter if (share and p in o.agents and rnd.random() < 0.9) else rnd.randrange(3)
            fl = cp.FORK_SHARE_RESIDUAL if share else 0
            so = o.fork(p, pl, nxt, ad, fl)
            sm, _ = _st(m.fork, p, pl, nxt, ad, fl)
            nxt += 1
        elif x < 0.42:
            toks = [rnd.randrange(3) for _ in range(rnd.randint(0, 3 * P))]
            ad = rnd.randrange(3)
            so, mo = o.fork_tokens(nxt, ad, toks)
            sm, mm = _st(m.fork_tokens, nxt, ad, toks)
            if so == 0:
                assert mm == mo
            nxt += 1
        elif x < 0.80:
            ags = rnd.sample(live, rnd.randint(1, min(3, len(live))))
            if rnd.random() < 0.05:
                ags = ags + [777777]
            ns = [rnd.randint(0, 2 * P) for _ in ags]
            toks = [rnd.randrange(3) for _ in range(sum(ns))]
            so = o.append(ags, ns, toks)
            sm, _ = _st(m.append, ags, ns, toks)
        elif x < 0.90:
            a = rnd.choice(live)
            s = rnd.randint(0, o.agents[a].seqlen)
            c = rnd.randint(0, o.agents[a].seqlen - s + (1 if rnd.random() < 0.1 else 0))
            mask = rnd.choice([15, 3, 12, 1])
            so = o.check_write([a], [s], [c], mask)
            sm, _ = _st(m.write_kv, 0, [a], [s], [c], None, None, None, None, mask)
        else:
            a = rnd.choice(live + [424242])
            so = o.release(a)
            sm, _ = _st(m.release, a)
        assert so == sm, (step, so, sm)
        assert m.dump() == o.dump(), step
        assert m.take_copy_log() == o.copies, step
        o.copies.clear()
        o.check_invariants()
    for a in o.agents:
        b, r, sl = m.get_table(a)
        assert (b, r, sl) == (o.agents[a].base, o.agents[a].res, o.agents[a].seqlen)
        assert m.get_agent(a) == (o.agents[a].adapter, o.agents[a].owner)


def test_plan_errors_host_only():
    m = _lib_ctx(4, 32, 32)
    m.create_root(0, 1)
    m.append([0], [5], list(range(5)))
    with pytest.raises(FkvError) as e:
        m.plan([(0, 1)], upload=False)
    assert e.value.code == L.E_INVALID           # adapter not registered
    m.register_adapter(1)
    with pytest.raises(FkvError) as e:
        m.plan([(0, 6)], upload=False)
    assert e.value.code == L.E_NO_KEYS
    with pytest.raises(FkvError) as e:
        m.plan([(0, 1)], flags=L.PLAN_CHECK_WRITTEN, upload=False)
    assert e.value.code == L.E_UNWRITTEN
    for layer in range(2):
        m.write_kv(layer, [0], [0], [5])
    pl = m.plan([(0, 1)], flags=L.PLAN_CHECK_WRITTEN, upload=False)
    assert pl.info.n_rows == 1 and pl.info.n_entries >= 2
    with pytest.raises(FkvError) as e:
        m.plan([(12, 1)], upload=False)
    assert e.value.code == L.E_UNKNOWN_AGENT


def test_plan_groups_shared_prefix():
    """Agents forked from one prefix form ONE shared segment whose base tile is
    read once for all their rows (the grouping of §8(a) a4)."""
    P, s = 16, 256
    m = ForkKV(n_layers=1, n_q_heads=32, n_kv_heads=8, head_dim=128, rank=16, page_size=P, n_base_pages=256,
               n_res_pages=512, device=None)
    m.register_adapter(0)
    m.create_root(0, 0)
    m.append([0], [s], list(range(s)))
    for a in range(1, 5):
        m.register_adapter(a)
        m.fork(0, s, a, a)
        m.append([a], [20], [a] * 20)
    pl = m.plan([(a, 1) for a in range(1, 5)], upload=False)
    # 1 shared segment + 4 private ones
    assert pl.info.n_segments == 5
    # algorithmic bytes: shared base once + 4 private bases + 4 residuals + adapters + Q/O
    el = 2
    shared = s * 8 * 128 * 2 * el
    private = 4 * 20 * 8 * 128 * 2 * el
    res = 4 * (s + 20) * 16 * 2 * el
    ad = 4 * 2 * 16 * 128 * 8 * el
    qo = 4 * 32 * 128 * 2 * el
    assert pl.info.alg_bytes == shared + private + res + ad + qo
    # the rank-proportional part (residual pages + adapters): what a rank r' < r adapter padded into the pool
    # scales by r'/r (bench.py alg_bytes_of, C-8)
    assert pl.info.alg_rank_bytes == res + ad


def test_partitioner():
    """§8(e): C4 shape at G=8 -> 2 kv-head shards x 4 agent shards."""
    from paper_2604_06370_b200.api import partition, partition_shard
    base = 131072 * 8 * 128 * 2 * 2          # shared base per layer
    res = 128 * 131072 * 16 * 2 * 2          # 128 agents' residual per layer
    assert partition(8, 8, base, res) == (2, 4)
    assert partition(1, 8, base, res) == (1, 1)
    seen = set()
    for rk in range(8):
        (h0, h1), (a0, a1) = partition_shard(rk, 2, 4, 8, 128)
        assert h1 - h0 == 4 and a1 - a0 == 32
        seen.add((h0, a0))
    assert len(seen) == 8


@pytest.mark.parametrize("seed", range(200))
def test_eviction_partial_hit_bit_exact(seed):
    """R10-R12 (decoupled eviction + partial hit): library vs oracle,
    bit-exact dumps (LRU clocks, insertion numbers, free-set order), status
    codes, evicted counts and partial-hit ranges over random scenarios, plus
    the decoupling property on the library itself (SPEC acceptance #7)."""
    rnd = random.Random(31000 + seed)
    P = rnd.choice([2, 4, 8])
    nb, nr = rnd.randint(12, 40), rnd.randint(12, 48)
    aseed = rnd.choice([0, 777])
    o = cp.ControlPlane(P, nb, nr, alloc_order_seed=aseed)
    m = _lib_ctx(P, nb, nr, seed=aseed)
    nxt = 0
    vocab = rnd.choice([2, 3])
    for step in range(80):
        live = sorted(o.agents)
        x = rnd.random()
        if x < 0.15 or not live:
            a, ad = nxt, rnd.randrange(3)
            so, (sm, _) = o.create_root(a, ad), _st(m.create_root, a, ad)
            nxt += 1
        elif x < 0.45:
            ags = rnd.sample(live, rnd.randint(1, min(2, len(live))))
            ns = [rnd.randint(0, 2 * P) for _ in ags]
            toks = [rnd.randrange(vocab) for _ in range(sum(ns))]
            so, (sm, _) = o.append(ags, ns, toks), _st(m.append, ags, ns, toks)
        elif x < 0.57:
            a = rnd.choice(live)
            so, (sm, _) = o.release(a), _st(m.release, a)
        elif x < 0.72:
            toks = [rnd.randrange(vocab) for _ in range(rnd.randint(0, 4 * P))]
            owner = rnd.choice([nxt] + sorted(o.res_roots) + live[:1])
            ad = o.res_adapter.get(owner, rnd.randrange(3)) if rnd.random() < 0.9 else rnd.randrange(3)
            so, ro = o.fork_resume(nxt, ad, owner, toks)
            sm, rm = _st(m.fork_resume, nxt, ad, owner, toks)
            if so == 0:
                assert rm == ro, (step, rm, ro)
            nxt += 1
        elif x < 0.77:
            toks = [rnd.randrange(vocab) for _ in range(rnd.randint(0, 3 * P))]
            ad = rnd.randrange(3)
            so, mo = o.fork_tokens(nxt, ad, toks)
            sm, mm = _st(m.fork_tokens, nxt, ad, toks)
            if so == 0:
                assert mm == mo
            nxt += 1
        else:
            kind = rnd.choice([cp.BASE, cp.RES])
            assert m.evictable_pages(kind) == o.evictable_pages(kind)
            n = rnd.randint(1, 3)
            before = m.dump()
            so, fo = o.evict(kind, n)
            sm, fm = _st(m.evict, kind, n)
            if so == 0:
                assert fm == fo == n
                after = _sections(m.dump())
                b4 = _sections(before)
                assert after[0] == b4[0], step                      # agent tables untouched
                other = 2 if kind == cp.BASE else 1
                assert after[other] == b4[other], step              # the other tree is bit-identical
        assert so == sm, (step, so, sm)
        assert m.dump() == o.dump(), step
        assert m.take_copy_log() == o.copies, step
        o.copies.clear()
        o.check_invariants()


@pytest.mark.parametrize("pingpong", [False, True])
def test_kernel2_plan_structure_c2(pingpong, monkeypatch):
    """The tcgen05 (kernel 2) planner on the C2 tree, on a host ctx (FKV_PLAN_ASSUME_TC: plan only, no GPU):
    the shared 32K segment of every kv head is split into 8 pieces of 32 tiles for each of its 4 row blocks
    (16 agents x 4 branches x 4 q heads = 256 rows per kv head, 64 per CTA), each sequence's 129-key tail is
    one 2-tile item, every slot gets 16 partial entries (32 with the ping-pong key warpgroups), and planning
    is deterministic."""
    from workloads import recipes
    monkeypatch.setenv("FKV_PLAN_ASSUME_TC", "1")
    if pingpong:
        monkeypatch.setenv("FKV_TC_PINGPONG", "1")
    scen = recipes.c2()
    nb, nr = scen.pages_needed(128)
    m = ForkKV(n_layers=1, n_q_heads=32, n_kv_heads=8, head_dim=128, rank=16, page_size=128, n_base_pages=nb + 8,
               n_res_pages=nr + 8, dtype="bf16", rope_mode="none", device=None)
    for ad in sorted({s.adapter for s in scen.agents}):
        m.register_adapter(ad)
    for s in scen.agents:
        if s.parent is None:
            m.create_root(s.id, s.adapter)
        else:
            m.fork(s.parent, s.fork_len, s.id, s.adapter, L.FORK_SHARE_RESIDUAL if s.share_res else 0)
        if s.n_private:
            m.append([s.id], [s.n_private], [1] * s.n_private)
    batch = scen.batch()
    pl = m.plan([(a, 1) for a in batch], upload=False)
    info = pl.info
    assert info.kernel == 2
    assert info.n_segments == 1 + 64                      # one shared prefix segment + 64 private tails
    hkv, shared_tiles, blocks, pieces = 8, 256, 4, 8
    assert info.n_items == hkv * (blocks * pieces + 64)    # 768
    assert info.key_tiles == hkv * (blocks * shared_tiles + 64 * 2)
    per_slot = 32 if pingpong else 16
    assert info.n_entries == hkv * (blocks * pieces * 4 + 64) * per_slot
    pl2 = m.plan([(a, 1) for a in batch], upload=False)
    for f in ("n_items", "n_entries", "key_tiles", "device_bytes", "workspace_bytes", "alg_bytes", "n_ctas"):
        assert getattr(pl2.info, f) == getattr(info, f), f
