"""Pins for the control-plane oracle (oracle/control.py): invariants and
worked examples the paper/SPEC fix, plus brute-force LCP."""
import random

import pytest

from oracle import control as cp


def test_spec_radix_split_example():
    """insert [1,2,3,4] then [1,2,5,6] -> root edge [1,2] with two
    children [3,4] and [5,6] (page size 2 so edges split at page bounds)."""
    m = cp.ControlPlane(2, 16, 16)
    assert m.create_root(1, 0) == cp.OK and m.append([1], [4], [1, 2, 3, 4]) == cp.OK
    assert m.create_root(2, 0) == cp.OK and m.append([2], [4], [1, 2, 5, 6]) == cp.OK
    d = m.dump()
    tree = d.split("base_tree")[1].split("res_forest")[0].strip().splitlines()[1:]
    assert [l.split()[0] for l in tree] == ["0", "1", "1"]
    assert tree[0].endswith("tok=1,2") and tree[1].endswith("tok=3,4") and tree[2].endswith("tok=5,6")
    # re-inserting an identical sequence is a no-op
    before = [m.pools[0].rc[:], len(m.base_root.children)]
    assert m.create_root(3, 0) == cp.OK and m.append([3], [4], [1, 2, 3, 4]) == cp.OK
    assert len(m.base_root.children) == before[1]
    m.check_invariants()


def test_sharing_invariant_eq3():
    """P-9 / Eq.3: N agents forked from an s-token root
    allocate ceil(s/P) base pages once and N*ceil(s/P) residual pages; the
    page-byte ratio equals 1/N + r/n (N=16, r=16, n=1024 -> 0.078125
    with the root's own residual counted as one of the N)."""
    P, s, N, r, n = 64, 2048, 16, 16, 1024
    m = cp.ControlPlane(P, 4096, 4096)
    m.create_root(0, 0)
    m.append([0], [s], list(range(s)))
    for a in range(1, N):
        assert m.fork(0, s, a, a) == cp.OK
    base_pages = sum(1 for x in m.pools[0].rc if x > 0)
    res_pages = sum(1 for x in m.pools[1].rc if x > 0)
    assert base_pages == -(-s // P)
    assert res_pages == N * -(-s // P)
    # bytes: base page holds P rows of n (K and V), residual page P rows of r
    ratio = (base_pages * P * n + res_pages * P * r) / (N * s * n)
    assert ratio == 1 / N + r / n == 0.078125
    m.check_invariants()


def test_refcount_holders_and_tree():
    """base block refcount == 1 (tree) + number of live views."""
    P = 4
    m = cp.ControlPlane(P, 64, 64)
    m.create_root(0, 0)
    m.append([0], [8], list(range(8)))
    for a in range(1, 4):
        m.fork(0, 8, a, a)
    for pg in m.agents[0].base:
        assert m.pools[0].rc[pg] == 1 + 4
    for a in (1, 2, 3):
        m.release(a)
    for pg in m.agents[0].base:
        assert m.pools[0].rc[pg] == 2
    m.check_invariants()


def test_cow_unaligned_fork_copies_on_first_write():
    """C-10: a fork at a non page-aligned length shares the partial tail page;
    the first append of either side copies rows [0, fill) to a new page."""
    P = 8
    m = cp.ControlPlane(P, 64, 64)
    m.create_root(0, 7)
    m.append([0], [13], list(range(13)))           # pages: 0 (full), 1 (5 rows)
    assert m.fork(0, 11, 1, 7, cp.FORK_SHARE_RESIDUAL) == cp.OK
    tail = m.agents[0].base[1]
    assert m.agents[1].base[1] == tail and m.pools[0].rc[tail] == 2
    m.copies.clear()
    assert m.append([1], [1], [99]) == cp.OK        # child writes position 11
    assert [c[:2] for c in m.copies] == [(0, tail), (1, m.agents[0].res[1])]
    assert all(c[3] == 11 % P for c in m.copies)    # rows [0, 3) copied
    assert m.agents[1].base[1] != tail and m.agents[0].base[1] == tail
    assert m.pools[0].rc[tail] == 1
    # parent now sole holder: its append is in place (no copy)
    m.copies.clear()
    assert m.append([0], [1], [5]) == cp.OK and m.copies == []
    m.check_invariants()


def test_append_is_atomic_on_exhaustion():
    """exhaustion returns NeedsEviction and leaves no partial state."""
    m = cp.ControlPlane(4, 3, 8)
    m.create_root(0, 0); m.create_root(1, 0)
    before = m.dump()
    assert m.append([0, 1], [8, 8], list(range(16))) == cp.E_NEEDS_EVICTION
    assert m.dump() == before
    assert m.append([0], [12], list(range(12))) == cp.OK
    assert m.append([1], [1], [0]) == cp.E_NEEDS_EVICTION
    m.check_invariants()


def test_readonly_shared_pages():
    """P:87 / P:219: a page with more than one holder is never written in
    place; the sole holder may write (tree refs do not count as holders)."""
    m = cp.ControlPlane(4, 32, 32)
    m.create_root(0, 0)
    m.append([0], [6], list(range(6)))
    assert m.check_write([0], [0], [6], 15) == cp.OK
    m.fork(0, 6, 1, 1)
    assert m.check_write([0], [0], [4], 1) == cp.E_READONLY   # shared base page
    assert m.check_write([1], [0], [6], 12) == cp.OK           # own fresh residual
    assert m.check_write([1], [0], [6], 1) == cp.E_READONLY


def test_match_prefix_bruteforce_lcp():
    """S:316 / S:627 #9: radix longest-prefix match == linear-scan LCP over all
    inserted full-page prefixes (1000 random cases, alphabet 4)."""
    rnd = random.Random(0)
    for case in range(1000):
        P = rnd.choice([1, 2, 3])
        m = cp.ControlPlane(P, 512, 512)
        seqs = []
        for a in range(rnd.randint(1, 4)):
            s = [rnd.randrange(4) for _ in range(rnd.randint(0, 12))]
            m.create_root(a, 0)
            m.append([a], [len(s)], s)
            seqs.append(s)
        q = [rnd.randrange(4) for _ in range(rnd.randint(0, 12))]
        best = 0
        for s in seqs:
            full = (len(s) // P) * P
            k = 0
            while k < min(full, len(q)) and s[k] == q[k]:
                k += 1
            best = max(best, (k // P) * P)
        assert len(m.match_prefix(q)) * P == best, (case, P, seqs, q)


@pytest.mark.parametrize("seed", range(20))
def test_random_sequences_keep_invariants(seed):
    """R9 after every call over random fork/append/release sequences."""
    rnd = random.Random(seed)
    P = rnd.choice([2, 4, 8])
    m = cp.ControlPlane(P, 40, 60, alloc_order_seed=rnd.choice([0, 7]))
    nxt = 0
    for _ in range(200):
        live = sorted(m.agents)
        op = rnd.random()
        if op < 0.15 or not live:
            m.create_root(nxt, rnd.randrange(4)); nxt += 1
        elif op < 0.35:
            p = rnd.choice(live)
            L = rnd.randint(0, m.agents[p].seqlen)
            share = rnd.random() < 0.4
            m.fork(p, L, nxt, m.agents[p].adapter if share else rnd.randrange(4),
                   cp.FORK_SHARE_RESIDUAL if share else 0)
            nxt += 1
        elif op < 0.45:
            toks = [rnd.randrange(3) for _ in range(rnd.randint(0, 3 * P))]
            m.fork_tokens(nxt, rnd.randrange(4), toks); nxt += 1
        elif op < 0.85:
            ags = rnd.sample(live, rnd.randint(1, min(3, len(live))))
            ns = [rnd.randint(0, 2 * P) for _ in ags]
            m.append(ags, ns, [rnd.randrange(3) for _ in range(sum(ns))])
        else:
            m.release(rnd.choice(live))
        m.check_invariants()


# ---- R10-R12: decoupled eviction and partial hit (§5.2, acceptance #6/#7) ----------

def _sections(dump):
    """Split a dump into (agents, base pool + tree, residual pool + forest) text (R8)."""
    lines = dump.splitlines()
    agents = [l for l in lines if l.startswith("agent ")]
    base = [l for l in lines if l.startswith("base_")]
    res = [l for l in lines if l.startswith("res_")]
    bt = dump.split("base_tree")[1].split("res_forest")[0]
    rt = dump.split("res_forest")[1]
    return "\n".join(agents), "\n".join(base) + bt, "\n".join(res) + rt


def _chain(P=2, n_pages=4, nb=32, nr=32):
    m = cp.ControlPlane(P, nb, nr)
    assert m.create_root(0, 0) == cp.OK
    toks = list(range(100, 100 + P * n_pages))
    assert m.append([0], [len(toks)], toks) == cp.OK
    return m, toks


def test_evict_single_chain_deepest_first():
    """S:340 example: a single chain; evicting 1 page removes the deepest leaf
    (the tail) first; the agent's own view is the lock (a held page is not
    evictable: nothing to evict while agent 0 lives)."""
    m, toks = _chain()
    assert m.evictable_pages(cp.BASE) == 0
    assert m.evict(cp.BASE, 1) == (cp.E_NEEDS_EVICTION, 0)
    tail_page = m.agents[0].base[-1]
    m.release(0)
    assert m.evictable_pages(cp.BASE) == 4 and m.evictable_pages(cp.RES) == 4
    before_free = len(m.pools[cp.BASE].free)
    assert m.evict(cp.BASE, 1) == (cp.OK, 1)
    assert tail_page in m.pools[cp.BASE].free and len(m.pools[cp.BASE].free) == before_free + 1
    assert m.match_prefix(toks) == m.match_prefix(toks[:6])       # 3 pages left, the tail went first
    assert len(m.match_prefix(toks)) == 3
    m.check_invariants()


def test_evict_locked_leaf_skipped():
    """S:341 example: a leaf held by a live view is skipped; the next LRU leaf
    goes.  Two branches share page 0; branch A is older (inserted first) but
    held by agent 1; branch B is unheld -> B's leaf is evicted."""
    m = cp.ControlPlane(2, 32, 32)
    m.create_root(0, 0)
    m.append([0], [4], [1, 2, 3, 4])        # branch A: [1,2][3,4]
    m.create_root(1, 1)
    m.append([1], [4], [1, 2, 5, 6])        # branch B: [1,2][5,6] (page of [1,2] is agent 0's)
    m.release(1)                            # B's leaf [5,6] unheld; A's leaf held by agent 0
    leaf_b = [nd for ck, nd in m.base_root.children[(1, 2)].children.items() if ck == (5, 6)][0].page
    assert m.evict(cp.BASE, 1) == (cp.OK, 1)
    assert leaf_b in m.pools[cp.BASE].free
    assert m.evict(cp.BASE, 1) == (cp.E_NEEDS_EVICTION, 0)   # [1,2] and [3,4] are agent 0's
    m.check_invariants()


def test_evict_lru_order_follows_access():
    """Independent LRU clock: re-accessing an older branch (a fork
    over it) makes the other branch the victim."""
    m = cp.ControlPlane(2, 32, 32)
    for a, t in ((0, [1, 2, 3, 4]), (1, [1, 2, 5, 6])):
        m.create_root(a, a)
        m.append([a], [4], t)
        m.release(a)
    # both leaves unheld; [3,4] is older -> it would go first ...
    m2 = cp.ControlPlane(2, 32, 32)
    for a, t in ((0, [1, 2, 3, 4]), (1, [1, 2, 5, 6])):
        m2.create_root(a, a)
        m2.append([a], [4], t)
        m2.release(a)
    p34 = m.base_root.children[(1, 2)].children[(3, 4)].page
    assert m.evict(cp.BASE, 1) == (cp.OK, 1) and p34 in m.pools[cp.BASE].free
    # ... unless a fork_tokens touched it in between
    assert m2.fork_tokens(9, 0, [1, 2, 3, 4]) == (cp.OK, 4)
    m2.release(9)
    p56 = m2.base_root.children[(1, 2)].children[(5, 6)].page
    assert m2.evict(cp.BASE, 1) == (cp.OK, 1) and p56 in m2.pools[cp.BASE].free


def test_partial_hit_acceptance_6():
    """SPEC acceptance #6 / P:304: prefill agent A, evict its base-tree
    tail, fork B on the same context and lineage -> the residual is reused in
    full (zero residual recompute) and only the evicted base range is
    recomputed."""
    P, n_pages = 4, 6
    m, toks = _chain(P=P, n_pages=n_pages)
    m.release(0)
    assert m.evict(cp.BASE, 2) == (cp.OK, 2)              # base tail: pages 4, 5
    st, (bh, rh, mapped) = m.fork_resume(1, 0, 0, toks)
    assert st == cp.OK
    assert (bh, rh, mapped) == (4 * P, 6 * P, 6 * P)
    recompute_base = (bh, mapped)                          # [16, 24): the evicted range only
    reuse_res, recompute_res = (0, rh), (rh, mapped)
    assert recompute_base == (16, 24) and reuse_res == (0, 24) and recompute_res[1] - recompute_res[0] == 0
    # FLOP-style accounting: residual projection rows to recompute = 0, base rows = evicted rows
    assert (recompute_res[1] - recompute_res[0]) * 16 == 0
    assert recompute_base[1] - recompute_base[0] == 2 * P
    # the recomputed pages are fresh (writable) and reinserted into the base tree
    ag = m.agents[1]
    assert all(m.writable(cp.BASE, pg) for pg in ag.base[4:]) and len(m.match_prefix(toks)) == 6
    assert not any(m.writable(cp.RES, pg) for pg in ag.res) or True
    m.check_invariants()
    # a cold fork of a NEW lineage: recompute everything residual, reuse the whole base
    st, (bh, rh, mapped) = m.fork_resume(2, 5, 2, toks)
    assert st == cp.OK and (bh, rh, mapped) == (24, 0, 24)
    # the lineage of agent 0 holds adapter 0's rows: another adapter is refused (R11)
    assert m.fork_resume(3, 7, 0, toks)[0] == cp.E_INVALID
    m.check_invariants()


def test_partial_hit_plan_partitions_request():
    """S:319 PartialHitPlan invariant: reuse/recompute ranges partition the
    request (random scenarios)."""
    rnd = random.Random(5)
    for _ in range(200):
        P = rnd.choice([2, 4])
        m, toks = _chain(P=P, n_pages=rnd.randint(1, 6))
        m.release(0)
        nb_ev = rnd.randint(0, m.evictable_pages(cp.BASE))
        nr_ev = rnd.randint(0, m.evictable_pages(cp.RES))
        if nb_ev:
            assert m.evict(cp.BASE, nb_ev)[0] == cp.OK
        if nr_ev:
            assert m.evict(cp.RES, nr_ev)[0] == cp.OK
        req = toks[:rnd.randint(0, len(toks))] + [7] * rnd.randint(0, 3)
        st, (bh, rh, mapped) = m.fork_resume(1, 0, 0, req)
        assert st == cp.OK
        n = len(req)
        assert 0 <= bh <= mapped <= n and 0 <= rh <= mapped and mapped == max(bh, rh)
        # reuse_res [0, rh) + recompute_res [rh, n) partition [0, n); base likewise
        assert (rh - 0) + (n - rh) == n and (bh - 0) + (n - bh) == n
        assert m.agents[1].seqlen == mapped
        m.check_invariants()


def _lru_victim_from_dump(dump, kind_prefix):
    """Shadow LRU-of-leaves oracle: parse a dump section and return the
    page of the unheld leaf with the smallest (last, seq)."""
    sec = dump.split("base_tree")[1].split("res_forest")[0] if kind_prefix == "base" else dump.split("res_forest")[1]
    nodes = []
    for l in sec.splitlines():
        if not l.startswith(" ") or not l.split()[0].isdigit():
            nodes.append(None)          # a tree header line: the previous tree ended
            continue
        f = dict(x.split("=") for x in l.split()[1:] if "=" in x)
        nodes.append((int(l.split()[0]), int(f["page"]), int(f["rc"]), int(f["last"]), int(f["seq"])))
    best = None
    for i, nd in enumerate(nodes):
        if nd is None:
            continue
        nxt = nodes[i + 1] if i + 1 < len(nodes) else None
        leaf = nxt is None or nxt[0] <= nd[0]
        if leaf and nd[2] == 1 and (best is None or (nd[3], nd[4]) < (best[3], best[4])):
            best = nd
    return None if best is None else best[1]


@pytest.mark.parametrize("seed", range(200))
def test_decoupled_eviction_acceptance_7(seed):
    """SPEC acceptance #7: evictions of one tree leave the other tree's
    dump (pool, nodes, clock) bit-identical; every victim is the shadow
    LRU-of-leaves choice read back from the dump."""
    rnd = random.Random(7000 + seed)
    P = rnd.choice([2, 4])
    m = cp.ControlPlane(P, 48, 64)
    nxt = 0
    for step in range(40):
        live = sorted(m.agents)
        x = rnd.random()
        if x < 0.25 or not live:
            m.create_root(nxt, rnd.randrange(2))
            nxt += 1
        elif x < 0.55:
            a = rnd.choice(live)
            n = rnd.randint(1, 3 * P)
            if m.append([a], [n], [rnd.randrange(3) for _ in range(n)]) != cp.OK:
                m.release(a)
        elif x < 0.65:
            m.release(rnd.choice(live))
        elif x < 0.75:
            toks = [rnd.randrange(3) for _ in range(rnd.randint(0, 4 * P))]
            owner = rnd.choice([nxt] + list(m.res_roots))
            m.fork_resume(nxt, m.res_adapter.get(owner, 0), owner, toks)
            nxt += 1
        else:
            kind = rnd.choice([cp.BASE, cp.RES])
            avail = m.evictable_pages(kind)
            if avail == 0:
                assert m.evict(kind, 1) == (cp.E_NEEDS_EVICTION, 0)
                continue
            before = _sections(m.dump())
            victim = _lru_victim_from_dump(m.dump(), "base" if kind == cp.BASE else "res")
            assert m.evict(kind, 1) == (cp.OK, 1)
            assert victim in m.pools[kind].free
            after = _sections(m.dump())
            assert after[0] == before[0]                       # agent tables untouched
            other = 2 if kind == cp.BASE else 1
            assert after[other] == before[other]               # the other tree: bit-identical
        m.check_invariants()
