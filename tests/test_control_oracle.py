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
    tree = d.split("base_tree\n")[1].split("res_tree")[0].strip().splitlines()
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
