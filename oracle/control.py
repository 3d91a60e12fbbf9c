"""ORACLE (test infrastructure): control-plane model of ForkKV's memory side.

A plain Python model of the two page pools, the per-agent block tables, the
fork-with-CoW semantics and the DualRadixTree, written from the paper:

  * disaggregated pools: bCache (base) and rCache (residual) are physically
    separate pools (§5.1, §6);
  * DualRadixTree: a base tree keyed by token ids and a residual tree keyed by
    (agent id, token ids) (§5.2, Fig design-cache-tree);
  * fork = Step 1 prefix match / inherit read-only base pages, Step 2
    copy-on-write allocation of exclusive residual pages (§5.2);
  * no page shared by more than one holder is ever written in place (the
    "in-place cache update" conflict of P:87 §1 / P:219 §3.3);
  * decoupled eviction: each radix tree has its own LRU state; evicting one
    tree never touches the other, and a fork over a context whose base pages
    were evicted while its residual pages survive is a *partial hit* that
    recomputes only the base rows (§5.2; rules R10-R12).

Where the paper is silent this follows the rule set R1-R9 and readings
C-9..C-12 listed in DESIGN.md ("Control-plane rules").  The C++ library in
the product implements the same rules independently; tests compare the two
bit-exactly through ``dump()`` and the per-agent tables.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

OK = 0
E_INVALID = 1
E_NEEDS_EVICTION = 2
E_UNKNOWN_AGENT = 3
E_STALE = 4
E_READONLY = 5
E_NO_KEYS = 6
E_UNWRITTEN = 7

FORK_SHARE_RESIDUAL = 1

BASE = 0
RES = 1

_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class Pool:
    """R1: refcounted pages; the free set is ordered by (rank, id)."""

    def __init__(self, n: int, seed: int):
        self.n = n
        self.seed = seed
        self.rc = [0] * n
        self.in_tree = [False] * n
        self.free = set(range(n))

    def rank(self, pid: int) -> Tuple[int, int]:
        return (pid if self.seed == 0 else splitmix64((self.seed ^ pid) & _M64), pid)

    def free_order(self) -> List[int]:
        return sorted(self.free, key=self.rank)

    def alloc(self) -> int:
        pid = min(self.free, key=self.rank)
        self.free.remove(pid)
        self.rc[pid] = 1
        self.in_tree[pid] = False
        return pid

    def retain(self, pid: int) -> None:
        self.rc[pid] += 1

    def release(self, pid: int) -> None:
        self.rc[pid] -= 1
        assert self.rc[pid] >= 0
        if self.rc[pid] == 0:
            self.in_tree[pid] = False
            self.free.add(pid)


@dataclass
class Agent:
    id: int
    adapter: int
    owner: int
    seqlen: int = 0
    base: List[int] = field(default_factory=list)
    res: List[int] = field(default_factory=list)
    tokens: List[int] = field(default_factory=list)


class Node:
    """One page-granular radix-tree node: a P-token chunk -> one page.  `last`
    is the tree's logical clock at the node's last access, `seq` its insertion
    number in that tree (LRU tie-break: older insertion first)."""
    __slots__ = ("page", "children", "last", "seq")

    def __init__(self, page: int, last: int = 0, seq: int = -1):
        self.page = page
        self.children: Dict[Tuple[int, ...], "Node"] = {}
        self.last = last
        self.seq = seq


class ControlPlane:
    def __init__(self, page_size: int, n_base_pages: int, n_res_pages: int, alloc_order_seed: int = 0):
        self.P = page_size
        self.pools = [Pool(n_base_pages, alloc_order_seed), Pool(n_res_pages, alloc_order_seed)]
        self.agents: Dict[int, Agent] = {}
        self.base_root = Node(-1)
        self.res_roots: Dict[int, Node] = {}
        self.res_adapter: Dict[int, int] = {}   # residual tree owner -> adapter whose xA_i it holds
        self.clock = [0, 0]                     # independent LRU clocks of the two trees (R10)
        self.nseq = [0, 0]                      # insertion counters of the two trees
        self.copies: List[Tuple[int, int, int, int]] = []  # (kind, src, dst, rows) CoW log

    def _lineage_ok(self, owner: int, adapter: int) -> bool:
        """R11: a residual lineage (tree key) holds the xA_i rows of ONE adapter:
        its surviving tree and every live view of it must use `adapter`."""
        if self.res_adapter.get(owner, adapter) != adapter:
            return False
        return all(ag.adapter == adapter for ag in self.agents.values() if ag.owner == owner)

    # ---- R3 -----------------------------------------------------------
    def create_root(self, a: int, adapter: int) -> int:
        if a in self.agents or a < 0 or adapter < 0 or not self._lineage_ok(a, adapter):
            return E_INVALID
        self.agents[a] = Agent(a, adapter, a)
        return OK

    # ---- R5 -----------------------------------------------------------
    def fork(self, parent: int, prefix_len: int, child: int, adapter: int, flags: int = 0) -> int:
        if parent not in self.agents:
            return E_UNKNOWN_AGENT
        p = self.agents[parent]
        if child in self.agents or child < 0 or adapter < 0 or prefix_len < 0 or prefix_len > p.seqlen:
            return E_INVALID
        share = bool(flags & FORK_SHARE_RESIDUAL)
        if share and adapter != p.adapter:
            return E_INVALID
        if not share and not self._lineage_ok(child, adapter):
            return E_INVALID
        k = -(-prefix_len // self.P)
        if not share and len(self.pools[RES].free) < k:
            return E_NEEDS_EVICTION
        c = Agent(child, adapter, p.owner if share else child, prefix_len)
        c.base = list(p.base[:k])
        for pg in c.base:
            self.pools[BASE].retain(pg)
        if share:
            c.res = list(p.res[:k])
            for pg in c.res:
                self.pools[RES].retain(pg)
        else:
            c.res = [self.pools[RES].alloc() for _ in range(k)]
        c.tokens = list(p.tokens[:prefix_len])
        self.agents[child] = c
        return OK

    # ---- R7: fork_tokens (Step 1 = longest full-page prefix match) ------
    def _match(self, root: Optional[Node], tokens: List[int]) -> List[Node]:
        """Longest full-page prefix of `tokens` stored under `root` (no touch)."""
        node, path = root, []
        if node is None:
            return path
        for s in range(len(tokens) // self.P):
            ch = node.children.get(tuple(tokens[s * self.P:(s + 1) * self.P]))
            if ch is None:
                break
            path.append(ch)
            node = ch
        return path

    def _touch(self, kind: int, path: List[Node]) -> None:
        """R10: one access of a tree = one tick of its own clock for every node on the path."""
        if path:
            self.clock[kind] += 1
            for nd in path:
                nd.last = self.clock[kind]

    def match_prefix(self, tokens: List[int]) -> List[int]:
        return [nd.page for nd in self._match(self.base_root, tokens)]

    def fork_tokens(self, child: int, adapter: int, tokens: List[int]) -> Tuple[int, int]:
        if child in self.agents or child < 0 or adapter < 0 or not self._lineage_ok(child, adapter):
            return E_INVALID, 0
        path = self._match(self.base_root, tokens)
        pages = [nd.page for nd in path]
        k = len(pages)
        if len(self.pools[RES].free) < k:
            return E_NEEDS_EVICTION, 0
        self._touch(BASE, path)
        c = Agent(child, adapter, child, k * self.P)
        c.base = list(pages)
        for pg in pages:
            self.pools[BASE].retain(pg)
        c.res = [self.pools[RES].alloc() for _ in range(k)]
        c.tokens = list(tokens[:k * self.P])
        self.agents[child] = c
        return OK, k * self.P

    # ---- R4 -----------------------------------------------------------
    def _dry_run_needs(self, agents: List[int], n_new: List[int]) -> Tuple[int, int]:
        rc_delta: Dict[Tuple[int, int], int] = {}
        need = [0, 0]
        for a, n in zip(agents, n_new):
            ag = self.agents[a]
            if n == 0:
                continue
            t0 = ag.seqlen
            if t0 % self.P != 0:
                slot = t0 // self.P
                for kind, table in ((BASE, ag.base), (RES, ag.res)):
                    pg = table[slot]
                    rc = self.pools[kind].rc[pg] + rc_delta.get((kind, pg), 0)
                    if rc > 1:
                        need[kind] += 1
                        rc_delta[(kind, pg)] = rc_delta.get((kind, pg), 0) - 1
            first_new = -(-t0 // self.P)  # first slot index that starts a new page
            last = t0 + n - 1
            new_pages = max(0, last // self.P - first_new + 1) if last >= first_new * self.P else 0
            need[BASE] += new_pages
            need[RES] += new_pages
        return need[BASE], need[RES]

    def append(self, agents: List[int], n_new: List[int], token_ids: List[int]) -> int:
        if len(agents) != len(n_new) or len(set(agents)) != len(agents):
            return E_INVALID
        for a, n in zip(agents, n_new):
            if a not in self.agents:
                return E_UNKNOWN_AGENT
            if n < 0:
                return E_INVALID
        if len(token_ids) != sum(n_new):
            return E_INVALID
        nb, nr = self._dry_run_needs(agents, n_new)
        if nb > len(self.pools[BASE].free) or nr > len(self.pools[RES].free):
            return E_NEEDS_EVICTION
        off_tok = 0
        for a, n in zip(agents, n_new):
            ag = self.agents[a]
            for i in range(n):
                t = ag.seqlen + i
                slot, off = divmod(t, self.P)
                if off == 0:
                    ag.base.append(self.pools[BASE].alloc())
                    ag.res.append(self.pools[RES].alloc())
                elif i == 0:
                    for kind, table in ((BASE, ag.base), (RES, ag.res)):
                        pg = table[slot]
                        if self.pools[kind].rc[pg] > 1:  # CoW (C-10)
                            new = self.pools[kind].alloc()
                            self.copies.append((kind, pg, new, off))
                            self.pools[kind].release(pg)
                            table[slot] = new
                ag.tokens.append(int(token_ids[off_tok + i]))
                if off == self.P - 1:
                    self._tree_insert(ag, slot)
            ag.seqlen += n
            off_tok += n
        return OK

    def _tree_insert(self, ag: Agent, slot: int) -> None:
        """R7: page `slot` of agent became full: insert chunks 0..slot (a
        chunk missing from the tree, e.g. evicted, is (re)inserted with the
        agent's page).  The walk is one access of each tree (R10)."""
        for kind, table in ((BASE, ag.base), (RES, ag.res)):
            if kind == BASE:
                node = self.base_root
            else:
                if ag.owner not in self.res_roots:
                    self.res_roots[ag.owner] = Node(-1)
                    self.res_adapter[ag.owner] = ag.adapter
                node = self.res_roots[ag.owner]
            self.clock[kind] += 1
            for k in range(slot + 1):
                chunk = tuple(ag.tokens[k * self.P:(k + 1) * self.P])
                ch = node.children.get(chunk)
                if ch is None:
                    pg = table[k]
                    ch = Node(pg, seq=self.nseq[kind])
                    self.nseq[kind] += 1
                    node.children[chunk] = ch
                    self.pools[kind].retain(pg)
                    self.pools[kind].in_tree[pg] = True
                ch.last = self.clock[kind]
                node = ch

    # ---- R11: fork with partial hit ------------------------------------------
    def fork_resume(self, child: int, adapter: int, owner: int, tokens: List[int]) -> Tuple[int, Tuple[int, int, int]]:
        """Fork `child` over `tokens` reusing what survives in BOTH trees
        (P:300 Step 1 + Step 2, P:304 partial hit).

        base hit  = longest full-page prefix in the base tree (pages mapped);
        res hit   = longest full-page prefix in the residual tree of `owner`
                    (the lineage whose xA_i rows it holds; must have been
                    produced with `adapter`);
        mapped    = max of the two (tokens).  Base pages [base hit, mapped) and
        residual pages [res hit, mapped) are fresh (unwritten) pages the
        engine fills by recomputing only xW resp. xA_i for those rows.
        All mapped pages are full, so they are inserted into both trees at
        once (R7).  Returns (status, (base_hit, res_hit, mapped)) in tokens."""
        if child in self.agents or child < 0 or adapter < 0 or owner < 0:
            return E_INVALID, (0, 0, 0)
        if not self._lineage_ok(owner, adapter):
            return E_INVALID, (0, 0, 0)
        bpath = self._match(self.base_root, tokens)
        rpath = self._match(self.res_roots.get(owner), tokens)
        bm, rm = len(bpath), len(rpath)
        k = max(bm, rm)
        if len(self.pools[BASE].free) < k - bm or len(self.pools[RES].free) < k - rm:
            return E_NEEDS_EVICTION, (0, 0, 0)
        c = Agent(child, adapter, owner, k * self.P)
        c.base = [nd.page for nd in bpath]
        c.res = [nd.page for nd in rpath]
        for pg in c.base:
            self.pools[BASE].retain(pg)
        for pg in c.res:
            self.pools[RES].retain(pg)
        c.base += [self.pools[BASE].alloc() for _ in range(k - bm)]
        c.res += [self.pools[RES].alloc() for _ in range(k - rm)]
        c.tokens = list(tokens[:k * self.P])
        self.agents[child] = c
        if k > 0:
            self._tree_insert(c, k - 1)
        return OK, (bm * self.P, rm * self.P, k * self.P)

    # ---- R12: decoupled eviction ----------------------------------------------
    def _roots(self, kind: int) -> List[Node]:
        return [self.base_root] if kind == BASE else [self.res_roots[o] for o in sorted(self.res_roots)]

    def evictable_pages(self, kind: int) -> int:
        """Pages `evict` could free: nodes whose whole subtree holds only
        tree-only pages (refcount 1), since only unheld leaves go, bottom-up."""
        pool = self.pools[kind]

        def walk(nd: Node) -> Tuple[int, bool]:
            tot, clean = 0, True
            for ch in nd.children.values():
                t, c = walk(ch)
                tot += t
                clean = clean and c
            if nd.page >= 0:
                clean = clean and pool.rc[nd.page] == 1
                tot += 1 if clean else 0
            return tot, clean

        return sum(walk(r)[0] for r in self._roots(kind))

    def evict(self, kind: int, n_pages: int) -> Tuple[int, int]:
        """Free `n_pages` pages of ONE tree: repeatedly drop the
        least recently used leaf (smallest (last, seq)) whose page no live
        view holds.  The other tree, its clock and every agent table are
        untouched.  Atomic: if fewer than n_pages can be freed, nothing is
        evicted and E_NEEDS_EVICTION is returned."""
        if kind not in (BASE, RES) or n_pages < 1:
            return E_INVALID, 0
        if self.evictable_pages(kind) < n_pages:
            return E_NEEDS_EVICTION, 0
        pool = self.pools[kind]
        freed = 0
        while freed < n_pages:
            best = None
            for ri, root in enumerate(self._roots(kind)):
                stack = [(root, None, None)]
                while stack:
                    nd, parent, key = stack.pop()
                    for ck, ch in nd.children.items():
                        stack.append((ch, nd, ck))
                    if nd.page >= 0 and not nd.children and pool.rc[nd.page] == 1:
                        if best is None or (nd.last, nd.seq) < (best[0].last, best[0].seq):
                            best = (nd, parent, key)
            nd, parent, key = best
            del parent.children[key]
            pool.release(nd.page)
            freed += 1
            if kind == RES:
                for o in [o for o, r in self.res_roots.items() if not r.children]:
                    del self.res_roots[o]
                    del self.res_adapter[o]
        return OK, freed

    # ---- R6 -----------------------------------------------------------
    def release(self, a: int) -> int:
        if a not in self.agents:
            return E_UNKNOWN_AGENT
        ag = self.agents.pop(a)
        for pg in ag.base:
            self.pools[BASE].release(pg)
        for pg in ag.res:
            self.pools[RES].release(pg)
        return OK

    # ---- write permission (R9 last bullet) ------------------------------
    def writable(self, kind: int, pg: int) -> bool:
        pool = self.pools[kind]
        return pool.rc[pg] - (1 if pool.in_tree[pg] else 0) == 1

    def check_write(self, agents, start, count, which_mask) -> int:
        """Status the library must return for fkv_write_kv (rows must be
        reserved; pages written must have exactly one holder)."""
        for a, s, c in zip(agents, start, count):
            if a not in self.agents:
                return E_UNKNOWN_AGENT
            ag = self.agents[a]
            if s < 0 or c < 0 or s + c > ag.seqlen:
                return E_INVALID
        for a, s, c in zip(agents, start, count):
            ag = self.agents[a]
            if c == 0:
                continue
            for slot in range(s // self.P, (s + c - 1) // self.P + 1):
                if which_mask & 3 and not self.writable(BASE, ag.base[slot]):
                    return E_READONLY
                if which_mask & 12 and not self.writable(RES, ag.res[slot]):
                    return E_READONLY
        return OK

    # ---- R8 -----------------------------------------------------------
    def dump(self) -> str:
        out = [f"P={self.P}"]
        for a in sorted(self.agents):
            ag = self.agents[a]
            out.append(f"agent {ag.id} adapter={ag.adapter} owner={ag.owner} seqlen={ag.seqlen} "
                       f"base={','.join(map(str, ag.base))} res={','.join(map(str, ag.res))}")
        for name, pool in (("base", self.pools[BASE]), ("res", self.pools[RES])):
            out.append(f"{name}_free {len(pool.free)} order={','.join(map(str, pool.free_order()))}")
            out.append(f"{name}_rc " + " ".join(f"{i}:{pool.rc[i]}" for i in range(pool.n) if pool.rc[i] > 0))

        def walk(node: Node, depth: int, kind: int):
            for chunk in sorted(node.children):
                ch = node.children[chunk]
                out.append(f" {depth} page={ch.page} rc={self.pools[kind].rc[ch.page]} last={ch.last} "
                           f"seq={ch.seq} tok={','.join(map(str, chunk))}")
                walk(ch, depth + 1, kind)

        out.append(f"base_tree clock={self.clock[BASE]} seq={self.nseq[BASE]}")
        walk(self.base_root, 0, BASE)
        out.append(f"res_forest clock={self.clock[RES]} seq={self.nseq[RES]}")
        for o in sorted(self.res_roots):
            out.append(f"res_tree owner={o} adapter={self.res_adapter[o]}")
            walk(self.res_roots[o], 0, RES)
        return "\n".join(out) + "\n"

    # ---- invariants (R9) -------------------------------------------------
    def check_invariants(self) -> None:
        for kind in (BASE, RES):
            pool = self.pools[kind]
            holders = [0] * pool.n
            for ag in self.agents.values():
                for pg in (ag.base if kind == BASE else ag.res):
                    holders[pg] += 1
            tree = [0] * pool.n
            roots = [self.base_root] if kind == BASE else list(self.res_roots.values())
            stack = list(roots)
            while stack:
                nd = stack.pop()
                for ch in nd.children.values():
                    tree[ch.page] += 1
                    stack.append(ch)
            for i in range(pool.n):
                assert pool.rc[i] == holders[i] + tree[i], (kind, i, pool.rc[i], holders[i], tree[i])
                assert tree[i] <= 1
                assert (pool.rc[i] == 0) == (i in pool.free)
            assert len(pool.free) + sum(1 for i in range(pool.n) if pool.rc[i] > 0) == pool.n
