"""§8(f) f4 — sequence split across GPUs with a log-sum-exp merge.

CPU: the merge oracle is pinned by softmax blocking invariance (P-6): merging the attention oracle's own
outputs over disjoint key subsets equals the oracle over all keys (NONE mode, decode rows: positions do not enter);
the key-range partitioner covers [0, L) with page-aligned disjoint ranges; a world-2 gloo run does the whole
host-side protocol (each rank its key range, all_gather of (O, lse), merge) on CPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import merge, ra


def _inputs(seed, L=300, hkv=2, g=2, d=16, r=4):
    rng = np.random.default_rng(seed)
    return dict(Kb=rng.standard_normal((L, hkv, d)), Vb=rng.standard_normal((L, hkv, d)),
                Rk=rng.standard_normal((L, r)), Rv=rng.standard_normal((L, r)),
                Bk=rng.standard_normal((hkv, r, d)) / 4, Bv=rng.standard_normal((hkv, r, d)) / 4,
                Q=rng.standard_normal((1, hkv * g, d)) * 2)


def _sub(inp, a, b):
    return dict(inp, Kb=inp["Kb"][a:b], Vb=inp["Vb"][a:b], Rk=inp["Rk"][a:b], Rv=inp["Rv"][a:b])


@pytest.mark.parametrize("seed", range(6))
def test_merge_of_key_subsets_equals_full_attention(seed):
    inp = _inputs(seed)
    full, lse_full = ra.residual_attention(inv_freq_=None, rope_mode=ra.ROPE_NONE, return_lse=True, **inp)
    cuts = sorted(np.random.default_rng(100 + seed).choice(np.arange(1, 300), size=3, replace=False))
    edges = [0] + list(cuts) + [300]
    parts = [ra.residual_attention(inv_freq_=None, rope_mode=ra.ROPE_NONE, return_lse=True, **_sub(inp, a, b))
             for a, b in zip(edges[:-1], edges[1:])]
    O, lse = merge.merge_lse([p[0] for p in parts], [p[1] for p in parts])
    np.testing.assert_allclose(O, full, atol=1e-12)
    np.testing.assert_allclose(lse, lse_full, atol=1e-12)


def test_merge_with_an_empty_part():
    inp = _inputs(9)
    full, lse_full = ra.residual_attention(inv_freq_=None, rope_mode=ra.ROPE_NONE, return_lse=True, **inp)
    O, lse = merge.merge_lse([full, np.zeros_like(full)], [lse_full, np.full_like(lse_full, -np.inf)])
    np.testing.assert_allclose(O, full, atol=1e-14)
    np.testing.assert_allclose(lse, lse_full, atol=1e-14)


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_partition_keys_covers_the_sequence(G):
    from paper_2604_06370_b200.api import partition_keys
    L, P = 131072 + 129, 128
    ranges = [partition_keys(L, G, P, r) for r in range(G)]
    assert ranges[0][0] == 0 and ranges[-1][1] is None
    for (a, b), (c, _) in zip(ranges[:-1], ranges[1:]):
        assert b == c and a % P == 0 and b % P == 0 and b > a
    sizes = [(b if b is not None else L) - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 2 * P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_06370_b200.api import partition_keys
        inp = _inputs(21, L=1000)
        kb, ke = partition_keys(1000, world, 64, rank)
        ke = 1000 if ke is None else ke
        O, lse = ra.residual_attention(inv_freq_=None, rope_mode=ra.ROPE_NONE, return_lse=True, **_sub(inp, kb, ke))
        Os = [torch.zeros(O.shape, dtype=torch.float64) for _ in range(world)]
        ls = [torch.zeros(lse.shape, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(Os, torch.from_numpy(O))
        dist.all_gather(ls, torch.from_numpy(lse))
        Om, _ = merge.merge_lse([o.numpy() for o in Os], [x.numpy() for x in ls])
        full = ra.residual_attention(inv_freq_=None, rope_mode=ra.ROPE_NONE, **inp)
        q.put((rank, float(np.abs(Om - full).max())))
    finally:
        dist.destroy_process_group()


def test_two_rank_sequence_split_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert max(res.values()) < 1e-12
