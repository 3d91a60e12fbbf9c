"""Multi-process host logic of the head x agent-batch partitioning (§8(e)),
world_size 2 over gloo on CPU: every rank derives its shard from the
partitioner, builds its own control plane for exactly its kv heads / agents
by the same deterministic call sequence, and the per-rank plans partition
the work with no data-path collective (only a final gather of metadata)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_06370_b200.api import ForkKV, partition, partition_shard
        from workloads import recipes
        n_kv, n_q, d, r, P, prefix, n_agents = 8, 32, 128, 16, 64, 512, 8
        scen = recipes.c5(prefix=prefix, n_agents=n_agents, private=20)
        base_bytes = prefix * n_kv * d * 2 * 2
        res_bytes = n_agents * prefix * r * 2 * 2
        if mode == "heads":
            H, D = world, 1
        elif mode == "agents":
            H, D = 1, world
        else:
            H, D = partition(world, n_kv, base_bytes, res_bytes)
        (h0, h1), (a0, a1) = partition_shard(rank, H, D, n_kv, n_agents)
        mine = [s.id for s in scen.agents if s.decode][a0:a1]
        nb, nr = scen.pages_needed(P)
        fkv = ForkKV(n_layers=1, n_q_heads=n_q, n_kv_heads=n_kv, head_dim=d, rank=r, page_size=P, n_base_pages=nb,
                     n_res_pages=nr, device=None, kv_heads=(h0, h1))
        # same deterministic call sequence on every rank (control plane is per rank)
        for s in scen.agents:
            fkv.register_adapter(s.adapter)
            if s.parent is None:
                fkv.create_root(s.id, s.adapter)
            else:
                fkv.fork(s.parent, s.fork_len, s.id, s.adapter)
            if s.n_private:
                fkv.append([s.id], [s.n_private], list(range(s.fork_len, s.fork_len + s.n_private)))
        pl = fkv.plan([(a, 1) for a in mine], upload=False)
        info = torch.tensor([h0, h1, a0, a1, pl.info.n_rows, pl.info.alg_bytes, pl.info.n_items], dtype=torch.int64)
        import hashlib
        dump_hash = torch.tensor([int(hashlib.sha1(fkv.dump().encode()).hexdigest()[:12], 16)], dtype=torch.int64)
        gathered = [torch.zeros_like(info) for _ in range(world)]
        hashes = [torch.zeros_like(dump_hash) for _ in range(world)]
        dist.all_gather(gathered, info)
        dist.all_gather(hashes, dump_hash)
        if rank == 0:
            q.put((H, D, [g.tolist() for g in gathered], [h.item() for h in hashes]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["heads", "agents", "auto"])
def test_two_rank_shards_partition_the_work(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    H, D, infos, hashes = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert H * D == world
    # shards are disjoint and cover all (head, agent) pairs
    covered = set()
    for h0, h1, a0, a1, *_ in infos:
        for h in range(h0, h1):
            for a in range(a0, a1):
                assert (h, a) not in covered
                covered.add((h, a))
    assert len(covered) == 8 * 8
    # every rank's query rows = its agents x its q heads (1 decode row each)
    for h0, h1, a0, a1, n_rows, alg, items in infos:
        assert n_rows == a1 - a0
        assert items > 0
    # control planes are identical per rank (deterministic call sequence)
    assert len(set(hashes)) == 1
    # head split divides the base bytes; agent split replicates the shared base
    if mode == "heads":
        assert infos[0][5] == infos[1][5]
    if mode == "agents":
        prefix_base = 512 * 8 * 128 * 2 * 2
        assert sum(i[5] for i in infos) > prefix_base * 2 - 1  # base replicated on both ranks


def _bench_worker(rank, world, port, q):
    """bench.py's N>1 host logic over gloo: the Workload each rank builds, the max-over-ranks step time and the
    whole-job token count (weak: every rank's own batch; strong c4: each sequence once)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        out = {}
        for cfg in ("c2", "c4"):
            wl = bench.Workload(cfg, world, rank)
            ms_rank = 2.0 + rank                       # a slower rank 1
            ms = bench._max_over_ranks(ms_rank, world)
            n_rows = len(wl.batch) * wl.C
            v = bench.tokens_value(n_rows, ms, world, wl.scaling, wl.kv[0] == 0,
                                   lambda x: bench._sum_over_ranks(x, world))
            out[cfg] = (wl.scaling, wl.kv, len(wl.batch), ms, v)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_bench_rank_logic_two_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    for cfg in ("c2", "c4"):
        a, b = res[0][cfg], res[1][cfg]
        assert a[3] == b[3] == 3.0                     # max over ranks
        assert a[4] == b[4]                            # every rank derives the same whole-job value
    # c2 weak scaling: each rank its own 64-sequence batch -> 2 x 64 tokens per step
    sc, kv, nb, ms, v = res[0]["c2"]
    assert sc == "weak" and nb == 64 and abs(v - 2 * 64 / (ms / 1e3)) < 1e-6
    # c4 strong scaling (partitioner H=2? D=?): the shards of ONE 128-agent batch count each sequence once
    sc, kv0, nb0, ms, v = res[0]["c4"]
    kv1, nb1 = res[1]["c4"][1], res[1]["c4"][2]
    assert sc == "strong"
    counted = (nb0 if kv0[0] == 0 else 0) + (nb1 if kv1[0] == 0 else 0)
    assert abs(v - counted / (ms / 1e3)) < 1e-6
    assert counted == 128                              # every agent's decode token exactly once
