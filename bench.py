#!/usr/bin/env python
"""bench.py — ResidualAttention throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5] [--mode deferred|none] [--page 128]

Default workload = BASELINE.json configs[1] (C2): Llama-3.1-8B shape, all 32
layers, 16 agents / 16 adapters forked from a 32K-token shared prefix, 4
same-agent branches each -> decode batch 64, r = 16, bf16.

Decode configs (c1, c2, c4, c5): one step = one decode step of the whole hot
path for the batch: append one token per sequence (control plane, CoW if
needed), plan (agent grouping + split) and plan upload, then for every layer
write the new K/V rows (kv_write) and run ResidualAttention (main kernel +
combine / late V fusion). Prefill config (c3): one step = one 1024-token chunk
per agent through every layer. Inputs are resident in HBM for `value`; `e2e`
repeats the step through the host-buffer C-ABI call with H2D/D2H copies in
the timed region. N > 1 (torchrun): c2/c5 run weak scaling (each rank its own
agent batch; no data-path collective), c4 is the head x agent-batch sharded
70B case (partitioner); time = max over ranks (CUDA events, all_reduce MAX).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ResidualAttention decode tokens/s and achieved HBM GB/s vs roofline, 1/2/4/8 B200"
METRIC_PREFILL = "ResidualAttention chunked-prefill tokens/s and tensor-pipe utilisation, B200"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1590.0)), float(
            d.get("bf16_tflops_sustained", d.get("bf16_tflops", 1400.0))), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=3)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class Workload:
    """A BASELINE.json config as seen by one rank."""

    def __init__(self, name, world=1, rank=0):
        from workloads import recipes
        self.name, self.kind, self.scaling = name, "decode", "weak"
        self.L, self.Hq, self.Hkv, self.d, self.r = 32, 32, 8, 128, 16
        self.kv = (0, 8)
        self.parallelism = f"agent-batch x{world} (partitioner H=1, D={world}): every rank its own agent batch"
        if name == "c1":
            self.scen, self.L = recipes.c1(), 1
            self.desc = "configs[0] C1: 1 layer Llama-3.1-8B shape, 4 agents forked from a 2K prefix + 128 private, r=16"
        elif name == "c3":
            self.scen, self.kind = recipes.c3(), "prefill"
            self.desc = ("configs[2] C3: Llama-3.1-8B all 32 layers, chunked prefill: 8 agents / 8 adapters over a 32K "
                         "shared prefix, 1024-token chunk of each 4K private context (keys 35,841..36,864), r=16")
        elif name == "c5":
            self.scen = recipes.c5()
            self.desc = "configs[4] point: Llama-3.1-8B 32 layers, 64 independent agents over a 32K prefix, r=16"
        elif name == "c4":
            from paper_2604_06370_b200.api import partition, partition_shard
            self.L, self.Hq, self.Hkv = 80, 64, 8
            n_agents, prefix = 128, 131072
            base_b = prefix * self.Hkv * self.d * 2 * 2
            res_b = n_agents * prefix * self.r * 2 * 2
            H, D = partition(world, self.Hkv, base_b, res_b)
            (h0, h1), (a0, a1) = partition_shard(rank, H, D, self.Hkv, n_agents)
            full = recipes.c5(prefix=prefix, n_agents=n_agents, private=128)
            keep = {s.id for s in full.agents if s.parent is None} | {s.id for s in full.agents[1:][a0:a1]}
            self.scen = recipes.Scenario("C4", [s for s in full.agents if s.id in keep])
            self.kv = (h0, h1)
            self.scaling = "strong"
            self.parallelism = f"kv-head x agent-batch (partitioner H={H}, D={D}) over {world} GPU(s)"
            self.desc = ("configs[3] C4: Llama-3.1-70B shape (80 layers, 64 q / 8 kv heads), r=16, 128 agents over a "
                         "128K shared prefix, KV heads and agent batch sharded")
        else:
            self.scen = recipes.c2()
            self.desc = ("configs[1] C2: Llama-3.1-8B all 32 layers, 16 agents / 16 adapters x 4 branches = decode "
                         "batch 64, 32K shared prefix, r=16")
        self.batch = self.scen.batch()
        self.C = self.scen.q_len

    def flops_per_layer(self, hkv_local, group):
        """Algorithmic FLOPs of one layer (minimal form): QK^T and PV over the
        visible keys of every query row, the rank-r rebuild per (owner, kv head,
        key), q.K_lora, P.R_v and the late fusion per row."""
        d, r = self.d, self.r
        tot = 0
        owners = {}
        for a in self.batch:
            L = self.scen.seqlen(a)
            vis = sum(L - self.C + i + 1 for i in range(self.C))  # causal visible keys over the chunk
            tot += hkv_local * group * vis * (2 * d + 2 * d + 2 * r) + hkv_local * group * self.C * 2 * r * d
            owners[a] = L
        tot += sum(owners.values()) * hkv_local * 2 * r * d  # rebuild K_lora (DEFERRED form)
        return tot


def _cpu_baseline(wl, mode, seed, max_seqs, budget_s=20.0):
    """The fp64 oracle, as it stands, on the host cores: a bounded sample of
    the workload at layer 0, extrapolated to every layer (and, for prefill,
    from a sample of the chunk's query rows to the whole chunk)."""
    from oracle import ra
    from workloads import recipes
    fr = ra.inv_freq(wl.d, 500000.0, llama3=True)
    threads = min(8, os.cpu_count() or 1)
    q_sample = min(wl.C, 4)
    done, spent = 0, 0.0
    for a in wl.batch[:max_seqs]:
        inp = recipes.oracle_inputs(wl.scen, seed, a, 0, wl.kv[1] - wl.kv[0], wl.d, wl.r,
                                    (wl.kv[1] - wl.kv[0]) * wl.Hq // wl.Hkv, q_sample, "bf16", kv_heads=wl.kv)
        t0 = time.perf_counter()
        ra.residual_attention(inv_freq_=fr, rope_mode=ra.ROPE_DEFERRED if mode == "deferred" else ra.ROPE_NONE,
                              threads=threads, **inp)
        spent += time.perf_counter() - t0
        done += 1
        if spent > budget_s:
            break
    # tokens: decode -> 1 per sequence; prefill -> C per sequence (sampled q_sample rows)
    per_token = spent / (done * q_sample) * wl.L
    return {"value": 1.0 / per_token, "unit": "tokens/s", "cores": threads, "kind": "oracle",
            "sample": f"{done} of {len(wl.batch)} sequences x {q_sample} query row(s), layer 0 of {wl.L} (full context, "
                      f"fp64, {threads} threads over kv heads), extrapolated x{wl.L} layers; oracle time {spent:.2f}s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = Workload(args.config)
    from oracle import ra
    from workloads import recipes
    fr = ra.inv_freq(wl.d, 500000.0, llama3=True)
    threads = min(8, os.cpu_count() or 1)
    a = wl.batch[0]
    q_sample = min(wl.C, 4)
    inp = recipes.oracle_inputs(wl.scen, args.seed, a, 0, wl.kv[1] - wl.kv[0], wl.d, wl.r,
                                (wl.kv[1] - wl.kv[0]) * wl.Hq // wl.Hkv, q_sample, "bf16", kv_heads=wl.kv)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ra.residual_attention(inv_freq_=fr, rope_mode=ra.ROPE_DEFERRED if args.mode == "deferred" else ra.ROPE_NONE,
                              threads=threads, **inp)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    per_step = sum(times) / len(times)
    value = q_sample / (per_step * wl.L)
    metric = METRIC_PREFILL if wl.kind == "prefill" else METRIC
    out = {"metric": metric, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": wl.scaling,
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": wl.desc, "rope_mode": args.mode},
           "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle",
                            "sample": f"each step: 1 sequence x {q_sample} query row(s) x layer 0 of {wl.L}, "
                                      f"extrapolated to tokens/s over all layers"},
           "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2604_06370_b200.api import ForkKV, synth_fill
    from workloads import driver, synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = Workload(args.config, world, rank)
    scen, batch, C = wl.scen, wl.batch, wl.C
    P = args.page
    B = len(batch)
    h0, h1 = wl.kv
    nb, nr = scen.pages_needed(P)
    nb += B + 8
    nr += B + 8
    max_pos = max(scen.seqlen(s.id) for s in scen.agents) + args.warmup + args.steps + 8
    t_setup = time.time()
    fkv = ForkKV(n_layers=wl.L, n_q_heads=wl.Hq, n_kv_heads=wl.Hkv, head_dim=wl.d, rank=wl.r, page_size=P,
                 n_base_pages=nb, n_res_pages=nr, dtype="bf16", rope_mode=args.mode, device=local, max_pos=max_pos,
                 rope_theta=500000.0, llama3=True, kv_heads=(h0, h1))
    hq = fkv.hq
    seed = args.seed + (1000 * rank if wl.scaling == "weak" else 0)
    driver.build(fkv, scen, seed, h0=h0)
    dev = torch.device("cuda", local)
    prefill = wl.kind == "prefill"
    n_q_rows = B * C
    Q = torch.empty(wl.L, n_q_rows, hq, wl.d, dtype=torch.bfloat16, device=dev)
    O = torch.empty_like(Q)
    for layer in range(wl.L):
        driver.make_queries(fkv, scen, seed, layer, step=1, h0=h0, out=Q[layer])
    kb = torch.empty(wl.L, B, fkv.hkv, wl.d, dtype=torch.bfloat16, device=dev)
    vb = torch.empty_like(kb)
    rk = torch.empty(wl.L, B, wl.r, dtype=torch.bfloat16, device=dev)
    rv = torch.empty_like(rk)
    for layer in range(wl.L):
        synth_fill(kb[layer], seed, synth.KIND_KBASE, 777, layer, 0, head0=h0)
        synth_fill(vb[layer], seed, synth.KIND_VBASE, 777, layer, 0, head0=h0)
        synth_fill(rk[layer], seed, synth.KIND_RK, 777, layer, 0)
        synth_fill(rv[layer], seed, synth.KIND_RV, 777, layer, 0)
    pl0 = fkv.plan([(a, C) for a in batch], upload=False)
    plan_buf = torch.empty(max(1 << 24, 2 * pl0.info.device_bytes), dtype=torch.uint8, device=dev)
    ws_buf = torch.empty(max(64, 2 * pl0.info.workspace_bytes // 4), dtype=torch.float32, device=dev)
    if prefill:
        fkv.plan_upload(pl0, dev=plan_buf, ws=ws_buf)
    torch.cuda.synchronize()
    t_setup = time.time() - t_setup
    stream = torch.cuda.current_stream()
    ones = [1] * B
    seqlens = {a: fkv.get_table(a)[2] for a in batch}   # host-side bookkeeping (no D2H)
    state = {"tok": 0, "events": [], "launches": 0, "info": pl0.info}

    def step(record=False, host=None):
        if prefill:
            pl = pl0                      # the chunk's K/V rows are resident; same plan every step
        else:
            toks = [(state["tok"] + i) % 32000 for i in range(B)]
            state["tok"] += 1
            fkv.append(batch, ones, toks)
            for a in batch:
                seqlens[a] += 1
            pl = fkv.plan([(a, 1) for a in batch], upload=False)
            fkv.plan_upload(pl, dev=plan_buf, ws=ws_buf)
            state["info"] = pl.info
        starts = [seqlens[a] - 1 for a in batch]
        for layer in range(wl.L):
            if host is None:
                if not prefill:
                    fkv.write_kv(layer, batch, starts, ones, kb[layer], vb[layer], rk[layer], rv[layer])
                    state["launches"] += 1
                if record:
                    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fkv.residual_attention_phases(pl, layer, Q[layer], O[layer], 1)
                    e1.record(stream)
                    state["events"].append((e0, e1))
                else:
                    fkv.residual_attention_phases(pl, layer, Q[layer], O[layer], 1)
                fkv.residual_attention_phases(pl, layer, Q[layer], O[layer], 2)
            else:
                if not prefill:
                    host["kv"](layer)
                    fkv.write_kv(layer, batch, starts, ones, host["dkb"], host["dvb"], host["drk"], host["drv"])
                    state["launches"] += 1
                fkv.residual_attention_host(pl, layer, host["q"][layer], host["o"][layer], host["dq"], host["do"])
            # tcgen05 path: stager + main kernel + combine; mma.sync / SIMT: main kernel + combine
            state["launches"] += 3 if pl.info.kernel == 2 else 2
        return pl

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    state["events"].clear()
    state["launches"] = 0
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(stream)
    for _ in range(args.steps):
        step(record=True)
    t1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = t0.elapsed_time(t1) / args.steps
    main_ms = [a.elapsed_time(b) for a, b in state["events"]]
    launches = state["launches"]
    info = state["info"]
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms = float(ms_t.item())
    tokens_per_step = n_q_rows
    if wl.scaling == "weak":
        value = tokens_per_step * world / (ms / 1e3)
    else:  # strong (c4): every rank holds a slice of the same batch; tokens counted once
        n_tok = torch.tensor([tokens_per_step if h0 == 0 else 0], device=dev)
        if world > 1:
            dist.all_reduce(n_tok)
        value = float(n_tok.item()) / (ms / 1e3)

    # ---- e2e: host buffers through the C-ABI ----------------------------------
    e2e = None
    if not args.no_e2e:
        qh = torch.empty(wl.L, n_q_rows, hq, wl.d, dtype=torch.bfloat16, pin_memory=True)
        qh.copy_(Q.cpu())
        oh = torch.empty_like(qh).pin_memory()
        kvh = [t.cpu().pin_memory() for t in (kb, vb, rk, rv)]
        dq = torch.empty(n_q_rows, hq, wl.d, dtype=torch.bfloat16, device=dev)
        do = torch.empty_like(dq)
        dkv = [torch.empty_like(t[0]) for t in (kb, vb, rk, rv)]

        def kv(layer):
            for dst, src in zip(dkv, kvh):
                dst.copy_(src[layer], non_blocking=True)

        host = {"q": qh, "o": oh, "dq": dq, "do": do, "kv": kv, "dkb": dkv[0], "dvb": dkv[1], "drk": dkv[2],
                "drv": dkv[3]}
        for _ in range(2):
            step(host=host)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(host=host)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        h2d = wl.L * (n_q_rows * hq * wl.d * 2 + (0 if prefill else sum(t[0].numel() * 2 for t in (kb, vb, rk, rv))))
        d2h = wl.L * n_q_rows * hq * wl.d * 2
        e2e = {"value": value * ms / float(ems.item()), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    hbm, tc, tc_sus, src = _peaks()
    avg_main = sum(main_ms) / len(main_ms)
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}_{args.mode}.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    if prefill:
        flops = wl.flops_per_layer(fkv.hkv, fkv.group)
        achieved = flops / (avg_main / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tc_sus, "unit": "TFLOP/s", "frac": achieved / tc_sus,
                "traffic": traffic, "peak_source": f"{src} (sustained bf16)", "alg_flops_per_launch": flops}
    else:
        achieved = info.alg_bytes / (avg_main / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "peak_source": src, "alg_bytes_per_launch": info.alg_bytes}
    roof.update({"kernel": "ResidualAttention main kernel (one launch per layer)", "avg_launch_ms": avg_main,
                 "share_of_step": sum(main_ms) / args.steps / ms})
    out = {
        "metric": METRIC_PREFILL if prefill else METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": wl.scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": wl.desc, "rope_mode": args.mode, "batch_per_gpu": B, "q_rows_per_seq": C,
                   "page_size": P, "keys_per_seq": max(scen.seqlen(a) for a in batch) + (0 if prefill else args.warmup),
                   "layers": wl.L, "kv_heads": [h0, h1], "parallelism": wl.parallelism,
                   "l2": "inputs larger than L2 (each step streams the whole per-layer cache, >>126 MB)",
                   "kernel": {0: "mma.sync grouped", 1: "simt", 2: "tcgen05"}.get(info.kernel, "?"),
                   "setup_s": round(t_setup, 1)},
        "roofline": roof,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if e2e:
        out["e2e"] = e2e
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = _cpu_baseline(wl, args.mode, seed, args.cpu_seqs)
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--mode", default="none", choices=["deferred", "none"],
                    help="none = the north-star split q(K_base + R_K B_K)^T = qK_base^T + (qB_K^T)R_K^T (default); "
                         "deferred = the paper's RoPE on the rebuilt residual (Alg.1), DESIGN.md C-1")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seqs", type=int, default=8)
    ap.add_argument("--page", type=int, default=128, help="tokens per KV page (DESIGN.md C-9)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
