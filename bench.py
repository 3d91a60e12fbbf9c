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

import numpy as np

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

    def __init__(self, name, world=1, rank=0, fanout_rank=(16, 64)):
        from workloads import recipes
        self.name, self.kind, self.scaling = name, "decode", "weak"
        self.L, self.Hq, self.Hkv, self.d, self.r = 32, 32, 8, 128, 16
        self.r_eff = None
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
        elif name == "sweep":
            # configs[4]: rank r x fork fan-out N. Ranks below 16 are zero-padded into a rank-16 pool (C-8: exact) so
            # the tcgen05 kernel runs them; the roofline counts the r-wide bytes only (the padding is overhead)
            R, N = int(fanout_rank[0]), int(fanout_rank[1])
            self.r_eff, self.r = R, (16 if R <= 16 else R)
            self.scen = recipes.fanout(N)
            self.desc = (f"configs[4] sweep point: Llama-3.1-8B 32 layers, fork fan-out {N} agents (distinct adapters, "
                         f"own residual) over a 32K prefix, LoRA rank {R}" +
                         (f" (zero-padded into a rank-{self.r} pool, C-8)" if self.r != R else ""))
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

    def flops_per_layer(self, hkv_local, group, mode="none"):
        """Algorithmic FLOPs of one layer (minimal form): QK^T and PV over the visible keys of every query row,
        the rank-r terms per (row, key) (NONE: q~.R_k and P.R_v; DEFERRED: q.K_lora and P.R_v), q~ and the late
        fusion per row, and for DEFERRED the rank-r rebuild K_lora = R_k B_k per (residual owner, kv head, key)."""
        d, r = self.d, self.r
        tot = 0
        owners = {}
        for a in self.batch:
            L = self.scen.seqlen(a)
            vis = sum(L - self.C + i + 1 for i in range(self.C))  # causal visible keys over the chunk
            rank_term = 2 * r + (2 * d if mode == "deferred" else 2 * r)
            tot += hkv_local * group * vis * (2 * d + 2 * d + rank_term) + hkv_local * group * self.C * 4 * r * d
            # a same-agent branch shares its parent's residual pages over the prefix (one owner there)
            s = self.scen.spec(a)
            key = s.parent if (s.share_res and s.parent is not None) else a
            owners[key] = max(owners.get(key, 0), L)
        if mode == "deferred":
            tot += sum(owners.values()) * hkv_local * 2 * r * d  # rebuild K_lora = R_k B_k
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
        inp = recipes.oracle_inputs(wl.scen, seed, a, 0, wl.kv[1] - wl.kv[0], wl.d, wl.r_eff or wl.r,
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
    return {"value": 1.0 / per_token, "unit": "tokens/s", "cores": threads, "kind": "oracle", "host": _host_cpu_info(),
            "sample": f"{done} of {len(wl.batch)} sequences x {q_sample} query row(s), layer 0 of {wl.L} (full context, "
                      f"fp64, {threads} threads over kv heads), extrapolated x{wl.L} layers; oracle time {spent:.2f}s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = Workload(args.config, 1, 0, (getattr(args, "rank", 16), getattr(args, "fanout", 64)))
    from oracle import ra
    from workloads import recipes
    fr = ra.inv_freq(wl.d, 500000.0, llama3=True)
    threads = min(8, os.cpu_count() or 1)
    a = wl.batch[0]
    q_sample = min(wl.C, 4)
    inp = recipes.oracle_inputs(wl.scen, args.seed, a, 0, wl.kv[1] - wl.kv[0], wl.d, wl.r_eff or wl.r,
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
                            "host": _host_cpu_info(),
                            "sample": f"each step: 1 sequence x {q_sample} query row(s) x layer 0 of {wl.L}, "
                                      f"extrapolated to tokens/s over all layers"},
           "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def _host_cpu_info():
    """nproc, the cgroup CPU quota and the CPU model of the host (SURVEY §8(d) oracle timing)."""
    info = {"nproc": os.cpu_count()}
    try:
        info["affinity"] = len(os.sched_getaffinity(0))
    except Exception:
        pass
    try:
        q, per = open("/sys/fs/cgroup/cpu.max").read().split()
        info["cgroup_cpu_quota"] = None if q == "max" else round(int(q) / int(per), 2)
    except Exception:
        info["cgroup_cpu_quota"] = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu_model"] = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return info


KERNEL_NAMES = {0: "mma.sync grouped (baseline)", 1: "simt", 2: "tcgen05 keys-on-lanes",
                3: "tcgen05 rows-on-lanes"}


def alg_bytes_of(info, wl):
    """The planner's algorithmic bytes per layer; for an adapter rank r_eff zero-padded into a rank-r pool only the
    r_eff-wide part of the rank-proportional bytes (residual pages + adapters) counts."""
    if wl.r_eff is None or wl.r_eff == wl.r:
        return info.alg_bytes
    return info.alg_bytes - info.alg_rank_bytes * (wl.r - wl.r_eff) // wl.r


def _launches_per_layer(kernel):
    """Our kernels per layer: main (+ the stager of kernel 2) + combine."""
    return 3 if kernel == 2 else 2


class Run:
    """One configured workload on this rank: the control plane, resident pools, Q/O and new-row buffers."""

    def __init__(self, args, wl, mode, world, rank, dev_index):
        import torch
        from paper_2604_06370_b200.api import ForkKV, synth_fill
        from workloads import driver, synth
        self.args, self.wl, self.mode = args, wl, mode
        scen, batch, C = wl.scen, wl.batch, wl.C
        P = args.page
        B = len(batch)
        self.B, self.C, self.P = B, C, P
        self.h0, self.h1 = wl.kv
        nb, nr = scen.pages_needed(P)
        nb += B + 8
        nr += B + 8
        # every timed / warm-up / e2e decode step appends one token per sequence (DEFERRED needs the RoPE table to
        # cover them: ADVICE r1)
        appends = args.warmup + 3 * args.steps + 4
        max_pos = max(scen.seqlen(s.id) for s in scen.agents) + appends + 16
        t_setup = time.time()
        self.fkv = fkv = ForkKV(n_layers=wl.L, n_q_heads=wl.Hq, n_kv_heads=wl.Hkv, head_dim=wl.d, rank=wl.r,
                                page_size=P, n_base_pages=nb, n_res_pages=nr, dtype="bf16", rope_mode=mode,
                                device=dev_index, max_pos=max_pos, rope_theta=500000.0, llama3=True,
                                kv_heads=(self.h0, self.h1))
        hq = fkv.hq
        self.hq = hq
        self.seed = seed = args.seed + (1000 * rank if wl.scaling == "weak" else 0)
        driver.build(fkv, scen, seed, h0=self.h0, r_eff=wl.r_eff)
        dev = self.dev = torch.device("cuda", dev_index)
        self.prefill = wl.kind == "prefill"
        self.n_q_rows = B * C
        self.Q = torch.empty(wl.L, self.n_q_rows, hq, wl.d, dtype=torch.bfloat16, device=dev)
        self.O = torch.empty_like(self.Q)
        for layer in range(wl.L):
            driver.make_queries(fkv, scen, seed, layer, step=1, h0=self.h0, out=self.Q[layer])
        self.kb = torch.empty(wl.L, B, fkv.hkv, wl.d, dtype=torch.bfloat16, device=dev)
        self.vb = torch.empty_like(self.kb)
        self.rk = torch.empty(wl.L, B, wl.r, dtype=torch.bfloat16, device=dev)
        self.rv = torch.empty_like(self.rk)
        for layer in range(wl.L):
            synth_fill(self.kb[layer], seed, synth.KIND_KBASE, 777, layer, 0, head0=self.h0)
            synth_fill(self.vb[layer], seed, synth.KIND_VBASE, 777, layer, 0, head0=self.h0)
            synth_fill(self.rk[layer], seed, synth.KIND_RK, 777, layer, 0)
            synth_fill(self.rv[layer], seed, synth.KIND_RV, 777, layer, 0)
        if wl.r_eff is not None and wl.r_eff < wl.r:
            self.rk[:, :, wl.r_eff:] = 0
            self.rv[:, :, wl.r_eff:] = 0
        self.pl0 = fkv.plan([(a, C) for a in batch], upload=False)
        self.plan_buf = torch.empty(max(1 << 24, 2 * self.pl0.info.device_bytes), dtype=torch.uint8, device=dev)
        self.ws_buf = torch.empty(max(64, 2 * self.pl0.info.workspace_bytes // 4), dtype=torch.float32, device=dev)
        if self.prefill:
            fkv.plan_upload(self.pl0, dev=self.plan_buf, ws=self.ws_buf)
        torch.cuda.synchronize()
        self.t_setup = time.time() - t_setup
        self.stream = torch.cuda.current_stream()
        self.batch_np = np.asarray(wl.batch, np.int64)
        self.ones_np = np.ones(len(wl.batch), np.int32)
        self.seqlens = {a: fkv.get_table(a)[2] for a in batch}   # host-side bookkeeping (no D2H)
        self.tok = 0
        self.events, self.launches, self.alg_bytes, self.info = [], 0, [], self.pl0.info
        self.pl = self.pl0

    def step(self, record=False, host=None, events=None):
        """One pass of the whole hot path over one batch: (decode) append + plan + upload, then per layer
        kv_write + main kernel + combine."""
        import torch
        fkv, wl, batch = self.fkv, self.wl, self.wl.batch
        B, ones = self.B, [1] * self.B
        if self.prefill:
            pl = self.pl0                     # the chunk's K/V rows are resident; same plan every step
        else:
            toks = [(self.tok + i) % 32000 for i in range(B)]
            self.tok += 1
            fkv.append(batch, ones, toks)
            for a in batch:
                self.seqlens[a] += 1
            pl = fkv.plan([(a, 1) for a in batch], upload=False)
            fkv.plan_upload(pl, dev=self.plan_buf, ws=self.ws_buf)
            self.info = pl.info
        self.pl = pl
        if record:
            self.alg_bytes.append(alg_bytes_of(pl.info, self.wl))
        # per-step host arrays built once (numpy, contiguous) and the stream passed explicitly: the per-layer calls
        # then skip the list -> array conversions and the current-stream lookup (host cost per layer ~63 -> ~40 us)
        starts = np.asarray([self.seqlens[a] - 1 for a in batch], np.int64)
        b_np, ones_np, st = self.batch_np, self.ones_np, self.stream
        Q, O = self.Q, self.O
        for layer in range(wl.L):
            if host is None:
                if not self.prefill:
                    fkv.write_kv(layer, b_np, starts, ones_np, self.kb[layer], self.vb[layer], self.rk[layer],
                                 self.rv[layer], stream=st)
                    self.launches += 1
                if record if events is None else events:
                    # the dominant kernel alone: kernel 2's operand stager is launched before the event window
                    # (FKV_PHASE_STAGE), the main kernel inside it (FKV_PHASE_MAIN | FKV_PHASE_NOSTAGE)
                    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                    split = pl.info.kernel == 2
                    if split:
                        fkv.residual_attention_phases(pl, layer, Q[layer], O[layer], 4, stream=st)
                    e0.record(self.stream)
                    fkv.residual_attention_phases(pl, layer, Q[layer], O[layer], 9 if split else 1, stream=st)
                    e1.record(self.stream)
                    self.events.append((e0, e1))
                else:
                    fkv.residual_attention_phases(pl, layer, Q[layer], O[layer], 1, stream=st)
                fkv.residual_attention_phases(pl, layer, Q[layer], O[layer], 2, stream=st)
            else:
                self._host_layer(host, pl, layer, starts)
            self.launches += _launches_per_layer(pl.info.kernel)
        if host is not None:
            self._host_drain(host)
        return pl

    def _host_layer(self, host, pl, layer, starts):
        """e2e leg, one layer: the public calls a serving loop makes (write_kv + residual_attention) on this step's
        device staging buffer, which the copy stream filled from pinned host memory while the previous step ran."""
        fkv, batch = self.fkv, self.wl.batch
        b = host["k"] & 1
        dv = host["dev"][b]
        if layer == 0:
            self.stream.wait_event(host["ev_in"][b])      # this step's inputs are on the device
        if not self.prefill:
            fkv.write_kv(layer, self.batch_np, starts, self.ones_np, dv["kb"][layer], dv["vb"][layer],
                         dv["rk"][layer], dv["rv"][layer], stream=self.stream)
            self.launches += 1
        fkv.residual_attention(pl, layer, dv["q"][layer], dv["o"][layer], stream=self.stream)

    def _host_h2d(self, host, k):
        """Step k's inputs (every layer's Q rows and new K/V/residual rows) pinned host -> device buffer k & 1, on
        the H2D copy stream, once step k - 2 (the buffer's previous user) and its D2H are done with it."""
        import torch
        b = k & 1
        dv, cs = host["dev"][b], host["cs_in"]
        with torch.cuda.stream(cs):
            for e in (host["done"][b], host["out"][b]):
                if e is not None:
                    cs.wait_event(e)
            dv["q"].copy_(host["q"], non_blocking=True)
            if not self.prefill:
                for key in ("kb", "vb", "rk", "rv"):
                    dv[key].copy_(host["kv"][key], non_blocking=True)
            host["ev_in"][b].record(cs)

    def _host_d2h(self, host, k):
        """Step k's result (every layer's O) device -> pinned host, on the D2H copy stream behind step k."""
        import torch
        b = k & 1
        cs = host["cs_out"]
        with torch.cuda.stream(cs):
            cs.wait_event(host["done"][b])
            host["o"].copy_(host["dev"][b]["o"], non_blocking=True)
            e = torch.cuda.Event()
            e.record(cs)
            host["out"][b] = e

    def _host_drain(self, host):
        """After step k's launches: its completion event; then step k + 1's inputs go H2D (they only wait for step
        k - 1) and step k's O goes D2H on a second copy stream, both while step k + 1 computes (steps pipelined as
        in a serving loop; PCIe is full duplex)."""
        import torch
        k = host["k"]
        e = torch.cuda.Event()
        e.record(self.stream)
        host["done"][k & 1] = e
        self._host_h2d(host, k + 1)
        self._host_d2h(host, k)
        host["k"] = k + 1

    def _host_join(self, host):
        """End of the timed steps: the compute stream waits for the last step's O to reach the host (and for the
        next step's inputs, already issued)."""
        import torch
        for cs in (host["cs_in"], host["cs_out"]):
            e = torch.cuda.Event()
            e.record(cs)
            self.stream.wait_event(e)

    def graph_median_ms(self, reps=25):
        """Main-kernel time of layer 0 as the median over `reps` CUDA-graph replays."""
        import torch
        try:
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            # kernel 2: the stager runs once outside the graph (its images stay valid for layer 0), the graph holds
            # the main kernel alone, as the event window does
            ph = 9 if self.pl.info.kernel == 2 else 1
            with torch.cuda.stream(s):
                self.fkv.residual_attention_phases(self.pl, 0, self.Q[0], self.O[0], 1)  # warm on the side stream
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=s):
                    self.fkv.residual_attention_phases(self.pl, 0, self.Q[0], self.O[0], ph)
            torch.cuda.synchronize()
            ts = []
            with torch.cuda.stream(s):                    # replay() launches on the current stream
                for _ in range(reps + 5):
                    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    g.replay()
                    e1.record(s)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
            return statistics.median(ts[5:])
        except Exception as e:  # capture is a measurement aid, not part of the hot path
            print(f"graph timing unavailable: {e}", file=sys.stderr)
            return None

    def free(self):
        import torch
        del self.fkv, self.Q, self.O, self.kb, self.vb, self.rk, self.rv, self.plan_buf, self.ws_buf
        torch.cuda.empty_cache()


def _timed(run, args, world, dist_ok, dev_index):
    """Warm-up, then exactly args.steps steps between barrier + synchronize; returns (ms per step, clocks)."""
    import torch
    import torch.distributed as dist
    for _ in range(args.warmup):
        run.step()
    torch.cuda.synchronize()
    if world > 1 and dist_ok:
        dist.barrier()
    clk = ClockSampler(dev_index)
    clk.start()
    time.sleep(0.3)
    run.events.clear()
    run.alg_bytes.clear()
    run.launches = 0
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(run.stream)
    # the timed steps carry no per-kernel events: an event recorded between two PDL-chained launches makes the
    # second wait for the first to drain (the overlap a serving loop gets); the kernel times for the roofline come
    # from the instrumented pass below (same steps, same inputs)
    nvtx = bool(os.environ.get("FKV_NVTX"))   # ncu --nvtx --nvtx-include "timed/": the launch list of these steps
    if nvtx:
        torch.cuda.nvtx.range_push("timed")
    for _ in range(args.steps):
        run.step(record=True, events=bool(os.environ.get("FKV_BENCH_EVENTS_IN_TIMED")))
    if nvtx:
        torch.cuda.nvtx.range_pop()
    t1.record(run.stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    if not run.events:
        launches = run.launches   # gpu_launches counts the timed steps only
        for _ in range(args.steps):
            run.step(record=False, events=True)
        torch.cuda.synchronize()
        run.launches = launches
    clocks = clk.stop()
    return ms, clocks


def _max_over_ranks(x, world):
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x, world):
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t)
    return float(t.item())


def tokens_value(tokens_per_step_rank, ms_max, world, scaling, counts_tokens, sum_fn=None):
    """Whole-job tokens/s: weak scaling counts every rank's own batch; strong scaling (c4: every rank holds a slice
    of ONE batch) counts each sequence once (the ranks of head shard 0). `sum_fn` sums over ranks."""
    sum_fn = sum_fn or (lambda x: x)
    if scaling == "weak":
        return tokens_per_step_rank * world / (ms_max / 1e3)
    return sum_fn(tokens_per_step_rank if counts_tokens else 0) / (ms_max / 1e3)


def _roofline(run, wl, ms, hbm, tc_sus, src, config_name, mode):
    main_ms = [a.elapsed_time(b) for a, b in run.events]
    avg_main = sum(main_ms) / len(main_ms)
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{config_name}_{mode}.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    kname = KERNEL_NAMES.get(run.info.kernel, "?")
    window = "main kernel only (kernel 2: its stager launched before the window)"
    if run.prefill:
        flops = wl.flops_per_layer(run.fkv.hkv, run.fkv.group, mode)
        achieved = flops / (avg_main / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tc_sus, "unit": "TFLOP/s", "frac": achieved / tc_sus,
                "traffic": traffic, "peak_source": f"{src} (sustained bf16)", "alg_flops_per_launch": flops}
    else:
        alg = statistics.mean(run.alg_bytes)   # the timed steps' own bytes (each step appends one token)
        achieved = alg / (avg_main / 1e3) / 1e9
        layer_ms = ms / wl.L
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "peak_source": src, "alg_bytes_per_launch": alg,
                "frac_whole_layer": alg / (layer_ms / 1e3) / 1e9 / hbm,
                "frac_vs_8tbs_spec": achieved / 8000.0}
        # the other roof (decode lines against both): algorithmic FLOPs of the layer (QK^T, PV, the
        # rank-r terms; the workload's sequence lengths) over the same launch time vs sustained bf16
        flops = wl.flops_per_layer(run.fkv.hkv, run.fkv.group, mode)
        roof["tensor_achieved_tflops"] = flops / (avg_main / 1e3) / 1e12
        roof["tensor_frac"] = roof["tensor_achieved_tflops"] / tc_sus
    roof.update({"kernel": f"ResidualAttention {kname} (one launch per layer)", "event_window": window,
                 "avg_launch_ms": avg_main, "share_of_step": sum(main_ms) / len(run.alg_bytes or [1]) / ms})
    return roof


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_dev = torch.cuda.device_count()
    if n_dev < 1:
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    dev_index = local % n_dev
    torch.cuda.set_device(dev_index)
    if world > 1:
        # the hot path has no data-path collective: ranks exchange only scalars (barrier, max time,
        # token counts), over gloo so that ranks sharing one GPU work too
        dist.init_process_group("gloo")
    wl = Workload(args.config, world, rank, (args.rank, args.fanout))
    run = Run(args, wl, args.mode, world, rank, dev_index)
    ms, clocks = _timed(run, args, world, True, dev_index)
    launches = run.launches
    ms = _max_over_ranks(ms, world)
    value = tokens_value(run.n_q_rows, ms, world, wl.scaling, run.h0 == 0, lambda x: _sum_over_ranks(x, world))
    graph_ms = run.graph_median_ms() if not args.no_graph else None

    # ---- e2e: host buffers through the C-ABI ----------------------------------
    e2e = None
    if not args.no_e2e:
        L_, hq, d = wl.L, run.hq, wl.d
        qh = torch.empty(L_, run.n_q_rows, hq, d, dtype=torch.bfloat16, pin_memory=True)
        qh.copy_(run.Q.cpu())
        oh = torch.empty_like(qh).pin_memory()
        kvh = {k: t.cpu().pin_memory() for k, t in zip(("kb", "vb", "rk", "rv"), (run.kb, run.vb, run.rk, run.rv))}
        # two step-sized device staging buffers (every layer's inputs and outputs): step k computes on buffer
        # k & 1 while the copy stream brings step k - 1's O to the host and step k + 1's inputs to the device
        devb = [{"q": torch.empty_like(run.Q), "o": torch.empty_like(run.Q),
                 **{k: torch.empty_like(t) for k, t in zip(("kb", "vb", "rk", "rv"),
                                                           (run.kb, run.vb, run.rk, run.rv))}} for _ in range(2)]
        host = {"q": qh, "o": oh, "kv": kvh, "dev": devb, "cs_in": torch.cuda.Stream(device=run.dev),
                "cs_out": torch.cuda.Stream(device=run.dev), "ev_in": [torch.cuda.Event(), torch.cuda.Event()],
                "done": [None, None], "out": [None, None], "k": 0}
        run._host_h2d(host, 0)
        for _ in range(2):
            run.step(host=host)
        run._host_join(host)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(run.stream)
        # the timed region holds every step's H2D and D2H: the first step's inputs were copied before e0 by the
        # warm-up's pipeline, so one extra step's inputs (the step after the last) go H2D inside it instead
        for _ in range(args.steps):
            run.step(host=host)
        run._host_join(host)
        e1.record(run.stream)
        torch.cuda.synchronize()
        ems = _max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
        h2d = L_ * (run.n_q_rows * hq * d * 2 + (0 if run.prefill else
                                                 sum(t[0].numel() * 2 for t in (run.kb, run.vb, run.rk, run.rv))))
        if not run.prefill:
            h2d += run.info.device_bytes   # the step's plan blob (fkv_plan_upload)
        d2h = L_ * run.n_q_rows * hq * d * 2
        e2e = {"value": value * ms / ems, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}

    hbm, tc, tc_sus, src = _peaks()
    roof = _roofline(run, wl, ms, hbm, tc_sus, src, args.config, args.mode)
    if graph_ms:
        roof["graph_median_launch_ms"] = graph_ms
        if not run.prefill:
            roof["frac_graph_median"] = statistics.mean(run.alg_bytes) / (graph_ms / 1e3) / 1e9 / hbm
    cfg = {"workload": wl.desc, "rope_mode": args.mode, "batch_per_gpu": run.B, "q_rows_per_seq": run.C,
           "page_size": run.P, "keys_per_seq": max(wl.scen.seqlen(a) for a in wl.batch) + (0 if run.prefill else
                                                                                         args.warmup),
           "layers": wl.L, "kv_heads": [run.h0, run.h1], "parallelism": wl.parallelism,
           "l2": "inputs larger than L2 (each step streams the whole per-layer cache, >>126 MB)",
           "kernel": KERNEL_NAMES.get(run.info.kernel, "?"), "setup_s": round(run.t_setup, 1)}
    deferred = None
    if args.mode == "none" and not args.no_deferred and args.config == "c2" and wl.kind == "decode":
        # the paper's own semantics (RoPE on the rebuilt residual, Alg1.335) timed in the same invocation
        run.free()
        drun = Run(args, wl, "deferred", world, rank, dev_index)
        dms, dclk = _timed(drun, args, world, True, dev_index)
        dms = _max_over_ranks(dms, world)
        droof = _roofline(drun, wl, dms, hbm, tc_sus, src, args.config, "deferred")
        deferred = {"value": tokens_value(drun.n_q_rows, dms, world, wl.scaling, drun.h0 == 0,
                                          lambda x: _sum_over_ranks(x, world)),
                    "unit": "tokens/s", "ms_per_step": dms, "kernel": KERNEL_NAMES.get(drun.info.kernel, "?"),
                    "roofline_frac": droof["frac"], "avg_launch_ms": droof["avg_launch_ms"], "clocks": dclk,
                    "gpu_launches": drun.launches}
        drun.free()
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    out = {
        "metric": METRIC_PREFILL if run.prefill else METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": wl.scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": cfg, "roofline": roof, "gpu_launches": launches, "clocks": clocks,
    }
    if e2e:
        out["e2e"] = e2e
    if deferred:
        out["deferred"] = deferred
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = _cpu_baseline(wl, args.mode, run.seed, args.cpu_seqs)
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
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "sweep"])
    ap.add_argument("--rank", type=int, default=16, help="sweep: LoRA rank (8 / 16 / 64)")
    ap.add_argument("--fanout", type=int, default=64, help="sweep: agents forked from the prefix (4..256)")
    ap.add_argument("--mode", default="none", choices=["deferred", "none"],
                    help="none = the north-star split q(K_base + R_K B_K)^T = qK_base^T + (qB_K^T)R_K^T (default); "
                         "deferred = the paper's RoPE on the rebuilt residual (Alg.1), DESIGN.md C-1")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-deferred", action="store_true", help="skip the DEFERRED (paper semantics) sub-result")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph median main-kernel timing")
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
