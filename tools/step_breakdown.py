"""Where one decode step's time goes (diagnostic, GPU): host time of append / plan / upload, and CUDA-event
durations of kv_write, phase 1 (stager + main), phase 2 (combine) per layer, plus the idle gap.

    python tools/step_breakdown.py [--config c2] [--mode none] [--steps 5]
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--mode", default="none")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--page", type=int, default=128)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    wl = bench.Workload(a.config, 1, 0)
    run = bench.Run(a, wl, a.mode, 1, 0, 0)
    for _ in range(a.warmup):
        run.step()
    torch.cuda.synchronize()
    fkv, batch, B = run.fkv, wl.batch, run.B
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    host = {"append": [], "plan": [], "upload": [], "enqueue": []}
    gpu = {"upload": [], "kv_write": [], "phase1": [], "phase2": [], "step": []}
    for _ in range(a.steps):
        torch.cuda.synchronize()
        s0 = E(); s0.record()
        t0 = time.perf_counter()
        fkv.append(batch, [1] * B, [7] * B)
        for x in batch:
            run.seqlens[x] += 1
        t1 = time.perf_counter()
        pl = fkv.plan([(x, 1) for x in batch], upload=False)
        t2 = time.perf_counter()
        u0 = E(); u0.record()
        fkv.plan_upload(pl, dev=run.plan_buf, ws=run.ws_buf)
        u1 = E(); u1.record()
        t3 = time.perf_counter()
        starts = [run.seqlens[x] - 1 for x in batch]
        ev = []
        for layer in range(wl.L):
            e = [E() for _ in range(4)]
            e[0].record()
            fkv.write_kv(layer, batch, starts, [1] * B, run.kb[layer], run.vb[layer], run.rk[layer], run.rv[layer])
            e[1].record()
            fkv.residual_attention_phases(pl, layer, run.Q[layer], run.O[layer], 1)
            e[2].record()
            fkv.residual_attention_phases(pl, layer, run.Q[layer], run.O[layer], 2)
            e[3].record()
            ev.append(e)
        t4 = time.perf_counter()
        s1 = E(); s1.record()
        torch.cuda.synchronize()
        host["append"].append((t1 - t0) * 1e3); host["plan"].append((t2 - t1) * 1e3)
        host["upload"].append((t3 - t2) * 1e3); host["enqueue"].append((t4 - t3) * 1e3)
        gpu["upload"].append(u0.elapsed_time(u1))
        gpu["kv_write"].append(sum(e[0].elapsed_time(e[1]) for e in ev))
        gpu["phase1"].append(sum(e[1].elapsed_time(e[2]) for e in ev))
        gpu["phase2"].append(sum(e[2].elapsed_time(e[3]) for e in ev))
        gpu["step"].append(s0.elapsed_time(s1))
    med = {k: statistics.median(v) for k, v in list(host.items()) + [("gpu_" + k, v) for k, v in gpu.items()]}
    L = wl.L
    print(f"config {a.config} mode {a.mode} kernel {pl.info.kernel} layers {L}")
    for k in host:
        print(f"  host {k:10s} {med[k]:8.3f} ms / step")
    for k in gpu:
        print(f"  gpu  {k:10s} {med['gpu_' + k]:8.3f} ms / step  {med['gpu_' + k] / L * 1e3:8.1f} us / layer")
    other = med["gpu_step"] - med["gpu_kv_write"] - med["gpu_phase1"] - med["gpu_phase2"]
    print(f"  gpu  other      {other:8.3f} ms / step  (append kernels, upload, host-bound idle)")


if __name__ == "__main__":
    main()
