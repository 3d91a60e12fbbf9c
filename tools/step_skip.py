"""Critical-path share of each side kernel in the C2 decode step (diagnostic, GPU, wrong output): times the bench
step with the combine, the kv_write and/or the stager launch skipped (FKV_DIAG_* set after the setup writes).

    python tools/step_skip.py [--steps 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    a.config, a.mode, a.page, a.seed, a.warmup = "c2", "none", 128, 0, 3
    torch.cuda.set_device(0)
    wl = bench.Workload("c2", 1, 0)
    run = bench.Run(a, wl, "none", 1, 0, 0)
    for _ in range(3):
        run.step()
    torch.cuda.synchronize()
    for name, envs in [("baseline", []), ("no combine", ["FKV_DIAG_NOCOMBINE"]), ("no kv_write", ["FKV_DIAG_NOKVWRITE"]),
                       ("no kv_write + combine", ["FKV_DIAG_NOCOMBINE", "FKV_DIAG_NOKVWRITE"]), ("baseline", [])]:
        for e in envs:
            os.environ[e] = "1"
        for _ in range(2):
            run.step()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.steps):
            run.step()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:24s} {e0.elapsed_time(e1) / a.steps:.3f} ms/step")
        for e in envs:
            del os.environ[e]


if __name__ == "__main__":
    main()
