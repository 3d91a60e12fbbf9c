"""Host-side cost of each per-layer API call of a decode step (diagnostic, GPU): the bench loop is host-bound when
these add up to more than the GPU time of a layer.

    python tools/host_overhead.py [--config c2]
"""
import argparse
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import numpy as np
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--mode", default="none")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--page", type=int, default=128)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--n", type=int, default=64)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    wl = bench.Workload(a.config, 1, 0)
    run = bench.Run(a, wl, a.mode, 1, 0, 0)
    run.step()
    torch.cuda.synchronize()
    fkv, batch, B, pl = run.fkv, wl.batch, run.B, run.pl
    starts = [run.seqlens[x] - 1 for x in batch]
    ones = [1] * B
    na, ns, no = np.asarray(batch, np.int64), np.asarray(starts, np.int64), np.ones(B, np.int32)
    st = torch.cuda.current_stream()
    calls = {
        "write_kv(lists)": lambda: fkv.write_kv(0, batch, starts, ones, run.kb[0], run.vb[0], run.rk[0], run.rv[0]),
        "write_kv(numpy,stream)": lambda: fkv.write_kv(0, na, ns, no, run.kb[0], run.vb[0], run.rk[0], run.rv[0],
                                                       stream=st),
        "phases(1)": lambda: fkv.residual_attention_phases(pl, 0, run.Q[0], run.O[0], 1),
        "phases(1,stream)": lambda: fkv.residual_attention_phases(pl, 0, run.Q[0], run.O[0], 1, stream=st),
        "phases(2)": lambda: fkv.residual_attention_phases(pl, 0, run.Q[0], run.O[0], 2),
        "current_stream": lambda: torch.cuda.current_stream(),
        "plan": lambda: fkv.plan([(x, 1) for x in batch], upload=False),
        "plan_upload": lambda: fkv.plan_upload(pl, dev=run.plan_buf, ws=run.ws_buf),
    }
    for name, f in calls.items():
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(a.n):
                f()
            ts.append((time.perf_counter() - t0) / a.n * 1e6)
        torch.cuda.synchronize()
        print(f"{name:26s} {statistics.median(ts):9.1f} us / call")
    # the raw C call without Python marshalling
    lib = fkv.lib
    pa, ps, pc = (na.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ns.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                  no.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    sh = ctypes.c_void_p(st.cuda_stream)
    args = [ctypes.c_void_p(t.data_ptr()) for t in (run.kb[0], run.vb[0], run.rk[0], run.rv[0])]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.n):
        lib.fkv_write_kv(fkv.ctx, 0, B, pa, ps, pc, *args, 15, sh)
    print(f"{'fkv_write_kv (raw ctypes)':26s} {(time.perf_counter() - t0) / a.n * 1e6:9.1f} us / call")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
