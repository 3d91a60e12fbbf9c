"""Pipeline timeline of one CTA of the rows-on-lanes tcgen05 kernel (ra_rows.cu; diagnostics).

    python tools/timeline_rows.py [--block B] [--config c2|c1|c5] [--tiles 12]

Builds one layer of the workload, times the main kernel, then runs it once with fkv_debug_timeline enabled
for CTA B and prints per-tile event times (clock64 cycles from the first event) plus the per-CTA durations."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EV = {0: "S:start", 1: "S:commit", 2: "PV:start", 3: "PV:commit", 4: "W0:sfull", 5: "W0:pfull", 6: "K:issue",
      16: "K:landed", 15: "V:issue", 17: "V:landed", 18: "Rk:issue", 19: "Rk:landed", 20: "Rv:issue", 21: "Rv:landed"}
COLS = [6, 16, 18, 19, 0, 1, 4, 5, 15, 17, 20, 21, 2, 3]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--tiles", type=int, default=16)
    ap.add_argument("--first", type=int, default=0)
    ap.add_argument("--page", type=int, default=128)
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2604_06370_b200 import _lib as L
    from paper_2604_06370_b200.api import ForkKV
    from workloads import driver, recipes
    scen = {"c2": recipes.c2, "c1": recipes.c1, "c5": recipes.c5}[a.config]()
    nb, nr = scen.pages_needed(a.page)
    fkv = ForkKV(n_layers=1, n_q_heads=32, n_kv_heads=8, head_dim=128, rank=16, page_size=a.page,
                 n_base_pages=nb, n_res_pages=nr, rope_mode="none", device=0, max_pos=40000, rope_theta=500000.0,
                 llama3=True)
    driver.build(fkv, scen, 0)
    pl = fkv.plan([(x, scen.q_len) for x in scen.batch()])
    Q = driver.make_queries(fkv, scen, 0, 0)
    O = torch.empty_like(Q)
    for _ in range(3):
        fkv.residual_attention(pl, 0, Q, O)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fkv.residual_attention_phases(pl, 0, Q, O, 1)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    print(f"kernel {pl.info.kernel} items={pl.info.n_items} main kernel avg {us:.1f} us; alg bytes/layer "
          f"{pl.info.alg_bytes / 1e6:.1f} MB -> {pl.info.alg_bytes / us / 1e3:.0f} GB/s")
    dbg = torch.zeros(32 * 512, dtype=torch.int64, device="cuda")
    lib = L.load()
    lib.fkv_debug_timeline(fkv.ctx, ctypes.c_void_p(dbg.data_ptr()), a.block)
    fkv.residual_attention_phases(pl, 0, Q, O, 1)
    torch.cuda.synchronize()
    lib.fkv_debug_timeline(fkv.ctx, None, 0)
    d = dbg.view(32, 512).cpu().numpy()
    ev = d[:22]
    t0 = ev[ev > 0].min()
    rel = lambda e, i: int(d[e, i] - t0) if d[e, i] else -1
    print("tile  " + " ".join(f"{EV[e]:>10s}" for e in COLS))
    for j in range(a.first, a.first + a.tiles):
        print(f"{j:4d}  " + " ".join(f"{rel(e, j):10d}" for e in COLS))
    n_items = int(d[31, a.block])
    for i in range(min(n_items, 16)):
        print(f"item {i}: S q_full {rel(8, i)}, S qt_full {rel(9, i)}, aux q~ done {rel(10, i)}, "
              f"epilogue start {rel(11, i)} done {rel(12, i)}")
    pf = np.array([d[5, j] for j in range(512) if d[5, j]])
    if len(pf) > 2:
        gaps = np.diff(pf)
        print(f"softmax p_full period: median {int(np.median(gaps))}, mean {gaps.mean():.0f}, n {len(pf)}")
    sc = np.array([d[1, j] for j in range(512) if d[1, j]])
    if len(sc) > 2:
        print(f"S commit period: median {int(np.median(np.diff(sc)))}")
    dur, ni = d[30, :148], d[31, :148]
    if dur.any():
        print(f"CTA cycles: min {dur.min()} median {int(np.median(dur))} max {dur.max()}; items min {ni.min()} "
              f"max {ni.max()}")
        o = np.argsort(dur)
        print("slowest CTAs (cta, cycles, items):", [(int(i), int(dur[i]), int(ni[i])) for i in o[-6:]])


if __name__ == "__main__":
    main()
