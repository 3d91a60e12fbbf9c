"""Pipeline timeline of one CTA of the tcgen05 kernel (diagnostics).

    python tools/timeline.py [--block B] [--mode deferred|none] [--layers 1]

Builds the C2 workload (1 layer by default), runs one ResidualAttention call
with fkv_debug_timeline enabled for CTA B and prints per-tile event times
(clock64 cycles relative to the CTA start)."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EV = {0: "prod:RK", 1: "prod:KB", 2: "prod:V", 3: "S:rkfull", 4: "S:base", 5: "S:done", 6: "PV:go",
      7: "W0:tile", 8: "W0:kl0", 9: "W0:rope_end", 10: "W0:sfull", 11: "W0:Pready", 12: "W0:pfull",
      13: "W1:tile", 14: "W1:kl0", 15: "W1:rope_end", 16: "W1:sfull", 17: "W1:Pready", 18: "W1:pfull"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--mode", default="deferred")
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--tiles", type=int, default=12)
    ap.add_argument("--page", type=int, default=64)
    a = ap.parse_args()
    import torch

    from paper_2604_06370_b200 import _lib as L
    from paper_2604_06370_b200.api import ForkKV
    from workloads import driver, recipes
    scen = recipes.c2()
    nb, nr = scen.pages_needed(a.page)
    fkv = ForkKV(n_layers=a.layers, n_q_heads=32, n_kv_heads=8, head_dim=128, rank=16, page_size=a.page,
                 n_base_pages=nb, n_res_pages=nr, rope_mode=a.mode, device=0, max_pos=33000, rope_theta=500000.0,
                 llama3=True)
    driver.build(fkv, scen, 0)
    pl = fkv.plan([(x, 1) for x in scen.batch()])
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
    print(f"items={pl.info.n_items} main kernel avg {e0.elapsed_time(e1) / 10 * 1e3:.1f} us; "
          f"alg bytes/layer {pl.info.alg_bytes / 1e6:.1f} MB")
    dbg = torch.zeros(32 * 256, dtype=torch.int64, device="cuda")
    lib = L.load()
    lib.fkv_debug_timeline(fkv.ctx, ctypes.c_void_p(dbg.data_ptr()), a.block)
    fkv.residual_attention_phases(pl, 0, Q, O, 1)
    torch.cuda.synchronize()
    lib.fkv_debug_timeline(fkv.ctx, None, 0)
    d = dbg.view(32, 256).cpu().numpy()
    t0 = d[20, 0]
    print(f"block {a.block}: setup {d[21, 0] - t0} cyc, total {d[22, 0] - t0} cyc")
    names = [EV[e] for e in sorted(EV)]
    print("tile " + " ".join(f"{n:>11s}" for n in names))
    for w in range(2):
        print(f"slow path W{w} tile0: enter {d[19, 128 * w] - t0} butterfly_done {d[23 + w, 0] - t0} "
              f"bar_done {d[29 + w, 0] - t0} resc_bar {d[27 + w, 0] - t0} recompute {d[25 + w, 0] - t0}")
    for j in range(a.tiles):
        row = [d[e, j] - t0 if d[e, j] else -1 for e in sorted(EV)]
        print(f"{j:4d} " + " ".join(f"{x:11d}" for x in row))


if __name__ == "__main__":
    main()
