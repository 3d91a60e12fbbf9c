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

EV = {0: "P:kslab", 1: "S:kfull", 8: "S:sfree", 2: "S:commit", 3: "W:sfull", 4: "W:pfull", 5: "PV:pfull",
      7: "P:vent", 6: "PV:vfull", 9: "P:Qitem", 10: "S:Qfull"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--mode", default="deferred")
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--tiles", type=int, default=12)
    ap.add_argument("--page", type=int, default=64)
    ap.add_argument("--detail", type=int, default=-1)
    ap.add_argument("--first", type=int, default=0)
    a = ap.parse_args()
    import torch
    import numpy as np

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
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fkv.residual_attention_phases(pl, 0, Q, O, 4)
    e2.record()
    for _ in range(10):
        fkv.residual_attention_phases(pl, 0, Q, O, 9)
    e3.record()
    torch.cuda.synchronize()
    print(f"main kernel alone (10 back to back): {e2.elapsed_time(e3) / 10 * 1e3:.1f} us")
    print(f"items={pl.info.n_items} main kernel avg {e0.elapsed_time(e1) / 10 * 1e3:.1f} us; "
          f"alg bytes/layer {pl.info.alg_bytes / 1e6:.1f} MB")
    dbg = torch.zeros(34 * 256, dtype=torch.int64, device="cuda")
    lib = L.load()
    lib.fkv_debug_timeline(fkv.ctx, ctypes.c_void_p(dbg.data_ptr()), a.block)
    fkv.residual_attention_phases(pl, 0, Q, O, 1)
    torch.cuda.synchronize()
    lib.fkv_debug_timeline(fkv.ctx, None, 0)
    d = dbg.view(34, 256).cpu().numpy()
    if not d[:30].any():
        print("no pipeline stamps: the product build compiles them out; build a timeline variant with\n"
              "  bash tools/variants.sh tl -DFKV_TIMELINE=1\nand run with "
              "FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_tl.so")
        dur = d[30, :148]
        if dur.any():
            print(f"CTA cycles: min {dur.min()} median {int(np.median(dur))} max {dur.max()}")
        return
    gs, ge = d[32, :148], d[33, :148]
    if gs.any():
        gs, ge = gs[gs > 0], ge[ge > 0]
        print(f"CTA globaltimer: start spread {(gs.max() - gs.min()) / 1e3:.1f} us, first start -> last end "
              f"{(ge.max() - gs.min()) / 1e3:.1f} us, first end {(ge.min() - gs.min()) / 1e3:.1f} us")
    t0 = d[:30][d[:30] > 0].min()
    print("per tile T (S/W/PV events) and per ring entry (K slab 3/tile, V entry 2/tile), cycles from first event")
    cols = [8, 2, 3, 4, 5]
    print("   T " + " ".join(f"{EV[e]:>9s}" for e in cols) + " |  n " + " ".join(f"{EV[e]:>9s}" for e in (0, 1, 7, 6)))
    for j in range(a.first, a.first + a.tiles):
        row = [d[e, j] - t0 if d[e, j] else -1 for e in cols]
        row2 = [d[e, j] - t0 if d[e, j] else -1 for e in (0, 1, 7, 6)]
        print(f"{j:4d} " + " ".join(f"{x:9d}" for x in row) + f" | {j:3d} " + " ".join(f"{x:9d}" for x in row2))
    print("items: P:Qitem / S:Qfull", [(int(d[9, i] - t0), int(d[10, i] - t0)) for i in range(64) if d[9, i]])
    print("items (NONE): key-warp start, end, reduced, | epilogue: start, TMEM loaded, done",
          [(int(d[25, i] - t0), int(d[26, i] - t0), int(d[13, i] - t0) if d[13, i] else -1,
            int(d[14, i] - t0) if d[14, i] else -1, int(d[15, i] - t0) if d[15, i] else -1,
            int(d[27, i] - t0) if d[27, i] else -1) for i in range(64) if d[25, i]])
    print("key warps per item: start / end / epilogue done", [(int(d[25, i] - t0), int(d[26, i] - t0), int(d[27, i] - t0) if d[27, i] else -1) for i in range(64) if d[25, i]])
    if a.detail >= 0:
        print("key-warp phases per tile (cycles from W:sfull): S loaded, pre-bar_or, post-bar_or, pfree wait/ok, P stored, "
              "fenced, pfull, next sfull")
        for T in range(a.detail, a.detail + 12):
            b0 = d[3, T]
            if not b0 or not d[3, T + 1]:
                break
            g = lambda e, i=T: int(d[e, i] - b0) if d[e, i] else -1
            print(f"  T{T}: {g(28)} {g(20)} {g(29)} {g(16)}/{g(17)} {g(11)} {g(12)} {g(4)} {int(d[3, T + 1] - b0)}")
        T = a.detail
        base = d[0, T]
        f = lambda e, i: int(d[e, i] - base) if d[e, i] else -1
        print(f"tile {T} (cycles from its K issue): K issue 0, S kfull {f(1, T)}, S sfree {f(8, T)}, S commit {f(2, T)}, "
              f"W sfull {f(3, T)}, W pfree-wait {f(16, T)} ok {f(17, T)}, W pfull {f(4, T)}, PV pfull {f(5, T)}, "
              f"PV commit {f(18, T)}")
        print(f"   key warps (NONE): sfull {f(3, T)}, S loaded {f(28, T)}, before bar_or {f(20, T)}, after bar_or {f(29, T)}, "
              f"pfree-wait {f(16, T)} ok {f(17, T)}, P stored {f(11, T)}, fenced {f(12, T)}, pfull {f(4, T)}")
        print(f"   key warps: sfull {f(3, T)}, before bar_or {f(20, T)}, slow {f(21, T)}, pre-atomic {f(22, T)}, "
              f"post-atomic {f(23, T)}, pre-recompute {f(24, T)}, pfree-wait {f(16, T)}")
        for h in range(2):
            n = 2 * T + h
            print(f"   V entry {n}: TMA issue {f(7, n)}, R_v issue {f(19, n)}, PV both full {f(6, n)}")
    if d[11].any():
        b0 = min(x for x in d[11] if x > 0)
        print("DEFERRED unit pipeline, tile 4 (cycles from first S-side ts wait): w, k: S rb-commit, S wait->ok | key pair wait-ok, pair done")
        for w in range(2):
            for k in range(8):
                i = 32 * w + k
                f = lambda e: (d[e, i] - b0) if d[e, i] else -1
                print(f"  w{w} k{k}: rb {f(15):7d}  ts-wait {f(11):7d} ok {f(12):7d} | keys ok {f(13):7d} done {f(14):7d}")
    pf = [int(d[4, j]) for j in range(256) if d[4, j]]
    if len(pf) > 1:
        gaps = np.diff(np.array(pf))
        print("W:pfull period per tile (cycles):", " ".join(str(int(g)) for g in gaps))
        print(f"  first W:pfull {pf[0] - t0}, median period {int(np.median(gaps))}, sum of periods > 1.5x median "
              f"{int(gaps[gaps > 1.5 * np.median(gaps)].sum())}")
    dur, nt = d[30, :148], d[31, :148]
    if dur.any():
        o = np.argsort(dur)
        print(f"CTA cycles: min {dur.min()} median {int(np.median(dur))} max {dur.max()}; "
              f"sum/148 {dur.sum() / 148:.0f}; tiles min {nt.min()} max {nt.max()}")
        print("slowest CTAs (cta, cycles, tiles):", [(int(i), int(dur[i]), int(nt[i])) for i in o[-6:]])
        print("fastest CTAs:", [(int(i), int(dur[i]), int(nt[i])) for i in o[:4]])
    last = max(j for j in range(256) if d[2, j]) if d[2].any() else 0
    print(f"tiles {last + 1}; last S:commit {d[2, last] - t0}, last W:pfull {d[4, last] - t0}, "
          f"cycles/tile overall {(d[4, last] - t0) / (last + 1):.0f}")


if __name__ == "__main__":
    main()
