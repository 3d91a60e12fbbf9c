import random, sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import test_gpu_parity as T
from oracle import ra
from workloads import driver, recipes
from paper_2604_06370_b200 import _lib as L
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 17
rnd = random.Random(seed)
P = rnd.choice([16, 64, 128]); mode = rnd.choice(["deferred", "none"])
dtype = "f32" if seed % 4 == 0 else "bf16"
scen = T._random_scenario(rnd, P)
print("P", P, mode, dtype, "q_len", scen.q_len, [(a.id, a.fork_len, a.n_private, a.decode) for a in scen.agents])
fkv = T._ctx(scen, 2, 8, 2, 128, 16, P, dtype, mode)
driver.build(fkv, scen, seed=seed)
batch = scen.batch(); C = scen.q_len
pl = fkv.plan([(a, C) for a in batch], flags=L.PLAN_CHECK_WRITTEN)
print("items", pl.info.n_items, "kernel", pl.info.kernel)
Q = driver.make_queries(fkv, scen, seed, 0)
O = fkv.residual_attention(pl, 0, Q); torch.cuda.synchronize(); O = O.float().cpu().numpy()
fr = ra.inv_freq(fkv.d, 10000.0, llama3=False)
for i, a in enumerate(batch):
    inp = recipes.oracle_inputs(scen, seed, a, 0, fkv.hkv, fkv.d, fkv.r, fkv.hq, C, dtype, kv_heads=(0, fkv.hkv))
    ref = ra.residual_attention(inv_freq_=fr, rope_mode=ra.ROPE_NONE if mode == "none" else ra.ROPE_DEFERRED, **inp)
    e = np.abs(O[i * C:(i + 1) * C] - ref)
    print("seq", a, "err", e.max(), "per row", e.reshape(C, fkv.hq, -1).max(axis=2).max(axis=1).round(3).tolist()[:16], "per head", e.reshape(C, fkv.hq, -1).max(axis=2).max(axis=0).round(3).tolist())
