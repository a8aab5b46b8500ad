"""K4 on AHA/SHA shard sizes (TP 2/4/8 of the 70B bench workload): per-layer
time in a plain CUDA graph of 80 back-to-back launches vs event-bracketed,
under several schedule parameters."""
import sys, itertools
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2502_15804_b200.cache as cm
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.decoder import rank_caches
from paper_2502_15804_b200.sharding import plan_layouts, synthetic_budgets
import bench

dev = torch.device('cuda:0')
L, bt, HQ, G = 80, 64, 64, 8
budgets = synthetic_budgets(L, bt, 8, 1024, window=32, alpha=0.2, seed=0, context=32768)
hkv_lens = budgets.reshape(L, -1)
qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
gen = torch.Generator(device=dev).manual_seed(7)
base = [LayerCache.allocate(hkv_lens[l], qrow, qrow, G, dev, fill="random", generator=gen) for l in range(L)]
q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)

def time_graph(fn, reps=5):
    g = bench.capture(fn)
    for _ in range(2): g.replay()
    return bench.timed(g.replay, reps) / reps

variants = [("default", dict()),
            ("pieces16", dict(MAX_PIECES_PER_SEGMENT=16)),
            ("pieces32_min2", dict(MAX_PIECES_PER_SEGMENT=32, MIN_TILES_PER_WORKER=2)),
            ("pieces8_min4", dict(MAX_PIECES_PER_SEGMENT=8))]
orig = {k: getattr(cm, k) for k in ("MAX_PIECES_PER_SEGMENT", "MIN_TILES_PER_WORKER")}
for tp, mode in [(1, "sha"), (2, "sha"), (4, "sha"), (8, "sha"), (8, "dp")]:
    plan, prof = bench.make_plan(budgets, tp, 8 if tp == 8 else 4, mode)
    shards, _ = plan_layouts(plan, budgets, G)
    for vname, kw in variants:
        for k, v in orig.items(): setattr(cm, k, v)
        for k, v in kw.items(): setattr(cm, k, v)
        worst = 0.0
        res = []
        for g in range(tp):
            caches = rank_caches([s[g] for s in shards], bt, HQ, G, tp, dev, base=base)
            sends = [torch.empty((max(c.n_segments, 1), G, ops.REC), device=dev) for c in caches]
            wss = [ops.DecodeWorkspace(c) for c in caches]
            def body():
                for l in range(L):
                    ops.decode_into(q[l], caches[l], wss[l], out_rec=sends[l])
            t = time_graph(body) / L
            kvb = np.mean([c.kv_bytes() for c in caches])
            res.append((t, kvb, np.mean([c.host["n_workers"] for c in caches]), np.mean([c.n_items for c in caches])))
        t = max(r[0] for r in res)
        print(f"tp{tp} {mode:4s} {vname:14s} per-layer max_g {t*1e6:6.1f} us  " +
              " ".join(f"[{r[0]*1e6:.1f}us {r[1]/r[0]/1e9:.0f}GB/s w{r[2]:.0f} it{r[3]:.0f}]" for r in res[:4]), flush=True)
        if tp == 1: break
