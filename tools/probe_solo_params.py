"""Sweep the per-warp planner's (whole, piece) tile thresholds on TP4/TP8 shards."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.decoder import rank_caches
from paper_2502_15804_b200.sharding import plan_layouts, synthetic_budgets
import bench
dev = torch.device('cuda:0')
L, bt, HQ, G = 80, 64, 64, 8
params = [(int(a), int(b)) for a, b in (x.split(',') for x in os.environ.get('SOLO_PARAMS', '8,8 12,8 16,8 16,12 24,16 32,16').split())]
for B in [int(x) for x in os.environ.get('SOLO_BUDGETS', '128 256 512').split()]:
    budgets = synthetic_budgets(L, bt, 8, B, window=32, alpha=0.2, seed=0, context=32768)
    qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
    os.environ["FKV_K4_SCHEDULE"] = "coop"
    base = [LayerCache.allocate(budgets.reshape(L, -1)[l], qrow, qrow, G, dev, fill="random") for l in range(L)]
    q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)
    for tp, mode in [(int(x[:-4] if False else x.split(':')[0]), x.split(':')[1]) for x in os.environ.get('SOLO_TPS', '4:sha 4:dp 8:sha 8:dp').split()]:
        plan, prof = bench.make_plan(budgets, tp, 8 if tp == 8 else 4, mode)
        shards, _ = plan_layouts(plan, budgets, G)
        line = f"B={B:4d} tp{tp} {mode:3s}"
        for sched, (wh, pc) in [("coop", (0, 0))] + [("solo", p) for p in params]:
            os.environ["FKV_K4_SCHEDULE"] = sched
            os.environ["FKV_SOLO_WHOLE"], os.environ["FKV_SOLO_PIECE"] = str(wh or 24), str(pc or 16)
            worst = 0.0
            for g in range(tp):
                caches = rank_caches([s[g] for s in shards], bt, HQ, G, tp, dev, base=base)
                sends = [torch.empty((max(c.n_segments, 1), G, ops.REC), device=dev) for c in caches]
                wss = [ops.DecodeWorkspace(c) for c in caches]
                def body():
                    for l in range(L):
                        ops.decode_into(q[l], caches[l], wss[l], out_rec=sends[l])
                gr = bench.capture(body)
                gr.replay()
                worst = max(worst, bench.timed(gr.replay, 3) / 3 / L)
            line += f" {sched}{'' if sched == 'coop' else f'({wh},{pc})'} {worst*1e6:5.1f}"
        print(line, flush=True)
    del base
    torch.cuda.empty_cache()
