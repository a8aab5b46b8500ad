"""K4 per-layer time of AHA/SHA shards (70B bench workload, 80 layers, each
rank's layers back to back in one graph) under the coop and solo schedules,
budgets 128-1024.  usage: python tools/probe_sched.py [budgets...]"""
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
budgets_list = [int(x) for x in sys.argv[1:]] or [128, 256, 512, 1024]
for B in budgets_list:
    budgets = synthetic_budgets(L, bt, 8, B, window=32, alpha=0.2, seed=0, context=32768)
    qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
    os.environ["FKV_K4_SCHEDULE"] = "coop"
    base = [LayerCache.allocate(budgets.reshape(L, -1)[l], qrow, qrow, G, dev, fill="random") for l in range(L)]
    q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)
    for tp, mode in [(1, "sha"), (2, "sha"), (4, "sha"), (8, "sha"), (8, "dp")]:
        plan, prof = bench.make_plan(budgets, tp, mode)
        shards, _ = plan_layouts(plan, budgets, G)
        line = f"B={B:5d} tp{tp} {mode:4s}"
        for sched in os.environ.get("SCHEDS", "coop wide solo auto").split():
            os.environ["FKV_K4_SCHEDULE"] = sched
            worst = 0.0
            for g in range(tp):
                caches = rank_caches([s[g] for s in shards], bt, HQ, G, tp, dev, base=base)
                sends = [ops.xrec_empty(max(c.n_segments, 1), G, dev)[0] for c in caches]
                wss = [ops.DecodeWorkspace(c) for c in caches]
                def body():
                    for l in range(L):
                        ops.decode_into(q[l], caches[l], wss[l], out_rec=sends[l])
                gr = bench.capture(body)
                gr.replay()
                t = bench.timed(gr.replay, 3) / 3 / L
                worst = max(worst, t)
            line += f"  {sched} {worst*1e6:6.1f}us"
        print(line, flush=True)
    del base
    torch.cuda.empty_cache()
