"""Small-shard K4 anatomy: the TP8 AHA-DP / SHA shards of the 70B workload at
B=128/256, 80 layers back to back: full vs loads-only vs compute-only, solo
vs coop schedule."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops, _native
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.decoder import rank_caches
from paper_2502_15804_b200.sharding import plan_layouts, synthetic_budgets
import bench
dev = torch.device('cuda:0')
L, bt, HQ, G = 80, 64, 64, 8
for B in (128, 256):
    budgets = synthetic_budgets(L, bt, 8, B, window=32, alpha=0.2, seed=0, context=32768)
    qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
    base = [LayerCache.allocate(budgets.reshape(L, -1)[l], qrow, qrow, G, dev, fill="random") for l in range(L)]
    q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)
    for mode in ("sha", "dp"):
        plan, prof = bench.make_plan(budgets, 8, 8, mode)
        shards, _ = plan_layouts(plan, budgets, G)
        for sched in ("solo", "coop"):
            os.environ["FKV_K4_SCHEDULE"] = sched
            caches = rank_caches([s[0] for s in shards], bt, HQ, G, 8, dev, base=base)
            sends = [torch.empty((max(c.n_segments, 1), G, ops.REC), device=dev) for c in caches]
            wss = [ops.DecodeWorkspace(c) for c in caches]
            res = []
            for probe in (0, 1, 2):
                def body():
                    for l in range(L):
                        _native.lib.fkv__decode_probe(probe)
                        ops.decode_into(q[l], caches[l], wss[l], out_rec=sends[l])
                gr = bench.capture(body)
                gr.replay()
                res.append(bench.timed(gr.replay, 3) / 3 / L)
            c = caches[0]
            print(f"B={B} tp8 {mode} {sched}: segs {c.n_segments} pieces {c.n_items} ctas {c.n_workers} "
                  f"kv {c.kv_bytes()/1e6:.1f}MB full {res[0]*1e6:.1f} loads {res[1]*1e6:.1f} compute {res[2]*1e6:.1f} us", flush=True)
