"""cfg2 (Llama-3.1-8B, G=4, B=256) per-layer K4 time by schedule, batch 16/64/256."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.sharding import synthetic_budgets
import bench
dev = torch.device('cuda')
L, hq, hkv, G, B = 32, 32, 8, 4, 256
for bt in (16, 64, 128, 256):
    budgets = synthetic_budgets(L, bt, hkv, B, window=32, alpha=0.2, seed=0, context=16384)
    qrow = np.array([b * hq + h * G for b in range(bt) for h in range(hkv)])
    line = f"batch {bt:3d}"
    for sched in os.environ.get("SCHEDS", "coop wide solo auto").split():
        os.environ["FKV_K4_SCHEDULE"] = sched
        try:
            caches = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, G, dev, fill="random") for l in range(L)]
        except ValueError as e:
            line += f"  {sched} n/a"
            continue
        q = torch.randn((L, bt, hq, 128), device=dev).to(torch.bfloat16)
        o = torch.empty_like(q)
        wss = [ops.DecodeWorkspace(c) for c in caches]
        def step():
            for l in range(L):
                ops.decode_into(q[l], caches[l], wss[l], out_bf16=o[l])
        g = bench.capture(step)
        g.replay()
        t = bench.timed(g.replay, 5) / 5 / L
        kv = np.mean([c.kv_bytes() for c in caches])
        line += f"  {sched} {t*1e6:6.1f}us ({kv/t/1e9/6549:4.2f})"
        del g, caches, wss
    print(line, flush=True)
