"""K4 per-layer time (16 chained layers, PDL graph) of the heaviest rank of
TP shards of the 70B workload: the automatic schedule vs the 8-warp ("wide")
CTA shape with whole segments packed longest-first (FKV_K4_SCHEDULE=wide
FKV_K4_WHOLE=1) and the wide shape under the automatic whole/split choice,
for caches of more segments than the wide shape is chosen for today.
usage: python tools/probe_wide.py [B ...]"""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.decoder import rank_caches
from paper_2502_15804_b200.sharding import plan_layouts, synthetic_budgets
import bench
dev = torch.device('cuda:0')
L, HQ, G = 16, 64, 8
bt = int(os.environ.get("PROBE_BT", 64))
VARIANTS = (("auto", {}), ("wide-whole", {"FKV_K4_SCHEDULE": "wide", "FKV_K4_WHOLE": "1"}),
            ("wide", {"FKV_K4_SCHEDULE": "wide"}))
for B in [int(x) for x in sys.argv[1:]] or [256, 512, 1024]:
    budgets = synthetic_budgets(L, bt, 8, B, window=32, alpha=0.2, seed=0, context=32768)
    qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
    base = [LayerCache.allocate(budgets.reshape(L, -1)[l], qrow, qrow, G, dev, fill="random") for l in range(L)]
    q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)
    for tp, mode in [(1, "sha"), (2, "sha"), (2, "dp"), (2, "dp-free"), (4, "sha"), (4, "dp"), (4, "dp-free")]:
        plan, prof = bench.make_plan(budgets, tp, mode)
        shards, _ = plan_layouts(plan, budgets, G)
        toks = [sum(int((s[g].seg_hi - s[g].seg_lo).sum()) for s in shards) for g in range(tp)]
        g = int(np.argmax(toks))
        line = f"bt={bt} B={B:5d} tp{tp} {mode:7s} {toks[g] * 512 / L / 1e6:6.1f} MB"
        for name, env in VARIANTS:
            for k, v in env.items():
                os.environ[k] = v
            caches = rank_caches([s[g] for s in shards], bt, HQ, G, tp, dev, base=base)
            for k in env:
                os.environ.pop(k)
            sends = [ops.xrec_empty(max(c.n_segments, 1), G, dev)[0] for c in caches]
            wss = [ops.DecodeWorkspace(c) for c in caches]
            gr = bench.capture(lambda: [ops.decode_into(q[l], caches[l], wss[l], out_rec=sends[l]) for l in range(L)])
            gr.replay()
            t = min(bench.timed(gr.replay, 1) for _ in range(5)) / L
            c = caches[0]
            line += f"  {name} {t * 1e6:6.2f}us (f{c.flags},n{c.n_segments},{c.n_workers}w,{c.n_items}i)"
        print(line, flush=True)
    del base
    torch.cuda.empty_cache()
