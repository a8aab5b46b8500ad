"""K4 per-layer time (16 chained layers, PDL graph) of the heaviest rank of
TP shards of the 70B workload with the whole-segment schedule's long-segment
cut off (FKV_HYBRID_SAVING=1e9) and always on (0), auto schedule choice
otherwise; with each case's segment count, longest segment and cut length
(tiles), to place the cut's saving threshold (cache.HYBRID_MIN_SAVING_US).
usage: python tools/probe_hybrid.py [bt ...]"""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops, cache as C
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.decoder import rank_caches
from paper_2502_15804_b200.sharding import plan_layouts, synthetic_budgets
import bench
dev = torch.device('cuda:0')
L, HQ, G = 16, 64, 8
for bt in [int(x) for x in sys.argv[1:]] or [1, 4, 16, 64]:
    for B in (256, 512, 1024):
        budgets = synthetic_budgets(L, bt, 8, B, window=32, alpha=0.2, seed=0, context=32768)
        qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
        base = [LayerCache.allocate(budgets.reshape(L, -1)[l], qrow, qrow, G, dev, fill="random") for l in range(L)]
        q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)
        for tp, mode in [(4, "sha"), (4, "dp"), (8, "sha"), (8, "dp"), (8, "dp-free")]:
            plan, prof = bench.make_plan(budgets, tp, mode)
            shards, _ = plan_layouts(plan, budgets, G)
            toks = [sum(int((s[g].seg_hi - s[g].seg_lo).sum()) for s in shards) for g in range(tp)]
            g = int(np.argmax(toks))
            line = f"bt={bt:3d} B={B:5d} tp{tp} {mode:7s} {toks[g] * 512 / L / 1e6:6.2f} MB"
            for sv in ("1e9", "0"):
                os.environ["FKV_HYBRID_SAVING"] = sv
                caches = rank_caches([s[g] for s in shards], bt, HQ, G, tp, dev, base=base)
                sends = [ops.xrec_empty(max(c.n_segments, 1), G, dev)[0] for c in caches]
                wss = [ops.DecodeWorkspace(c) for c in caches]
                gr = bench.capture(lambda: [ops.decode_into(q[l], caches[l], wss[l], out_rec=sends[l])
                                            for l in range(L)])
                gr.replay()
                t = min(bench.timed(gr.replay, 1) for _ in range(5)) / L
                c = caches[0]
                lens = c.host["seg_len"]
                piece = int(((c.item_t1 - c.item_t0).max().item() + 15) // 16) if c.n_items else 0
                line += (f" | {'off' if sv == '1e9' else 'on '} {t * 1e6:6.2f}us f{c.flags} n{len(lens)} "
                         f"items{c.n_items} long{int((lens.max() + 15) // 16) if len(lens) else 0}t piece{piece}t")
            print(line, flush=True)
        del base
        torch.cuda.empty_cache()
os.environ.pop("FKV_HYBRID_SAVING", None)
