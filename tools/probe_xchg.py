"""Per-layer K4 time of one TP rank's shard (70B bench workload, 80 layers
back to back in one graph): local outputs vs one local record block vs the
fused loopback exchange (epoch-tagged XLL records to all tp receive areas)
and the exchange plus every rank's merge_wait.
usage: python tools/probe_xchg.py [B] [tp...]"""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.decoder import rank_caches
from paper_2502_15804_b200.exchange import P2PGroup, exchange_buffer
from paper_2502_15804_b200.sharding import plan_layouts, synthetic_budgets
import bench
dev = torch.device('cuda:0')
L, bt, HQ, G = 80, 64, 64, 8
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
tps = [int(x) for x in sys.argv[2:]] or [1, 2, 8]
budgets = synthetic_budgets(L, bt, 8, B, window=32, alpha=0.2, seed=0, context=32768)
qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
base = [LayerCache.allocate(budgets.reshape(L, -1)[l], qrow, qrow, G, dev, fill="random") for l in range(L)]
q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)
o = torch.empty((bt, HQ, 128), device=dev, dtype=torch.bfloat16)
for tp in tps:
    for mode in (["sha"] if tp == 1 else ["sha", "dp"]):
        plan, prof = bench.make_plan(budgets, tp, mode)
        shards, finals = plan_layouts(plan, budgets, G)
        res = {"local": 0.0, "rec": 0.0, "xchg": 0.0, "xchg+k5": 0.0}
        grp = P2PGroup.loopback(tp, max(f.slots for f in finals), G) if tp > 1 else None
        for g in range(tp):
            caches = rank_caches([s[g] for s in shards], bt, HQ, G, tp, dev, base=base)
            sends = [ops.xrec_empty(max(c.n_segments, 1), G, dev)[0] for c in caches]
            wss = [ops.DecodeWorkspace(c) for c in caches]
            bodies = {"local": lambda: [ops.decode_into(q[l], caches[l], wss[l], out_bf16=o) for l in range(L)],
                      "rec": lambda: [ops.decode_into(q[l], caches[l], wss[l], out_rec=sends[l]) for l in range(L)]}
            if grp is not None:
                bodies["xchg"] = lambda: [ops.decode_exchange(q[l], caches[l], grp.endpoints[g], exchange_buffer(l, L), wss[l])
                                          for l in range(L)]
            if grp is not None and g == 0:
                tabs = [tuple(torch.as_tensor(x, device=dev) for x in (f.grp_ptr, f.src_idx, f.out_row)) for f in finals]
                allc = [rank_caches([s[r] for s in shards], bt, HQ, G, tp, dev, base=base) for r in range(tp)]
                allw = [[ops.DecodeWorkspace(c) for c in cs] for cs in allc]
                def k45():
                    for l in range(L):
                        for r in range(tp):
                            ops.decode_exchange(q[l], allc[r][l], grp.endpoints[r], exchange_buffer(l, L), allw[r][l])
                        for r in range(tp):
                            ops.merge_wait(grp.endpoints[r], exchange_buffer(l, L), *tabs[l], G, out_bf16=o)
                def k4():
                    for l in range(L):
                        for r in range(tp):
                            ops.decode_exchange(q[l], allc[r][l], grp.endpoints[r], exchange_buffer(l, L), allw[r][l])
                g45, g4 = bench.capture(k45), bench.capture(k4)
                g45.replay()
                t45 = min(bench.timed(g45.replay, 1) for _ in range(3))
                t4 = min(bench.timed(g4.replay, 1) for _ in range(3))
                res["xchg+k5"] = (t45 - t4) / (L * tp)
            for name, body in bodies.items():
                gr = bench.capture(body)
                gr.replay()
                t = min(bench.timed(gr.replay, 3) for _ in range(3)) / 3 / L
                res[name] = max(res[name], t)
        if grp is not None:
            grp.close()
        print(f"B={B} tp{tp} {mode}: " + "  ".join(f"{k} {v*1e6:6.2f}us" for k, v in res.items()), flush=True)

