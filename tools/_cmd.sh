FKV_K4_SCHEDULE=auto python - <<'PY'
import sys, os, json, argparse
sys.path.insert(0, '.')
import torch, bench
a = argparse.Namespace(seed=0)
r = bench.cfg2_sweep(a, torch.device('cuda'), 6549.1)
print("auto", {k: (round(v['ms_per_step']*1e3/32, 2), round(v['hbm_frac'], 3), v['schedule']) for k, v in r.items()})
PY
python - <<'PY'
import sys, os
sys.path.insert(0, '.')
import numpy as np, torch, bench
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.sharding import synthetic_budgets
dev = torch.device('cuda')
L, bt, HQ, G = 80, 64, 64, 8
for B in (256, 512, 1024):
    budgets = synthetic_budgets(L, bt, 8, B, window=32, alpha=0.2, seed=0, context=32768)
    qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
    line = f"70B TP1 B={B}"
    for sched in ("auto", "coop"):
        os.environ["FKV_K4_SCHEDULE"] = sched
        caches = [LayerCache.allocate(budgets.reshape(L, -1)[l], qrow, qrow, G, dev, fill="random") for l in range(L)]
        q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16); o = torch.empty_like(q)
        wss = [ops.DecodeWorkspace(c) for c in caches]
        def body():
            for l in range(L):
                ops.decode_into(q[l], caches[l], wss[l], out_bf16=o[l])
        g = bench.capture(body); g.replay()
        t = bench.timed(g.replay, 3) / 3 / L
        line += f"  {sched}({'solo' if caches[0].flags else 'coop'}) {t*1e6:.1f}us"
        del g, caches, wss; torch.cuda.empty_cache()
    print(line, flush=True)
PY
