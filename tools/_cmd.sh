python - <<'PY' 2>&1 | tail -12
import sys, os, json, argparse, time
sys.path.insert(0, '.')
import torch, bench
a = argparse.Namespace(seed=0, budget=1024, batch=64, layers=80, context=32768, ch=4)
budgets, _ = bench.workload(a)
t0 = time.time()
r = bench.full_layer(a, budgets, torch.device('cuda'))
print("elapsed", time.time() - t0)
for k, v in r.items(): print(k, v if k == "note" else {m: {x: round(y, 3) for x, y in d.items() if y is not None} for m, d in v.items()})
PY
