"""TP=8: AHA free-split DP with few copies (CH=1..4) vs uniform TP at small
budgets (emulated exactly as bench.py's emulate_tp)."""
import sys, copy
sys.path.insert(0, '.')
import torch
import bench
sys.argv = [sys.argv[0]]
base = bench.parse()
dev = torch.device("cuda")
for B in (128, 256):
    for ch in (1, 2, 3, 4):
        a = copy.copy(base)
        a.budget, a.ch = B, ch
        budgets, _ = bench.workload(a)
        r = bench.emulate_tp(a, budgets, dev, calibrate=False, tps=(8,), modes_tp8=("sha", "dp-free"))["tp8"]
        print(f"B={B} CH={ch}: sha {r['sha']['tokens_per_s']:.0f}  dp-free {r['dp-free']['tokens_per_s']:.0f} "
              f"({r['dp-free']['gain_vs_sha']:.3f}), kv max/mean {r['dp-free']['kv_max_over_mean']:.3f}", flush=True)
