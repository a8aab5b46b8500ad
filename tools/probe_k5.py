"""K5 (polling merge) marginal cost per layer and the emulated TP step, from
bench.py's emulation on a 16-layer slice of the 70B workload (batch 64).
usage: python tools/probe_k5.py [B ...]"""
import sys
import types
sys.path.insert(0, '.')
import torch
import bench
from paper_2502_15804_b200.sharding import synthetic_budgets

dev = torch.device("cuda:0")
for B in [int(x) for x in sys.argv[1:]] or [256, 1024]:
    budgets = synthetic_budgets(16, 64, 8, B, window=32, alpha=0.2, seed=0, context=32768)
    base, q = bench._alloc_base(budgets, dev)
    res = bench.emulate_tp(types.SimpleNamespace(ch=4), budgets, dev, base, q, tps=(2, 8), modes=("sha", "dp"))
    for tp in ("tp2", "tp8"):
        for m in ("sha", "dp"):
            x = res[tp][m]
            print(f"B={B} {tp} {m:4s}: k4x {x['k4x_us_per_layer_max_rank']:6.2f} us + k5 {x['k5_us_per_layer']:5.2f} us"
                  f" -> {x['tokens_per_s']:8.0f} tok/s", flush=True)
