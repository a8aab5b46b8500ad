"""K4 on the bench workload (70B, TP=1, 80 layers back to back in a graph):
full kernel vs loads-only (probe 1) vs compute-only (probe 2)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops, _native
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.sharding import synthetic_budgets
import bench
dev = torch.device('cuda')
L, bt, HQ, G = 80, 64, 64, 8
budgets = synthetic_budgets(L, bt, 8, 1024, window=32, alpha=0.2, seed=0, context=32768)
qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
caches = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, G, dev, fill="random") for l in range(L)]
q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)
o = torch.empty_like(q)
wss = [ops.DecodeWorkspace(c) for c in caches]
kv = np.mean([c.kv_bytes() for c in caches])
for probe in (0, 1, 2):
    def body():
        for l in range(L):
            _native.lib.fkv__decode_probe(probe)
            ops.decode_into(q[l], caches[l], wss[l], out_bf16=o[l])
    g = bench.capture(body)
    g.replay()
    t = bench.timed(g.replay, 5) / 5 / L
    print(f"probe {probe}: {t*1e6:6.2f} us per layer, {kv/t/1e9:6.0f} GB/s (K+V)", flush=True)
