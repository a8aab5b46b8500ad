"""K4 per-layer time of small-batch decode (Llama-3.1-8B shape: 8 KV heads,
G=4, B=256, 32 layers back to back in one PDL graph) under every schedule
override, plus an (almost) empty cache: the launch-chain floor.
usage: python tools/probe_small_batch.py [batch ...]"""
import os
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.sharding import synthetic_budgets

dev = torch.device('cuda:0')
L, HQ, G = 32, 32, 4
B = int(os.environ.get("PROBE_B", 256))


def per_layer(bt, lens_fn, env):
    for k, v in env.items():
        os.environ[k] = v
    qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
    caches = [LayerCache.allocate(lens_fn(l), qrow, qrow, G, dev, fill="random") for l in range(L)]
    for k in env:
        os.environ.pop(k)
    q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)
    o = torch.empty_like(q)
    wss = [ops.DecodeWorkspace(c) for c in caches]
    gr = bench.capture(lambda: [ops.decode_into(q[l], caches[l], wss[l], out_bf16=o[l]) for l in range(L)])
    gr.replay()
    t = min(bench.timed(gr.replay, 5) for _ in range(3)) / 5 / L
    return t * 1e6, caches[0].flags, caches[0].n_workers


for bt in [int(x) for x in sys.argv[1:]] or [1, 4, 16]:
    budgets = synthetic_budgets(L, bt, 8, B, window=32, alpha=0.2, seed=0, context=16384)
    line = f"batch {bt:3d}:"
    for name, env in (("auto", {}), ("coop", {"FKV_K4_SCHEDULE": "coop"}), ("wide", {"FKV_K4_SCHEDULE": "wide"}),
                      ("solo", {"FKV_K4_SCHEDULE": "solo"}), ("wide-split", {"FKV_K4_SCHEDULE": "wide", "FKV_K4_WHOLE": "0"}),
                      ("wide-whole", {"FKV_K4_SCHEDULE": "wide", "FKV_K4_WHOLE": "1"}),
                      ("coop-whole", {"FKV_K4_SCHEDULE": "coop", "FKV_K4_WHOLE": "1"})):
        us, fl, w = per_layer(bt, lambda l: budgets[l].reshape(-1), env)
        line += f"  {name} {us:5.2f}us(f{fl},{w}w)"
    print(line, flush=True)
us, fl, w = per_layer(1, lambda l: np.full(8, 16), {})
print(f"floor (8 segments x 16 tokens): {us:5.2f} us/layer (f{fl},{w}w)", flush=True)
us, fl, w = per_layer(1, lambda l: np.full(8, 16), {"FKV_K4_SCHEDULE": "solo"})
print(f"floor solo: {us:5.2f} us/layer (f{fl},{w}w)", flush=True)
