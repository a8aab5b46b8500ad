"""K4 fixed cost: per-layer time of tiny caches, 80 launches back to back in a graph."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
import bench
dev = torch.device('cuda:0')
G, HQ, L = 8, 64, 80
for n_seg, ln in [(8, 16), (64, 16), (64, 64), (64, 128), (64, 256), (512, 16), (512, 128)]:
    bt = max(1, n_seg // 8)
    qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])[:n_seg]
    caches = [LayerCache.allocate(np.full(n_seg, ln), qrow, qrow, G, dev, fill='random') for _ in range(L)]
    q = torch.randn(L, bt, HQ, 128, device=dev).to(torch.bfloat16)
    o = torch.empty_like(q)
    wss = [ops.DecodeWorkspace(c) for c in caches]
    def body():
        for l in range(L):
            ops.decode_into(q[l], caches[l], wss[l], out_bf16=o[l])
    g = bench.capture(body)
    g.replay()
    t = bench.timed(g.replay, 5) / 5 / L
    print(f"nseg={n_seg:4d} len={ln:4d} ctas={caches[0].n_workers:4d} solo={caches[0].flags} per-layer {t*1e6:6.2f} us", flush=True)
