"""K4 timing probe: one layer of the 70B shape at TP=1, several chunk sizes,
partial-record mode vs fused merge, CUDA-graph timed (20 launches)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
dev = torch.device('cuda:0')
bt = int(sys.argv[1]) if len(sys.argv) > 1 else 64
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
hkv = int(sys.argv[3]) if len(sys.argv) > 3 else 8
G = 8
rng = np.random.default_rng(0)
lens = np.maximum(64, (B * rng.dirichlet(np.full(hkv, 8.0), size=bt) * hkv).round()).astype(int).ravel()
hq = hkv * G
qrow = [b * hq + h * G for b in range(bt) for h in range(hkv)]
q = torch.randn(bt, hq, 128, device=dev).to(torch.bfloat16)
o = torch.empty_like(q)
for chunk in (None, 128, 256, 512, 1024):
    cache = LayerCache.allocate(lens, qrow, qrow, G, dev, chunk=chunk, fill='random')
    ws = ops.DecodeWorkspace(cache)
    for mode in ("partial", "fused"):
        fn = (lambda: ops.decode_partial(q, cache, ws)) if mode == "partial" else \
             (lambda: ops.decode_into(q, cache, ws, out_bf16=o))
        for _ in range(3): fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20): fn()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 20 * 1e-3
        byts = cache.kv_bytes()
        print(f"bt={bt} B={B} chunk={str(cache.host['chunk']):>5s} items={cache.n_items:5d} {mode:7s} "
              f"kv={byts/1e6:.1f}MB t={t*1e6:.1f}us {byts/t/1e9:.0f} GB/s (KV only)")
