"""Quick K4 timing probe: one layer of the 70B shape at TP=1."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
dev = torch.device('cuda:0')
bt, hkv, G, B = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 8, 8, int(sys.argv[2]) if len(sys.argv) > 2 else 1024
rng = np.random.default_rng(0)
lens = np.maximum(64, (B * rng.dirichlet(np.full(hkv, 8.0), size=bt) * hkv).round()).astype(int).ravel()
hq = hkv * G
qrow = [b * hq + h * G for b in range(bt) for h in range(hkv)]
for chunk in (None, 256, 512, 1024):
    cache = LayerCache.allocate(lens, qrow, qrow, G, dev, chunk=chunk, fill='random')
    q = torch.randn(bt, hq, 128, device=dev).to(torch.bfloat16)
    ws = ops.DecodeWorkspace(cache)
    for _ in range(3): ops.decode_partial(q, cache, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 50
    e0.record()
    for _ in range(n): ops.decode_partial(q, cache, ws)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / n * 1e-3
    byts = cache.kv_bytes() + q.numel() * 2 + ws.part_o.numel() * 4
    print(f"bt={bt} B={B} chunk={cache.host['chunk']} items={cache.n_items} kv={cache.kv_bytes()/1e6:.1f}MB t={t*1e6:.1f}us {byts/t/1e9:.0f} GB/s")
