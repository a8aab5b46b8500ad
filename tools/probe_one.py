"""Single K4 configuration (for ncu): python tools/probe_one.py BT B CHUNK MODE [REPEAT]"""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
dev = torch.device('cuda:0')
bt, B, chunk, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
rep = int(sys.argv[5]) if len(sys.argv) > 5 else 3
hkv, G = 8, 8
rng = np.random.default_rng(0)
lens = np.maximum(64, (B * rng.dirichlet(np.full(hkv, 8.0), size=bt) * hkv).round()).astype(int).ravel()
hq = hkv * G
qrow = [b * hq + h * G for b in range(bt) for h in range(hkv)]
q = torch.randn(bt, hq, 128, device=dev).to(torch.bfloat16)
o = torch.empty_like(q)
cache = LayerCache.allocate(lens, qrow, qrow, G, dev, chunk=chunk or None, fill='random')
ws = ops.DecodeWorkspace(cache)
for _ in range(rep):
    if mode == "partial":
        ops.decode_partial(q, cache, ws)
    elif mode == "fused":
        ops.decode_into(q, cache, ws, out_bf16=o)
    else:  # streaming-read reference: reduce the whole cache
        cache.k.view(torch.int16).sum(dtype=torch.int64); cache.v.view(torch.int16).sum(dtype=torch.int64)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20):
    if mode == "partial": ops.decode_partial(q, cache, ws)
    elif mode == "fused": ops.decode_into(q, cache, ws, out_bf16=o)
    else: cache.k.view(torch.int16).sum(dtype=torch.int64); cache.v.view(torch.int16).sum(dtype=torch.int64)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 20 * 1e-3
print(f"{mode} chunk={cache.host['chunk']} items={cache.n_items} t={t*1e6:.1f}us kv {cache.kv_bytes()/t/1e9:.0f} GB/s rows {cache.k.shape[0]}")
