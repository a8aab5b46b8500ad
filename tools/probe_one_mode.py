"""One K4 launch config for ncu: argv = n_seg len probe_mode."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops, _native
from paper_2502_15804_b200.cache import LayerCache
dev = torch.device('cuda:0')
G, HQ = 8, 64
n_seg, ln, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
bt = max(1, n_seg // 8)
qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])[:n_seg]
cache = LayerCache.allocate(np.full(n_seg, ln), qrow, qrow, G, dev, fill='random')
q = torch.randn(bt, HQ, 128, device=dev).to(torch.bfloat16)
o = torch.empty_like(q)
ws = ops.DecodeWorkspace(cache)
for _ in range(3):
    _native.lib.fkv__decode_probe(mode)
    ops.decode_into(q, cache, ws, out_bf16=o)
torch.cuda.synchronize()
