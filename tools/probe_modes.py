"""K4 diagnostics: full kernel vs loads-only (probe 1) vs compute-only (probe 2)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops, _native
from paper_2502_15804_b200.cache import LayerCache
import bench
dev = torch.device('cuda:0')
G, HQ = 8, 64
for n_seg, ln in [(64, 1024), (64, 4096), (512, 1024), (512, 4096)]:
    bt = max(1, n_seg // 8)
    qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])[:n_seg]
    cache = LayerCache.allocate(np.full(n_seg, ln), qrow, qrow, G, dev, fill='random')
    q = torch.randn(bt, HQ, 128, device=dev).to(torch.bfloat16)
    o = torch.empty_like(q)
    ws = ops.DecodeWorkspace(cache)
    res = []
    for mode in (0, 1, 2):
        def fn():
            _native.lib.fkv__decode_probe(mode)
            ops.decode_into(q, cache, ws, out_bf16=o)
        fn(); torch.cuda.synchronize()
        def body():
            for _ in range(20): fn()
        g = bench.capture(body)
        g.replay()
        res.append(bench.timed(g.replay, 5) / 100)
    kv = cache.kv_bytes()
    print(f"nseg={n_seg:4d} len={ln:5d} workers={cache.n_workers:5d} tiles/worker={n_seg*ln/16/cache.n_workers:5.1f} "
          f"full={res[0]*1e6:6.1f}us loads-only={res[1]*1e6:6.1f}us compute-only={res[2]*1e6:6.1f}us", flush=True)
