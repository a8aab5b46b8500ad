"""K4 time vs size: uniform segments (n_seg x len), graph of 20 launches vs
single event-timed launch.  argv[1] = 'ncu' -> run each config 3x untimed (for ncu)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache
import bench
dev = torch.device('cuda:0')
G, HQ = 8, 64
under_ncu = len(sys.argv) > 1 and sys.argv[1] == 'ncu'
for n_seg, ln in [(64, 64), (64, 256), (64, 1024), (128, 1024), (256, 1024), (512, 1024), (64, 4096), (512, 4096)]:
    bt = max(1, n_seg // 8)
    qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])[:n_seg]
    cache = LayerCache.allocate(np.full(n_seg, ln), qrow, qrow, G, dev, fill='random')
    q = torch.randn(bt, HQ, 128, device=dev).to(torch.bfloat16)
    o = torch.empty_like(q)
    ws = ops.DecodeWorkspace(cache)
    fn = lambda: ops.decode_into(q, cache, ws, out_bf16=o)
    if under_ncu:
        for _ in range(3): fn()
        torch.cuda.synchronize(); continue
    for _ in range(3): fn()
    t1 = min(bench.timed(fn, 1) for _ in range(10))
    def body():
        for _ in range(20): fn()
    g = bench.capture(body)
    g.replay()
    tg = bench.timed(g.replay, 5) / 100
    kv = cache.kv_bytes()
    print(f"nseg={n_seg:4d} len={ln:5d} kv={kv/1e6:7.1f}MB workers={cache.host['n_workers']:5d} items={cache.n_items:5d} "
          f"single={t1*1e6:6.1f}us graph={tg*1e6:6.1f}us  {kv/tg/1e9:6.0f} GB/s", flush=True)
