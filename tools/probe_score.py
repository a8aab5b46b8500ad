"""K1..K3 timing probe: one layer of prefill compression."""
import sys, math
sys.path.insert(0, '.')
import torch
from paper_2502_15804_b200 import ops
dev = torch.device('cuda:0')

def timeit(fn, n=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e-3

for (bt, hq, hkv, T, B) in [(1, 32, 8, 16384, 256), (4, 32, 8, 16384, 256), (1, 64, 8, 32768, 1024), (1, 64, 8, 131072, 1024)]:
    w = 32
    q = torch.randn(bt, hq, w, 128, device=dev).to(torch.bfloat16)
    k = torch.randn(bt, hkv, T, 128, device=dev).to(torch.bfloat16)
    v = torch.randn(bt, hkv, T, 128, device=dev).to(torch.bfloat16)
    ws = torch.empty(int(ops._lib.fkv_score_workspace_bytes(bt, hkv, T, w, hq // hkv)), dtype=torch.uint8, device=dev)
    t_s = timeit(lambda: ops.score(q, k, workspace=ws))
    sc = ops.score(q, k, workspace=ws)
    t_b = timeit(lambda: ops.budgets(sc, B, w))
    hb = ops.budgets(sc, B, w)
    t_k = timeit(lambda: ops.select(sc, hb, w, total=bt * hkv * B))
    t_f = timeit(lambda: ops.ada_select(sc, B, w))
    hb2, off2, idx2 = ops.ada_select(sc, B, w)
    off1, idx1 = ops.select(sc, hb, w, total=bt * hkv * B)
    same = bool((hb2 == hb).all() and (idx2 == idx1).all())
    flops = 2 * 2 * hq * w * T * 128 * bt  # two passes
    kbytes = bt * hkv * T * 256
    print(f"bt={bt} Hq={hq} T={T}: score {t_s*1e6:.0f}us  {flops/t_s/1e12:.0f} TFLOP/s (2 passes)  K-read {kbytes/t_s/1e9:.0f} GB/s (1x K)  "
          f"budgets {t_b*1e6:.0f}us  select {t_k*1e6:.0f}us  fused ada_select {t_f*1e6:.0f}us (same={same})")
