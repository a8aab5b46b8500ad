"""Fused K1+A18+K2 vs score + grid select across batch sizes (8B shape, 16k):
where the fused grid (Bt*Hkv x chunks <= #SMs) leaves SMs idle."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2502_15804_b200 import ops
import bench
dev = torch.device("cuda")
for bt in (1, 2, 4, 5, 8, 10, 12, 16, 18):
    hq, hkv, T, B, w = 32, 8, 16384, 256, 32
    q = torch.randn((bt, hq, w, 128), device=dev).to(torch.bfloat16)
    k = torch.randn((bt, hkv, T, 128), device=dev).to(torch.bfloat16)
    ws = torch.empty(int(ops._lib.fkv_score_workspace_bytes(bt, hkv, T, w, hq // hkv)), dtype=torch.uint8, device=dev)
    wsel = torch.empty(int(ops._lib.fkv_ada_select_workspace_bytes(bt, hkv, T - w)), dtype=torch.uint8, device=dev)
    def fused():
        ops.score_select(q, k, B, w, workspace=ws)
    def split():
        sc = ops.score(q, k, workspace=ws)
        ops.ada_select(sc, B, w, workspace=wsel)
    res = []
    for fn in (fused, split):
        g = bench.capture(lambda: [fn() for _ in range(5)])
        g.replay()
        res.append(bench.timed(g.replay, 1) / 5 * 1e6)
    print(f"batch {bt:3d} heads {bt*hkv:4d}: fused {res[0]:7.1f} us   score+select {res[1]:7.1f} us", flush=True)
