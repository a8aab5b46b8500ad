"""Standalone A18+K2 (grid_select_kernel) timings + per-phase stamps of CTA 0."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2502_15804_b200 import ops, _native

dev = torch.device("cuda")
for (bt, hkv, n, B) in [(1, 8, 16352, 256), (4, 8, 16352, 256), (1, 8, 32736, 1024), (1, 8, 131040, 1024),
                        (64, 8, 16352, 256)]:
    if "--real" in sys.argv:  # pooled Ada-SnapKV scores of random q / k
        hq = 32 if B == 256 else 64
        q = torch.randn((bt, hq, 32, 128), device=dev).to(torch.bfloat16)
        k = torch.randn((bt, hkv, n + 32, 128), device=dev).to(torch.bfloat16)
        sc = ops.score(q, k)
        del q, k
    else:
        sc = torch.rand((bt, hkv, n), device=dev)
    ws = torch.empty(int(ops._lib.fkv_ada_select_workspace_bytes(bt, hkv, n)), dtype=torch.uint8, device=dev)
    for _ in range(3):
        ops.ada_select(sc, B, 32, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ops.ada_select(sc, B, 32, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    # same calls captured in a CUDA graph (no host launch overhead)
    g = torch.cuda.CUDAGraph()
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        with torch.cuda.graph(g, stream=s_):
            for _ in range(20):
                ops.ada_select(sc, B, 32, workspace=ws)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us_g = e0.elapsed_time(e1) / 20 * 1e3
    print(f"  graph: {us_g:.1f} us/call")
    buf = (C.c_ulonglong * 32)()
    ops.ada_select(sc, B, 32, workspace=ws)
    torch.cuda.synchronize()
    _native.lib.fkv__select_stamps(buf)
    st = np.array(buf, dtype=np.float64)
    t0 = st[0]
    names = {0: "start"}
    for p in range(4):
        names[1 + 3 * p] = f"h{p}"; names[2 + 3 * p] = f"b{p}"; names[3 + 3 * p] = f"g{p}"
    names.update({20: "counted", 21: "cbar", 22: "written"})
    print(f"bt={bt} n={n} B={B}: {us:.1f} us/call |", " ".join(f"{names[i]} {(st[i]-t0)/1e3:.1f}" for i in sorted(names)))
