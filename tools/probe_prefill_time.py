"""Prefill compression timings: fused K1+A18+K2 vs score + ada_select."""
import sys, json
sys.path.insert(0, '.')
import bench
peaks = json.load(open('MEASURED_PEAKS.json')) if __import__('os').path.exists('MEASURED_PEAKS.json') else {}
for k, v in bench.prefill_compress(peaks).items():
    print(k, {a: (round(b, 2) if isinstance(b, float) else b) for a, b in v.items()})

import ctypes as C, numpy as np, torch
from paper_2502_15804_b200 import ops, _native
for (bt, hq, hkv, T, B) in [(1, 32, 8, 16384, 256), (1, 64, 8, 32768, 1024), (1, 64, 8, 131072, 1024)]:
    dev = torch.device("cuda")
    q = torch.randn((bt, hq, 32, 128), device=dev).to(torch.bfloat16)
    k = torch.randn((bt, hkv, T, 128), device=dev).to(torch.bfloat16)
    buf = (C.c_ulonglong * 64)()
    for _ in range(3):
        ops.score_select(q, k, B, 32)
    torch.cuda.synchronize()
    ctypes_zero = (C.c_ulonglong * 64)()
    ops.score_select(q, k, B, 32)
    torch.cuda.synchronize()
    _native.lib.fkv__score_stamps(buf)
    st = np.array(buf, dtype=np.float64)
    t0 = st[0]
    names = {0: "start", 40: "pre-stats-bar", 41: "post-stats-bar", 42: "pre-raw-bar", 43: "post-raw-bar", 1: "select-start",
             30: "search-done", 31: "pre-count-bar", 32: "post-count-bar", 33: "written"}
    for p in range(4):
        names[2 + 2 * p] = f"pass{p}-pre-bar"; names[3 + 2 * p] = f"pass{p}-post-bar"
        names[12 + 3 * p] = f"p{p}-floor-done"; names[13 + 3 * p] = f"p{p}-global-done"
    print(f"T={T} B={B}:", ", ".join(f"{names[i]} {(st[i]-t0)/1e3:.1f}" for i in sorted(names) if st[i] >= t0 and st[i] - t0 < 1e7))
