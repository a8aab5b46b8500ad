"""Phase timeline of the grid-wide A18+K2 select (fkv_ada_select) from CTA
0's %globaltimer stamps, plus the graph-replay time of the launch, at the
8B 16k and 70B 128k prefill shapes (batch 1) and batch 4 at 16k.
usage: python tools/probe_select_phases.py"""
import ctypes as C
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2502_15804_b200 import ops, _native
import bench
dev = torch.device("cuda:0")
for bt, n, B in ((1, 16384 - 32, 256), (1, 131072 - 32, 1024)):
    s = torch.rand(bt, 8, n, generator=torch.Generator().manual_seed(0)).to(dev)
    ws = torch.empty(int(_native.lib.fkv_ada_select_workspace_bytes(bt, 8, n)), dtype=torch.uint8, device=dev)
    ops.ada_select(s, B, workspace=ws)
    g = bench.capture(lambda: ops.ada_select(s, B, workspace=ws))
    g.replay()
    t = min(bench.timed(g.replay, 10) for _ in range(3)) / 10
    ops.ada_select(s, B, workspace=ws)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 32)()
    _native.lib.fkv__select_stamps(buf)
    st = np.array(buf, dtype=np.float64)
    t0 = st[0]
    rel = lambda i: (st[i] - t0) / 1e3 if st[i] else float("nan")  # noqa: E731
    phases = []
    for p in range(4):
        phases.append(f"p{p}: start {rel(23 + 2 * p):5.2f} keys {rel(24 + 2 * p):5.2f} hist {rel(1 + 3 * p):5.2f} "
                      f"bar {rel(2 + 3 * p):5.2f} dec {rel(3 + 3 * p):5.2f}")
    print(f"bt={bt} n={n + 32} B={B}: graph replay {t * 1e6:6.2f} us; CTA0 (us from its start): "
          + " | ".join(phases) + f" | counts {rel(20):5.2f} bar {rel(21):5.2f} end {rel(22):5.2f}", flush=True)

