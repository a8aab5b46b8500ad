"""Phase timeline of the fused K1+A18+K2 launch (fkv_snapkv_select) from CTA
0's %globaltimer stamps (one-wave shapes), plus the graph-replay time of the
call, at the 8B 16k and 70B 32k / 128k prefill shapes.
usage: python tools/probe_prefill_time.py [bt ...]"""
import ctypes as C
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2502_15804_b200 import ops, _native
import bench
dev = torch.device("cuda:0")
for bt in [int(x) for x in sys.argv[1:]] or [1]:
    for hq, T, B in ((32, 16384, 256), (64, 32768, 1024), (64, 131072, 1024)):
        if bt * T > 32 * 16384:
            continue
        g = torch.Generator().manual_seed(0)
        q = (torch.randn(bt, hq, 32, 128, generator=g) * 2).to(torch.bfloat16).to(dev)
        k = torch.randn(bt, 8, T, 128, generator=g).to(torch.bfloat16).to(dev)
        need = int(_native.lib.fkv_score_workspace_bytes(bt, 8, T, 32, hq // 8))
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
        ops.score_select(q, k, B, workspace=ws)
        gr = bench.capture(lambda: ops.score_select(q, k, B, workspace=ws))
        gr.replay()
        t = min(bench.timed(gr.replay, 5) for _ in range(3)) / 5
        gs = bench.capture(lambda: ops.score(q, k, workspace=ws))
        gs.replay()
        ts = min(bench.timed(gs.replay, 5) for _ in range(3)) / 5
        ops.score_select(q, k, B, workspace=ws)
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * 64)()
        _native.lib.fkv__score_stamps(buf)
        st = np.array(buf, dtype=np.float64)
        rel = lambda i: (st[i] - st[0]) / 1e3 if st[i] else float("nan")  # noqa: E731
        line = (f"bt={bt} hq={hq} T={T} B={B}: select graph {t * 1e6:7.2f} us, score-only {ts * 1e6:7.2f} us"
                f" | w0 p1 done {rel(40):6.2f} bar {rel(41):6.2f} | all p2 done {rel(42):6.2f} bar {rel(43):6.2f}")
        if st[1] > st[0]:
            line += f" | sel start {rel(1):6.2f}"
            for p in range(4):
                line += f" | s{p}: hist {rel(2 + 2 * p):6.2f} bar {rel(3 + 2 * p):6.2f} dec {rel(13 + 3 * p):6.2f}"
            line += f" | counts {rel(31):6.2f} bar {rel(32):6.2f} write {rel(33):6.2f}"
        print(line, flush=True)
