"""Host-time phases of ops.compress_stack over L layers: queueing the fused
score+select launches, the one budgets read-back (waits for them), queueing
the compactions (LayerCache build + K3), the final drain; plus the GPU time
of the same stack's kernels alone.  usage: python tools/probe_stack_phases.py [layers]"""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2502_15804_b200 import ops, cache as C

dev = torch.device("cuda:0")
L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for bt, hq, T, B in ((1, 32, 16384, 256), (1, 64, 32768, 1024), (8, 64, 32768, 1024)):
    g = torch.Generator(device=dev).manual_seed(0)
    q = (torch.randn((bt, hq, 32, 128), generator=g, device=dev) * 2).to(torch.bfloat16)
    k = torch.randn((bt, 8, T, 128), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((bt, 8, T, 128), generator=g, device=dev).to(torch.bfloat16)
    hkv, group = 8, hq // 8
    need = int(ops._lib.fkv_score_workspace_bytes(bt, hkv, T, 32, group))
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    res = {}
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sel = [ops.score_select(q, k, B, workspace=ws) for _ in range(L)]
        t1 = time.perf_counter()
        hbs = torch.stack([x[1] for x in sel])
        hb_host = hbs.cpu().numpy()
        t2 = time.perf_counter()
        bh = np.arange(bt * hkv)
        qrow = (bh // hkv) * hq + (bh % hkv) * group
        caches = []
        tb = 0.0
        for l in range(L):
            x = sel[l]
            s = time.perf_counter()
            lens = hb_host[l].reshape(-1)
            cache = C.LayerCache.allocate(lens, qrow, qrow, group, dev)
            tb += time.perf_counter() - s
            caches.append(ops.compact(k, v, x[2], x[3], bh, np.zeros_like(bh), lens, qrow, qrow, group))
        t3 = time.perf_counter()
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        res = dict(queue_select=(t1 - t0), readback=(t2 - t1), queue_compact=(t3 - t2) - tb,
                   allocate_only=tb, drain=(t4 - t3), total=(t4 - t0) - tb)
    # GPU time of the kernels alone (graph-free: events around the queued work)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(L):
        ops.score_select(q, k, B, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    res["gpu_select"] = e0.elapsed_time(e1) * 1e-3
    print(f"bt={bt} T={T} B={B}: " + ", ".join(f"{a} {b / L * 1e6:.1f}" for a, b in res.items()) + " us/layer",
          flush=True)
