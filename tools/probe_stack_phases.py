"""Host-time phases of ops.compress_stack over L layers (8B 16k batch 1,
70B 32k batch 1 / 8): queueing the fused score+select launches, the per-layer
layout (waiting for each layer's budgets, then planning it), the stack's K/V
allocation + one table copy, the compaction launches, the drain -- and the
GPU time of the same selects alone.  usage: python tools/probe_stack_phases.py [layers]"""
import sys
import time
sys.path.insert(0, '.')
import torch
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.cache import LayerCache

dev = torch.device("cuda:0")
L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
orig = LayerCache.allocate_many
stamps = {}


def timed_allocate_many(layers, *a, **kw):
    stamps["enter"] = time.perf_counter()
    waits, plans = [], []

    def it():
        for x in layers:  # the generator blocks on the layer's budgets
            t = time.perf_counter()
            waits.append(t)
            yield x
    res = orig(it(), *a, **kw)
    stamps["leave"] = time.perf_counter()
    stamps["yields"] = waits
    return res


LayerCache.allocate_many = staticmethod(timed_allocate_many)
for bt, hq, T, B in ((1, 32, 16384, 256), (1, 64, 32768, 1024), (8, 64, 32768, 1024)):
    g = torch.Generator(device=dev).manual_seed(0)
    q = (torch.randn((bt, hq, 32, 128), generator=g, device=dev) * 2).to(torch.bfloat16)
    k = torch.randn((bt, 8, T, 128), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((bt, 8, T, 128), generator=g, device=dev).to(torch.bfloat16)
    for _ in range(3):
        ops.compress_stack([q] * L, [k] * L, [v] * L, B)
    best = None
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ops.compress_stack([q] * L, [k] * L, [v] * L, B)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        y = stamps["yields"]
        row = dict(total=t2 - t0, queue_selects=stamps["enter"] - t0, first_budgets=y[0] - stamps["enter"],
                   layout_loop=y[-1] - y[0], after_last=stamps["leave"] - y[-1], compactions=t1 - stamps["leave"],
                   drain=t2 - t1)
        if best is None or row["total"] < best["total"]:
            best = row
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(L):
        ops.score_select(q, k, B)
    e1.record()
    torch.cuda.synchronize()
    best["gpu_selects"] = e0.elapsed_time(e1) * 1e-3
    print(f"bt={bt} T={T} B={B} L={L}: " + ", ".join(f"{a} {b * 1e6:.0f}" for a, b in best.items()) + " us",
          flush=True)
