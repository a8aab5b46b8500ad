"""Fused K1+A18+K2 with a head below its floor (the window soaks up all of its
attention) vs without: the floor path's cost at 16k and 128k."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2502_15804_b200 import ops

dev = torch.device("cuda")


def timeit(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for (bt, hq, hkv, T, B) in [(1, 32, 8, 16384, 256), (1, 64, 8, 131072, 1024)]:
    for flat in (False, True):
        g = torch.Generator(device=dev).manual_seed(3)
        q = (torch.randn((bt, hq, 32, 128), generator=g, device=dev) * 2).to(torch.bfloat16)
        k = torch.randn((bt, hkv, T, 128), generator=g, device=dev).to(torch.bfloat16)
        if flat:
            G = hq // hkv
            u = torch.full((128,), 0.5, dtype=torch.bfloat16, device=dev)
            q[:, 3 * G:4 * G] = u
            k[:, 3] = 0
            k[:, 3, T - 32:] = 20 * u
        ws = torch.empty(int(ops._lib.fkv_score_workspace_bytes(bt, hkv, T, 32, hq // hkv)), dtype=torch.uint8,
                         device=dev)
        t_f = timeit(lambda: ops.score_select(q, k, B, 32, workspace=ws))
        sc, hb, _, _ = ops.score_select(q, k, B, 32, workspace=ws)
        t_s = timeit(lambda: ops.ada_select(sc, B, 32))
        print(f"T={T} B={B} flat={flat}: fused {t_f:.1f} us, standalone select {t_s:.1f} us, "
              f"budgets {hb[0].tolist()}")
