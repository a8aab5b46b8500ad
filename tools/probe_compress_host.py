"""Host-visible time of a layer stack's prefill compression: compress_layer
per layer (one host round trip each) vs compress_stack (one round trip),
per layer, at the 8B 16k and 70B 32k shapes.  FKV_PY_SCHEDULE=1 selects the
Python schedule planner for comparison.
usage: python tools/probe_compress_host.py [layers]"""
import sys
import time
sys.path.insert(0, '.')
import torch
from paper_2502_15804_b200 import ops

dev = torch.device("cuda:0")
L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for bt, hq, T, B in ((1, 32, 16384, 256), (4, 32, 16384, 256), (1, 64, 32768, 1024), (8, 64, 32768, 1024)):
    g = torch.Generator(device=dev).manual_seed(0)
    q = (torch.randn((bt, hq, 32, 128), generator=g, device=dev) * 2).to(torch.bfloat16)
    k = torch.randn((bt, 8, T, 128), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((bt, 8, T, 128), generator=g, device=dev).to(torch.bfloat16)
    for _ in range(2):
        ops.compress_layer(q, k, v, B)
        ops.compress_stack([q] * L, [k] * L, [v] * L, B)
    torch.cuda.synchronize()
    res = {}
    for name, fn in (("per_layer", lambda: [ops.compress_layer(q, k, v, B) for _ in range(L)]),
                     ("stack", lambda: ops.compress_stack([q] * L, [k] * L, [v] * L, B))):
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        res[name] = best / L * 1e6
    print(f"bt={bt} hq={hq} T={T} B={B}: compress_layer {res['per_layer']:7.1f} us/layer, "
          f"compress_stack {res['stack']:7.1f} us/layer", flush=True)
