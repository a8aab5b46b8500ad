"""Host cost of queueing one fused score+select launch (fkv_snapkv_select
through ctypes) and of the pieces around it in compress_stack, measured
while the GPU is busy (launches only queue).  usage: python tools/probe_launch_host.py"""
import math
import sys
import time
sys.path.insert(0, '.')
import torch
from paper_2502_15804_b200 import ops

dev = torch.device("cuda:0")
bt, hq, hkv, T, B, w = 1, 32, 8, 16384, 256, 32
g = torch.Generator(device=dev).manual_seed(0)
q = (torch.randn((bt, hq, w, 128), generator=g, device=dev) * 2).to(torch.bfloat16)
k = torch.randn((bt, hkv, T, 128), generator=g, device=dev).to(torch.bfloat16)
BH = bt * hkv
need = int(ops._lib.fkv_score_workspace_bytes(bt, hkv, T, w, hq // hkv))
ws = torch.empty(need, dtype=torch.uint8, device=dev)
sc = torch.empty((bt, hkv, T - w), dtype=torch.float32, device=dev)
hb = torch.empty((bt, hkv), dtype=torch.int32, device=dev)
off = torch.empty(BH + 1, dtype=torch.int64, device=dev)
idx = torch.empty(BH * B, dtype=torch.int32, device=dev)
st = torch.cuda.current_stream().cuda_stream
args = (q.data_ptr(), k.data_ptr(), bt, hq, hkv, T, w, 7, 1 / math.sqrt(128), B, ops.ada_floor(B, w, 0.2),
        sc.data_ptr(), hb.data_ptr(), off.data_ptr(), idx.data_ptr(), ws.data_ptr(), st)
fn = ops._lib.fkv_snapkv_select
big = torch.empty(1 << 28, device=dev)
N = 20


def busy():
    for _ in range(20):
        big.mul_(1.0)  # ~ms of GPU work ahead of the launches


def timed(name, f):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        busy()
        t = time.perf_counter()
        for _ in range(N):
            f()
        best = min(best, (time.perf_counter() - t) / N)
        torch.cuda.synchronize()
    print(f"{name:34s} {best * 1e6:7.1f} us", flush=True)


timed("fkv_snapkv_select (ctypes)", lambda: fn(*args))
timed("fkv_snapkv_score (ctypes)", lambda: ops._lib.fkv_snapkv_score(
    q.data_ptr(), k.data_ptr(), bt, hq, hkv, T, w, 7, 1 / math.sqrt(128), sc.data_ptr(), ws.data_ptr(), st))
timed("ops.score_select", lambda: ops.score_select(q, k, B, workspace=ws))
timed("torch.cuda.Event() + record", lambda: torch.cuda.Event().record())
side = torch.cuda.Stream()
pin = torch.empty(BH, dtype=torch.int32, pin_memory=True)


def d2h():
    e = torch.cuda.Event()
    e.record()
    side.wait_event(e)
    with torch.cuda.stream(side):
        pin.copy_(hb.view(-1), non_blocking=True)
        e2 = torch.cuda.Event()
        e2.record(side)


timed("side-stream budgets copy", d2h)
timed("cudaMemsetAsync (torch zero_ 256B)", lambda: ws[:256].zero_())
