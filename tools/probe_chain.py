"""Timeline of four chained K4 launches (PDL, one CUDA graph) of one TP rank
of the 70B bench workload, from per-CTA %globaltimer stamps (probe 3, one
stamp block per launch): when each launch's CTAs enter, get their first
K/V tile, finish streaming and exit, relative to the first launch's first
CTA.  Shows how much of a layer is launch/ramp, streaming and tail, and how
far consecutive layers overlap.
usage: python tools/probe_chain.py [tp] [mode] [B] [xchg]"""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops, _native
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.decoder import rank_caches
from paper_2502_15804_b200.exchange import P2PGroup, exchange_buffer
from paper_2502_15804_b200.sharding import plan_layouts, synthetic_budgets
import bench
dev = torch.device('cuda:0')
tp = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mode = sys.argv[2] if len(sys.argv) > 2 else "sha"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
xchg = len(sys.argv) > 4 and sys.argv[4] == "xchg"
L, bt, HQ, G, N = 16, 64, 64, 8, 4  # 16 chained layers; timestamps of the first N launches
budgets = synthetic_budgets(L, bt, 8, B, window=32, alpha=0.2, seed=0, context=32768)
qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
base = [LayerCache.allocate(budgets.reshape(L, -1)[l], qrow, qrow, G, dev, fill="random") for l in range(L)]
q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)
plan, prof = bench.make_plan(budgets, tp, mode)
shards, finals = plan_layouts(plan, budgets, G)
caches = rank_caches([s[0] for s in shards], bt, HQ, G, tp, dev, base=base)
wss = [ops.DecodeWorkspace(c) for c in caches]
sends = [ops.xrec_empty(max(c.n_segments, 1), G, dev)[0] for c in caches]
grp = P2PGroup.loopback(tp, max(f.slots for f in finals), G) if xchg else None
tabs = [tuple(torch.as_tensor(x, device=dev) for x in (f.grp_ptr, f.src_idx, f.out_row)) for f in finals]
o5 = torch.empty((bt, HQ, 128), device=dev, dtype=torch.bfloat16)


def body(probe):
    for l in range(L):
        if probe and l < N:
            _native.lib.fkv__decode_probe(3 + 16 * l)
        if xchg:  # this rank's K4 + exchange, then its merge (other ranks' records pre-filled below)
            ops.decode_exchange(q[l], caches[l], grp.endpoints[0], exchange_buffer(l, L), wss[l])
        else:
            ops.decode_into(q[l], caches[l], wss[l], out_rec=sends[l])


def body_mode(mode):
    for l in range(L):
        _native.lib.fkv__decode_probe(mode)
        ops.decode_into(q[l], caches[l], wss[l], out_rec=sends[l])


g_plain = bench.capture(lambda: body(False))
gp = bench.capture(lambda: [ops.decode_partial(q[l], caches[l], wss[l]) for l in range(L)])
gp.replay()
print(f"  chained partial records only (no split merges): {min(bench.timed(gp.replay, 1) for _ in range(5)) / L * 1e6:.2f} us/layer")
for mode, nm in ((1, "loads only"), (2, "compute only")):
    gm = bench.capture(lambda: body_mode(mode))
    gm.replay()
    print(f"  chained {nm}: {min(bench.timed(gm.replay, 1) for _ in range(5)) / L * 1e6:.2f} us/layer")
g_probe = bench.capture(lambda: body(True))
for _ in range(3):
    g_probe.replay()
torch.cuda.synchronize()
t_plain = min(bench.timed(g_plain.replay, 1) for _ in range(5)) / L
n = caches[0].n_workers
buf = (C.c_ulonglong * (4 * 1024 * 16))()
_native.lib.fkv__decode_stamps(buf, 4 * 1024 * 16)
st = np.array(buf, dtype=np.float64).reshape(4, 1024, 16)[:, :n, :]  # launches 0..N-1
times = st[:, :, 1:].copy()
times[times == 0] = np.nan
t0 = np.nanmin(times[0, :, 11])  # entry stamp (index 12 -> 11 here)
rel = (times - t0) / 1e3
print(f"tp{tp} {mode} B={B} {'xchg' if xchg else 'rec'}: workers {n}, kv {caches[0].kv_bytes()/1e6:.1f} MB/layer, "
      f"flags {caches[0].flags}, chained graph {t_plain*1e6:.2f} us/layer (no probe)")
cols = {"entry": 11, "pdl-wait": 0, "combine": 2, "pre-atomic": 5, "post-atomic": 6, "merge0": 12, "merge1": 13,
        "exit": 4}
for l in range(N):
    line = f"  launch {l}:"
    for nm, i in cols.items():
        x = rel[l, :, i]
        x = x[~np.isnan(x)]
        if len(x):
            line += f"  {nm} {x.min():6.2f}/{np.median(x):6.2f}/{x.max():6.2f}"
    print(line)
print("  (min/median/max over CTAs, us from launch 0's first CTA entry)")
