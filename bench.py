"""FairKV decode benchmark on B200 (driver contract: one JSON line on rank 0).

Metric (BASELINE.json): decode tokens/s of the Llama-3.3-70B-shaped attention
sub-stack -- 80 layers x (K4 split-KV decode over the Ada-compressed,
AHA-sharded cache, fused per-segment LSE merge [+ the per-layer all-gather
and the K5 merge of DP copies at N > 1]) -- for AHA and for uniform
head-sharded TP, plus per-GPU KV load max/mean.  QKV / o_proj / MLP GEMMs are
excluded by definition (the 70B weights would bury AHA's
effect); the reference itself measured "a single layer ... decoding one
token".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fairkv|reference]

* ``value``: tokens/s with q and the cache resident in HBM, the 80-layer step
  captured in a CUDA graph and timed with CUDA events, max over ranks.  At
  N > 1 every placement (uniform TP = ``sha``; AHA ``nodp`` / ``dp`` equal
  split / ``dp-free`` free split) is built and timed on the same cache; the
  value is the best AHA placement and ``modes`` lists all of them.  Before
  timing, rank 0 checks one step's gathered o of every placement against a
  local single-GPU decode of the same layers.
* ``e2e``: the same metric through the public API with q copied from pinned
  host memory and o copied back every step (inside the timed region).
* ``roofline``: K4 alone (graph of its 80 launches), algorithmic bytes
  (retained K+V + q + o + split-segment records) / mean launch time vs the
  measured HBM bandwidth.
* ``cpu_baseline``: the float64 oracle (oracle/workload.py) decoding one full
  80-layer step of the same workload on all host cores (rank 0, N = 1).
* ``emulated_tp`` (N = 1): AHA vs uniform TP at 2/4/8 GPUs emulated on this
  GPU -- every rank's K4 + fused exchange stores of every layer timed alone,
  span = sum_l max_g t(l, g) + the K5 merge (the reference simulator's
  synchronous per-layer barrier, simulate.py:118-136); NVLink latency is not
  included (one GPU).
``--impl reference`` times the CPU reference path on the same config: the
oracle port of the decode (the reference has no decode) over the
budgets built with the reference's own generate_profile; it never imports
this package.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

L_LAYERS, HQ, HKV, GROUP, HEAD_DIM = 80, 64, 8, 8, 128
WINDOW, ALPHA = 32, 0.2
METRIC = "decode tokens/s (Llama-3.3-70B attention sub-stack, Ada-compressed KV, AHA-sharded)"
AHA_MODES = ("nodp", "dp", "dp-free")


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["fairkv", "reference"], default="fairkv")
    p.add_argument("--budget", type=int, default=1024)
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--layers", type=int, default=L_LAYERS)
    p.add_argument("--context", type=int, default=32768)
    p.add_argument("--ch", type=int, default=4)
    p.add_argument("--modes", default="sha,nodp,dp,dp-free", help="placements timed at N > 1")
    p.add_argument("--no-emulate", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                   help="N>1 per-layer exchange: fused NVLink P2P stores (default) or NCCL all-gather")
    return p.parse_args(argv)


# --------------------------------------------------------- workload -----
def workload_name(args) -> str:
    return (f"llama-3.3-70b attention sub-stack decode: {args.layers} layers, {HQ}Q/{HKV}KV heads, "
            f"d={HEAD_DIM}, Ada-SnapKV avg budget {args.budget}/head (dirichlet a=8 head skew, "
            f"w={WINDOW}, alpha={ALPHA}), context {args.context}, batch {args.batch}")


def workload_config(args, world: int) -> dict:
    """The config both arms print (identical keys and values)."""
    return {
        "workload": workload_name(args),
        "global_batch": args.batch,
        "layers": args.layers,
        "avg_budget": args.budget,
        "context": args.context,
        "parallelism": f"tp{world}" + ("" if world == 1 else " (AHA placements vs uniform head-sharded TP)"),
        "l2": "inputs larger than L2: the retained K/V read every step is GBs per GPU (126 MB L2)",
    }


def ref_headbalance():
    """The unmodified reference package (baseline/_ref, else its sources), or None."""
    for d in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (d / "headbalance" / "__init__.py").exists():
            if str(d) not in sys.path:
                sys.path.append(str(d))
            try:
                import headbalance
                return headbalance
            except Exception:
                return None
    return None


def workload_budgets(args):
    from paper_2502_15804_b200.sharding import synthetic_budgets
    return synthetic_budgets(args.layers, args.batch, HKV, args.budget, window=WINDOW, alpha=ALPHA,
                             seed=args.seed, context=args.context)


def make_plan(budgets, tp, mode, ch=4, workers=8):
    """AHA placement of the workload's profile (KV-head planning unit):
    sha = uniform head-sharded TP (allocate.sha_plan); nodp = no copies;
    dp = equal split (CH=8 at TP=8, where CH=4 degenerates to SHA, SURVEY
    §0.4); dp-free = free split, CH=4."""
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200.sharding import budgets_profile
    prof = budgets_profile(budgets, int(budgets.mean()))
    if tp == 1 or mode == "sha":
        return fk.sha_plan(prof, tp), prof
    if mode == "nodp":
        return fk.optimize_plan(prof, tp, fk.EnumerationConfig(0, 1, True, tp), workers=workers), prof
    if mode == "dp-free":
        return fk.optimize_plan(prof, tp, fk.EnumerationConfig(ch, 2, True, tp), equal_split=False,
                                workers=workers), prof
    ch_eq = 8 if tp == 8 else ch
    return fk.optimize_plan(prof, tp, fk.EnumerationConfig(ch_eq, 2, True, tp), workers=workers), prof


def mode_label(tp, mode, ch=4):
    if tp == 1 or mode == "sha":
        return "uniform head-sharded TP (sha_plan)"
    if mode == "nodp":
        return "AHA-NoDP"
    if mode == "dp-free":
        return f"AHA-DP free split CH={ch}"
    return f"AHA-DP equal split CH={8 if tp == 8 else ch}"


# ------------------------------------------------------------- clocks -----
class ClockSampler:
    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 5 and self.proc.poll() is None:
                time.sleep(0.02)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# -------------------------------------------------------------- timing ----
def timed(fn, steps, stream=None):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def _dist_dev():
    import torch.distributed as dist
    return "cpu" if dist.get_backend() == "gloo" else "cuda"


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_dist_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def capture(fn):
    import torch
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()  # warm (allocations, attributes) outside capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fn()
    return g


def k4_bytes(c):
    """Algorithmic bytes of one K4 launch over cache c: retained K+V, q in and
    o out per segment (bf16), fp32 partial records of split segments written
    and read back."""
    import numpy as np
    from paper_2502_15804_b200 import ops
    per_seg = np.diff(c.grp_ptr.cpu().numpy())
    multi = int(per_seg[per_seg > 1].sum())
    return (c.kv_bytes() + 2 * c.n_segments * GROUP * HEAD_DIM * 2 + 2 * multi * GROUP * ops.REC * 4)


# ------------------------------------------------------- CPU baseline -----
def cpu_step_sample(budgets, hb_note: str):
    """One full step (every layer) of the float64 oracle decode on all host
    cores: (tokens/s, sample text, cores)."""
    from oracle.workload import CpuDecodeStack
    st = CpuDecodeStack(budgets, HQ)
    st.step(layers=1)  # warm the pool / BLAS
    t0 = time.perf_counter()
    st.step()
    dt = time.perf_counter() - t0
    st.close()
    bt = budgets.shape[1]
    return bt / dt, (f"one full decode step ({budgets.shape[0]} layers x batch {bt} x {HKV} KV heads, "
                     f"float64 oracle/workload.py, {st.threads} threads; {hb_note})"), st.threads


# --------------------------------------------------------- our arm --------
class Placement:
    """One placement of the workload on this rank: caches (views of the shared
    base cache), decoder, captured step graph."""

    def __init__(self, mode, tp, rank, budgets, base, args, dev):
        import torch
        from paper_2502_15804_b200.decoder import StackDecoder, rank_caches
        from paper_2502_15804_b200.sharding import imbalance_ratio, plan_layouts, rank_loads
        self.mode = mode
        self.plan, self.prof = make_plan(budgets, tp, mode, args.ch)
        shards, finals = plan_layouts(self.plan, budgets, GROUP)
        self.caches = rank_caches([s[rank] for s in shards], args.batch, HQ, GROUP, tp, dev, base=base)
        self.endpoint = None
        self.exchange = args.exchange if tp > 1 else None
        if tp > 1 and args.exchange == "p2p":
            from paper_2502_15804_b200.exchange import P2PGroup
            self.group = P2PGroup.connect(rank, tp, finals[0].slots, GROUP)
            self.endpoint = self.group.endpoints[0]
        self.dec = StackDecoder(self.caches, finals if tp > 1 else None, tp=tp, bt=args.batch, hq=HQ,
                                group=GROUP, exchange=args.exchange if tp > 1 else "nccl",
                                endpoint=self.endpoint)
        loads = rank_loads(self.plan, budgets, GROUP)
        self.kv = {"max_over_mean": imbalance_ratio(loads), "per_gpu_tokens": loads.sum(axis=0).tolist()}
        self.extra_copies = int(sum(len(g) for la in self.plan.layers for g in la.groups) - args.layers * HKV)
        self.use_graph = tp == 1 or args.exchange == "p2p"  # the P2P flag protocol is replay-safe

    def build(self, q, o):
        self.step = lambda: self.dec.step(q, o)
        if self.use_graph:
            self.graph = capture(self.step)
            self.run = self.graph.replay
        else:
            self.run = self.step


def run_fairkv(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    args.gpus = world
    # FKV_SHARED_DEVICE=1 (protocol check only, timings meaningless): every
    # rank on cuda:0 with gloo plumbing -- the N > 1 code path on a 1-GPU box
    shared = os.environ.get("FKV_SHARED_DEVICE") == "1"
    if shared:
        local = 0
        args.exchange = "p2p"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    tp = world
    budgets = workload_budgets(args)

    # The full per-head cache of every layer, identical on every rank (same
    # seed); each placement's rank cache is a view of it (DP copies = 16-row
    # aligned sub-ranges), so rank 0 can recompute any layer locally.
    qrow = np.array([b * HQ + h * GROUP for b in range(args.batch) for h in range(HKV)])
    gen = torch.Generator(device=dev).manual_seed(1000 + args.seed)
    base = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, GROUP, dev, fill="random", generator=gen)
            for l in range(args.layers)]
    gq = torch.Generator(device=dev).manual_seed(123)
    q = torch.randn((args.layers, args.batch, HQ, HEAD_DIM), generator=gq, device=dev).to(torch.bfloat16)
    o = torch.empty_like(q)

    modes = ["sha"] if tp == 1 else [m for m in args.modes.split(",") if m]
    if tp > 1 and args.exchange == "p2p":
        # every rank must take the same exchange path: probe CUDA IPC / peer access once
        ok = 1
        try:
            from paper_2502_15804_b200.exchange import P2PGroup
            P2PGroup.connect(rank, tp, 1, GROUP).close()
        except Exception as exc:
            print(f"rank {rank}: P2P exchange unavailable ({exc}); using NCCL all-gather", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=_dist_dev())
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0 and not shared:
            args.exchange = "nccl"
    places = {m: Placement(m, tp, rank, budgets, base, args, dev) for m in modes}
    for p in places.values():
        p.build(q, o)

    # ---- rank 0 checks each placement's gathered o against a local decode
    check = {}
    if tp > 1:
        ref = torch.stack([ops.decode(q[l], base[l])[0] for l in (0, args.layers - 1)])
        for m, p in places.items():
            o.zero_()
            p.run()
            torch.cuda.synchronize()
            got = torch.stack([o[0], o[args.layers - 1]])
            err = float((got.float() - ref.float()).abs().max())
            good = bool(torch.allclose(got.float(), ref.float(), rtol=2e-2, atol=4e-3))
            flag = torch.tensor([int(good)], dtype=torch.int32, device=_dist_dev())
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            check[m] = {"max_abs_err_vs_local": err, "ok": bool(flag.item())}
            if not flag.item():
                raise RuntimeError(f"placement {m}: gathered o differs from the local decode (err {err})")

    for p in places.values():
        for _ in range(args.warmup):
            p.run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    res = {}
    with ClockSampler(local) as clk:
        # hold the clocks under load for ~1 s before timing.  The replay count
        # must be the same on every rank: the exchange's flags are counters,
        # so a rank that ran one replay more than its peers would wait for
        # flags that never come.
        first = places[modes[0]]
        t_one = max(timed(first.run, 1), 1e-6)
        n_load = max(1, int(1.0 / t_one))
        if world > 1:
            cnt = torch.tensor([n_load], dtype=torch.int64, device=_dist_dev())
            dist.all_reduce(cnt, op=dist.ReduceOp.MIN)
            n_load = int(cnt.item())
        for _ in range(n_load):
            first.run()
        torch.cuda.synchronize()
        for m, p in places.items():
            if world > 1:
                dist.barrier()
            t = max_over_ranks(timed(p.run, args.steps), world)
            res[m] = t
    best = "sha" if tp == 1 else max((m for m in modes if m != "sha"), key=lambda m: -res[m], default="sha")
    t = res[best]
    tok_s = args.batch * args.steps / t
    bp = places[best]
    launches = bp.dec.kernel_launches_per_step * args.steps

    # ---- roofline of the dominant kernel (K4 with its fused merge), best placement
    if tp == 1:
        t4 = t / (args.steps * args.layers)  # the step is exactly the 80 K4 launches
    else:
        send = [ops.xrec_empty(max(c.n_segments, 1), GROUP, dev)[0] for c in bp.caches]

        def k4_only():
            for l in range(args.layers):
                ops.decode_into(q[l], bp.caches[l], bp.dec.ws[l], out_rec=send[l])
        g4 = capture(k4_only)
        for _ in range(2):
            g4.replay()
        t4 = timed(g4.replay, args.steps) / (args.steps * args.layers)
    bytes_k4 = float(np.mean([k4_bytes(c) for c in bp.caches]))
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bytes_k4 / t4 / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "k4_traffic.json"
    if tfile.exists() and tp == 1:
        traffic = json.loads(tfile.read_text()).get("bytes_per_launch")

    # ---- e2e through the public API with host buffers: per-layer-group H2D of
    # q, decode, D2H of o, pipelined over two copy streams, one CUDA graph ----
    qh = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
    qh.copy_(q)
    oh = torch.empty(o.shape, dtype=o.dtype, pin_memory=True)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    # layers per copy group: "sym" (default; 17.4k -> 17.8k tokens/s against
    # uniform groups of 4, the best of 1-40) or a fixed group size
    cg = os.environ.get("FKV_E2E_GROUP", "sym")
    if cg.startswith("sym"):
        # copy groups growing geometrically from each end (1, 2, 4, ...
        # layers): the first upload and the last download stay short, and the
        # middle needs few event nodes (each one breaks the layers'
        # programmatic-launch chain); "sym:<first>:<factor>"
        w0, fac = (int(x) for x in (cg.split(":")[1:] + ["1", "2"])[:2]) if ":" in cg else (1, 2)
        cuts, a, b, w = {0, args.layers}, 0, args.layers, w0
        while a < b:
            a, b = min(a + w, b), max(b - w, a)
            cuts |= {a, b}
            w *= fac
        cuts = sorted(cuts)
    else:
        cg = int(cg)
        cuts = sorted({0, min(1, args.layers), max(args.layers - 1, 0), args.layers,
                       *range(1, args.layers - 1, cg)})
    groups = [(a, b) for a, b in zip(cuts, cuts[1:]) if b > a]
    ev_in = [torch.cuda.Event() for _ in groups]
    ev_out = [torch.cuda.Event() for _ in groups]

    def e2e_body():
        cur = torch.cuda.current_stream()
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        with torch.cuda.stream(s_in):
            for gi, (a, b) in enumerate(groups):
                q[a:b].copy_(qh[a:b], non_blocking=True)
                ev_in[gi].record(s_in)
        for gi, (a, b) in enumerate(groups):
            cur.wait_event(ev_in[gi])
            for l in range(a, b):
                bp.dec.layer(l, q[l], o[l])
            ev_out[gi].record(cur)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_out[gi])
                oh[a:b].copy_(o[a:b], non_blocking=True)
        cur.wait_stream(s_in)
        cur.wait_stream(s_out)
    e2e_run = capture(e2e_body).replay if bp.use_graph else e2e_body
    for _ in range(2):
        e2e_run()
    if world > 1:
        dist.barrier()
    te = max_over_ranks(timed(e2e_run, args.steps), world)

    out = {
        "metric": METRIC,
        "value": tok_s,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init N(0,1) bf16 K/V/q; Ada-shaped per-head budgets)",
        "config": workload_config(args, world),
        "placement": mode_label(tp, best, args.ch) + (f", exchange {args.exchange}" if tp > 1 else ""),
        "kv_load": places[best].kv,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "fkv decode_kernel<8> (K4 with fused LSE merge)",
                     "bytes_per_launch": bytes_k4, "us_per_launch": t4 * 1e6,
                     "k4_share_of_step": (t4 * args.layers) / (t / args.steps),
                     "bytes_note": "retained K+V + q + o + split-segment partial records (write+read); "
                                   "at N > 1 this rank's shard of the best placement",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"},
        "e2e": {"value": args.batch * args.steps / te, "unit": "tokens/s",
                "h2d_bytes_per_step": q.numel() * 2, "d2h_bytes_per_step": o.numel() * 2},
        "clocks": clk.summary(),
    }
    if tp > 1:
        out["modes"] = {m: {"tokens_per_s": args.batch * args.steps / res[m], "ms_per_step": res[m] / args.steps * 1e3,
                            "placement": mode_label(tp, m, args.ch), "kv_load_max_over_mean": places[m].kv["max_over_mean"],
                            "extra_copies": places[m].extra_copies,
                            "gain_vs_sha": (res["sha"] / res[m]) if "sha" in res else None}
                        for m in modes}
        out["check"] = check
    if rank == 0 and world == 1 and not args.no_cpu:
        v, sample, cores = cpu_step_sample(budgets, "budgets from the product's generator")
        out["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port",
                               "sample": sample}
    del places
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_emulate:
        out["emulated_tp"] = emulate_tp(args, budgets, dev, base, q)
        out["calibration"] = calibrate_reference(args, budgets, dev, base, q)
        del base
        torch.cuda.empty_cache()
        out["emulated_tp_budget_sweep"] = budget_sweep(args, dev)
        out["cfg4_tp8_batch_sweep"] = cfg4_batch_sweep(args, dev)
        out["cfg5_tp8_skew_B1024"] = cfg5_skew(args, dev)
        out["cfg2_llama3.1-8b_b256_T16k"] = cfg2_sweep(args, dev, peak)
        out["full_layer"] = full_layer(args, budgets, dev)
        out["append"] = append_cost(args, budgets, dev)
        out["prefill"] = prefill_compress(peaks)
    if rank == 0 and world == 1 and not args.no_cpu:
        out["planner"] = planner_compare(budgets)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------- emulated TP (N = 1) -----
EMU_REPLAYS = 3  # replays per back-to-back emulated timing (min)
# replays of the event-bracketed graph: CUDA event timestamps are quantised
# (~0.5 us), so a per-(layer, rank) median of a few replays is a multiple of
# the quantum and the max over similar ranks picks whichever rounded up; the
# mean over many replays resolves below the quantum (natural jitter dithers)
EMU_SPAN_REPLAYS = 16
EMU_ROUNDS = 5   # interleaved rounds over the placements; the median round is reported


def _alloc_base(budgets, dev, seed=7):
    import numpy as np
    import torch
    from paper_2502_15804_b200.cache import LayerCache
    L, bt = budgets.shape[0], budgets.shape[1]
    qrow = np.array([b * HQ + h * GROUP for b in range(bt) for h in range(HKV)])
    gen = torch.Generator(device=dev).manual_seed(seed)
    base = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, GROUP, dev, fill="random", generator=gen)
            for l in range(L)]
    q = torch.randn((L, bt, HQ, HEAD_DIM), device=dev, generator=gen).to(torch.bfloat16)
    return base, q


def emulate_tp(args, budgets, dev, base, q, tps=(2, 4, 8), modes=("sha",) + AHA_MODES):
    """AHA vs uniform TP at 2/4/8 GPUs on this GPU.  Per placement and rank
    g: K4 with the fused exchange (``decode_exchange`` into loopback
    endpoints: every record stored to all tp receive areas as epoch-tagged XLL units)
    over the rank's shard of every layer, timed alone (event nodes in one
    CUDA graph) and corrected by the rank's 80 layers back to back; then the
    K5 merge of the gathered records.  Layer span = max_g t(l, g) + K5(l)."""
    import numpy as np
    import torch
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.decoder import rank_caches
    from paper_2502_15804_b200.exchange import P2PGroup, exchange_buffer
    from paper_2502_15804_b200.sharding import imbalance_ratio, plan_layouts, rank_loads

    hb = ref_headbalance()
    L, bt = budgets.shape[0], budgets.shape[1]
    results = {}
    for tp in tps:
        row, st = {}, {}
        for mode in modes:
            plan, prof = make_plan(budgets, tp, mode, args.ch)
            shards, finals = plan_layouts(plan, budgets, GROUP)
            per_rank = [rank_caches([s[g] for s in shards], bt, HQ, GROUP, tp, dev, base=base) for g in range(tp)]
            grp = P2PGroup.loopback(tp, finals[0].slots, GROUP)
            wss = [[ops.DecodeWorkspace(c) for c in pr] for pr in per_rank]
            evs = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(tp + 1)] for _ in range(L)]
            bufs = [exchange_buffer(l, L) for l in range(L)]

            def body(per_rank=per_rank, wss=wss, evs=evs, grp=grp, bufs=bufs):
                for l in range(L):
                    for g in range(tp):
                        evs[l][g].record()
                        ops.decode_exchange(q[l], per_rank[g][l], grp.endpoints[g], bufs[l], wss[g][l])
                    evs[l][tp].record()
            gph = capture(body)
            ggs = []
            for g in range(tp):
                def run_g(g=g, per_rank=per_rank, wss=wss, grp=grp, bufs=bufs):
                    for l in range(L):
                        ops.decode_exchange(q[l], per_rank[g][l], grp.endpoints[g], bufs[l], wss[g][l])
                ggs.append(capture(run_g))
            # K5: the marginal cost of every rank's merge_wait (polls its XLL
            # records, merges, advances the epoch) -- all ranks' K4 + K5 per
            # layer minus the same K4 sequence alone, per (layer, rank)
            tabs = [tuple(torch.as_tensor(x, device=dev) for x in (f.grp_ptr, f.src_idx, f.out_row))
                    for f in finals]
            o5 = torch.empty((bt, HQ, HEAD_DIM), dtype=torch.bfloat16, device=dev)

            def run_k4(per_rank=per_rank, wss=wss, grp=grp, bufs=bufs):
                for l in range(L):
                    for g in range(tp):
                        ops.decode_exchange(q[l], per_rank[g][l], grp.endpoints[g], bufs[l], wss[g][l])

            def run_k45(per_rank=per_rank, wss=wss, grp=grp, bufs=bufs, tabs=tabs, o5=o5):
                for l in range(L):
                    for g in range(tp):
                        ops.decode_exchange(q[l], per_rank[g][l], grp.endpoints[g], bufs[l], wss[g][l])
                    for g in range(tp):
                        ops.merge_wait(grp.endpoints[g], bufs[l], *tabs[l], GROUP, out_bf16=o5)
            g4, g45 = capture(run_k4), capture(run_k45)
            g5 = (g4, g45)
            st[mode] = dict(plan=plan, prof=prof, keep=(per_rank, wss, grp, tabs, o5), evs=evs, gph=gph,
                            ggs=ggs, g5=g5, rounds=[])

        def measure(m):
            gph, evs, ggs = m["gph"], m["evs"], m["ggs"]
            span = []
            for _ in range(EMU_SPAN_REPLAYS):
                gph.replay()
                torch.cuda.synchronize()
                span.append(np.array([[evs[l][g].elapsed_time(evs[l][g + 1]) for g in range(tp)]
                                      for l in range(L)]) * 1e-3)
            t_br = np.mean(np.stack(span), axis=0)  # [L, tp], each launch event-bracketed
            t = np.empty_like(t_br)
            for g in range(tp):
                ggs[g].replay()
                tot = min(timed(ggs[g].replay, 1) for _ in range(EMU_REPLAYS))
                c_g = max(0.0, (t_br[:, g].sum() - tot) / L)
                t[:, g] = np.maximum(t_br[:, g] - c_g, 0.0)
            g4, g45 = m["g5"]
            g45.replay()
            t4 = min(timed(g4.replay, 1) for _ in range(EMU_REPLAYS))
            t45 = min(timed(g45.replay, 1) for _ in range(EMU_REPLAYS))
            k5 = max(0.0, t45 - t4) / (L * tp)
            return t, t_br, k5

        for _ in range(EMU_ROUNDS):
            for mode in modes:
                st[mode]["rounds"].append(measure(st[mode]))
        for mode in modes:
            m = st[mode]
            steps = [r[0].max(axis=1).sum() + L * r[2] for r in m["rounds"]]
            t, t_br, k5 = m["rounds"][int(np.argsort(steps)[len(steps) // 2])]
            step = t.max(axis=1).sum() + L * k5
            loads = rank_loads(m["plan"], budgets, GROUP)
            r = {"tokens_per_s": bt / step, "stack_ms": step * 1e3,
                 "tokens_per_s_k4_only": bt / t.max(axis=1).sum(),
                 "k5_us_per_layer": k5 * 1e6,
                 "k4x_us_per_layer_max_rank": float(t.max(axis=1).mean() * 1e6),
                 "busy_rate": float(t.sum() / (t.max(axis=1).sum() * tp)),
                 "kv_max_over_mean": imbalance_ratio(loads),
                 "extra_copies": int(sum(len(g) for la in m["plan"].layers for g in la.groups) - L * HKV),
                 "rounds_tokens_per_s": [round(bt / x, 1) for x in steps],
                 "placement": mode_label(tp, mode, args.ch)}
            # the reference's load efficiency of the plan (allocate.py:418-424: mean
            # per-GPU load / bottleneck load), beside the measured busy rate
            import paper_2502_15804_b200 as fk
            r["efficiency"] = float((hb or fk).efficiency(m["plan"], m["prof"]))
            if hb is not None:  # the reference simulator's prediction (pure-cache latency law)
                model = hb.LatencyModel(0.0, 0.0, 1.0, 0.0)
                r["sim_throughput"] = hb.simulate(m["prof"], m["plan"], model, hb.SimulationConfig(1, 1, tp)).throughput
            row[mode] = r
        del st
        torch.cuda.empty_cache()
        for mode in modes[1:]:
            row[mode]["gain_vs_sha"] = row[mode]["tokens_per_s"] / row["sha"]["tokens_per_s"]
            if "sim_throughput" in row[mode]:
                row[mode]["sim_gain_vs_sha"] = row[mode]["sim_throughput"] / row["sha"]["sim_throughput"]
        aha = max(modes[1:], key=lambda m_: row[m_]["tokens_per_s"])
        row["best_aha"] = {"placement": aha, "gain_vs_sha": row[aha]["gain_vs_sha"]}
        results[f"tp{tp}"] = row
    results["note"] = ("per placement and rank: K4 with the fused exchange stores into loopback endpoints "
                       "(decode_exchange: XLL records tagged with the layer's epoch to all tp receive areas) "
                       "of every layer timed alone on this GPU (event nodes in one CUDA graph) minus the "
                       "per-launch bracketing overhead (each rank's 80 layers back to back); layer span = max "
                       "over ranks + K5 (merge_wait: polls the records, merges, advances the epoch; its "
                       "marginal cost per launch) (synchronous per-layer barrier, reference "
                       "simulate.py:118-136); NVLink latency not included (one GPU); placements timed in 3 "
                       "interleaved rounds, median round; sim = reference simulator, pure-cache latency law")
    return results


def calibrate_reference(args, budgets, dev, base, q):
    """measured per-layer decode latencies -> the reference's
    own latency.calibrate (OLS on c0 + c1 B + c2 C + c3 B C, C = retained
    tokens per request on one GPU-layer) -> the reference's compare()
    predicting the AHA gains at TP 2/4/8.  Samples: whole TP1 layers over the
    first `nh` KV heads of the first `sub` requests, batch 1/4/16/64 x
    1/2/4/8 heads (batch and load vary independently, as the law needs),
    plus the same batches over all 8 heads cut to their first 16 / 64
    retained tokens: small per-request loads expose the per-request cost
    (q, o, one segment per head) that the c1 term models -- without them the
    OLS has nothing to pin c1 and returns it slightly negative (rejected)."""
    import numpy as np
    import torch
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache
    from paper_2502_15804_b200.sharding import budgets_profile
    hb = ref_headbalance()
    if hb is None:
        return {"unavailable": "reference package not installed (baseline/_ref)"}
    L = budgets.shape[0]
    samples = []
    for i, sub in enumerate((1, 4, 16, 64)):
        for j, nh in enumerate((1, 2, 4, 8)):
            l = (7 * i + 3 * j) % L
            heads = [b * HKV + h for b in range(sub) for h in range(nh)]
            lens = budgets[l].reshape(-1)[heads]
            qrow = np.array([b * HQ + h * GROUP for b in range(sub) for h in range(nh)])
            c = LayerCache.view(base[l].k, base[l].v, base[l].host["seg_row0"][heads], lens, qrow, qrow, GROUP)
            qq = q[l, :sub].contiguous()
            oo = torch.empty_like(qq)
            ws = ops.DecodeWorkspace(c)
            g = capture(lambda: [ops.decode_into(qq, c, ws, out_bf16=oo) for _ in range(10)])
            g.replay()
            tt = min(timed(g.replay, 1) for _ in range(3)) / 10
            samples.append(hb.MeasurementSample(sub, float(lens.sum()) / sub, tt))
    for i, sub in enumerate((1, 4, 16, 64)):
        for cap in (16, 64):
            l = (5 * i + cap) % L
            heads = [b * HKV + h for b in range(sub) for h in range(HKV)]
            lens = np.minimum(budgets[l].reshape(-1)[heads], cap)
            qrow = np.array([b * HQ + h * GROUP for b in range(sub) for h in range(HKV)])
            c = LayerCache.view(base[l].k, base[l].v, base[l].host["seg_row0"][heads], lens, qrow, qrow, GROUP)
            qq = q[l, :sub].contiguous()
            oo = torch.empty_like(qq)
            ws = ops.DecodeWorkspace(c)
            g = capture(lambda: [ops.decode_into(qq, c, ws, out_bf16=oo) for _ in range(10)])
            g.replay()
            tt = min(timed(g.replay, 1) for _ in range(3)) / 10
            samples.append(hb.MeasurementSample(sub, float(lens.sum()) / sub, tt))
    out = {"samples": [[s.batch, s.kv_load, s.latency] for s in samples]}
    try:
        fit = hb.calibrate(samples)
        out["reference_calibrate"] = "accepted"
    except hb.CalibrationError as exc:
        out["reference_calibrate"] = f"rejected: {exc}"
        out["why"] = ("K4 is a launch floor (~3 us for a few hundred KB, ~7 us for a few MB) and then "
                      "bandwidth-bound with ~zero per-request cost: max(floor, a + b*B*C), not the reference's "
                      "c0 + c1 B + c2 C + c3 B C with every c >= 0 -- its OLS over these samples (and over every "
                      "bandwidth-regime subset tried) puts c1 slightly below zero, which calibrate() rejects")
        return out
    m = fit.model
    out.update(residual_rms_s=fit.residual_rms, model={"c0": m.c0, "c1": m.c1, "c2": m.c2, "c3": m.c3})
    prof = budgets_profile(budgets, int(budgets.mean()))
    rp = hb.ModelProfile(prof.model_name, prof.kv_budget, prof.num_layers, prof.heads_per_layer, prof.weights)
    pred = {}
    for tp in (2, 4, 8):
        ch = 8 if tp == 8 else args.ch
        c = hb.compare(rp, tp, hb.EnumerationConfig(ch, 2, True, tp), m,
                       hb.SimulationConfig(batch=budgets.shape[1], decode_steps=1, tp=tp), workers=8)
        pred[f"tp{tp}"] = {r.name: r.throughput_gain for r in c.results}
    out["predicted_gain_vs_sha"] = pred
    out["note"] = "reference latency.calibrate + simulate.compare (baseline/_ref), DP at TP8 = equal split CH=8"
    return out


def budget_sweep(args, dev):
    """cfg3 of BASELINE.json: AHA placements vs uniform TP at budgets 128-1024."""
    import copy
    import torch
    rows = {}
    for B in (128, 256, 512):
        a = copy.copy(args)
        a.budget = B
        budgets = workload_budgets(a)
        base, q = _alloc_base(budgets, dev)
        res = emulate_tp(a, budgets, dev, base, q)
        rows[f"B{B}"] = {tp: {m: {"tokens_per_s": round(v["tokens_per_s"], 1),
                                  "gain_vs_sha": round(v.get("gain_vs_sha", 1.0), 4),
                                  "kv_max_over_mean": round(v["kv_max_over_mean"], 4)}
                              for m, v in r.items() if m != "best_aha"} | {"best_aha": r["best_aha"]}
                         for tp, r in res.items() if tp.startswith("tp")}
        del base, q
        torch.cuda.empty_cache()
    return rows


def cfg4_batch_sweep(args, dev):
    """BASELINE configs[3]: 70B shape, AHA-DP copy heads CH=4 (free split; the
    equal split needs CH=8 at TP=8, reported too), batch sweep 1-64 at 8 GPUs."""
    import torch
    rows = {}
    budgets = workload_budgets(args)
    for bt in (1, 4, 16, 64):
        b = budgets[:, :bt].copy()
        base, q = _alloc_base(b, dev)
        res = emulate_tp(args, b, dev, base, q, tps=(8,))["tp8"]
        rows[f"batch{bt}"] = {m: {"tokens_per_s": round(v["tokens_per_s"], 1),
                                  "gain_vs_sha": round(v.get("gain_vs_sha", 1.0), 4),
                                  "kv_max_over_mean": round(v["kv_max_over_mean"], 4)}
                              for m, v in res.items() if m != "best_aha"} | {"best_aha": res["best_aha"]}
        del base, q
        torch.cuda.empty_cache()
    return rows


def cfg5_skew(args, dev):
    """BASELINE configs[4]: budget 1024 (128k context), strongly skewed
    per-head budgets (dirichlet alpha=1, zipf s=1.2 -- the reference's
    acceptance profile shape), AHA vs uniform TP at 8 GPUs (emulated)."""
    import torch
    from paper_2502_15804_b200.sharding import synthetic_budgets
    rows = {}
    for dist_, param in (("dirichlet", 1.0), ("zipf", 1.2)):
        bud = synthetic_budgets(args.layers, args.batch, HKV, 1024, window=WINDOW, alpha=ALPHA,
                                distribution=dist_, param=param, seed=7, context=131072)
        base, q = _alloc_base(bud, dev)
        res = emulate_tp(args, bud, dev, base, q, tps=(8,))["tp8"]
        rows[f"{dist_}{param:g}"] = {m: {"tokens_per_s": round(v["tokens_per_s"], 1),
                                        "gain_vs_sha": round(v.get("gain_vs_sha", 1.0), 4),
                                        "kv_max_over_mean": round(v["kv_max_over_mean"], 4),
                                        "busy_rate": round(v["busy_rate"], 4)}
                                    for m, v in res.items() if m != "best_aha"} | {"best_aha": res["best_aha"]}
        del base, q
        torch.cuda.empty_cache()
    return rows


def cfg2_sweep(args, dev, peak):
    """BASELINE configs[1]: Llama-3.1-8B shape (32 layers, 32Q/8KV heads, G=4),
    Ada budget 256 (w=32, alpha=0.2, dirichlet skew), decode on one GPU,
    batch sweep 1-256: tokens/s and K4 GB/s vs HBM peak."""
    import numpy as np
    import torch
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache
    from paper_2502_15804_b200.sharding import synthetic_budgets
    L, hq, hkv, G, B = 32, 32, 8, 4, 256
    rows = {}
    for bt in (1, 16, 64, 256):
        budgets = synthetic_budgets(L, bt, hkv, B, window=WINDOW, alpha=ALPHA, seed=args.seed, context=16384)
        qrow = np.array([b * hq + h * G for b in range(bt) for h in range(hkv)])
        gen = torch.Generator(device=dev).manual_seed(11)
        caches = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, G, dev, fill="random", generator=gen)
                  for l in range(L)]
        q = torch.randn((L, bt, hq, HEAD_DIM), device=dev).to(torch.bfloat16)
        o = torch.empty_like(q)
        wss = [ops.DecodeWorkspace(c) for c in caches]

        def step():
            for l in range(L):
                ops.decode_into(q[l], caches[l], wss[l], out_bf16=o[l])
        g = capture(step)
        for _ in range(3):
            g.replay()
        t = timed(g.replay, 10) / 10
        kv = sum(c.kv_bytes() for c in caches)
        rows[f"batch{bt}"] = {"tokens_per_s": bt / t, "ms_per_step": t * 1e3,
                              "kv_GBs": kv / t / 1e9, "hbm_frac": kv / t / 1e9 / peak,
                              "kv_MB_per_step": kv / 1e6,
                              "schedule": {0: "coop", 1: "solo", 2: "wide"}[caches[0].flags]}
        del g, caches, wss
        torch.cuda.empty_cache()
    return rows


def full_layer(args, budgets, dev):
    """the decode layer with its weight GEMMs -- per layer and
    rank: QKV projection x[Bt, 8192] @ W_qkv (the rank's q heads + K/V heads,
    replicated rows for AHA-DP copies; cuBLAS bf16), K4 over the rank's shard,
    o_proj o[Bt, 8192] @ W_o[:, rank's 1/tp of the columns] (column-parallel
    after the all-gather).  Random-init weights; each rank's layers timed as
    in emulate_tp (event-bracketed minus the back-to-back correction), span =
    sum over layers of the max over ranks.  Shows how much of AHA's attention
    gain survives once the weights (302 MB per layer at TP=1) are streamed too."""
    import numpy as np
    import torch
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.decoder import rank_caches
    from paper_2502_15804_b200.sharding import plan_layouts
    L, bt = budgets.shape[0], budgets.shape[1]
    hidden = HQ * HEAD_DIM
    base, _ = _alloc_base(budgets, dev, seed=17)
    gen = torch.Generator(device=dev).manual_seed(17)
    w_qkv = [torch.randn((hidden, (HQ + 2 * HKV) * HEAD_DIM), device=dev, generator=gen).to(torch.bfloat16)
             for _ in range(L)]
    w_o = [torch.randn((hidden, hidden), device=dev, generator=gen).to(torch.bfloat16) for _ in range(L)]
    x = torch.randn((bt, hidden), device=dev, generator=gen).to(torch.bfloat16)
    q = torch.randn((L, bt, HQ, HEAD_DIM), device=dev, generator=gen).to(torch.bfloat16)
    o_full = torch.randn((bt, hidden), device=dev, generator=gen).to(torch.bfloat16)
    qkv_out = torch.empty((bt, (HQ + 2 * HKV) * HEAD_DIM), device=dev, dtype=torch.bfloat16)
    y = torch.empty((bt, hidden), device=dev, dtype=torch.bfloat16)
    results = {}
    for tp, modes in ((1, ["sha"]), (2, ["sha", "nodp"]), (4, ["sha", "nodp", "dp"]), (8, ["sha", "dp"])):
        row = {}
        for mode in modes:
            plan, _ = make_plan(budgets, tp, mode, args.ch)
            shards, _ = plan_layouts(plan, budgets, GROUP)
            t = np.zeros((L, tp))
            attn = np.zeros((L, tp))
            for g in range(tp):
                caches = rank_caches([s[g] for s in shards], bt, HQ, GROUP, tp, dev, base=base)
                sends = [ops.xrec_empty(max(c.n_segments, 1), GROUP, dev)[0] for c in caches]
                wss = [ops.DecodeWorkspace(c) for c in caches]
                cols = [len(plan.layers[l].groups[g]) * (GROUP + 2) * HEAD_DIM for l in range(L)]
                ocols = hidden // tp
                evs = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)] for _ in range(L)]

                def layer(l, ev=None):
                    if ev:
                        ev[0].record()
                    torch.mm(x, w_qkv[l][:, :cols[l]], out=qkv_out[:, :cols[l]])
                    if ev:
                        ev[1].record()
                    ops.decode_into(q[l], caches[l], wss[l], out_rec=sends[l])
                    if ev:
                        ev[2].record()
                    torch.mm(o_full, w_o[l][:, :ocols], out=y[:, :ocols])
                    if ev:
                        ev[3].record()

                gb = capture(lambda: [layer(l, evs[l]) for l in range(L)])
                gs = capture(lambda: [layer(l) for l in range(L)])
                gb.replay()
                gs.replay()
                torch.cuda.synchronize()
                tot = timed(gs.replay, 3) / 3
                gb.replay()
                torch.cuda.synchronize()
                tb = np.array([evs[l][0].elapsed_time(evs[l][3]) for l in range(L)]) * 1e-3
                ta = np.array([evs[l][1].elapsed_time(evs[l][2]) for l in range(L)]) * 1e-3
                c_g = max(0.0, (tb.sum() - tot) / L)
                t[:, g] = np.maximum(tb - c_g, 0.0)
                attn[:, g] = ta
                del gb, gs, caches, sends, wss
            step = t.max(axis=1).sum()
            row[mode] = {"tokens_per_s": bt / step, "ms_per_step": step * 1e3,
                         "attention_share_bracketed": float(attn.sum() / t.sum()) if t.sum() else None}
        for mode in modes[1:]:
            row[mode]["gain_vs_sha"] = row[mode]["tokens_per_s"] / row["sha"]["tokens_per_s"]
        results[f"tp{tp}"] = row
    results["note"] = ("per layer: QKV GEMM + K4 + o_proj GEMM (cuBLAS bf16 for the GEMMs, random-init "
                       "weights, 302 MB per layer at TP=1), all-gather excluded; "
                       "attention_share_bracketed = K4 time (event-bracketed, uncorrected) / corrected "
                       "layer time -- an upper bound")
    del base, w_qkv, w_o
    torch.cuda.empty_cache()
    return results


def append_cost(args, budgets, dev):
    """Decode-time append (ops.append: the step's new K/V row into every
    segment's headroom, work table grown on the device) on one 70B layer of
    the workload: microseconds per layer-step, next to the layer's K4."""
    import numpy as np
    import torch
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache
    bt = budgets.shape[1]
    qrow = np.array([b * HQ + h * GROUP for b in range(bt) for h in range(HKV)])
    c = LayerCache.allocate(budgets[0].reshape(-1), qrow, qrow, GROUP, dev, fill="random", reserve=64)
    kn = torch.randn((bt, HKV, HEAD_DIM), device=dev).to(torch.bfloat16)
    vn = torch.randn_like(kn)
    ops.append(c, kn, vn)
    g = capture(lambda: [ops.append(c, kn, vn) for _ in range(20)])  # device time, not launch cost
    g.replay()
    t = timed(g.replay, 1) / 20
    return {"us_per_layer_step": t * 1e6, "segments": c.n_segments,
            "note": "one launch per layer and step (20 back to back in a CUDA graph); 64-row headroom "
                    "per segment; the 20 appends overflow nothing (headroom 64)"}


def prefill_compress(peaks):
    """Per-layer prefill compression on the GPU (K1 score -> A18+K2 -> K3),
    cfg2 (Llama-3.1-8B shape, 16k context, budget 256) and the 70B shape at
    32k / 128k, timed with CUDA events around back-to-back API calls (host
    launch cost included) and, under "graph_replay", the same calls replayed
    from a CUDA graph (device time); K1 against the MUFU (ex2) bound."""
    import torch
    from paper_2502_15804_b200 import ops
    dev = torch.device("cuda")
    rows = {}
    mufu_path = ROOT / "profiles" / "mufu_peak.json"
    mufu_rate = json.loads(mufu_path.read_text())["ex2_per_s"] if mufu_path.exists() else 4.62e12
    for name, (bt, hq, hkv, T, B) in {"llama-3.1-8b_T16k_B256": (1, 32, 8, 16384, 256),
                                     "llama-3.1-8b_T16k_B256_batch4": (4, 32, 8, 16384, 256),
                                     "llama-3.1-8b_T16k_B256_batch32": (32, 32, 8, 16384, 256),
                                     "llama-3.3-70b_T32k_B1024": (1, 64, 8, 32768, 1024),
                                     "llama-3.3-70b_T128k_B1024": (1, 64, 8, 131072, 1024)}.items():
        w = WINDOW
        g = torch.Generator(device=dev).manual_seed(5)
        q = torch.randn((bt, hq, w, HEAD_DIM), generator=g, device=dev).to(torch.bfloat16)
        k = torch.randn((bt, hkv, T, HEAD_DIM), generator=g, device=dev).to(torch.bfloat16)
        v = torch.randn((bt, hkv, T, HEAD_DIM), generator=g, device=dev).to(torch.bfloat16)
        ws = torch.empty(int(ops._lib.fkv_score_workspace_bytes(bt, hkv, T, w, hq // hkv)),
                         dtype=torch.uint8, device=dev)
        sc = ops.score(q, k, workspace=ws)
        wsel = torch.empty(int(ops._lib.fkv_ada_select_workspace_bytes(bt, hkv, T - w)), dtype=torch.uint8,
                           device=dev)
        hb, off, idx = ops.ada_select(sc, B, w, workspace=wsel)
        for _ in range(3):  # warm: first launches set attributes / encode tensor maps
            ops.score(q, k, workspace=ws)
            ops.ada_select(sc, B, w, workspace=wsel)
            ops.score_select(q, k, B, w, workspace=ws)
        t_score = timed(lambda: ops.score(q, k, workspace=ws), 10) / 10
        t_sel = timed(lambda: ops.ada_select(sc, B, w, workspace=wsel), 10) / 10
        t_fused = timed(lambda: ops.score_select(q, k, B, w, workspace=ws), 10) / 10
        cache, _, _ = ops.compress_layer(q, k, v, B, w)
        sbh, slo, shi = cache.host["compact_args"]
        mx = int(hb.max().item())
        ops.compact_into(cache, k, v, off, idx, sbh, slo, shi, mx)  # warm (first-launch setup)
        t_cmp = timed(lambda: ops.compact_into(cache, k, v, off, idx, sbh, slo, shi, mx), 5) / 5

        def graph_us(fn, n=10):  # the same calls replayed from a CUDA graph: device time only
            g = capture(lambda: [fn() for _ in range(n)])
            g.replay()
            t = timed(g.replay, 1) / n
            del g
            return t * 1e6
        dev_us = {"score_us": graph_us(lambda: ops.score(q, k, workspace=ws)),
                  "ada_select_us": graph_us(lambda: ops.ada_select(sc, B, w, workspace=wsel)),
                  "score_select_us": graph_us(lambda: ops.score_select(q, k, B, w, workspace=ws)),
                  "compact_us": graph_us(lambda: ops.compact_into(cache, k, v, off, idx, sbh, slo, shi, mx))}
        # a whole layer stack's compression (8 layers, host-visible wall time):
        # per layer compress_layer (the host waits for each layer's budgets
        # before its compaction) vs compress_stack (all fused launches queued,
        # each layer laid out as its budgets land in pinned host memory, one
        # table copy, then every compaction); stack8_gpu_us_per_layer = the
        # same layers' fused launches + compactions alone
        Ls = 8

        def per_layer():
            for _ in range(Ls):
                ops.compress_layer(q, k, v, B, w)
            torch.cuda.synchronize()

        def stacked():
            ops.compress_stack([q] * Ls, [k] * Ls, [v] * Ls, B, w)
            torch.cuda.synchronize()
        per_layer()
        stacked()
        t_pl = min(timed(per_layer, 1) for _ in range(3)) / Ls
        t_st = min(timed(stacked, 1) for _ in range(3)) / Ls
        hbm_bps = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
        flops = 2 * 2.0 * bt * hq * w * T * HEAD_DIM  # two passes of Q_win.K^T
        exps = 2.0 * bt * hq * w * T  # one ex2 per score per pass (MUFU)
        kbytes = bt * hkv * T * HEAD_DIM * 2
        tf_peak = float(peaks.get("bf16_tflops", 1590.0))
        rows[name] = {
            "score_us": t_score * 1e6, "ada_select_us": t_sel * 1e6, "compact_us": t_cmp * 1e6,
            "score_select_fused_us": t_fused * 1e6,
            "score_select_path": ("one persistent cooperative launch (per-chunk select)"
                                  if bt * hkv <= 148 else
                                  "one persistent cooperative launch (items dealt round robin, grid-wide select)"),
            "score_tflops": flops / t_score / 1e12, "score_tflops_frac": flops / t_score / 1e12 / tf_peak,
            "score_K_read_GBs_per_pass": kbytes / (t_score / 2) / 1e9,
            "roofline_us": max(flops / (tf_peak * 1e12), 2 * kbytes / (float(peaks.get("hbm_gbs", 6650.0)) * 1e9)) * 1e6,
            "graph_replay": dev_us,
            "stack8_compress_layer_us_per_layer": t_pl * 1e6,
            "stack8_compress_stack_us_per_layer": t_st * 1e6,
            "stack8_gpu_us_per_layer": dev_us["score_select_us"] + dev_us["compact_us"],
            # K1 is bound by the special-function unit, not the tensor cores:
            # two exponentials per (query row, key), at the measured ex2 rate
            "mufu_bound_us": exps / mufu_rate * 1e6,
            "score_mufu_frac": exps / mufu_rate / (dev_us["score_us"] * 1e-6),
            # the two passes in sequence (pass 2 needs every chunk's pass-1
            # statistics): pass 1 streams K from HBM and exponentiates, pass 2
            # exponentiates again over K re-read from L2 when it fits (the one-
            # item-per-CTA schedule keeps it there), else from HBM
            "two_pass_bound_us": (max(kbytes / hbm_bps, exps / 2 / mufu_rate)
                                  + max(kbytes / hbm_bps if kbytes > 96e6 else 0.0, exps / 2 / mufu_rate)) * 1e6,
        }
        rows[name]["score_two_pass_frac"] = rows[name]["two_pass_bound_us"] / dev_us["score_us"]
    return rows


def planner_compare(budgets):
    """AHA placement of this workload's profile: the native C++ planner vs the
    reference's own optimize_plan (baseline/_ref, compiled Cython equal-split
    kernel; its free split is pure Python), same workers, identical plans."""
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200.sharding import budgets_profile
    prof = budgets_profile(budgets, int(budgets.mean()))
    ref = ref_headbalance()
    workers = os.cpu_count() or 1
    rows = {}
    for tp, ch, eq in ((4, 4, True), (8, 8, True), (8, 4, False)):
        t0 = time.perf_counter()
        mine = fk.optimize_plan(prof, tp, fk.EnumerationConfig(ch, 2, True, tp), equal_split=eq,
                                workers=workers)
        t_native = time.perf_counter() - t0
        row = {"native_s": t_native}
        if ref is not None:
            rp = ref.ModelProfile(prof.model_name, prof.kv_budget, prof.num_layers,
                                  prof.heads_per_layer, prof.weights)
            t0 = time.perf_counter()
            theirs = ref.optimize_plan(rp, tp, ref.EnumerationConfig(ch, 2, True, tp), equal_split=eq,
                                       workers=workers)
            row["reference_s"] = time.perf_counter() - t0
            row["identical"] = all(
                [[(c.head_id, c.replica_count) for c in g] for g in a.groups] ==
                [[(c.head_id, c.replica_count) for c in g] for g in b.groups] and a.delta == b.delta
                for a, b in zip(mine.layers, theirs.layers))
            row["speedup"] = row["reference_s"] / t_native
        rows[f"tp{tp}_ch{ch}_{'equal' if eq else 'free'}"] = row
    return {"workers": workers, "layers": prof.num_layers, "heads": prof.heads_per_layer,
            "kind": "reference" if ref is not None else "unavailable", "results": rows}


# ------------------------------------------------------ reference arm -----
def run_reference(args):
    """The reference CPU path on the same workload, rank 0 only: budgets from
    the reference's own generate_profile (oracle/workload.py), then K timed
    steps of the float64 decode of every layer on all host threads (the
    reference has no decode; the oracle port restates it).  Never imports
    this package."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    hb = ref_headbalance()
    if hb is None:
        print(json.dumps({"impl": "reference", "unavailable": "reference package not installed in baseline/_ref"}))
        return
    from oracle.workload import CpuDecodeStack, synthetic_budgets
    budgets = synthetic_budgets(hb, args.layers, args.batch, HKV, args.budget, window=WINDOW, alpha=ALPHA,
                                seed=args.seed)
    st = CpuDecodeStack(budgets, HQ)
    for _ in range(args.warmup):
        st.step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        st.step()
        times.append(time.perf_counter() - t0)
    st.close()
    step_s = sum(times) / len(times)
    value = args.batch / step_s
    sample = (f"every step: all {args.layers} layers x batch {args.batch} x {HKV} KV heads ({HQ} query heads) "
              f"decoded in float64 (oracle/workload.py; the reference has no decode, SPEC.md:8), budgets from "
              f"the reference's generate_profile ({hb.__file__})")
    out = {
        "impl": "reference",
        "metric": METRIC,
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (N(0,1) float64 K/V/q; Ada-shaped per-head budgets)",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": st.threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_fairkv(a)
