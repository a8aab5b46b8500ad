"""The fused NVLink all-gather across real processes: two OS processes (one
rank each, torch.distributed over gloo for the plumbing) share the single
GPU of this environment, map each other's receive areas with CUDA IPC
(exchange.P2PGroup.connect) and run StackDecoder with the P2P exchange.
Every rank's o must equal the single-GPU decode of the same layers.  This is
the multi-process path bench.py takes at N > 1 (IPC handles, cross-process
epoch-tagged XLL records polled across processes), minus NVLink itself."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, tp: int, port: int, mode: str, out_dir: str):
    import torch.distributed as dist
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache
    from paper_2502_15804_b200.decoder import StackDecoder, rank_caches
    from paper_2502_15804_b200.exchange import P2PGroup
    from paper_2502_15804_b200.sharding import budgets_profile, plan_layouts, synthetic_budgets

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=tp)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    L, bt, hkv, G, B = 3, 4, 8, 8, 256
    hq = hkv * G
    budgets = synthetic_budgets(L, bt, hkv, B, seed=11)
    prof = budgets_profile(budgets, B)
    plan = fk.sha_plan(prof, tp) if mode == "sha" else \
        fk.optimize_plan(prof, tp, fk.EnumerationConfig(4, 2, True, tp))
    shards, finals = plan_layouts(plan, budgets, G)
    qrow = np.array([b * hq + h * G for b in range(bt) for h in range(hkv)])
    gen = torch.Generator(device=dev).manual_seed(5)  # identical base cache in every process
    base = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, G, dev, fill="random", generator=gen)
            for l in range(L)]
    caches = rank_caches([s[rank] for s in shards], bt, hq, G, tp, dev, base=base)
    grp = P2PGroup.connect(rank, tp, finals[0].slots, G)
    dec = StackDecoder(caches, finals, tp=tp, bt=bt, hq=hq, group=G, exchange="p2p",
                       endpoint=grp.endpoints[0])
    gq = torch.Generator(device=dev).manual_seed(9)
    q = torch.randn((L, bt, hq, 128), generator=gq, device=dev).to(torch.bfloat16)
    o = torch.zeros_like(q)
    ref = torch.stack([ops.decode(q[l], base[l])[0] for l in range(L)])
    ok, err = True, 0.0
    # several steps of an odd layer count, checked after every step: the last
    # layer of step s and layer 0 of step s+1 must not share a receive area
    # (exchange_buffer), or a fast peer overwrites records being merged
    for s in range(4):
        o.zero_()
        q_s = q * (1 + s)  # a different q per step: a stale record cannot pass
        dec.step(q_s, o)
        torch.cuda.synchronize()
        ref_s = torch.stack([ops.decode(q_s[l], base[l])[0] for l in range(L)])
        err = max(err, float((o.float() - ref_s.float()).abs().max()))
        ok = ok and bool(torch.allclose(o.float(), ref_s.float(), rtol=2e-2, atol=4e-3))
    del ref
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
        f.write(f"{int(ok)} {err}\n")
    dist.barrier()
    grp.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("tp,mode", [(2, "sha"), (2, "dp")])
def test_two_process_p2p_exchange(cuda_device, tmp_path, tp, mode):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, tp, port, mode, str(tmp_path))) for r in range(tp)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
            pytest.fail("multi-process exchange timed out")
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    for r in range(tp):
        ok, err = (tmp_path / f"rank{r}.txt").read_text().split()
        assert ok == "1", f"rank {r}: max |o - ref| = {err}"


def test_bench_two_ranks_shared_device(cuda_device):
    """bench.py's N > 1 path end to end (torchrun, P2P exchange through CUDA
    IPC, graph capture, max-over-ranks timing) with both ranks on the one GPU
    (FKV_SHARED_DEVICE=1: gloo plumbing; timings meaningless)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, FKV_SHARED_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--layers", "3", "--batch", "4", "--steps", "2", "--warmup", "3", "--no-emulate", "--no-cpu"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert "exchange p2p" in line["placement"]
    # every placement was checked against a local decode before timing
    assert set(line["check"]) == set(line["modes"]) == {"sha", "nodp", "dp", "dp-free"}
    assert all(c["ok"] for c in line["check"].values())
