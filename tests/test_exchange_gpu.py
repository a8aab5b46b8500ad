"""Fused NVLink all-gather protocol (fkv_decode_exchange + fkv_merge_wait),
exercised with tp virtual ranks on one GPU ("loopback": every peer pointer
is local memory, same kernels, same epoch/buffer-rotation protocol).  Every rank's
o must equal the single-GPU (TP=1) decode, layer after layer, including DP
copies split along the token axis and a CUDA-graph replay."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(tp, mode, dev, L=3, bt=4, B=256, G=8):
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200.cache import LayerCache
    from paper_2502_15804_b200.decoder import rank_caches
    from paper_2502_15804_b200.sharding import budgets_profile, plan_layouts, synthetic_budgets
    hkv = 8
    hq = G * hkv
    budgets = synthetic_budgets(L, bt, hkv, B, seed=tp)
    prof = budgets_profile(budgets, B)
    if mode == "sha":
        plan = fk.sha_plan(prof, tp)
    else:
        plan = fk.optimize_plan(prof, tp, fk.EnumerationConfig(4, 2, True, tp), equal_split=(mode == "dp"))
    shards, finals = plan_layouts(plan, budgets, G)
    qrow = np.array([b * hq + h * G for b in range(bt) for h in range(hkv)])
    gen = torch.Generator(device=dev).manual_seed(1)
    base = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, G, dev, fill="random", generator=gen)
            for l in range(L)]
    per_rank = [rank_caches([s[r] for s in shards], bt, hq, G, tp, dev, base=base) for r in range(tp)]
    return base, per_rank, finals, bt, hq, G


@pytest.mark.parametrize("tp,mode,G", [(2, "sha", 8), (2, "dp", 8), (4, "dp", 8), (8, "free", 8), (4, "dp", 4),
                                        (8, "sha", 4)])
def test_loopback_exchange_matches_single_gpu(cuda_device, tp, mode, G):
    """G = 8: Llama-3.3-70B heads; G = 4: Llama-3.1-8B heads."""
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.exchange import P2PGroup, exchange_buffer
    base, per_rank, finals, bt, hq, G = _setup(tp, mode, cuda_device, G=G)
    L = len(base)
    slots = max(f.slots for f in finals)
    grp = P2PGroup.loopback(tp, slots, G)
    q = torch.randn(L, bt, hq, 128, device=cuda_device).to(torch.bfloat16)
    tabs = [tuple(torch.as_tensor(x, device=cuda_device) for x in (f.grp_ptr, f.src_idx, f.out_row))
            for f in finals]
    outs = torch.zeros(tp, L, bt, hq, 128, dtype=torch.bfloat16, device=cuda_device)

    def step():
        for l in range(L):
            for r in range(tp):
                ops.decode_exchange(q[l], per_rank[r][l], grp.endpoints[r], exchange_buffer(l, L))
            for r in range(tp):
                ptr, src, row = tabs[l]
                ops.merge_wait(grp.endpoints[r], exchange_buffer(l, L), ptr, src, row, G, out_bf16=outs[r, l])

    step()
    torch.cuda.synchronize()
    ref = torch.stack([ops.decode(q[l], base[l])[0] for l in range(L)])
    for r in range(tp):
        torch.testing.assert_close(outs[r].float(), ref.float(), rtol=2e-2, atol=4e-3)
    # graph replay: epochs are monotonic, arrival counters self-resetting
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        step()
    outs.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for r in range(tp):
        torch.testing.assert_close(outs[r].float(), ref.float(), rtol=2e-2, atol=4e-3)
    grp.close()


@pytest.mark.parametrize("tp,mode", [(2, "dp"), (4, "dp")])
def test_sharded_append_then_exchange(cuda_device, tp, mode):
    """Decode steps append one token per (request, head): on a sharded cache
    only the copy that owns the end of the head's token axis grows (views
    over the base storage: the same rows the TP=1 cache appends into), and the
    fused exchange + LSE merge still equals the single-GPU decode."""
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache
    from paper_2502_15804_b200.decoder import rank_caches
    from paper_2502_15804_b200.exchange import P2PGroup, exchange_buffer
    from paper_2502_15804_b200.sharding import budgets_profile, plan_layouts, synthetic_budgets
    G, hkv, L, bt, B = 8, 8, 2, 4, 256
    hq = G * hkv
    budgets = synthetic_budgets(L, bt, hkv, B, seed=3)
    plan = fk.optimize_plan(budgets_profile(budgets, B), tp, fk.EnumerationConfig(4, 2, True, tp))
    shards, finals = plan_layouts(plan, budgets, G)
    qrow = np.array([b * hq + h * G for b in range(bt) for h in range(hkv)])
    gen = torch.Generator(device=cuda_device).manual_seed(2)
    base = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, G, cuda_device, fill="random",
                                generator=gen, reserve=8) for l in range(L)]
    per_rank = [rank_caches([s[r] for s in shards], bt, hq, G, tp, cuda_device, base=base) for r in range(tp)]
    slots = max(f.slots for f in finals)
    grp = P2PGroup.loopback(tp, slots, G)
    tabs = [tuple(torch.as_tensor(x, device=cuda_device) for x in (f.grp_ptr, f.src_idx, f.out_row))
            for f in finals]
    q = torch.randn(L, bt, hq, 128, device=cuda_device).to(torch.bfloat16)
    out = torch.zeros(tp, L, bt, hq, 128, dtype=torch.bfloat16, device=cuda_device)
    for step in range(3):
        for l in range(L):
            kn = torch.randn(bt, hkv, 128, device=cuda_device).to(torch.bfloat16)
            vn = torch.randn(bt, hkv, 128, device=cuda_device).to(torch.bfloat16)
            for r in range(tp):
                ops.append(per_rank[r][l], kn, vn)  # owning copies only
            ops.append(base[l], kn, vn)  # writes the same rows again; grows the TP=1 view
            for r in range(tp):
                ops.decode_exchange(q[l], per_rank[r][l], grp.endpoints[r], exchange_buffer(l, L))
            for r in range(tp):
                ptr, src, row = tabs[l]
                ops.merge_wait(grp.endpoints[r], exchange_buffer(l, L), ptr, src, row, G, out_bf16=out[r, l])
        torch.cuda.synchronize()
        ref = torch.stack([ops.decode(q[l], base[l])[0] for l in range(L)])
        for r in range(tp):
            torch.testing.assert_close(out[r].float(), ref.float(), rtol=2e-2, atol=4e-3)
    grown = sum(int(c.sync_lengths().sum()) for pr in per_rank for c in pr)
    assert grown == sum(int(c.sync_lengths().sum()) for c in base)
    grp.close()


@pytest.mark.parametrize("tp,mode", [(2, "dp"), (4, "dp"), (8, "free")])
def test_nccl_path_loopback_allgather(cuda_device, tp, mode):
    """The NCCL fallback of StackDecoder (K4 -> exchange-record send block ->
    all_gather_into_tensor -> K5) with tp virtual ranks on this GPU: each
    layer every rank produces, a loopback all-gather stacks the send blocks
    into every rank's receive area exactly as NCCL's all_gather_into_tensor
    lays them out (rank r's block at r * block), every rank consumes.  Each
    rank's o equals the single-GPU decode; a CUDA graph replays it."""
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.decoder import StackDecoder
    base, per_rank, finals, bt, hq, G = _setup(tp, mode, cuda_device, L=4)
    L = len(base)
    decs = [StackDecoder(per_rank[r], finals, tp=tp, bt=bt, hq=hq, group=G, exchange="nccl")
            for r in range(tp)]
    q = torch.randn(L, bt, hq, 128, device=cuda_device).to(torch.bfloat16)
    outs = torch.zeros(tp, L, bt, hq, 128, dtype=torch.bfloat16, device=cuda_device)

    def step():
        for l in range(L):
            for r in range(tp):
                decs[r].produce(l, q[l])
            gathered = torch.stack([decs[r].send[l] for r in range(tp)])
            for r in range(tp):
                decs[r].recv[l].copy_(gathered)
            for r in range(tp):
                decs[r].consume(l, outs[r, l])

    step()
    torch.cuda.synchronize()
    ref = torch.stack([ops.decode(q[l], base[l])[0] for l in range(L)])
    for r in range(tp):
        torch.testing.assert_close(outs[r].float(), ref.float(), rtol=2e-2, atol=4e-3)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        step()
    outs.zero_()
    g.replay()
    torch.cuda.synchronize()
    for r in range(tp):
        torch.testing.assert_close(outs[r].float(), ref.float(), rtol=2e-2, atol=4e-3)


def test_nccl_allgather_of_exchange_blocks(cuda_device, tmp_path):
    """The real NCCL call on the exchange-record blocks (world size 1 in a
    subprocess: one GPU here): all_gather_into_tensor of a uint8 send block
    into the [tp, block] receive area the K5 merge reads."""
    import subprocess
    import sys
    from pathlib import Path
    code = r'''
import os, torch, torch.distributed as dist
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=os.environ["PORT"])
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
from paper_2502_15804_b200 import ops
send = ops.xrec_empty(3, 8, "cuda")[0].random_(0, 255)
recv = ops.xrec_empty(3, 8, "cuda", ranks=1)
dist.all_gather_into_tensor(recv.view(-1), send)
torch.cuda.synchronize()
assert torch.equal(recv[0], send)
dist.destroy_process_group()
print("ok")
'''
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    import os
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, PORT=str(port), PYTHONPATH=str(root))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
