"""Fused NVLink all-gather protocol (fkv_decode_exchange + fkv_merge_wait),
exercised with tp virtual ranks on one GPU ("loopback": every peer pointer
is local memory, same kernels, same flags/parity protocol).  Every rank's
o must equal the single-GPU (TP=1) decode, layer after layer, including DP
copies split along the token axis and a CUDA-graph replay."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(tp, mode, dev, L=3, bt=4, B=256):
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200.cache import LayerCache
    from paper_2502_15804_b200.decoder import rank_caches
    from paper_2502_15804_b200.sharding import budgets_profile, plan_layouts, synthetic_budgets
    G, hkv = 8, 8
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


@pytest.mark.parametrize("tp,mode", [(2, "sha"), (2, "dp"), (4, "dp"), (8, "free")])
def test_loopback_exchange_matches_single_gpu(cuda_device, tp, mode):
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.exchange import P2PGroup, exchange_buffer
    base, per_rank, finals, bt, hq, G = _setup(tp, mode, cuda_device)
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
        torch.testing.assert_close(outs[r].float(), ref.float(), rtol=2e-2, atol=1e-2)
    # graph replay: flags and counters are monotonic / self-resetting
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
        torch.testing.assert_close(outs[r].float(), ref.float(), rtol=2e-2, atol=1e-2)
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
            torch.testing.assert_close(out[r].float(), ref.float(), rtol=2e-2, atol=1e-2)
    grown = sum(int(c.sync_lengths().sum()) for pr in per_rank for c in pr)
    assert grown == sum(int(c.sync_lengths().sum()) for c in base)
    grp.close()
