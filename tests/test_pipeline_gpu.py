"""End-to-end parity of the north-star pipeline on the GPU against the CPU
oracle chain.

* Selection on *separated* inputs: Q/K are redrawn until every
  selection boundary of the float64 oracle's scores is wider than the score
  tolerance (oracle/gaps.py), then the GPU's budgets and selected indices,
  computed from its own fp32 scores, must equal the oracle's exactly.
* cfg1 (BASELINE configs[0]): one 32Q/8KV layer, 4k context, Ada budget 128,
  AHA placement for TP=2 -- GPU prefill (K1+A18+K2) -> budgets ->
  ModelProfile -> optimize_plan (identical to the reference planner) ->
  per-rank compaction of the owned copies (K3, DP copies split along tokens)
  -> sharded decode with the fused exchange (loopback: both ranks on this
  GPU) -> LSE merge, against oracle scores -> oracle budgets -> oracle
  selection -> float64 attention over whole heads.
* The bench's exact headline configuration (Llama-3.3-70B, batch 64, Ada
  budget 1024, dirichlet head skew, its schedule) decoded inside a CUDA graph
  of back-to-back programmatic-dependent launches, every layer checked.
"""

import numpy as np
import pytest
import torch

from oracle import gaps
from oracle import kv as okv

pytestmark = pytest.mark.gpu

S_RTOL, S_ATOL_ROW = 1e-4, 1e-6
O_TOL = dict(rtol=2e-2, atol=4e-3)  # bf16; atol: half a bf16 ulp at the unit scale of V
LSE_TOL = dict(rtol=1e-4, atol=1e-5)


def _draw(bt, hq, hkv, T, seed, temp=2.0):
    g = torch.Generator().manual_seed(seed)
    q = (torch.randn(bt, hq, 32, 128, generator=g) * temp).to(torch.bfloat16)
    k = torch.randn(bt, hkv, T, 128, generator=g).to(torch.bfloat16)
    v = torch.randn(bt, hkv, T, 128, generator=g).to(torch.bfloat16)
    return q, k, v


def separated_inputs(bt, hq, hkv, T, budget, seed0=0, tries=40):
    """First draw whose oracle scores have every selection boundary
    separated by more than the score tolerance; -> (q, k, v, s_ref, draws)."""
    for i in range(tries):
        q, k, v = _draw(bt, hq, hkv, T, seed0 + i)
        s = okv.snapkv_scores(q.double().numpy(), k.double().numpy())
        if gaps.separated(s, budget, 32, S_RTOL, S_ATOL_ROW):
            return q, k, v, s, i + 1
    pytest.fail(f"no separated draw in {tries} tries")


@pytest.mark.parametrize("bt,hq,T,budget", [(1, 32, 4096, 128), (3, 32, 4096, 256), (2, 64, 6000, 512),
                                            (1, 64, 2100, 1024)])
def test_selection_exact_on_separated_inputs(cuda_device, bt, hq, T, budget):
    from paper_2502_15804_b200 import ops
    q, k, v, s_ref, draws = separated_inputs(bt, hq, 8, T, budget, seed0=bt * 100 + T)
    ref_b = okv.ada_budgets(s_ref, budget, 32, 0.2)
    ref_off, ref_idx = okv.topk_select(s_ref, ref_b, 32)
    qd, kd = q.to(cuda_device), k.to(cuda_device)
    # the fused launch and the two-launch path (score, then grid-wide select)
    sc, hb, off, idx = ops.score_select(qd, kd, budget, 32)
    hb2, off2, idx2 = ops.ada_select(ops.score(qd, kd), budget, 32)
    torch.cuda.synchronize()
    for b_, o_, i_ in ((hb, off, idx), (hb2, off2, idx2)):
        np.testing.assert_array_equal(b_.cpu().numpy(), ref_b)
        np.testing.assert_array_equal(o_.cpu().numpy(), ref_off)
        np.testing.assert_array_equal(i_.cpu().numpy(), ref_idx)
    print(f"separated after {draws} draw(s): budgets and {len(ref_idx)} indices identical")


def test_cfg1_end_to_end_tp2(cuda_device):
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.exchange import P2PGroup
    from paper_2502_15804_b200.sharding import plan_layouts
    from oracle import planner as oplan
    from conftest import reference_headbalance

    bt, hq, hkv, T, w, B, tp = 1, 32, 8, 4096, 32, 128, 2
    G = hq // hkv
    cfg = fk.EnumerationConfig(4, 2, True, tp)
    # a draw whose selection boundaries are separated *and* whose AHA-DP plan
    # replicates a head (so the token-split copies and their merge run)
    for seed0 in range(0, 400, 40):
        q, k, v, s_ref, _ = separated_inputs(bt, hq, hkv, T, B, seed0=seed0)
        b0 = okv.ada_budgets(s_ref, B, w, 0.2)
        p0 = fk.optimize_plan(fk.profile_from_budgets(b0[None], B), tp, cfg)
        if any(c.replica_count > 1 for g in p0.layers[0].groups for c in g):
            break
    dev = cuda_device
    kd, vd = k.to(dev), v.to(dev)

    # ---- GPU prefill: scores, Ada budgets, per-head selection (one launch)
    sc, hb, off, idx = ops.score_select(q.to(dev), kd, B, w)
    torch.cuda.synchronize()
    ref_b = okv.ada_budgets(s_ref, B, w, 0.2)
    ref_off, ref_idx = okv.topk_select(s_ref, ref_b, w)
    budgets = hb.cpu().numpy()
    np.testing.assert_array_equal(budgets, ref_b)
    np.testing.assert_array_equal(idx.cpu().numpy(), ref_idx)

    # ---- placement: profile -> AHA plan, identical to the reference's
    prof = fk.profile_from_budgets(budgets[None], B)
    plan = fk.optimize_plan(prof, tp, cfg)
    la = plan.layers[0]
    ref = reference_headbalance()
    if ref is not None:
        rp = ref.optimize_plan(ref.ModelProfile(prof.model_name, prof.kv_budget, 1, hkv, prof.weights), tp,
                               ref.EnumerationConfig(4, 2, True, tp))
        want = [[(c.head_id, c.replica_count) for c in g] for g in rp.layers[0].groups]
        assert want == [[(c.head_id, c.replica_count) for c in g] for g in la.groups]
        assert rp.layers[0].delta == la.delta
    else:
        delta, reps, hc, rgs = oplan.select_best(list(prof.weights[0]), tp, 4, 2, True)
        assert delta == la.delta
        want = oplan.groups_of(reps, hc, rgs, tp)
        assert want == [tuple((c.head_id, c.replica_count) for c in g) for g in la.groups]
    assert any(c.replica_count > 1 for g in la.groups for c in g), "cfg1 plan should copy a head"

    # ---- per-rank compaction of the owned copies, sharded decode, exchange
    shards, finals = plan_layouts(plan, budgets[None], G)
    caches = []
    for r in range(tp):
        sh = shards[0][r]
        bh = sh.seg_b * hkv + sh.seg_h
        qrow = sh.seg_b * hq + sh.seg_h * G
        caches.append(ops.compact(kd, vd, off, idx, bh, sh.seg_lo, sh.seg_hi, qrow,
                                  np.arange(sh.n_segments) * G, G))
    grp = P2PGroup.loopback(tp, finals[0].slots, G)
    tabs = tuple(torch.as_tensor(x, device=dev) for x in (finals[0].grp_ptr, finals[0].src_idx,
                                                          finals[0].out_row))
    qdec = torch.randn(bt, hq, 128, generator=torch.Generator().manual_seed(99)).to(torch.bfloat16)
    outs = torch.zeros(tp, bt, hq, 128, dtype=torch.bfloat16, device=dev)
    lses = torch.zeros(tp, bt, hq, device=dev)
    for step in range(3):  # buffers rotate: steps 2 and 3 reuse the receive areas
        outs.zero_()
        for r in range(tp):
            ops.decode_exchange(qdec.to(dev), caches[r], grp.endpoints[r], step % 2)
        for r in range(tp):
            ops.merge_wait(grp.endpoints[r], step % 2, *tabs, G, out_bf16=outs[r], out_lse=lses[r])
        torch.cuda.synchronize()
        # ---- oracle: float64 attention of each whole head over its oracle-selected rows
        kn, vn = k.double().numpy(), v.double().numpy()
        ks = [kn[b, h, ref_idx[ref_off[b * hkv + h]:ref_off[b * hkv + h + 1]]] for b in range(bt) for h in range(hkv)]
        vs = [vn[b, h, ref_idx[ref_off[b * hkv + h]:ref_off[b * hkv + h + 1]]] for b in range(bt) for h in range(hkv)]
        o_ref, lse_ref = okv.decode_heads(qdec.double().numpy(), ks, vs, G)
        for r in range(tp):
            torch.testing.assert_close(outs[r].float().cpu().double(), torch.from_numpy(o_ref), **O_TOL)
            torch.testing.assert_close(lses[r].cpu().double(), torch.from_numpy(lse_ref), **LSE_TOL)
    grp.close()


def _host_rows(cache, s):
    """Logical (unswizzled) K and V rows of segment s, float64."""
    r0, n = int(cache.host["seg_row0"][s]), int(cache.host["seg_len"][s])
    kk = okv.unswizzle_rows(cache.k[r0:r0 + n].cpu().view(torch.int16).numpy(), r0)
    vv = okv.unswizzle_rows(cache.v[r0:r0 + n].cpu().view(torch.int16).numpy(), r0)
    f = lambda a: torch.from_numpy(a).view(torch.bfloat16).double().numpy()  # noqa: E731
    return f(kk), f(vv)


def test_bench_config_layers_in_graph(cuda_device):
    """The headline bench configuration (bench.py defaults: 70B shape, batch
    64, budget 1024, dirichlet a=8 skew, TP=1 schedule) -- four layers
    captured back to back in one CUDA graph with programmatic dependent
    launch, replayed twice; every layer's o and lse against the oracle."""
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache
    from paper_2502_15804_b200.sharding import synthetic_budgets
    L, bt, hq, hkv, G, B = 4, 64, 64, 8, 8, 1024
    budgets = synthetic_budgets(80, bt, hkv, B, seed=0, context=32768)[[0, 27, 53, 79]]
    qrow = np.array([b * hq + h * G for b in range(bt) for h in range(hkv)])
    gen = torch.Generator(device=cuda_device).manual_seed(3)
    caches = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, G, cuda_device, fill="random",
                                  generator=gen) for l in range(L)]
    assert caches[0].flags == 0  # the cooperative schedule, as in the bench
    q = torch.randn((L, bt, hq, 128), generator=gen, device=cuda_device).to(torch.bfloat16)
    o = torch.zeros_like(q)
    lse = torch.zeros((L, bt, hq), device=cuda_device)
    wss = [ops.DecodeWorkspace(c) for c in caches]

    def step():
        for l in range(L):
            ops.decode_into(q[l], caches[l], wss[l], out_bf16=o[l], out_lse=lse[l])
    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        step()
    o.zero_()
    lse.zero_()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    qn = q.double().cpu().numpy()
    for l in range(L):
        segs = [_host_rows(caches[l], i) for i in range(bt * hkv)]
        o_ref, lse_ref = okv.decode_heads(qn[l], [x[0] for x in segs], [x[1] for x in segs], G)
        torch.testing.assert_close(o[l].float().cpu().double(), torch.from_numpy(o_ref), **O_TOL)
        torch.testing.assert_close(lse[l].cpu().double(), torch.from_numpy(lse_ref), **LSE_TOL)
