"""Compression path parity on the GPU (K1 score, A18 budgets, K2 select, K3
compact) against the float64 oracle (oracle/kv.py).

Tolerances: scores are fp32 (bf16 operands, tcgen05 fp32 accumulation,
ex2.approx): elementwise |s - ref| <= 1e-4 |ref| + 1e-6 max_t |ref| (north_star
fp32 rtol 1e-4; the atol floor is for scores many orders below their row's
peak, where the flush-to-zero exponential underflows).  Long contexts (32k,
128k) are checked on sampled heads against the float64 oracle.
Budgets, offsets, selected indices and compacted rows are BIT-EXACT functions
of the score tensor: the oracle is fed the GPU's own fp32 scores (exact in
float64), so any mismatch is a selection/tie-rule bug, not rounding; and
end to end (GPU scores vs oracle scores) on inputs whose every selection
boundary is separated by more than the score tolerance.
"""

import numpy as np
import pytest
import torch

from oracle import kv as okv

pytestmark = pytest.mark.gpu

S_RTOL, S_ATOL_ROW = 1e-4, 1e-6


def check_scores(s, ref):
    """Elementwise score tolerance; returns the worst |err| / allowed."""
    s, ref = np.asarray(s, np.float64), np.asarray(ref, np.float64)
    assert s.shape == ref.shape
    allowed = S_RTOL * np.abs(ref) + S_ATOL_ROW * np.abs(ref).max(axis=-1, keepdims=True)
    worst = float((np.abs(s - ref) / allowed).max())
    assert worst <= 1.0, f"score error {worst:.3g} x the tolerance"
    return worst


def sampled_head_scores(qn, kn, heads):
    """float64 oracle scores of the listed (b, h) only: [len(heads), T-w]."""
    hq, hkv = qn.shape[1], kn.shape[1]
    G = hq // hkv
    return np.stack([okv.snapkv_scores(qn[b:b + 1, h * G:(h + 1) * G], kn[b:b + 1, h:h + 1])[0, 0]
                     for b, h in heads])


def _inputs(bt, hq, hkv, T, w, seed, dev, temp=1.0):
    g = torch.Generator().manual_seed(seed)
    q = (torch.randn(bt, hq, w, 128, generator=g) * temp).to(torch.bfloat16)
    k = torch.randn(bt, hkv, T, 128, generator=g).to(torch.bfloat16)
    v = torch.randn(bt, hkv, T, 128, generator=g).to(torch.bfloat16)
    return q.to(dev), k.to(dev), v.to(dev), q.double().numpy(), k.double().numpy(), v.double().numpy()


@pytest.mark.parametrize("bt,hq,hkv,T", [(1, 32, 8, 4096), (2, 32, 8, 1000), (1, 64, 8, 2100), (2, 16, 4, 333),
                                         (20, 32, 8, 300), (3, 64, 8, 20000)])
def test_score_matches_oracle(cuda_device, bt, hq, hkv, T):
    """Covers the fused cooperative launch (Bt*Hkv*chunks <= #SMs) and the
    three-launch path (20 x 8 = 160 heads > 148 SMs)."""
    from paper_2502_15804_b200 import ops
    q, k, _, qn, kn, _ = _inputs(bt, hq, hkv, T, 32, 1, cuda_device, temp=2.0)
    s = ops.score(q, k).cpu().double().numpy()
    print(f"score error {check_scores(s, okv.snapkv_scores(qn, kn)):.3g} x tolerance")


@pytest.mark.parametrize("bt,hq,T,fused", [(1, 64, 32768, True), (1, 64, 131072, True), (2, 64, 32768, False),
                                           (1, 32, 131072, False)])
def test_score_long_context_sampled(cuda_device, bt, hq, T, fused):
    """cfg4 (32k) and cfg5 (128k): many key chunks per head and the
    multi-chunk softmax-statistics combine, checked elementwise on sampled
    heads against the float64 oracle (both the score-only and the fused
    score+select launch)."""
    from paper_2502_15804_b200 import ops
    q, k, _, qn, kn, _ = _inputs(bt, hq, 8, T, 32, 17, cuda_device, temp=2.0)
    if fused:
        s = ops.score_select(q, k, 1024, 32)[0]
    else:
        s = ops.score(q, k)
    s = s.cpu().double().numpy()
    heads = [(0, 0), (bt - 1, 5)]
    ref = sampled_head_scores(qn, kn, heads)
    got = np.stack([s[b, h] for b, h in heads])
    print(f"T={T}: score error {check_scores(got, ref):.3g} x tolerance")


def _gpu_select(sc, budget, w, alpha=0.2):
    from paper_2502_15804_b200 import ops
    hb = ops.budgets(sc, budget, w, alpha)
    off, idx = ops.select(sc, hb, w, total=sc.shape[0] * sc.shape[1] * budget)
    torch.cuda.synchronize()
    return hb.cpu().numpy(), off.cpu().numpy(), idx.cpu().numpy()


@pytest.mark.parametrize("budget", [64, 128, 1024])
def test_budgets_and_select_bit_exact(cuda_device, budget):
    from paper_2502_15804_b200 import ops
    q, k, _, _, _, _ = _inputs(3, 32, 8, 4096, 32, 2, cuda_device, temp=3.0)
    sc = ops.score(q, k)
    hb, off, idx = _gpu_select(sc, budget, 32)
    s64 = sc.cpu().double().numpy()
    ref_b = okv.ada_budgets(s64, budget, 32, 0.2)
    np.testing.assert_array_equal(hb, ref_b)
    assert (hb.sum(axis=1) == 8 * budget).all()
    ref_off, ref_idx = okv.topk_select(s64, ref_b, 32)
    np.testing.assert_array_equal(off, ref_off)
    np.testing.assert_array_equal(idx, ref_idx)


@pytest.mark.parametrize("bt,hkv,n,ties", [(3, 8, 5000, False), (2, 16, 3000, True), (600, 8, 168, False),
                                           (1, 8, 70000, True), (4, 4, 0, False), (50, 8, 3, True)])
def test_topk_select_any_budgets(cuda_device, bt, hkv, n, ties):
    """K2 with budgets that are not an Ada split (window-only heads, whole-head
    heads, random sizes): per-head top-k == the oracle's."""
    from paper_2502_15804_b200 import ops
    g = torch.Generator().manual_seed(bt + hkv + n)
    sc = torch.randint(0, 6, (bt, hkv, n), generator=g).float() if ties else torch.rand(bt, hkv, n, generator=g)
    hb = torch.randint(32, 32 + n + 1, (bt, hkv), generator=g, dtype=torch.int32)
    hb[0, 0] = 32           # window only
    hb[-1, -1] = 32 + n     # every token
    off, idx = ops.select(sc.to(cuda_device), hb.to(cuda_device), 32)
    torch.cuda.synchronize()
    ref_off, ref_idx = okv.topk_select(sc.double().numpy(), hb.numpy(), 32)
    np.testing.assert_array_equal(off.cpu().numpy(), ref_off)
    np.testing.assert_array_equal(idx.cpu().numpy(), ref_idx)
    if n:
        rb = okv.ada_budgets(sc.double().numpy(), 32 + n // 2, 32, 0.2)
        np.testing.assert_array_equal(ops.budgets(sc.to(cuda_device), 32 + n // 2, 32).cpu().numpy(), rb)


def test_select_with_exact_ties(cuda_device):
    """Integer-valued scores: massive exact ties exercise both tie rules."""
    from paper_2502_15804_b200 import ops
    g = torch.Generator().manual_seed(3)
    sc = torch.randint(0, 4, (2, 8, 3000), generator=g).float()
    sc[1, 3] = 0.0  # a whole head of zeros
    hb, off, idx = _gpu_select(sc.to(cuda_device), 256, 32)
    s64 = sc.double().numpy()
    ref_b = okv.ada_budgets(s64, 256, 32, 0.2)
    np.testing.assert_array_equal(hb, ref_b)
    ref_off, ref_idx = okv.topk_select(s64, ref_b, 32)
    np.testing.assert_array_equal(off, ref_off)
    np.testing.assert_array_equal(idx, ref_idx)


def test_compact_rows_exact(cuda_device):
    from paper_2502_15804_b200 import ops
    bt, hq, hkv, T, w, B = 2, 32, 8, 2048, 32, 200
    q, k, v, _, kn, vn = _inputs(bt, hq, hkv, T, w, 4, cuda_device)
    cache, hb, sc = ops.compress_layer(q, k, v, B, w)
    torch.cuda.synchronize()
    hb = hb.cpu().numpy().reshape(-1)
    off, idx = okv.topk_select(sc.cpu().double().numpy(), hb.reshape(bt, hkv), w)
    kc = cache.k.cpu().view(torch.int16).numpy()
    vc = cache.v.cpu().view(torch.int16).numpy()
    k16 = k.cpu().view(torch.int16).numpy()
    v16 = v.cpu().view(torch.int16).numpy()
    row0 = cache.host["seg_row0"]
    for s in range(bt * hkv):
        b, h = divmod(s, hkv)
        sel = idx[off[s]:off[s + 1]]
        n = len(sel)
        np.testing.assert_array_equal(okv.unswizzle_rows(kc[row0[s]:row0[s] + n], row0[s]), k16[b, h, sel])
        np.testing.assert_array_equal(okv.unswizzle_rows(vc[row0[s]:row0[s] + n], row0[s]), v16[b, h, sel])
        pad = okv.page_rows(n)
        assert (kc[row0[s] + n:row0[s] + pad] == 0).all()


def test_compress_then_decode_end_to_end(cuda_device):
    """Prefill (score -> budgets -> select -> compact) then decode, against
    the oracle decoding the oracle-gathered rows."""
    from paper_2502_15804_b200 import ops
    bt, hq, hkv, T, w, B = 2, 64, 8, 3000, 32, 256
    G = hq // hkv
    q, k, v, _, kn, vn = _inputs(bt, hq, hkv, T, w, 5, cuda_device, temp=2.0)
    cache, hb, sc = ops.compress_layer(q, k, v, B, w)
    qd = torch.randn(bt, hq, 128, generator=torch.Generator().manual_seed(6)).to(torch.bfloat16)
    o, lse = ops.decode(qd.to(cuda_device), cache)
    torch.cuda.synchronize()
    off, idx = okv.topk_select(sc.cpu().double().numpy(), hb.cpu().numpy(), w)
    ks = [kn[b, h, idx[off[b * hkv + h]:off[b * hkv + h + 1]]] for b in range(bt) for h in range(hkv)]
    vs = [vn[b, h, idx[off[b * hkv + h]:off[b * hkv + h + 1]]] for b in range(bt) for h in range(hkv)]
    o_ref, lse_ref = okv.decode_heads(qd.double().numpy(), ks, vs, G)
    torch.testing.assert_close(o.float().cpu().double(), torch.from_numpy(o_ref), rtol=2e-2, atol=4e-3)
    torch.testing.assert_close(lse.cpu().double(), torch.from_numpy(lse_ref), rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("seed", range(8))
def test_score_select_random_shapes(cuda_device, seed):
    """Random shapes through the persistent fused launch (one item per CTA or
    several, G*w 128 / 256, T not a multiple of the tile, budgets near the
    floor and near T): budgets and indices bit-exact against the oracle fed
    the kernel's own scores, scores within tolerance on a sampled head."""
    from paper_2502_15804_b200 import ops
    rng = np.random.default_rng(1000 + seed)
    hq = int(rng.choice([32, 64]))
    bt = int(rng.choice([1, 2, 5, 19, 23]))
    T = int(rng.integers(200, 3000))
    budget = int(rng.integers(33, min(T - 32, 1024) + 1))
    q, k, _, qn, kn, _ = _inputs(bt, hq, 8, T, 32, 70 + seed, cuda_device, temp=float(rng.uniform(0.5, 3)))
    sc, hb, off, idx = ops.score_select(q, k, budget, 32)
    torch.cuda.synchronize()
    s64 = sc.cpu().double().numpy()
    heads = [(bt - 1, int(rng.integers(8)))]
    check_scores(np.stack([s64[b, h] for b, h in heads]), sampled_head_scores(qn, kn, heads))
    ref_b = okv.ada_budgets(s64, budget, 32, 0.2)
    np.testing.assert_array_equal(hb.cpu().numpy(), ref_b)
    ref_off, ref_idx = okv.topk_select(s64, ref_b, 32)
    np.testing.assert_array_equal(off.cpu().numpy(), ref_off)
    np.testing.assert_array_equal(idx.cpu().numpy(), ref_idx)


@pytest.mark.parametrize("bt,T", [(2, 2500), (20, 900)])  # per-chunk select; grid-wide select (> 148 heads)
def test_compress_stack_matches_per_layer(cuda_device, bt, T):
    """compress_stack (all layers' fused launches queued, budgets written to
    pinned host memory by the kernels, each layer laid out as they arrive,
    one table copy, then every compaction) builds the same caches as
    compress_layer per layer: budgets, scores, tables and the compacted K/V
    bytes bit for bit, and the caches decode identically."""
    from paper_2502_15804_b200 import ops
    L, hq, hkv, B = 3, 32, 8, 256
    layers = [_inputs(bt, hq, hkv, T, 32, 40 + l, cuda_device, temp=2.0)[:3] for l in range(L)]
    caches, hbs, scs = ops.compress_stack([x[0] for x in layers], [x[1] for x in layers],
                                          [x[2] for x in layers], B)
    torch.cuda.synchronize()
    for l, (q, k, v) in enumerate(layers):
        # the composition of the public stages, one host round trip
        sc, hb, offsets, idx = ops.score_select(q, k, B)
        hb_host = hb.cpu().numpy().reshape(-1)
        bh = np.arange(bt * hkv)
        qrow = (bh // hkv) * hq + (bh % hkv) * (hq // hkv)
        cache = ops.compact(k, v, offsets, idx, bh, np.zeros_like(bh), hb_host, qrow, qrow, hq // hkv)
        torch.cuda.synchronize()
        one, hb1, sc1 = ops.compress_layer(q, k, v, B)
        assert torch.equal(hb1, hb) and torch.equal(sc1, sc) and torch.equal(one.k, cache.k)
        assert torch.equal(hbs[l], hb) and torch.equal(scs[l], sc)
        assert torch.equal(caches[l].k, cache.k) and torch.equal(caches[l].v, cache.v)
        assert torch.equal(caches[l].work, cache.work)
        for name in ("seg_row0", "seg_len", "seg_qrow", "warp_ptr", "work_list", "grp_ptr", "src_idx"):
            assert torch.equal(getattr(caches[l], name), getattr(cache, name)), name
        # the stacked caches (views of one K/V allocation) decode identically
        qd = torch.randn((bt, hq, 128), device=cuda_device).to(torch.bfloat16)
        (o1, l1), (o2, l2) = ops.decode(qd, caches[l]), ops.decode(qd, cache)
        assert torch.equal(o1, o2) and torch.equal(l1, l2)


def test_selection_agreement_with_oracle_scores(cuda_device):
    """Unconstrained inputs: index sets chosen from GPU scores vs from the
    float64 oracle scores agree except at near-ties (reported, >= 98%)."""
    from paper_2502_15804_b200 import ops
    q, k, _, qn, kn, _ = _inputs(1, 32, 8, 4096, 32, 7, cuda_device, temp=3.0)
    sc = ops.score(q, k)
    hb, off, idx = _gpu_select(sc, 256, 32)
    ref_s = okv.snapkv_scores(qn, kn)
    rb = okv.ada_budgets(ref_s, 256, 32, 0.2)
    roff, ridx = okv.topk_select(ref_s, rb, 32)
    a = {(h, int(t)) for h in range(8) for t in idx[off[h]:off[h + 1]]}
    r = {(h, int(t)) for h in range(8) for t in ridx[roff[h]:roff[h + 1]]}
    agree = len(a & r) / len(r)
    print(f"selection agreement GPU-scores vs oracle-scores: {agree:.4f}")
    assert agree >= 0.98


@pytest.mark.parametrize("bt,T,budget,ties,hkv,alpha", [
    (3, 4096, 256, False, 8, 0.2), (2, 2048, 64, True, 8, 0.2), (1, 65600, 1024, False, 8, 0.2),
    (2, 40000, 512, True, 8, 0.2), (2, 3000, 256, "zero-head", 8, 0.2), (1, 1000, 32, False, 8, 0.2),
    (1, 131104, 1024, False, 8, 0.2),      # cfg5 length: many chunks per head
    (3, 5000, 300, "zero-head", 16, 0.2),  # 16 KV heads
    (5, 3000, 200, True, 1, 0.2),          # one KV head: the floor is the whole story
    (2, 3000, 256, True, 8, 1.0),          # floor = budget - window: no global picks
    (2, 3000, 256, "zero-head", 8, 0.0),   # no floor
    (600, 200, 64, False, 8, 0.2),         # 4800 heads: more than one launch
    (64, 16384, 256, False, 8, 0.2),       # batch 64 at 16k: pieces across heads
    (3, 32, 32, False, 8, 0.2),            # n = 0: the window only
    (7, 300, 100, "zero-head", 8, 0.2),    # heads shorter than a CTA's key range
    (40, 40, 36, True, 8, 0.2),            # 8 keys per head: many heads per CTA range
])
def test_fused_ada_select_bit_exact(cuda_device, bt, T, budget, ties, hkv, alpha):
    """The one-launch grid-wide split + select == oracle budgets + selection."""
    from paper_2502_15804_b200 import ops
    g = torch.Generator().manual_seed(bt * 7 + T)
    n = T - 32
    sc = torch.randint(0, 5, (bt, hkv, n), generator=g).float() if ties is True \
        else torch.rand(bt, hkv, n, generator=g)
    if ties == "zero-head":  # a head that can only keep its floor
        sc[:, 2] = 0.0
        sc[:, 5] *= 1e-3
    hb, off, idx = ops.ada_select(sc.to(cuda_device), budget, 32, alpha)
    torch.cuda.synchronize()
    s64 = sc.double().numpy()
    ref_b = okv.ada_budgets(s64, budget, 32, alpha)
    np.testing.assert_array_equal(hb.cpu().numpy(), ref_b)
    ref_off, ref_idx = okv.topk_select(s64, ref_b, 32)
    np.testing.assert_array_equal(off.cpu().numpy(), ref_off)
    np.testing.assert_array_equal(idx.cpu().numpy(), ref_idx)
    # the same workspace again (reset inside the call)
    ws = torch.empty(int(ops._lib.fkv_ada_select_workspace_bytes(bt, hkv, n)), dtype=torch.uint8,
                     device=cuda_device).fill_(0xAB)
    for _ in range(2):
        hb2, off2, idx2 = ops.ada_select(sc.to(cuda_device), budget, 32, alpha, workspace=ws)
    assert torch.equal(hb2, hb) and torch.equal(off2, off) and torch.equal(idx2, idx)


@pytest.mark.parametrize("bt,hq,hkv,T,budget,temp,flat_head", [
    (1, 32, 8, 4096, 128, 3.0, False),    # 8B shape, fused grid
    (2, 64, 8, 6000, 256, 2.0, False),    # 70B shape (G*w = 256)
    (1, 32, 8, 20000, 1024, 3.0, False),  # long context, several chunks per head
    (2, 32, 8, 3000, 256, 2.0, True),     # a head whose window soaks up all attention: below its floor
    (1, 32, 8, 40000, 1024, 3.0, True),   # the same over many chunks per head (joint floor search)
    (20, 32, 8, 600, 64, 2.0, False),     # 160 heads > 148 SMs: two waves, grid-wide select in the launch
    (1, 64, 8, 131072, 1024, 2.0, False),  # cfg5: 128k context, B=1024, 70B shape (four L2 waves)
    (32, 32, 8, 16384, 256, 3.0, False),  # batch 32 at 16k: several items per CTA, one launch
    (20, 64, 8, 900, 128, 2.0, True),     # G*w = 256 with several items per CTA (Q_win reloads), a flat head
])
def test_fused_score_select_bit_exact(cuda_device, bt, hq, hkv, T, budget, temp, flat_head):
    """K1 + A18 + K2 in one persistent launch at any batch (one wave with the
    per-chunk selection, or several L2-sized waves with the grid-wide search):
    scores within tolerance of the oracle;
    budgets / offsets / indices bit-exact against the oracle fed the kernel's
    own pooled scores (max-pooling makes exact ties common)."""
    from paper_2502_15804_b200 import ops
    q, k, _, qn, kn, _ = _inputs(bt, hq, hkv, T, 32, 13, cuda_device, temp=temp)
    if flat_head:
        # KV head 3: constant queries u, zero keys outside the window and window
        # keys 20u -> the window takes all attention mass, every other score of
        # the head ties at ~e^-57: the head keeps exactly its floor (lowest tokens)
        G = hq // hkv
        u = torch.full((128,), 0.5, dtype=torch.bfloat16, device=cuda_device)
        q[:, 3 * G:4 * G] = u
        k[:, 3] = 0
        k[:, 3, T - 32:] = 20 * u
        qn, kn = q.cpu().double().numpy(), k.cpu().double().numpy()
    sc, hb, off, idx = ops.score_select(q, k, budget, 32)
    torch.cuda.synchronize()
    s64 = sc.cpu().double().numpy()
    if T <= 6000:
        check_scores(s64, okv.snapkv_scores(qn, kn))
    else:
        heads = [(0, 0), (bt - 1, 3 if flat_head else 6)]
        check_scores(np.stack([s64[b, h] for b, h in heads]), sampled_head_scores(qn, kn, heads))
    ref_b = okv.ada_budgets(s64, budget, 32, 0.2)
    np.testing.assert_array_equal(hb.cpu().numpy(), ref_b)
    if flat_head:
        assert (ref_b[:, 3] == 32 + int(0.2 * (budget - 32))).all()  # kept exactly its floor
    ref_off, ref_idx = okv.topk_select(s64, ref_b, 32)
    np.testing.assert_array_equal(off.cpu().numpy(), ref_off)
    np.testing.assert_array_equal(idx.cpu().numpy(), ref_idx)
    # repeated launches reuse the workspace (counters / histograms re-zeroed)
    sc2, hb2, off2, idx2 = ops.score_select(q, k, budget, 32)
    torch.cuda.synchronize()
    assert torch.equal(idx2, idx) and torch.equal(hb2, hb)


def test_compress_stack_rejects_bad_inputs(cuda_device):
    """compress_stack validates every layer before queueing anything: a
    missing tensor, a layer of another shape, a window that is not q_win's."""
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.errors import NativeError
    q, k, v = _inputs(1, 32, 8, 600, 32, 3, cuda_device)[:3]
    with pytest.raises(NativeError):
        ops.compress_stack([q], [k], [], 256)
    with pytest.raises(NativeError):
        ops.compress_stack([q, q], [k, k[:, :, :-16].contiguous()], [v, v[:, :, :-16].contiguous()], 256)
    with pytest.raises(NativeError):
        ops.compress_stack([q], [k], [v.float()], 256)
    with pytest.raises(NativeError):
        ops.compress_stack([q], [k], [v], 256, window=16)
