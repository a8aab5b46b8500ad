"""K4 + K5 parity: CUDA split-KV decode over the ragged swizzled cache vs the
float64 oracle (oracle/kv.py).  Tolerances (north_star): o is bf16 -> rtol
2e-2 (atol 4e-3, half a bf16 ulp at the unit scale of V, for entries that cancel to near zero); lse is fp32 -> rtol 1e-4 (atol 1e-5
for lse near zero)."""

import numpy as np
import pytest
import torch

from oracle import kv as okv

pytestmark = pytest.mark.gpu

O_TOL = dict(rtol=2e-2, atol=4e-3)    # bf16 output; atol = half a bf16 ulp at |V| ~ 1
LSE_TOL = dict(rtol=1e-4, atol=1e-5)  # fp32 log-sum-exp


def check_o_lse(o, lse, o_ref, lse_ref):
    torch.testing.assert_close(o.float().cpu().double(), torch.from_numpy(np.asarray(o_ref)), **O_TOL)
    lse_c = lse.cpu().double()
    ref = torch.from_numpy(np.asarray(lse_ref))
    empty = torch.isneginf(ref)
    assert torch.isneginf(lse_c[empty]).all()
    torch.testing.assert_close(lse_c[~empty], ref[~empty], **LSE_TOL)


def _bf16(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16)


def build_cache(seg_lens, group, hkv, bt, device, seed=0, chunk=None):
    from paper_2502_15804_b200.cache import LayerCache, segment_offsets
    g = torch.Generator().manual_seed(seed)
    hq = hkv * group
    seg_qrow = [b * hq + h * group for b in range(bt) for h in range(hkv)]
    cache = LayerCache.allocate(seg_lens, seg_qrow, seg_qrow, group, device, chunk=chunk)
    row0, _ = segment_offsets(seg_lens)
    ks, vs = [], []
    kh = torch.zeros(cache.k.shape, dtype=torch.bfloat16)
    vh = torch.zeros(cache.v.shape, dtype=torch.bfloat16)
    for r0, n in zip(row0, seg_lens):
        k = _bf16(torch.randn(n, 128, generator=g))
        v = _bf16(torch.randn(n, 128, generator=g))
        ks.append(k.float().numpy().astype(np.float64))
        vs.append(v.float().numpy().astype(np.float64))
        # store swizzled rows (pure permutation of 16-byte chunks)
        kh[r0:r0 + n] = torch.from_numpy(okv.swizzle_rows(k.view(torch.int16).numpy(), r0)).view(torch.bfloat16)
        vh[r0:r0 + n] = torch.from_numpy(okv.swizzle_rows(v.view(torch.int16).numpy(), r0)).view(torch.bfloat16)
    cache.k.copy_(kh)
    cache.v.copy_(vh)
    q = _bf16(torch.randn(bt, hq, 128, generator=g))
    return cache, q, ks, vs


@pytest.mark.parametrize("group", [8, 4])
@pytest.mark.parametrize("chunk", [None, 64, 128])
@pytest.mark.parametrize("schedule", ["auto", "coop", "wide", "solo"])
def test_decode_matches_oracle(cuda_device, group, chunk, schedule, monkeypatch):
    """Both K4 schedules (CTA-cooperative pieces / per-warp pieces) and the
    host's automatic choice."""
    from paper_2502_15804_b200 import ops
    monkeypatch.setenv("FKV_K4_SCHEDULE", schedule)
    rng = np.random.default_rng(group * 100 + (chunk or 0))
    hkv, bt = 8, 3
    seg_lens = rng.integers(1, 700, size=bt * hkv).tolist()
    seg_lens[0] = 1
    seg_lens[1] = 16
    seg_lens[2] = 17
    seg_lens[3] = 64
    seg_lens[4] = 65
    cache, q, ks, vs = build_cache(seg_lens, group, hkv, bt, cuda_device, chunk=chunk)
    if schedule != "auto" and chunk is None:
        assert cache.flags == {"coop": 0, "solo": 1, "wide": 2}[schedule]
    o, lse = ops.decode(q.to(cuda_device), cache)
    torch.cuda.synchronize()
    o_ref, lse_ref = okv.decode_heads(q.float().numpy().astype(np.float64), ks, vs, group)
    check_o_lse(o, lse, o_ref, lse_ref)


@pytest.mark.parametrize("schedule", ["coop", "wide", "solo"])
def test_decode_many_segments_split(cuda_device, schedule, monkeypatch):
    """Many long segments: pieces split across CTAs / warps, merged by the
    fused K5 (several pieces per segment, the last CTA's cooperative merge)."""
    from paper_2502_15804_b200 import ops
    monkeypatch.setenv("FKV_K4_SCHEDULE", schedule)
    rng = np.random.default_rng(11)
    hkv, bt, group = 8, 8, 8
    seg_lens = rng.integers(900, 2600, size=bt * hkv).tolist()
    cache, q, ks, vs = build_cache(seg_lens, group, hkv, bt, cuda_device, seed=5)
    assert int(np.diff(cache.grp_ptr.cpu().numpy()).max()) > 1  # some segments are split
    o, lse = ops.decode(q.to(cuda_device), cache)
    torch.cuda.synchronize()
    o_ref, lse_ref = okv.decode_heads(q.float().numpy().astype(np.float64), ks, vs, group)
    check_o_lse(o, lse, o_ref, lse_ref)


@pytest.mark.parametrize("schedule,bt", [("wide", 8), ("coop", 8), ("coop", 24)])
def test_decode_whole_segment_schedule(cuda_device, schedule, bt, monkeypatch):
    """Whole-segment schedule: up to one segment per SM, the longest cut into
    equal pieces (>= 32 tiles) so that every piece has an SM of its own
    (only those segments merge); bt=24 under coop puts 192 segments on 148
    SMs: no segment is split, the longest get an SM alone, the rest pair
    longest with shortest.  Every CTA's pieces are combined by all its warps."""
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import (HYBRID_MIN_SAVING_US, NUM_SMS, WHOLE_MODEL, _whole_owners,
                                             plan_work_hybrid)
    monkeypatch.setenv("FKV_K4_SCHEDULE", schedule)
    monkeypatch.setenv("FKV_K4_WHOLE", "1")
    rng = np.random.default_rng(bt)
    hkv, group = 8, 8
    seg_lens = rng.integers(0, 900, size=bt * hkv).tolist()
    seg_lens[:4] = [0, 1, 16, 17]
    cache, q, ks, vs = build_cache(seg_lens, group, hkv, bt, cuda_device, seed=bt)
    ptr = cache.grp_ptr.cpu().numpy()
    if len(seg_lens) <= NUM_SMS:  # one piece per CTA, the longest segments cut
        want = plan_work_hybrid(np.asarray(seg_lens), NUM_SMS, WHOLE_MODEL[schedule][2], HYBRID_MIN_SAVING_US)
        np.testing.assert_array_equal(ptr, want[3])
        np.testing.assert_array_equal(cache.item_t1.cpu().numpy(), want[2])
        assert int(np.diff(ptr).max()) > 1 and len(want[0]) <= NUM_SMS
        assert int(np.diff(cache.warp_ptr.cpu().numpy()).max()) == 1
    else:
        assert int(np.diff(ptr).max()) == 1  # no segment is split
    assert cache.flags == {"coop": 0, "wide": 2}[schedule]
    o, lse = ops.decode(q.to(cuda_device), cache)
    torch.cuda.synchronize()
    o_ref, lse_ref = okv.decode_heads(q.float().numpy().astype(np.float64), ks, vs, group)
    check_o_lse(o, lse, o_ref, lse_ref)
    if bt == 24:  # 192 segments on 148 SMs: one CTA each, heavy paired with light
        tiles = (np.asarray(seg_lens) + 15) // 16
        own = _whole_owners(tiles, 2 * NUM_SMS, NUM_SMS)
        assert sorted(own.tolist()) == list(range(len(seg_lens)))


def test_decode_large_scores_stable(cuda_device):
    """Large-magnitude logits must not overflow the online softmax."""
    from paper_2502_15804_b200 import ops
    hkv, bt, group = 8, 1, 8
    seg_lens = [300] * hkv
    cache, q, ks, vs = build_cache(seg_lens, group, hkv, bt, cuda_device, seed=3)
    q = (q.float() * 30).to(torch.bfloat16)
    o, lse = ops.decode(q.to(cuda_device), cache)
    o_ref, lse_ref = okv.decode_heads(q.float().numpy().astype(np.float64), ks, vs, group)
    assert torch.isfinite(o).all()
    check_o_lse(o, lse, o_ref, lse_ref)


def test_lse_merge_of_token_split_equals_whole(cuda_device):
    """AHA-DP: a head split along tokens into r copies, merged by LSE, equals
    attention over the whole head (the identity the sharded decode relies on)."""
    from paper_2502_15804_b200 import ops
    group, hkv = 8, 1
    n = 1000
    cuts = [0, 333, 334, 1000]  # includes an empty copy
    lens = [cuts[i + 1] - cuts[i] for i in range(3)]
    g = torch.Generator().manual_seed(7)
    k = _bf16(torch.randn(n, 128, generator=g))
    v = _bf16(torch.randn(n, 128, generator=g))
    q = _bf16(torch.randn(1, group, 128, generator=g)).to(cuda_device)
    from paper_2502_15804_b200.cache import LayerCache, segment_offsets
    cache = LayerCache.allocate(lens, [0, 0, 0], [0, group, 2 * group], group, cuda_device)
    row0, _ = segment_offsets(lens)
    kh = torch.zeros(cache.k.shape, dtype=torch.bfloat16)
    vh = torch.zeros(cache.v.shape, dtype=torch.bfloat16)
    for i, r0 in enumerate(row0):
        a, b = cuts[i], cuts[i + 1]
        kh[r0:r0 + b - a] = torch.from_numpy(okv.swizzle_rows(k[a:b].view(torch.int16).numpy(), r0)).view(torch.bfloat16)
        vh[r0:r0 + b - a] = torch.from_numpy(okv.swizzle_rows(v[a:b].view(torch.int16).numpy(), r0)).view(torch.bfloat16)
    cache.k.copy_(kh)
    cache.v.copy_(vh)
    # per-copy (bf16 o, f32 lse) exchange records into 3 slots, then merge them
    dev = cuda_device
    slots = ops.xrec_empty(3, group, dev)
    ops.decode_into(q, cache, out_rec=slots[0])
    ro, rl = ops.xrec_view(slots, group)
    for i in range(3):  # each copy's record is its own attention (bf16 o, fp32 lse)
        oi, li = okv.attend(q[0].float().cpu().numpy(), k[cuts[i]:cuts[i + 1]].float().numpy(),
                            v[cuts[i]:cuts[i + 1]].float().numpy())
        check_o_lse(ro[0, i * group:(i + 1) * group], rl[0, i * group:(i + 1) * group], oi, li)
    o = torch.empty(1, group, 128, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(1, group, device=dev)
    ops.merge_lse(slots,
                  torch.tensor([0, 3], dtype=torch.int32, device=dev),
                  torch.arange(3, dtype=torch.int32, device=dev),
                  torch.zeros(1, dtype=torch.int32, device=dev), group, out_bf16=o, out_lse=lse)
    o_ref, lse_ref = okv.attend(q[0].float().cpu().numpy(), k.float().numpy(), v.float().numpy())
    check_o_lse(o[0], lse[0], o_ref, lse_ref)


@pytest.mark.parametrize("schedule", ["coop", "wide", "solo"])
def test_decode_empty_and_tiny_segments(cuda_device, schedule, monkeypatch):
    """Zero-token segments (an AHA-DP copy can own no tokens) give o = 0 and
    lse = -inf; 1..17-token segments exercise the masked tails."""
    from paper_2502_15804_b200 import ops
    monkeypatch.setenv("FKV_K4_SCHEDULE", schedule)
    group, hkv, bt = 8, 8, 2
    seg_lens = [0, 1, 2, 15, 16, 17, 0, 31, 33, 0, 5, 64, 65, 0, 7, 128]
    cache, q, ks, vs = build_cache(seg_lens, group, hkv, bt, cuda_device, seed=9)
    o, lse = ops.decode(q.to(cuda_device), cache)
    torch.cuda.synchronize()
    o_ref, lse_ref = okv.decode_heads(q.float().numpy().astype(np.float64), ks, vs, group)
    check_o_lse(o, lse, o_ref, lse_ref)


@pytest.mark.parametrize("schedule", ["coop", "wide", "solo"])
def test_append_then_decode(cuda_device, schedule, monkeypatch):
    """Decode-time appends: each step writes the new token's K/V into every
    segment's headroom (device-side length + work-table update); decode after
    every step equals the oracle over the grown rows; capacity overflow is
    counted, not written."""
    from paper_2502_15804_b200 import ops
    monkeypatch.setenv("FKV_K4_SCHEDULE", schedule)
    from paper_2502_15804_b200.cache import LayerCache, segment_offsets
    group, hkv, bt = 8, 8, 2
    rng = np.random.default_rng(21)
    seg_lens = rng.integers(1, 900, size=bt * hkv)
    seg_lens[3] = 63  # one row short of a page: overflows after one append with reserve 0...
    hq = hkv * group
    qrow = [b * hq + h * group for b in range(bt) for h in range(hkv)]
    reserve = 3
    cache = LayerCache.allocate(seg_lens, qrow, qrow, group, cuda_device, reserve=reserve)
    row0 = cache.host["seg_row0"]
    g = torch.Generator().manual_seed(22)
    ks = [torch.randn(int(n), 128, generator=g).to(torch.bfloat16) for n in seg_lens]
    vs = [torch.randn(int(n), 128, generator=g).to(torch.bfloat16) for n in seg_lens]
    kh = torch.zeros(cache.k.shape, dtype=torch.bfloat16)
    vh = torch.zeros(cache.v.shape, dtype=torch.bfloat16)
    for r0, k, v in zip(row0, ks, vs):
        kh[r0:r0 + len(k)] = torch.from_numpy(okv.swizzle_rows(k.view(torch.int16).numpy(), r0)).view(torch.bfloat16)
        vh[r0:r0 + len(v)] = torch.from_numpy(okv.swizzle_rows(v.view(torch.int16).numpy(), r0)).view(torch.bfloat16)
    cache.k.copy_(kh)
    cache.v.copy_(vh)
    cap = cache.host["seg_cap"]
    q = torch.randn(bt, hq, 128, generator=g).to(torch.bfloat16)
    steps = int((cap - seg_lens).min()) + 2  # the tightest segment overflows twice
    for step in range(steps):
        kn = torch.randn(bt, hkv, 128, generator=g).to(torch.bfloat16)
        vn = torch.randn(bt, hkv, 128, generator=g).to(torch.bfloat16)
        ops.append(cache, kn.to(cuda_device), vn.to(cuda_device))
        for s in range(bt * hkv):
            if len(ks[s]) < cap[s]:
                b, h = divmod(s, hkv)
                ks[s] = torch.cat([ks[s], kn[b, h][None]])
                vs[s] = torch.cat([vs[s], vn[b, h][None]])
        o, lse = ops.decode(q.to(cuda_device), cache)
        torch.cuda.synchronize()
        kk = [x.float().numpy().astype(np.float64) for x in ks]
        vv = [x.float().numpy().astype(np.float64) for x in vs]
        o_ref, lse_ref = okv.decode_heads(q.float().numpy().astype(np.float64), kk, vv, group)
        check_o_lse(o, lse, o_ref, lse_ref)
    assert np.array_equal(cache.sync_lengths(), np.array([len(x) for x in ks]))
    assert int(cache.overflow_t.item()) >= 2


def test_append_on_stacked_caches(cuda_device):
    """Caches laid out together (LayerCache.allocate_many: one K/V
    allocation, every layer's tables in one device buffer) grow and decode
    independently: appends to layer 1 change neither layer 0's nor layer 2's
    outputs, and every layer matches the oracle over its own rows."""
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache
    group, hkv, bt, L = 4, 8, 2, 3
    hq = hkv * group
    qrow = np.array([b * hq + h * group for b in range(bt) for h in range(hkv)])
    rng = np.random.default_rng(5)
    lens = [rng.integers(1, 700, size=bt * hkv) for _ in range(L)]
    caches, _ = LayerCache.allocate_many([(n, qrow, qrow) for n in lens], group, cuda_device, reserve=5)
    g = torch.Generator().manual_seed(6)
    rows = []
    for c, n in zip(caches, lens):
        ks = [torch.randn(int(x), 128, generator=g).to(torch.bfloat16) for x in n]
        vs = [torch.randn(int(x), 128, generator=g).to(torch.bfloat16) for x in n]
        kh = torch.zeros(c.k.shape, dtype=torch.bfloat16)
        vh = torch.zeros(c.v.shape, dtype=torch.bfloat16)
        for r0, k, v in zip(c.host["seg_row0"], ks, vs):
            kh[r0:r0 + len(k)] = torch.from_numpy(okv.swizzle_rows(k.view(torch.int16).numpy(), r0)).view(torch.bfloat16)
            vh[r0:r0 + len(v)] = torch.from_numpy(okv.swizzle_rows(v.view(torch.int16).numpy(), r0)).view(torch.bfloat16)
        c.k.copy_(kh)
        c.v.copy_(vh)
        rows.append((ks, vs))
    q = torch.randn(bt, hq, 128, generator=g).to(torch.bfloat16)
    before = [ops.decode(q.to(cuda_device), c) for c in (caches[0], caches[2])]
    for _ in range(3):  # grow layer 1 only
        kn = torch.randn(bt, hkv, 128, generator=g).to(torch.bfloat16)
        vn = torch.randn(bt, hkv, 128, generator=g).to(torch.bfloat16)
        ops.append(caches[1], kn.to(cuda_device), vn.to(cuda_device))
        ks, vs = rows[1]
        for s in range(bt * hkv):
            b, h = divmod(s, hkv)
            ks[s] = torch.cat([ks[s], kn[b, h][None]])
            vs[s] = torch.cat([vs[s], vn[b, h][None]])
    after = [ops.decode(q.to(cuda_device), c) for c in (caches[0], caches[2])]
    for (o0, l0), (o1, l1) in zip(before, after):
        assert torch.equal(o0, o1) and torch.equal(l0, l1)
    for c, (ks, vs) in zip(caches, rows):
        o, lse = ops.decode(q.to(cuda_device), c)
        torch.cuda.synchronize()
        kk = [x.float().numpy().astype(np.float64) for x in ks]
        vv = [x.float().numpy().astype(np.float64) for x in vs]
        o_ref, lse_ref = okv.decode_heads(q.float().numpy().astype(np.float64), kk, vv, group)
        check_o_lse(o, lse, o_ref, lse_ref)
    assert np.array_equal(caches[1].sync_lengths(), np.array([len(x) for x in rows[1][0]]))


def test_decode_long_segments_wide_shape(cuda_device):
    """A TP=2-like shard at B=1024 (256 segments of ~65 tiles): the
    automatic schedule takes the 8-warp CTA shape with whole segments packed
    longest-first (two per CTA on most SMs); o / lse match the oracle."""
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import FKV_DECODE_WIDE
    rng = np.random.default_rng(17)
    group, hkv, bt = 8, 4, 64
    seg_lens = rng.integers(700, 1400, size=bt * hkv).tolist()
    cache, q, ks, vs = build_cache(seg_lens, group, hkv, bt, cuda_device, seed=17)
    assert cache.flags == FKV_DECODE_WIDE and cache.n_items == len(seg_lens)
    o, lse = ops.decode(q.to(cuda_device), cache)
    torch.cuda.synchronize()
    o_ref, lse_ref = okv.decode_heads(q.float().numpy().astype(np.float64), ks, vs, group)
    check_o_lse(o, lse, o_ref, lse_ref)
