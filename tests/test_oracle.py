"""The CPU oracle (oracle/kv.py) checked against independent implementations.

The reference has no scoring / selection / decode code, so these
pieces are "parity unpinned" against it; this file pins the oracle to
independent formulations instead: torch float64 attention (F.softmax /
scaled_dot_product_attention), a direct torch restatement of SnapKV scoring,
and brute-force definitions of the Ada split and top-k tie rules.
"""

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import kv as okv


def test_attend_matches_torch_sdpa():
    g = torch.Generator().manual_seed(0)
    for n in (1, 7, 300):
        q = torch.randn(8, 128, generator=g, dtype=torch.float64)
        k = torch.randn(n, 128, generator=g, dtype=torch.float64)
        v = torch.randn(n, 128, generator=g, dtype=torch.float64)
        o, lse = okv.attend(q.numpy(), k.numpy(), v.numpy())
        ref = F.scaled_dot_product_attention(q[None, :, None, :], k[None, None].expand(1, 8, n, 128),
                                             v[None, None].expand(1, 8, n, 128))[0, :, 0]
        np.testing.assert_allclose(o, ref.numpy(), rtol=1e-10, atol=1e-12)
        lse_ref = torch.logsumexp(q @ k.T / math.sqrt(128), dim=-1)
        np.testing.assert_allclose(lse, lse_ref.numpy(), rtol=1e-12)


def test_attend_empty_segment():
    o, lse = okv.attend(np.ones((4, 128)), np.zeros((0, 128)), np.zeros((0, 128)))
    assert (o == 0).all() and np.isneginf(lse).all()


def test_lse_merge_identity():
    rng = np.random.default_rng(1)
    q = rng.standard_normal((8, 128))
    k = rng.standard_normal((500, 128))
    v = rng.standard_normal((500, 128))
    o, lse = okv.attend(q, k, v)
    parts = [okv.attend(q, k[a:b], v[a:b]) for a, b in ((0, 0), (0, 123), (123, 400), (400, 500))]
    mo, ml = okv.lse_merge([p[0] for p in parts], [p[1] for p in parts])
    np.testing.assert_allclose(mo, o, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(ml, lse, rtol=1e-12)


def _snapkv_torch(q_win, k, pool_k=7):
    """Independent restatement with torch ops (mask via triu, F.max_pool1d)."""
    q = torch.from_numpy(q_win)
    kk = torch.from_numpy(k)
    bt, hq, w, d = q.shape
    hkv, T = kk.shape[1], kk.shape[2]
    G = hq // hkv
    kx = kk.repeat_interleave(G, dim=1)  # [bt, hq, T, d]
    logits = q @ kx.transpose(-1, -2) / math.sqrt(d)
    mask = torch.ones(w, T, dtype=torch.bool)
    mask[:, T - w:] = torch.triu(torch.ones(w, w, dtype=torch.bool), diagonal=1)
    mask[:, :T - w] = False
    logits = logits.masked_fill(mask, float("-inf"))
    p = logits.softmax(-1)[..., :T - w].sum(-2)  # [bt, hq, T-w]
    p = p.view(bt, hkv, G, T - w).mean(2)
    return F.max_pool1d(p, pool_k, stride=1, padding=pool_k // 2).numpy()


def test_snapkv_matches_torch_restatement():
    rng = np.random.default_rng(2)
    q = rng.standard_normal((2, 8, 6, 128))
    k = rng.standard_normal((2, 2, 70, 128))
    np.testing.assert_allclose(okv.snapkv_scores(q, k), _snapkv_torch(q, k), rtol=1e-12, atol=1e-15)


def _brute_budgets(s, budget, window, alpha):
    hkv, n = s.shape
    f = math.floor(alpha * (budget - window))
    floor = set()
    for h in range(hkv):
        order = sorted(range(n), key=lambda t: (-s[h, t], t))
        floor |= {(h, t) for t in order[:f]}
    rest = [(h, t) for h in range(hkv) for t in range(n) if (h, t) not in floor]
    rest.sort(key=lambda x: (-s[x], x[0], x[1]))
    R = hkv * (budget - window) - hkv * f
    chosen = rest[:R]
    return [window + f + sum(1 for x in chosen if x[0] == h) for h in range(hkv)]


@pytest.mark.parametrize("seed", range(6))
def test_ada_budgets_brute_force(seed):
    rng = np.random.default_rng(seed)
    hkv, n = 4, 40
    s = rng.integers(0, 6, size=(2, hkv, n)).astype(np.float64)  # many exact ties
    if seed % 2:
        s = rng.random((2, hkv, n))
    for budget in (32, 40, 50, 72):
        got = okv.ada_budgets(s, budget, window=32, alpha=0.2)
        for b in range(2):
            assert got[b].tolist() == _brute_budgets(s[b], budget, 32, 0.2)
            assert got[b].sum() == hkv * budget


def test_topk_select_tie_rule_and_window():
    s = np.array([[[3.0, 1.0, 3.0, 2.0, 3.0, 0.0]]])
    off, idx = okv.topk_select(s, np.array([[2 + 3]]), window=2)
    assert off.tolist() == [0, 5]
    assert idx.tolist() == [0, 2, 4, 6, 7]  # the three 3.0s (token asc), then window 6,7
    off, idx = okv.topk_select(s, np.array([[2 + 2]]), window=2)
    assert idx.tolist() == [0, 2, 6, 7]


def test_ada_selection_equals_floor_plus_global():
    """Per-head top-(b_h - w) == floor set + globally chosen."""
    rng = np.random.default_rng(9)
    s = rng.random((1, 8, 300))
    b = okv.ada_budgets(s, 128, 32, 0.2)
    _, idx = okv.topk_select(s, b, 32)
    assert idx.shape[0] == 8 * 128


def test_swizzle_roundtrip():
    rows = np.arange(40 * 128, dtype=np.int16).reshape(40, 128)
    for r0 in (0, 16, 64, 3):
        st = okv.swizzle_rows(rows, r0)
        assert not np.array_equal(st, rows) or r0 % 8 == 0
        np.testing.assert_array_equal(okv.unswizzle_rows(st, r0), rows)
