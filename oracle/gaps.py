"""Selection-boundary margins of the Ada split + top-k -- TEST
INFRASTRUCTURE ONLY.

End-to-end index equality between the GPU path (fp32 scores) and the oracle
(float64 scores) can only be asserted where no selection boundary is closer
than the score tolerance (SURVEY §7 "hard parts").  ``boundary_margins``
lists, for one request, every place the selection turns on the order of two
scores -- each head's floor boundary, the global Ada threshold, each head's
top-(b_h - w) boundary -- as (v_in, v_out): the last score kept and the
first one left out.  ``separated`` accepts a boundary when the two scores
differ by more than both tolerances, or are exactly equal (a max-pooling
plateau: both sides come from the same raw peak and tie the same way in
fp32).
"""

from __future__ import annotations

import math

import numpy as np

from .kv import _order_desc


def boundary_margins(s: np.ndarray, budget: int, window: int, alpha: float = 0.2):
    """s [Hkv, n] float64 scores of one request -> list of (v_in, v_out)."""
    hkv, n = s.shape
    sel = budget - window
    f = int(math.floor(alpha * sel))
    R = hkv * sel - hkv * f
    out = []
    orders = [_order_desc(s[h]) for h in range(hkv)]
    cs, ch, ct = [], [], []
    for h in range(hkv):
        o = orders[h]
        if 0 < f < n:
            out.append((s[h, o[f - 1]], s[h, o[f]]))
        rest = o[f:]
        cs.append(s[h, rest])
        ch.append(np.full(len(rest), h))
        ct.append(rest)
    cs, ch, ct = map(np.concatenate, (cs, ch, ct))
    g = np.lexsort((ct, ch, -cs))
    if 0 < R < len(g):
        out.append((cs[g[R - 1]], cs[g[R]]))
    counts = np.bincount(ch[g[:R]], minlength=hkv)
    for h in range(hkv):
        k = f + int(counts[h])
        if 0 < k < n:
            out.append((s[h, orders[h][k - 1]], s[h, orders[h][k]]))
    return out


def separated(s: np.ndarray, budget: int, window: int, rtol: float, atol_row: float,
              alpha: float = 0.2) -> bool:
    """Every boundary of every request is exactly tied or wider than the
    score tolerance (rtol |v| + atol_row * that head's max) on both sides."""
    for b in range(s.shape[0]):
        floor_abs = atol_row * np.abs(s[b]).max()
        for v_in, v_out in boundary_margins(s[b], budget, window, alpha):
            if v_in == v_out:
                continue
            tol = rtol * (abs(v_in) + abs(v_out)) + 2 * floor_abs
            if v_in - v_out <= tol:
                return False
    return True
