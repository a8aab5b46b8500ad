"""float64 numpy restatement of the compression + decode path -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).  PARITY UNPINNED vs the
reference, which has no implementation of any of this.

Definitions (fixed once, documented in DESIGN.md §"Algorithm definitions"):

Ada-SnapKV scoring (SnapKV, Li et al. 2024; GQA handling as in Ada-KV):
    window queries i = 0..w-1 sit at positions T-w+i and see keys t <= T-w+i;
    P[g,i,:] = softmax_t(q[g,i] . k[t] / sqrt(d))           (full-row softmax)
    raw[t]   = (1/G) * sum_g sum_i P[g,i,t]                 for t < T-w
    s[t]     = max(raw[t-3 .. t+3] clipped to [0, T-w))      (max-pool k=7)

Ada budget split (Ada-KV, Feng et al. 2024; safeguard alpha):
    f   = floor(alpha * (B - w))        per-head floor
    F_h = top-f of s[h] by (score desc, token asc)
    R   = Hkv*(B - w) - Hkv*f           slots left after the floors
    global top-R over {(h,t) not in F_h} by (score desc, head asc, token asc)
    b_h = w + f + (#globally chosen of head h);  sum_h b_h = Hkv*B

Selection: head h keeps its top-(b_h - w) tokens by (score desc, token asc)
(== F_h + its globally chosen tokens), sorted ascending, then the window
tokens T-w..T-1.

Decode: o = softmax(q . K_sel^T / sqrt(d)) V_sel per (request, query head),
with lse = log sum exp(q . k / sqrt(d)).  LSE merge of partials (o_c, lse_c):
lse = log sum_c e^{lse_c};  o = sum_c e^{lse_c - lse} o_c.
"""

from __future__ import annotations

import math

import numpy as np

HEAD_DIM = 128
PAGE = 64


# ------------------------------------------------------------------ scoring --
def snapkv_scores(q_win: np.ndarray, k: np.ndarray, pool_k: int = 7) -> np.ndarray:
    """q_win [Bt,Hq,w,d], k [Bt,Hkv,T,d] -> pooled scores [Bt,Hkv,T-w] (float64)."""
    q_win = np.asarray(q_win, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    bt, hq, w, d = q_win.shape
    _, hkv, T, _ = k.shape
    G = hq // hkv
    n = T - w
    out = np.empty((bt, hkv, n), dtype=np.float64)
    pos_q = (T - w) + np.arange(w)
    causal = np.arange(T)[None, :] <= pos_q[:, None]  # [w, T]
    for b in range(bt):
        for h in range(hkv):
            kk = k[b, h]
            raw = np.zeros(n, dtype=np.float64)
            for g in range(G):
                logits = q_win[b, h * G + g] @ kk.T / math.sqrt(d)  # [w, T]
                logits = np.where(causal, logits, -np.inf)
                logits -= logits.max(axis=1, keepdims=True)
                p = np.exp(logits)
                p /= p.sum(axis=1, keepdims=True)
                raw += p[:, :n].sum(axis=0)
            raw /= G
            out[b, h] = maxpool1d(raw, pool_k)
    return out


def maxpool1d(x: np.ndarray, k: int) -> np.ndarray:
    r = k // 2
    n = x.shape[-1]
    out = np.full_like(x, -np.inf)
    for off in range(-r, r + 1):
        lo, hi = max(0, -off), min(n, n - off)
        out[..., lo:hi] = np.maximum(out[..., lo:hi], x[..., lo + off:hi + off])
    return out


# ----------------------------------------------------------- budget split --
def _order_desc(scores_row: np.ndarray) -> np.ndarray:
    """Token order by (score desc, token asc)."""
    return np.lexsort((np.arange(scores_row.shape[0]), -scores_row))


def ada_budgets(scores: np.ndarray, budget: int, window: int, alpha: float = 0.2) -> np.ndarray:
    """scores [Bt,Hkv,n] (n = T - w) -> int32 budgets [Bt,Hkv] incl. the window."""
    s = np.asarray(scores, dtype=np.float64)
    bt, hkv, n = s.shape
    sel = budget - window
    if sel < 0 or sel > n:
        raise ValueError(f"budget {budget} needs 0 <= budget - window <= T - window ({n})")
    f = int(math.floor(alpha * sel))
    R = hkv * sel - hkv * f
    out = np.zeros((bt, hkv), dtype=np.int32)
    for b in range(bt):
        cand_s, cand_h, cand_t = [], [], []
        for h in range(hkv):
            order = _order_desc(s[b, h])
            rest = order[f:]
            cand_s.append(s[b, h, rest])
            cand_h.append(np.full(rest.shape[0], h))
            cand_t.append(rest)
        cs, ch, ct = map(np.concatenate, (cand_s, cand_h, cand_t))
        glob = np.lexsort((ct, ch, -cs))[:R]
        counts = np.bincount(ch[glob], minlength=hkv)
        out[b] = window + f + counts
    return out


def topk_select(scores: np.ndarray, budgets: np.ndarray, window: int):
    """-> (offsets int64 [Bt*Hkv+1], idx int32 [sum b]) in (b, h) order; each
    head's list = ascending top-(b_h - w) tokens then the window tokens."""
    s = np.asarray(scores, dtype=np.float64)
    bt, hkv, n = s.shape
    lists = []
    for b in range(bt):
        for h in range(hkv):
            kk = int(budgets[b, h]) - window
            top = np.sort(_order_desc(s[b, h])[:kk])
            lists.append(np.concatenate([top, n + np.arange(window)]).astype(np.int32))
    offsets = np.zeros(len(lists) + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([x.shape[0] for x in lists])
    return offsets, (np.concatenate(lists) if lists else np.zeros(0, np.int32))


# ---------------------------------------------------------- cache layout --
def swizzle_rows(rows: np.ndarray, row0: int = 0) -> np.ndarray:
    """Logical rows [R,128] -> stored rows with 16-B chunk c at c ^ (r & 7)
    where r = row0 + i is the absolute cache row (include/fairkv.h)."""
    R = rows.shape[0]
    ch = rows.reshape(R, 16, 8)
    out = np.empty_like(ch)
    r = (row0 + np.arange(R)) & 7
    for c in range(16):
        out[np.arange(R), c ^ r] = ch[:, c]
    return out.reshape(R, 128)


def unswizzle_rows(stored: np.ndarray, row0: int = 0) -> np.ndarray:
    R = stored.shape[0]
    ch = stored.reshape(R, 16, 8)
    r = (row0 + np.arange(R)) & 7
    out = np.empty_like(ch)
    for c in range(16):
        out[:, c] = ch[np.arange(R), c ^ r]
    return out.reshape(R, 128)


def page_rows(n_tok: int) -> int:
    return (n_tok + PAGE - 1) // PAGE * PAGE


# ------------------------------------------------------------------ decode --
def attend(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float | None = None):
    """q [G,d], k/v [n,d] -> (o [G,d], lse [G]) in float64; n == 0 -> (0, -inf)."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    G, d = q.shape
    if k.shape[0] == 0:
        return np.zeros((G, d)), np.full(G, -np.inf)
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    logits = q @ k.T * scale
    m = logits.max(axis=1, keepdims=True)
    p = np.exp(logits - m)
    l = p.sum(axis=1, keepdims=True)
    return (p @ v) / l, (m + np.log(l))[:, 0]


def lse_merge(parts_o: list, parts_lse: list):
    """Merge partials of one head group: lists of ([G,d], [G])."""
    lse = np.stack(parts_lse)  # [c, G]
    o = np.stack(parts_o)      # [c, G, d]
    M = lse.max(axis=0)
    finite = np.isfinite(M)
    Ms = np.where(finite, M, 0.0)
    w = np.where(np.isfinite(lse), np.exp(lse - Ms), 0.0)
    S = w.sum(axis=0)
    out = np.where(S[:, None] > 0, (w[:, :, None] * o).sum(axis=0) / np.maximum(S, 1e-300)[:, None], 0.0)
    out_lse = np.where(S > 0, Ms + np.log(np.maximum(S, 1e-300)), -np.inf)
    return out, out_lse


def decode_heads(q: np.ndarray, seg_k: list, seg_v: list, group: int):
    """q [Bt,Hq,d]; seg_k/seg_v lists over (b, kv head) in (b, h) order of
    logical [n_tok, d] arrays -> (o [Bt,Hq,d], lse [Bt,Hq])."""
    q = np.asarray(q, np.float64)
    bt, hq, d = q.shape
    hkv = hq // group
    o = np.zeros((bt, hq, d))
    lse = np.zeros((bt, hq))
    for b in range(bt):
        for h in range(hkv):
            i = b * hkv + h
            oo, ll = attend(q[b, h * group:(h + 1) * group], seg_k[i], seg_v[i])
            o[b, h * group:(h + 1) * group] = oo
            lse[b, h * group:(h + 1) * group] = ll
    return o, lse
