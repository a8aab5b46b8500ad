"""Restatement of the reference AHA search -- TEST INFRASTRUCTURE ONLY.

Checker for the native planner (paper_2502_15804_b200/csrc/planner.cpp).
Written independently of the reference's recursive code: the branch-and-bound
runs on an explicit stack, so agreement on spreads, groupings *and node
counts* between this file, the reference and the C++ planner is a real
cross-check of the search order and the bound arithmetic.

Follows:
  _greedy            reference pkg/src/headbalance/_kernel/reference.py:47-77
  solve_equal_split  reference.py:80-235  (bounds 159-181, branch rules 183-221,
                     precedence 225-235)
  solve_free_split   reference.py:238-340
  canonical_copies   reference allocate.py:85-98
  ordered_schemes    reference allocate.py:186-197 + schemes.py:64-96
  sha_hint           reference allocate.py:214-233
  select_best        reference allocate.py:236-277
PINNED by tests/golden/planner_golden.json (produced by the reference itself,
tests/golden/make_golden.py) and, where /root/reference exists, by live
comparison.
"""

from __future__ import annotations

import itertools
import math

INF = math.inf
NODE_BUDGET = 200_000


def _guard(x: float) -> float:
    return 1e-12 * (1.0 + abs(x))


def _rgs(labels):
    seen = {}
    return [seen.setdefault(g, len(seen)) for g in labels]


def greedy(weights, heads, tp, k):
    load = [0.0] * tp
    size = [0] * tp
    occupied = [set() for _ in range(tp)]
    labels = []
    for w, h in zip(weights, heads):
        ok = [j for j in range(tp) if size[j] < k and h not in occupied[j]]
        if not ok:
            return None
        j = min(ok, key=lambda g: (load[g], g))  # first index among equal loads
        load[j] += w
        size[j] += 1
        occupied[j].add(h)
        labels.append(j)
    return max(load) - min(load), _rgs(labels)


def _spread(sums):
    return max(sums) - min(sums)


def solve_equal_split(weights, heads, tp, cutoff, node_budget=NODE_BUDGET, hint=None):
    m = len(weights)
    k = m // tp
    pre = [0.0]
    for w in weights:
        pre.append(pre[-1] + w)
    avg = pre[m] / tp
    hi_avg, lo_avg = avg + _guard(avg), avg - _guard(avg)
    tail_same = [0] * m
    for t in range(m - 2, -1, -1):
        tail_same[t] = tail_same[t + 1] + 1 if heads[t + 1] == heads[t] else 0
    g = greedy(weights, heads, tp, k)
    seed = INF
    for cand in (g, hint):
        if cand is not None and cand[0] < seed:
            seed = cand[0]

    sums = [0.0] * tp
    counts = [0] * tp
    last = {}
    assign = [0] * m
    best = [cutoff, None]
    nodes = 0

    def bound(t, opened):
        ub_min, lb_max = hi_avg, lo_avg
        for j in range(min(opened + 1, tp)):
            s, need = (sums[j], k - counts[j]) if j < opened else (0.0, k)
            hi = s + (pre[t + need] - pre[t])
            hi += _guard(hi)
            lo = s + (pre[m] - pre[m - need])
            lo -= _guard(lo)
            if hi < ub_min:
                ub_min = hi
            if lo > lb_max:
                lb_max = lo
        return lb_max - ub_min, ub_min

    def child_ok(t, opened, j, ub_min):
        cnt, base = (counts[j], sums[j]) if j < opened else (0, 0.0)
        if cnt >= k:
            return False
        trailing = tail_same[t]
        if trailing:
            free = sum(1 for j2 in range(j + 1, tp) if j2 >= opened or counts[j2] < k)
            if trailing > free:
                return False
        fill = k - cnt - 1
        forced = base + weights[t] + (pre[m] - pre[m - fill])
        forced -= _guard(forced)
        blb = forced - ub_min
        return not (blb >= best[0] or blb > seed)

    def leaf_spread():
        hi = lo = sums[0]
        for s in sums[1:]:
            if s > hi:
                hi = s
            elif s < lo:
                lo = s
        return hi - lo

    def enter(t, opened):
        nonlocal nodes
        if nodes >= node_budget:
            return "abort"
        nodes += 1
        if t == m:
            d = leaf_spread()
            if d < best[0] and d <= seed:
                best[0], best[1] = d, assign.copy()
            return None
        lb, ub_min = bound(t, opened)
        if lb >= best[0] or lb > seed:
            return None
        start = last.get(heads[t], -1) + 1
        return {"t": t, "opened": opened, "j": start, "start": start, "ub": ub_min,
                "placed": None, "saved": None}

    stack = []
    fr = enter(0, 0)
    aborted = fr == "abort"
    if isinstance(fr, dict):
        stack.append(fr)
    while stack and not aborted:
        fr = stack[-1]
        t, opened = fr["t"], fr["opened"]
        h = heads[t]
        if fr["placed"] is not None:  # undo the previous child
            sums[fr["placed"]], counts[fr["placed"]] = fr["saved"]
            last[h] = fr["start"] - 1
            fr["placed"] = None
        limit = opened if opened < tp else tp - 1
        pick = None
        j = fr["j"]
        while j <= limit:
            if child_ok(t, opened, j, fr["ub"]):
                pick = j
                break
            j += 1
        if pick is None:
            stack.pop()
            continue
        base = sums[pick] if pick < opened else 0.0
        cnt = counts[pick] if pick < opened else 0
        fr["j"], fr["placed"], fr["saved"] = pick + 1, pick, (base, cnt)
        sums[pick] = base + weights[t]
        counts[pick] = cnt + 1
        last[h] = pick
        assign[t] = pick
        child = enter(t + 1, opened + 1 if pick == opened else opened)
        if child == "abort":
            aborted = True
        elif child is not None:
            stack.append(child)

    result = None
    if best[1] is not None:
        result = (best[0], best[1])
    if hint is not None and hint[0] < cutoff and (result is None or hint[0] < result[0]):
        result = (hint[0], list(hint[1]))
    if g is not None and g[0] < cutoff and (result is None or g[0] < result[0]):
        result = g
    return result, nodes


def solve_free_split(weights, heads, tp, cutoff, node_budget=NODE_BUDGET, hint=None):
    m = len(weights)
    if m < tp:
        return None, 0
    total = 0.0
    for w in weights:
        total += w
    avg = total / tp
    hi_avg, lo_avg = avg + _guard(avg), avg - _guard(avg)
    tail_same = [0] * m
    for t in range(m - 2, -1, -1):
        tail_same[t] = tail_same[t + 1] + 1 if heads[t + 1] == heads[t] else 0
    seed = INF if hint is None else hint[0]
    sums = [0.0] * tp
    last = {}
    assign = [0] * m
    best = [cutoff, None]
    nodes = 0

    def enter(t, opened):
        nonlocal nodes
        if nodes >= node_budget:
            return "abort"
        nodes += 1
        if t == m:
            if opened < tp:
                return None
            hi = lo = sums[0]
            for s in sums[1:]:
                if s > hi:
                    hi = s
                elif s < lo:
                    lo = s
            d = hi - lo
            if d < best[0] and d <= seed:
                best[0], best[1] = d, assign.copy()
            return None
        if m - t < tp - opened:
            return None
        cur = 0.0
        for s in sums[:opened]:
            if s > cur:
                cur = s
        lb = (cur if cur > lo_avg else lo_avg) - hi_avg
        if lb >= best[0] or lb > seed:
            return None
        start = last.get(heads[t], -1) + 1
        return {"t": t, "opened": opened, "j": start, "start": start, "placed": None, "old": 0.0}

    stack = []
    fr = enter(0, 0)
    aborted = fr == "abort"
    if isinstance(fr, dict):
        stack.append(fr)
    while stack and not aborted:
        fr = stack[-1]
        t, opened = fr["t"], fr["opened"]
        h = heads[t]
        if fr["placed"] is not None:
            sums[fr["placed"]] = fr["old"]
            last[h] = fr["start"] - 1
            fr["placed"] = None
        limit = opened if opened < tp else tp - 1
        pick = None
        j = fr["j"]
        while j <= limit:
            nxt_open = opened + 1 if j == opened else opened
            if tail_same[t] > tp - 1 - j or m - t - 1 < tp - nxt_open:
                j += 1
                continue
            ns = sums[j] + weights[t]
            blb = ns - _guard(ns) - hi_avg
            if blb >= best[0] or blb > seed:
                j += 1
                continue
            pick = j
            break
        if pick is None:
            stack.pop()
            continue
        fr["j"], fr["placed"], fr["old"] = pick + 1, pick, sums[pick]
        sums[pick] = sums[pick] + weights[t]
        last[h] = pick
        assign[t] = pick
        child = enter(t + 1, opened + 1 if pick == opened else opened)
        if child == "abort":
            aborted = True
        elif child is not None:
            stack.append(child)

    result = None
    if best[1] is not None:
        result = (best[0], best[1])
    if hint is not None and hint[0] < cutoff and (result is None or hint[0] < result[0]):
        result = (hint[0], list(hint[1]))
    return result, nodes


# ------------------------------------------------------------ scheme loop --
def ordered_schemes(n, ch_budget, r_max, divisible, tp):
    out = []
    for vec in itertools.product(range(1, r_max + 1), repeat=n):
        extra = sum(vec) - n
        if extra > ch_budget:
            continue
        if divisible and sum(vec) % tp:
            continue
        out.append(tuple(vec))
    out.sort(key=lambda v: (sum(v), v))
    return out


def canonical_copies(replicas, weights):
    pairs = []
    for h, (r, w) in enumerate(zip(replicas, weights)):
        pairs += [(w / r, h)] * r
    pairs.sort(key=lambda p: (-p[0], p[1]))
    return [p[0] for p in pairs], [p[1] for p in pairs]


def sha_hint(wc, hc, n, tp):
    per = n // tp
    labels = _rgs([h // per for h in hc])
    sums = [0.0] * tp
    for lab, w in sorted(zip(labels, wc), key=lambda x: (x[0], -x[1])):
        sums[lab] += w
    return _spread(sums), labels


def select_best(weights, tp, ch_budget, r_max, equal_split=True, node_budget=NODE_BUDGET):
    """-> (delta, replicas, heads_c, rgs) with the reference tie rule."""
    n = len(weights)
    solve = solve_equal_split if equal_split else solve_free_split
    best = None
    for reps in ordered_schemes(n, ch_budget, r_max, equal_split, tp):
        if max(reps) > tp:
            continue
        wc, hc = canonical_copies(reps, weights)
        hint = sha_hint(wc, hc, n, tp) if (equal_split and sum(reps) == n and n % tp == 0) else None
        res, _ = solve(wc, hc, tp, INF if best is None else best[0], node_budget, hint)
        if res is not None:
            best = (res[0], reps, hc, res[1])
    return best


def groups_of(replicas, heads_c, rgs, tp):
    """RGS -> sorted ((head, replicas), ...) per GPU, as reference allocate.py:200-211."""
    buckets = [[] for _ in range(tp)]
    for i, g in enumerate(rgs):
        buckets[g].append(heads_c[i])
    return [tuple((h, replicas[h]) for h in b) for b in sorted((sorted(b) for b in buckets), key=tuple)]
