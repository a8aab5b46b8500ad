"""AHA-sharded decode across GPUs of one node (north_star subsystem 4).

An ``AllocationPlan`` (allocate.optimize_plan / sha_plan; reference
allocate.py:60-67, group position = GPU index per allocate.py:403-404) says
which KV-head copies each GPU holds per layer.  This module turns it into:

* per-rank segment tables: copy c of head h (c = rank order among the GPUs
  that hold h, r copies in total) owns retained tokens [cut_c, cut_{c+1}) of
  every request, cut_c = round(floor(c*b/r) / 16) * 16 capped at floor16(b) (DP copies split the
  token axis; the reference's adjusted weight w/r is this equal share,
  allocate.py:3-4,70-82);
* fixed per-rank send slots (one per local segment, padded to the max over
  ranks) and the final merge tables every rank uses after the all-gather:
  head (b, h) = LSE merge of the slots of its copies, in rank order.

Per layer and GPU the decode is K4 (partials) -> K5 (chunks -> slots) ->
all-gather of the slot records (NCCL over NVLink) -> K5 (copies -> o bf16
[Bt, Hq, 128] on every rank, ready for o_proj).  TP = 1 skips the exchange.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .allocate import AllocationPlan
from .profiles import ModelProfile, SyntheticSpec, generate_profile

SPLIT = 16  # FKV_SPLIT


# ----------------------------------------------------------- budgets ------
def apportion(total: int, shares: np.ndarray) -> np.ndarray:
    """Largest-remainder rounding of total * shares to ints summing to total
    (ties to the lower index)."""
    q = total * np.asarray(shares, dtype=np.float64)
    base = np.floor(q).astype(np.int64)
    rem = int(total - base.sum())
    if rem > 0:
        frac = q - base
        order = np.lexsort((np.arange(len(q)), -frac))
        base[order[:rem]] += 1
    return base


def synthetic_budgets(num_layers: int, batch: int, hkv: int, budget: int, *, window: int = 32,
                      alpha: float = 0.2, distribution: str = "dirichlet", param: float = 8.0,
                      concentration: float = 400.0, seed: int = 0,
                      context: int | None = None) -> np.ndarray:
    """Ada-shaped per-(layer, request, head) retained-token counts [L, Bt, Hkv].

    Layer shape: ``generate_profile`` (reference profiles.py:105-137) with
    ``distribution``/``param`` -- dirichlet alpha=8 over 8 KV heads matches
    the paper's SHA busy rates.  Per request the shares are
    redrawn from Dirichlet(concentration * share) (Ada budgets vary by
    request; the profile is their mean).  Each head keeps the window plus
    the Ada floor floor(alpha*(B-w)); the remaining Hkv*(B-w-floor) tokens
    are apportioned by share, so every request sums to exactly Hkv*B."""
    prof = generate_profile(SyntheticSpec(distribution, param, float(hkv * budget), seed),
                            num_layers, hkv)
    rng = np.random.default_rng(seed + 1)
    floor_ = int(math.floor(alpha * (budget - window)))
    base = window + floor_
    rest = hkv * (budget - base)
    out = np.empty((num_layers, batch, hkv), dtype=np.int32)
    for l, row in enumerate(prof.weights):
        share = np.asarray(row) / sum(row)
        for b in range(batch):
            s = rng.dirichlet(concentration * share + 1e-3)
            out[l, b] = base + apportion(rest, s)
    if context is not None and int(out.max()) > context:
        raise ValueError(f"a head budget {int(out.max())} exceeds the context {context}")
    return out


def budgets_profile(budgets: np.ndarray, kv_budget: int) -> ModelProfile:
    """Mean over requests -> the planner's ModelProfile (profiles.profile_from_budgets)."""
    from .profiles import profile_from_budgets
    return profile_from_budgets(budgets, kv_budget)


# ------------------------------------------------------------ DP cuts -----
def dp_cuts(n: int, r: int) -> list[int]:
    """Token cut points of r copies of a head with n retained tokens."""
    cuts = [0]
    for c in range(1, r):
        x = (c * n) // r
        cuts.append(min(n // SPLIT * SPLIT, (x + SPLIT // 2) // SPLIT * SPLIT))
    cuts.append(n)
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return cuts


# ------------------------------------------------------------- layouts ----
@dataclass
class LayerShard:
    """One layer on one rank."""

    seg_b: np.ndarray      # request of each local segment
    seg_h: np.ndarray      # KV head
    seg_copy: np.ndarray   # copy index c of that head
    seg_lo: np.ndarray     # first retained token (logical index within the head)
    seg_hi: np.ndarray

    @property
    def n_segments(self) -> int:
        return int(self.seg_b.shape[0])

    def tokens(self) -> int:
        return int((self.seg_hi - self.seg_lo).sum())


@dataclass
class FinalMerge:
    """Tables (identical on every rank) turning gathered slots into o rows."""

    slots: int               # per-rank slot count (max local segments over ranks)
    grp_ptr: np.ndarray      # [Bt*Hkv + 1]
    src_idx: np.ndarray      # rank * slots + slot
    out_row: np.ndarray      # b*Hq + h*G


def head_copies(plan: AllocationPlan, layer: int) -> dict[int, list[int]]:
    """head -> ranks holding a copy, in rank order (copy index = position)."""
    out: dict[int, list[int]] = {}
    for g, group in enumerate(plan.layers[layer].groups):
        for c in group:
            out.setdefault(c.head_id, []).append(g)
    return out


def layer_layout(plan: AllocationPlan, layer: int, budgets_l: np.ndarray, group: int,
                 slots: int | None = None) -> tuple[list[LayerShard], FinalMerge]:
    """budgets_l: [Bt, Hkv] retained tokens of this layer.  ``slots`` fixes
    the per-rank slot count (default: this layer's maximum)."""
    bt, hkv = budgets_l.shape
    hq = hkv * group
    owners = head_copies(plan, layer)
    missing = [h for h in range(hkv) if h not in owners]
    if missing:
        raise ValueError(f"layer {layer}: heads {missing} have no GPU")
    shards = []
    slot_of: dict[tuple[int, int, int], int] = {}
    for g, grp in enumerate(plan.layers[layer].groups):
        sb, sh, sc, lo, hi = [], [], [], [], []
        for copy in sorted(grp, key=lambda c: c.head_id):
            h = copy.head_id
            c = owners[h].index(g)
            r = len(owners[h])
            for b in range(bt):
                cuts = dp_cuts(int(budgets_l[b, h]), r)
                slot_of[(g, b, h)] = len(sb)
                sb.append(b)
                sh.append(h)
                sc.append(c)
                lo.append(cuts[c])
                hi.append(cuts[c + 1])
        shards.append(LayerShard(*(np.asarray(x, dtype=np.int64) for x in (sb, sh, sc, lo, hi))))
    need = max(1, max(s.n_segments for s in shards))
    slots = need if slots is None else slots
    if slots < need:
        raise ValueError(f"layer {layer}: {need} slots needed, {slots} given")
    ptr = [0]
    src = []
    out_row = []
    for b in range(bt):
        for h in range(hkv):
            for g in owners[h]:
                src.append(g * slots + slot_of[(g, b, h)])
            ptr.append(len(src))
            out_row.append(b * hq + h * group)
    fm = FinalMerge(slots, np.asarray(ptr, np.int32), np.asarray(src, np.int32),
                    np.asarray(out_row, np.int32))
    return shards, fm


def plan_layouts(plan: AllocationPlan, budgets: np.ndarray, group: int):
    """All layers: ([per-layer list over ranks of LayerShard], [per-layer
    FinalMerge]); one slot count for every layer (the receive areas of the
    fused all-gather are sized once)."""
    L = budgets.shape[0]
    slots = 1
    for l in range(L):
        for g, grp in enumerate(plan.layers[l].groups):
            slots = max(slots, len(grp) * budgets.shape[1])
    shards, finals = [], []
    for l in range(L):
        s, f = layer_layout(plan, l, budgets[l], group, slots)
        shards.append(s)
        finals.append(f)
    return shards, finals


def rank_loads(plan: AllocationPlan, budgets: np.ndarray, group: int) -> np.ndarray:
    """Actual retained tokens per (layer, rank) summed over the batch (the
    load the K4 kernel streams), shape [L, tp]."""
    L = budgets.shape[0]
    out = np.zeros((L, plan.tp), dtype=np.int64)
    for l in range(L):
        shards, _ = layer_layout(plan, l, budgets[l], group)
        for g, s in enumerate(shards):
            out[l, g] = s.tokens()
    return out


def imbalance_ratio(loads: np.ndarray) -> float:
    """sum_l max_g load / sum_l mean_g load (>= 1, 1 = balanced)."""
    return float(loads.max(axis=1).sum() / loads.mean(axis=1).sum())
