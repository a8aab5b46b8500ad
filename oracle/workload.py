"""The benchmark workload and the CPU decode step of the reference arm --
TEST / BENCH INFRASTRUCTURE ONLY (bench.py ``--impl reference`` and
``cpu_baseline``, tests).  Never imports the product package.

``synthetic_budgets`` restates ``paper_2502_15804_b200.sharding.
synthetic_budgets`` on top of the *reference's own* ``generate_profile``
(pkg/src/headbalance/profiles.py:105-137, passed in as ``hb``), so the
reference arm builds the identical per-(layer, request, head) budgets
without the product (tests/test_bench_cpu.py pins the two bit for bit).

``decode_layer`` is the reference CPU path of one decode layer: float64
attention of every (request, KV head) over its retained tokens, G query
heads per KV head (oracle/kv.py ``attend``), requests spread over host
threads.  The reference has no decode of its own; this is the
oracle restatement, ``cpu_baseline.kind = "port"``.
"""

from __future__ import annotations

import math

import numpy as np

from . import kv


def apportion(total: int, shares) -> np.ndarray:
    """Largest-remainder rounding of total * shares to ints summing to total,
    ties to the lower index."""
    q = total * np.asarray(shares, dtype=np.float64)
    base = np.floor(q).astype(np.int64)
    rem = int(total - base.sum())
    if rem > 0:
        frac = q - base
        order = np.lexsort((np.arange(len(q)), -frac))
        base[order[:rem]] += 1
    return base


def synthetic_budgets(hb, num_layers: int, batch: int, hkv: int, budget: int, *, window: int = 32,
                      alpha: float = 0.2, distribution: str = "dirichlet", param: float = 8.0,
                      concentration: float = 400.0, seed: int = 0) -> np.ndarray:
    """[L, Bt, Hkv] int32 retained tokens: the layer's head shares from the
    reference's ``generate_profile``, per request redrawn from
    Dirichlet(concentration * share), each head keeping the window plus the
    Ada floor floor(alpha (B - w)) and the rest apportioned by share."""
    prof = hb.generate_profile(hb.SyntheticSpec(distribution, param, float(hkv * budget), seed),
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
    return out


class CpuDecodeStack:
    """Synthetic float64 K/V for every (request, KV head) -- one pool sized to
    the longest budget of that pair over the layers; layer l attends over its
    first budgets[l, b, h] rows (the values do not change the work) -- and
    the per-layer decode over host threads."""

    def __init__(self, budgets: np.ndarray, hq: int, head_dim: int = 128, seed: int = 1,
                 threads: int | None = None):
        import os
        self.budgets = np.asarray(budgets)
        L, bt, hkv = self.budgets.shape
        self.group = hq // hkv
        rng = np.random.default_rng(seed)
        longest = self.budgets.max(axis=0)  # [bt, hkv]
        self.k = [[rng.standard_normal((int(longest[b, h]), head_dim)) for h in range(hkv)]
                  for b in range(bt)]
        self.v = [[rng.standard_normal((int(longest[b, h]), head_dim)) for h in range(hkv)]
                  for b in range(bt)]
        self.q = rng.standard_normal((bt, hq, head_dim))
        self.threads = threads or os.cpu_count() or 1
        from concurrent.futures import ThreadPoolExecutor
        self.pool = ThreadPoolExecutor(self.threads)

    def _request(self, l: int, b: int) -> np.ndarray:
        G = self.group
        out = np.empty((self.q.shape[1], self.q.shape[2]))
        for h in range(self.budgets.shape[2]):
            n = int(self.budgets[l, b, h])
            o, _ = kv.attend(self.q[b, h * G:(h + 1) * G], self.k[b][h][:n], self.v[b][h][:n])
            out[h * G:(h + 1) * G] = o
        return out

    def decode_layer(self, l: int) -> np.ndarray:
        """o [Bt, Hq, d] of layer l (float64)."""
        jobs = [self.pool.submit(self._request, l, b) for b in range(self.budgets.shape[1])]
        return np.stack([j.result() for j in jobs])

    def step(self, layers: int | None = None) -> float:
        """Decode every layer once; returns a checksum of the outputs.  BLAS
        runs single-threaded inside each worker thread (the parallelism is
        over requests; nested BLAS threads would oversubscribe the cores)."""
        from threadpoolctl import threadpool_limits
        acc = 0.0
        with threadpool_limits(1):
            for l in range(layers or self.budgets.shape[0]):
                acc += float(self.decode_layer(l)[:, :, 0].sum())
        return acc

    def close(self):
        self.pool.shutdown()
