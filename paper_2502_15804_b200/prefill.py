"""Prefill-side producer of the planner's input.

Per layer, the fused K1 + A18 + K2 launch (``ops.score_select``) yields the
Ada budgets of every (request, KV head); ``ada_profile`` stacks them over
layers and aggregates them over requests into the reference's
``ModelProfile`` (reference profiles.py:25-70; weights = mean retained KV
entries per head, profiles.py:4-6), which ``save_profile`` writes in the
reference's JSON format -- so ``headbalance optimize`` consumes profiles
measured on the B200.  ``profile_similarity`` of two disjoint request sets is
the paper's invariance check (reference profiles.py:159-161).

``skewed_prefill_inputs`` makes synthetic prefill inputs whose Ada budgets
are skewed across heads the way trained models' are: random q / k give
near-uniform budgets, so every (layer, KV head) gets a fixed attention
temperature beta_{l,h} (its queries are scaled by beta), drawn once per model
from a seeded generator and shared by all requests.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops
from .profiles import ModelProfile, profile_from_budgets

HEAD_DIM = 128


def head_temperatures(num_layers: int, hkv: int, seed: int = 0, sigma: float = 0.35,
                      mean: float = 1.5) -> np.ndarray:
    """beta [L, Hkv] = mean * exp(sigma * N(0,1)), fixed per model (seeded)."""
    rng = np.random.default_rng(seed)
    return mean * np.exp(sigma * rng.standard_normal((num_layers, hkv)))


def skewed_prefill_inputs(layer: int, beta: np.ndarray, batch: int, hq: int, hkv: int, T: int,
                          window: int = 32, seed: int = 0, device="cuda"):
    """(q_win bf16 [Bt, Hq, w, 128], k bf16 [Bt, Hkv, T, 128]) of one layer:
    N(0,1) keys, queries N(0,1) scaled by the layer's per-KV-head temperature."""
    g = torch.Generator(device=device).manual_seed(seed * 7919 + layer)
    G = hq // hkv
    q = torch.randn((batch, hq, window, HEAD_DIM), generator=g, device=device)
    scale = torch.as_tensor(np.repeat(beta[layer], G), dtype=torch.float32, device=device)
    q = (q * scale[None, :, None, None]).to(torch.bfloat16)
    k = torch.randn((batch, hkv, T, HEAD_DIM), generator=g, device=device).to(torch.bfloat16)
    return q, k


def layer_budgets(q_win: torch.Tensor, k: torch.Tensor, budget: int, window: int = 32,
                  alpha: float = 0.2, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """int32 [Bt, Hkv] Ada budgets of one layer (one fused launch)."""
    _, hb, _, _ = ops.score_select(q_win, k, budget, window, alpha, workspace=workspace)
    return hb


def ada_profile(budgets_per_layer, kv_budget: int, model_name: str = "b200-ada-snapkv") -> ModelProfile:
    """[L] x [Bt, Hkv] GPU budgets -> ModelProfile (mean over requests)."""
    return profile_from_budgets([b.cpu().numpy() if isinstance(b, torch.Tensor) else b
                                 for b in budgets_per_layer], kv_budget, model_name)


def measure_profile(num_layers: int, batch: int, hq: int, hkv: int, T: int, budget: int, *,
                    window: int = 32, alpha: float = 0.2, seed: int = 0, request_seed: int = 0,
                    device="cuda", model_name: str = "b200-ada-snapkv"):
    """Run the fused scoring + Ada split over ``num_layers`` synthetic skewed
    layers for ``batch`` requests; -> (ModelProfile, budgets int32 [L, Bt, Hkv]).
    ``seed`` fixes the model (head temperatures), ``request_seed`` the requests."""
    beta = head_temperatures(num_layers, hkv, seed)
    out = []
    for l in range(num_layers):
        q, k = skewed_prefill_inputs(l, beta, batch, hq, hkv, T, window, request_seed, device)
        out.append(layer_budgets(q, k, budget, window, alpha).cpu().numpy())
    arr = np.stack(out)
    return ada_profile(arr, budget, model_name), arr
