"""AHA sharding host logic (north_star subsystem 4) on CPU.

* layout invariants: every retained token of every (request, head) is owned by
  exactly one (rank, segment); DP cuts are 16-aligned; final merge tables
  reference each copy once;
* a world_size-2 gloo run of the exact exchange the GPU decoder performs:
  each rank computes its slot records (with the oracle standing in for the
  CUDA kernels, which cannot run here), all-gathers them over a real process
  group, and merges with the shared final tables -> must equal the oracle's
  unsharded decode.
"""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2502_15804_b200 as fk
from paper_2502_15804_b200.sharding import (
    dp_cuts, imbalance_ratio, plan_layouts, rank_loads, synthetic_budgets, budgets_profile,
)
from oracle import kv as okv

REC = 132


def _plan(budgets, tp, mode):
    prof = budgets_profile(budgets, int(budgets.mean()))
    if mode == "sha":
        return fk.sha_plan(prof, tp)
    if mode == "free":
        return fk.optimize_plan(prof, tp, fk.EnumerationConfig(4, 2, True, tp), equal_split=False)
    return fk.optimize_plan(prof, tp, fk.EnumerationConfig(4, 2, True, tp))


def test_synthetic_budgets_shape_and_sum():
    b = synthetic_budgets(6, 5, 8, 256, window=32, alpha=0.2, seed=3)
    assert b.shape == (6, 5, 8)
    assert (b.sum(axis=2) == 8 * 256).all()
    assert b.min() >= 32 + int(0.2 * (256 - 32))


def test_dp_cuts():
    for n in (0, 1, 15, 16, 17, 100, 1000, 4097):
        for r in (1, 2, 3, 4):
            c = dp_cuts(n, r)
            assert c[0] == 0 and c[-1] == n and len(c) == r + 1
            assert all(x % 16 == 0 for x in c[1:-1])
            assert all(a <= b for a, b in zip(c, c[1:]))
            if n >= 64 * r:
                assert max(b - a for a, b in zip(c, c[1:])) - n / r <= 16


@pytest.mark.parametrize("tp,mode", [(1, "sha"), (2, "sha"), (2, "dp"), (4, "dp"), (8, "sha"), (8, "free"), (4, "free")])
def test_layout_covers_every_token_once(tp, mode):
    budgets = synthetic_budgets(3, 4, 8, 256, seed=tp)
    plan = _plan(budgets, tp, mode)
    shards, finals = plan_layouts(plan, budgets, group=8)
    for l in range(3):
        covered = {}
        for g, sh in enumerate(shards[l]):
            for b, h, lo, hi in zip(sh.seg_b, sh.seg_h, sh.seg_lo, sh.seg_hi):
                covered.setdefault((int(b), int(h)), []).append((int(lo), int(hi)))
        for (b, h), ranges in covered.items():
            ranges.sort()
            assert ranges[0][0] == 0 and ranges[-1][1] == budgets[l, b, h]
            assert all(x[1] == y[0] for x, y in zip(ranges, ranges[1:]))
        assert len(covered) == 4 * 8
        f = finals[l]
        assert f.grp_ptr[-1] == len(f.src_idx)
        assert len(set(f.src_idx.tolist())) == len(f.src_idx)
    loads = rank_loads(plan, budgets, 8)
    assert loads.sum() == budgets.sum()
    assert imbalance_ratio(loads) >= 1.0


def test_aha_reduces_imbalance_vs_sha():
    budgets = synthetic_budgets(40, 8, 8, 512, seed=0)
    for tp, mode in ((2, "dp"), (4, "dp"), (8, "free")):
        sha = imbalance_ratio(rank_loads(_plan(budgets, tp, "sha"), budgets, 8))
        aha = imbalance_ratio(rank_loads(_plan(budgets, tp, mode), budgets, 8))
        assert aha < sha


# ------------------------------------------------------ gloo exchange ----
def _rank_main(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        G, hkv, bt, L = 4, 8, 3, 2
        hq = G * hkv
        budgets = synthetic_budgets(L, bt, hkv, 128, seed=11)
        plan = _plan(budgets, world, "dp")
        shards, finals = plan_layouts(plan, budgets, G)
        rng = np.random.default_rng(5)  # identical data on every rank
        K = [[[rng.standard_normal((int(budgets[l, b, h]), 128)) for h in range(hkv)] for b in range(bt)]
             for l in range(L)]
        V = [[[rng.standard_normal(k.shape) for k in row] for row in lay] for lay in K]
        q = rng.standard_normal((L, bt, hq, 128))
        max_err = 0.0
        for l in range(L):
            sh, f = shards[l][rank], finals[l]
            send = torch.zeros((f.slots, G, REC), dtype=torch.float64)
            for s in range(sh.n_segments):
                b, h, lo, hi = (int(x[s]) for x in (sh.seg_b, sh.seg_h, sh.seg_lo, sh.seg_hi))
                o, lse = okv.attend(q[l, b, h * G:(h + 1) * G], K[l][b][h][lo:hi], V[l][b][h][lo:hi])
                send[s, :, :128] = torch.from_numpy(o)
                send[s, :, 128] = torch.from_numpy(lse)
            recv = [torch.zeros_like(send) for _ in range(world)]
            dist.all_gather(recv, send)
            recv = torch.cat(recv).numpy()
            out = np.zeros((bt * hq, 128))
            for grp in range(len(f.out_row)):
                src = f.src_idx[f.grp_ptr[grp]:f.grp_ptr[grp + 1]]
                o, _ = okv.lse_merge([recv[i, :, :128] for i in src], [recv[i, :, 128] for i in src])
                out[f.out_row[grp]:f.out_row[grp] + G] = o
            ref, _ = okv.decode_heads(q[l], [K[l][b][h] for b in range(bt) for h in range(hkv)],
                                      [V[l][b][h] for b in range(bt) for h in range(hkv)], G)
            max_err = max(max_err, float(np.abs(out.reshape(bt, hq, 128) - ref).max()))
        result_q.put((rank, max_err))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_exchange_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, err in res:
        assert err < 1e-10


def test_rank_cache_tables_for_exchange():
    """Host tables of a rank's caches (built on CPU tensors here): slot i's
    record rows are i*G .. i*G+G-1 and the final merge sources address
    rank*slots + slot -- the layout both exchanges (NCCL / P2P) rely on."""
    from paper_2502_15804_b200.decoder import rank_caches
    G, hkv, bt = 8, 8, 3
    budgets = synthetic_budgets(2, bt, hkv, 128, seed=4)
    plan = _plan(budgets, 4, "dp")
    shards, finals = plan_layouts(plan, budgets, G)
    for r in range(4):
        caches = rank_caches([s[r] for s in shards], bt, G * hkv, G, 4, "cpu", fill="zeros")
        for l, c in enumerate(caches):
            n = c.n_segments
            assert c.host["seg_out_row"].tolist() == [i * G for i in range(n)]
            assert n <= finals[l].slots
    f = finals[0]
    assert f.src_idx.max() < 4 * f.slots
