"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck).

One invocation exercises one kernel family at shapes the sanitizer finishes
in seconds; ``tools/sanitize.sh`` runs every part under every tool and writes
the summaries to ``gpurun_out/sanitize/``.  Each part also checks its result
against the float64 oracle, so a run that "passes" the sanitizer with wrong
numbers is caught too.

  python tools/sanitize_run.py {score_fused,score_multi,score_fused256,score_multi256,select,compact,
                                decode_coop,decode_wide,decode_solo,exchange,append}
"""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import kv as okv  # noqa: E402


def _inputs(bt, hq, hkv, T, seed=0):
    g = torch.Generator().manual_seed(seed)
    q = (torch.randn(bt, hq, 32, 128, generator=g) * 2).to(torch.bfloat16)
    k = torch.randn(bt, hkv, T, 128, generator=g).to(torch.bfloat16)
    v = torch.randn(bt, hkv, T, 128, generator=g).to(torch.bfloat16)
    return q, k, v


def score(bt, hq, hkv, T):
    from paper_2502_15804_b200 import ops
    q, k, _ = _inputs(bt, hq, hkv, T)
    dev = torch.device("cuda:0")
    sc, hb, off, idx = ops.score_select(q.to(dev), k.to(dev), 128)
    torch.cuda.synchronize()
    s = sc.cpu().double().numpy()
    ref = okv.snapkv_scores(q.double().numpy(), k.double().numpy())
    err = float((np.abs(s - ref) / (1e-4 * np.abs(ref) + 1e-6 * np.abs(ref).max(-1, keepdims=True))).max())
    assert err <= 1.0, err
    rb = okv.ada_budgets(s, 128, 32, 0.2)
    assert np.array_equal(hb.cpu().numpy(), rb)
    ro, ri = okv.topk_select(s, rb, 32)
    assert np.array_equal(off.cpu().numpy(), ro) and np.array_equal(idx.cpu().numpy(), ri)
    return f"score_select bt={bt} T={T}: err/tol {err:.3f}, budgets+indices exact"


def select():
    from paper_2502_15804_b200 import ops
    dev = torch.device("cuda:0")
    g = torch.Generator().manual_seed(3)
    s = torch.rand(3, 8, 3000, generator=g)
    hb, off, idx = ops.ada_select(s.to(dev), 256)
    torch.cuda.synchronize()
    sn = s.double().numpy()
    rb = okv.ada_budgets(sn, 256, 32, 0.2)
    ro, ri = okv.topk_select(sn, rb, 32)
    assert np.array_equal(hb.cpu().numpy(), rb)
    assert np.array_equal(off.cpu().numpy(), ro) and np.array_equal(idx.cpu().numpy(), ri)
    return "ada_select 3x8x3000 B=256: exact"


def compress_decode():
    """K1+A18+K2 fused, K3 compact, K4 (schedule from FKV_K4_SCHEDULE) + fused K5."""
    from paper_2502_15804_b200 import ops
    dev = torch.device("cuda:0")
    bt, hq, hkv, T, B = 2, 32, 8, 1024, 128
    G = hq // hkv
    q, k, v = _inputs(bt, hq, hkv, T, seed=5)
    cache, hb, sc = ops.compress_layer(q.to(dev), k.to(dev), v.to(dev), B)
    qd = torch.randn(bt, hq, 128, generator=torch.Generator().manual_seed(6)).to(torch.bfloat16)
    o, lse = ops.decode(qd.to(dev), cache)
    torch.cuda.synchronize()
    s = sc.cpu().double().numpy()
    rb = okv.ada_budgets(s, B, 32, 0.2)
    off, idx = okv.topk_select(s, rb, 32)
    kn, vn = k.double().numpy(), v.double().numpy()
    o_ref = np.empty((bt, hq, 128))
    lse_ref = np.empty((bt, hq))
    for b in range(bt):
        ks = [kn[b, h, idx[off[b * hkv + h]:off[b * hkv + h + 1]]] for h in range(hkv)]
        vs = [vn[b, h, idx[off[b * hkv + h]:off[b * hkv + h + 1]]] for h in range(hkv)]
        o_ref[b], lse_ref[b] = okv.decode_heads(qd[b:b + 1].double().numpy(), ks, vs, G)
    torch.testing.assert_close(o.float().cpu().double(), torch.from_numpy(o_ref), rtol=2e-2, atol=4e-3)
    torch.testing.assert_close(lse.cpu().double(), torch.from_numpy(lse_ref), rtol=1e-4, atol=1e-5)
    return f"compress+decode ({cache.flags=}): o/lse within tolerance"


def decode_sched(schedule):
    """K4 on a synthetic ragged cache: long segments split across CTAs
    (split-segment records + fused merge) and short ones."""
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache
    os.environ["FKV_K4_SCHEDULE"] = schedule
    dev = torch.device("cuda:0")
    G, hkv, bt = 8, 8, 2
    hq = G * hkv
    rng = np.random.default_rng(1)
    seg_len = rng.integers(1, 3000, size=bt * hkv)
    seg_len[0] = 9000
    qrow = np.array([b * hq + h * G for b in range(bt) for h in range(hkv)])
    gen = torch.Generator(device=dev).manual_seed(1)
    cache = LayerCache.allocate(seg_len, qrow, qrow, G, dev, fill="random", generator=gen)
    q = torch.randn(bt, hq, 128, device=dev).to(torch.bfloat16)
    o, lse = ops.decode(q, cache)
    torch.cuda.synchronize()
    kc = cache.k.cpu().view(torch.int16).numpy()
    vc = cache.v.cpu().view(torch.int16).numpy()
    row0 = cache.seg_row0.cpu().numpy()
    as_f = lambda a: torch.from_numpy(a.copy()).view(torch.bfloat16).double().numpy()  # noqa: E731
    o_ref = np.empty((bt, hq, 128))
    lse_ref = np.empty((bt, hq))
    for b in range(bt):
        ks, vs = [], []
        for h in range(hkv):
            s = b * hkv + h
            n = int(seg_len[s])
            ks.append(as_f(okv.unswizzle_rows(kc[row0[s]:row0[s] + n], row0[s])))
            vs.append(as_f(okv.unswizzle_rows(vc[row0[s]:row0[s] + n], row0[s])))
        o_ref[b], lse_ref[b] = okv.decode_heads(q[b:b + 1].double().cpu().numpy(), ks, vs, G)
    torch.testing.assert_close(o.float().cpu().double(), torch.from_numpy(o_ref), rtol=2e-2, atol=4e-3)
    torch.testing.assert_close(lse.cpu().double(), torch.from_numpy(lse_ref), rtol=1e-4, atol=1e-5)
    return f"decode schedule={schedule} flags={cache.flags}: o/lse within tolerance"


def exchange():
    """K4 + fused P2P exchange into loopback endpoints, K5 merge_wait, append."""
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache
    from paper_2502_15804_b200.decoder import rank_caches
    from paper_2502_15804_b200.exchange import P2PGroup, exchange_buffer
    from paper_2502_15804_b200.sharding import budgets_profile, plan_layouts, synthetic_budgets
    dev = torch.device("cuda:0")
    G, hkv, L, bt, B, tp = 8, 8, 3, 2, 256, 4
    hq = G * hkv
    budgets = synthetic_budgets(L, bt, hkv, B, seed=3)
    plan = fk.optimize_plan(budgets_profile(budgets, B), tp, fk.EnumerationConfig(4, 2, True, tp))
    shards, finals = plan_layouts(plan, budgets, G)
    qrow = np.array([b * hq + h * G for b in range(bt) for h in range(hkv)])
    gen = torch.Generator(device=dev).manual_seed(2)
    base = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, G, dev, fill="random",
                                generator=gen, reserve=8) for l in range(L)]
    per_rank = [rank_caches([s[r] for s in shards], bt, hq, G, tp, dev, base=base) for r in range(tp)]
    grp = P2PGroup.loopback(tp, max(f.slots for f in finals), G)
    tabs = [tuple(torch.as_tensor(x, device=dev) for x in (f.grp_ptr, f.src_idx, f.out_row)) for f in finals]
    q = torch.randn(L, bt, hq, 128, device=dev).to(torch.bfloat16)
    out = torch.zeros(tp, L, bt, hq, 128, dtype=torch.bfloat16, device=dev)
    for _ in range(2):
        for l in range(L):
            kn = torch.randn(bt, hkv, 128, device=dev).to(torch.bfloat16)
            vn = torch.randn(bt, hkv, 128, device=dev).to(torch.bfloat16)
            for r in range(tp):
                ops.append(per_rank[r][l], kn, vn)
            ops.append(base[l], kn, vn)
            for r in range(tp):
                ops.decode_exchange(q[l], per_rank[r][l], grp.endpoints[r], exchange_buffer(l, L))
            for r in range(tp):
                ops.merge_wait(grp.endpoints[r], exchange_buffer(l, L), *tabs[l], G, out_bf16=out[r, l])
    torch.cuda.synchronize()
    ref = torch.stack([ops.decode(q[l], base[l])[0] for l in range(L)])
    for r in range(tp):
        torch.testing.assert_close(out[r].float(), ref.float(), rtol=2e-2, atol=4e-3)
    grp.close()
    return f"exchange tp={tp} L={L} x2 steps with append: every rank == TP1 decode"


PARTS = {
    "score_fused": lambda: score(1, 32, 8, 2048),
    "score_multi": lambda: score(20, 32, 8, 300),  # 160 heads: several items per CTA, grid-wide select
    "score_fused256": lambda: score(1, 64, 8, 2048),  # G*w = 256 (70B shape)
    "score_multi256": lambda: score(20, 64, 8, 300),
    "select": select,
    "compress_decode": compress_decode,
    "decode_coop": lambda: decode_sched("coop"),
    "decode_wide": lambda: decode_sched("wide"),
    "decode_solo": lambda: decode_sched("solo"),
    "exchange": exchange,
}

if __name__ == "__main__":
    part = sys.argv[1]
    print(f"[{part}] {PARTS[part]()}")
