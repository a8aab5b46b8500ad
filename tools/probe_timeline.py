"""Per-CTA timeline of one K4 launch (probe 3 stamps): TP8 SHA shard of the
bench workload and the TP1 layer.  Prints percentiles of each phase (us from
the earliest CTA entry)."""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2502_15804_b200 import ops, _native
from paper_2502_15804_b200.cache import LayerCache
from paper_2502_15804_b200.decoder import rank_caches
from paper_2502_15804_b200.sharding import plan_layouts, synthetic_budgets
import bench
dev = torch.device('cuda:0')
L, bt, HQ, G = 2, 64, 64, 8
budgets = synthetic_budgets(L, bt, 8, 1024, window=32, alpha=0.2, seed=0, context=32768)
qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
base = [LayerCache.allocate(budgets.reshape(L, -1)[l], qrow, qrow, G, dev, fill="random") for l in range(L)]
q = torch.randn((bt, HQ, 128), device=dev).to(torch.bfloat16)
o = torch.empty_like(q)
names = ["entry", "pdl-wait", "first-data", "rounds-done(last piece)", "combine-start", "exit", "pre-atomic", "post-atomic", "merge:lse-loaded", "merge:weights", "merge:records-loaded", "merge:stored"]
for tp in (1, 8):
    plan, prof = bench.make_plan(budgets, tp, "sha")
    shards, _ = plan_layouts(plan, budgets, G)
    cache = rank_caches([s[0] for s in shards], bt, HQ, G, tp, dev, base=base)[0]
    ws = ops.DecodeWorkspace(cache)
    send = ops.xrec_empty(max(cache.n_segments, 1), G, dev)[0]
    for _ in range(3):
        ops.decode_into(q, cache, ws, out_rec=send)
    torch.cuda.synchronize()
    import ctypes
    _native.lib.fkv__decode_probe(3)
    ops.decode_into(q, cache, ws, out_rec=send)
    torch.cuda.synchronize()
    n = cache.n_workers
    buf = (C.c_ulonglong * (n * 16))()
    _native.lib.fkv__decode_stamps(buf, n * 16)
    st = np.array(buf, dtype=np.float64).reshape(n, 16)[:, :12]
    sm0 = st[:, 0].copy()
    st[st == 0] = np.nan
    st[:, 0] = sm0
    smid = st[:, 0].copy()
    t0 = np.nanmin(st[:, 1])
    st = (st - t0) / 1e3
    st[:, 0] = smid
    done = st[:, 3]
    print("   rounds-done by CTA id (16 buckets):", np.round([np.nanmean(x) for x in np.array_split(done, 16)], 1).tolist())
    wk = cache.work.cpu().numpy()
    npieces = (wk[:, :, 7] > 0).sum(1)
    nsplit = ((wk[:, :, 7] > 1)).sum(1)
    for k in sorted(set(npieces.tolist())):
        sel = npieces == k
        print(f"   CTAs with {k} pieces: n={sel.sum():3d} mean done {np.nanmean(done[sel]):6.2f} exit {np.nanmean(st[sel,5]):6.2f}  "
              + " ".join(f"{names[i]}={np.nanmean(st[sel, i]):.2f}" for i in (1, 2, 4, 6, 7, 8, 9, 10, 11) if i < st.shape[1]))
    for k in sorted(set(nsplit.tolist())):
        sel = nsplit == k
        print(f"   CTAs with {k} split pieces: n={sel.sum():3d} mean done {np.nanmean(done[sel]):6.2f} exit {np.nanmean(st[sel,5]):6.2f}")
    order = np.argsort(smid)
    print("   rounds-done by SM id (16 buckets):", np.round([np.nanmean(x) for x in np.array_split(done[order], 16)], 1).tolist())
    cnt = np.bincount(smid.astype(int), minlength=148)
    pair = {}
    for c in range(n):
        pair.setdefault(int(smid[c]), []).append(done[c])
    solo = [v[0] for v in pair.values() if len(v) == 1]
    print("   CTAs per SM histogram:", np.bincount(cnt).tolist(), " solo-CTA mean done:", np.round(np.mean(solo), 1) if solo else None)
    print(f"tp{tp}: workers {n}, pieces {cache.n_items}, kv {cache.kv_bytes()/1e6:.1f} MB, span {np.nanmax(st[:,5]):.2f} us")
    for i, nm in enumerate(names):
        x = st[:, i][~np.isnan(st[:, i])]
        if len(x): print(f"   {nm:26s} n={len(x):4d} p0 {np.percentile(x,0):6.2f}  p50 {np.percentile(x,50):6.2f}  p90 {np.percentile(x,90):6.2f}  max {x.max():6.2f}")
    late = np.argsort(-st[:, 5])[:5]
    for c in late:
        print("   late CTA", c, np.round(st[c], 2).tolist())
    # per-CTA cost model: exit time vs (tiles, pieces, split pieces); per-SM totals
    tiles = ((np.maximum(wk[:, :, 2], 0) + 15) // 16).sum(1)
    A = np.stack([tiles, npieces, nsplit, np.ones(n)], 1).astype(float)
    ex = st[:, 5]
    ok = ~np.isnan(ex)
    coef, *_ = np.linalg.lstsq(A[ok], ex[ok], rcond=None)
    print(f"   exit ~ {coef[0]*1e3:.1f} ns/tile + {coef[1]:.2f} us/piece + {coef[2]:.2f} us/split + {coef[3]:.2f}"
          f"  (resid rms {np.sqrt(np.mean((A[ok] @ coef - ex[ok])**2)):.2f} us)")
    sm_t = {}
    for c in range(n):
        sm_t.setdefault(int(smid[c]), []).append((tiles[c], ex[c]))
    tot = np.array([sum(t for t, _ in v) for v in sm_t.values()])
    last = np.array([max(e for _, e in v) for v in sm_t.values()])
    print(f"   per-SM tiles min/mean/max {tot.min()}/{tot.mean():.1f}/{tot.max()}  per-SM last exit p0/p50/max "
          f"{np.percentile(last,0):.1f}/{np.percentile(last,50):.1f}/{last.max():.1f}")
    print(f"   corr(per-SM tiles, last exit) = {np.corrcoef(tot, last)[0,1]:.2f}")
    if n > 148:
        same = np.mean([smid[i] == smid[i + 148] for i in range(n - 148)])
        print(f"   CTA i and i+148 on the same SM: {same:.2f};  smid[:8] {smid[:8].astype(int).tolist()} smid[148:156] {smid[148:156].astype(int).tolist()}")
