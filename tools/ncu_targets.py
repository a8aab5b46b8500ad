"""Small drivers for ncu captures (run under ncu by tools/ncu_profile.sh):
  tp8       K4 + fused XLL exchange of the heaviest TP=8 rank (SHA, then
            AHA-DP) of the 70B bench workload, B=1024, batch 64: 4 layers each
  prefill   fused K1+A18+K2 (score_kernel<4,*>) + K3 at the 8B shape (16k,
            B=256) and the 70B shape at 128k (B=1024), batch 1
  select    standalone grid-wide A18+K2 (fkv_ada_select) at 128k, batch 1
usage: python tools/ncu_targets.py {tp8,prefill,select}"""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch

dev = torch.device("cuda:0")


def tp8():
    import bench
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.cache import LayerCache
    from paper_2502_15804_b200.decoder import rank_caches
    from paper_2502_15804_b200.exchange import P2PGroup, exchange_buffer
    from paper_2502_15804_b200.sharding import plan_layouts, synthetic_budgets
    L, bt, HQ, G = 4, 64, 64, 8
    budgets = synthetic_budgets(80, bt, 8, 1024, window=32, alpha=0.2, seed=0, context=32768)[:L]
    qrow = np.array([b * HQ + h * G for b in range(bt) for h in range(8)])
    base = [LayerCache.allocate(budgets.reshape(L, -1)[l], qrow, qrow, G, dev, fill="random") for l in range(L)]
    q = torch.randn((L, bt, HQ, 128), device=dev).to(torch.bfloat16)
    for mode in ("sha", "dp"):
        plan, _ = bench.make_plan(budgets, 8, mode)
        shards, finals = plan_layouts(plan, budgets, G)
        toks = [sum(int((s[g].seg_hi - s[g].seg_lo).sum()) for s in shards) for g in range(8)]
        g = int(np.argmax(toks))
        caches = rank_caches([s[g] for s in shards], bt, HQ, G, 8, dev, base=base)
        grp = P2PGroup.loopback(8, max(f.slots for f in finals), G)
        for l in range(L):
            ops.decode_exchange(q[l], caches[l], grp.endpoints[g], exchange_buffer(l, L))
        torch.cuda.synchronize()
        print(f"tp8 {mode}: rank {g}, {[c.kv_bytes() / 1e6 for c in caches]} MB, flags {caches[0].flags}, "
              f"workers {caches[0].n_workers}, items {caches[0].n_items}")
        grp.close()


def prefill():
    from paper_2502_15804_b200 import ops
    for hq, T, B in ((32, 16384, 256), (64, 131072, 1024)):
        g = torch.Generator().manual_seed(0)
        qw = torch.randn(1, hq, 32, 128, generator=g).to(torch.bfloat16).to(dev)
        k = torch.randn(1, 8, T, 128, generator=g).to(torch.bfloat16).to(dev)
        v = torch.randn(1, 8, T, 128, generator=g).to(torch.bfloat16).to(dev)
        ops.compress_layer(qw, k, v, B)
        torch.cuda.synchronize()
        print(f"prefill hq={hq} T={T} B={B} done")


def select():
    from paper_2502_15804_b200 import ops
    s = torch.rand(1, 8, 131072 - 32, generator=torch.Generator().manual_seed(0)).to(dev)
    for _ in range(2):
        ops.ada_select(s, 1024)
    torch.cuda.synchronize()
    print("select done")


if __name__ == "__main__":
    {"tp8": tp8, "prefill": prefill, "select": select}[sys.argv[1]]()
