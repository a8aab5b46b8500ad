"""Full decode layer with its weight GEMMs (decoder.DecodeLayer)
against a float64 reference: x -> QKV projection -> append the new K/V ->
attention over the cache + the new token -> o_proj, per rank of an AHA /
uniform-TP placement (tp virtual ranks on one GPU, the fused exchange in
loopback), two layers (layer 1's input = the all-gathered layer-0 output)
over two decode steps.  The reference rounds q/k/v and o to bf16 where the
GPU stores them in bf16 (cuBLAS bf16 GEMMs); tolerance = the bf16 output
tolerance of the decode tests (rtol 2e-2, atol 1e-2 at O(1) magnitudes)."""

import numpy as np
import pytest
import torch

from oracle import kv as okv

pytestmark = pytest.mark.gpu


def _bf(x):
    return torch.as_tensor(x).to(torch.bfloat16).double()


@pytest.mark.parametrize("tp,mode", [(1, "sha"), (2, "sha"), (2, "dp"), (4, "dp")])
def test_decode_layer_matches_reference(cuda_device, tp, mode):
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200.cache import LayerCache
    from paper_2502_15804_b200.decoder import DecodeLayer, rank_caches
    from paper_2502_15804_b200.exchange import P2PGroup, exchange_buffer
    from paper_2502_15804_b200.sharding import budgets_profile, plan_layouts, synthetic_budgets
    dev = cuda_device
    G, hkv, bt, L, B, d = 4, 8, 2, 2, 128, 128
    hq = G * hkv
    hidden = hq * d
    budgets = synthetic_budgets(L, bt, hkv, B, seed=tp)
    prof = budgets_profile(budgets, B)
    plan = fk.sha_plan(prof, tp) if mode == "sha" else \
        fk.optimize_plan(prof, tp, fk.EnumerationConfig(4, 2, True, tp), equal_split=True)
    shards, finals = plan_layouts(plan, budgets, G)
    qrow = np.array([b * hq + h * G for b in range(bt) for h in range(hkv)])
    gen = torch.Generator(device=dev).manual_seed(7)
    base = [LayerCache.allocate(budgets[l].reshape(-1), qrow, qrow, G, dev, fill="random", generator=gen,
                                reserve=4) for l in range(L)]
    caches = [rank_caches([s[r] for s in shards], bt, hq, G, tp, dev, base=base) for r in range(tp)]
    g = torch.Generator().manual_seed(3)
    w_qkv = [(torch.randn(hidden, (hq + 2 * hkv) * d, generator=g) / hidden ** 0.5).to(torch.bfloat16)
             for _ in range(L)]
    w_o = [(torch.randn(hidden, hidden, generator=g) / hidden ** 0.5).to(torch.bfloat16) for _ in range(L)]
    grp = P2PGroup.loopback(tp, max(f.slots for f in finals), G) if tp > 1 else None
    layers = [[DecodeLayer(w_qkv[l].to(dev), w_o[l].to(dev), caches[r][l], shards[l][r], finals[l], tp=tp,
                           rank=r, bt=bt, hq=hq, group=G, endpoint=grp.endpoints[r] if grp else None,
                           buf=exchange_buffer(l, L)) for r in range(tp)] for l in range(L)]
    lens = [budgets[l].reshape(-1).astype(np.int64).copy() for l in range(L)]
    for step in range(2):
        x = (torch.randn(bt, hidden, generator=g)).to(torch.bfloat16).to(dev)
        for l in range(L):
            for r in range(tp):
                layers[l][r].produce(x)
            y = torch.cat([layers[l][r].consume().clone() for r in range(tp)], dim=1)
            torch.cuda.synchronize()
            # ---- reference: bf16 q/k/v from the float64 projection, attention in
            # float64 over the stored cache rows + the new token, o rounded to bf16
            qkv = _bf(x.cpu().double() @ w_qkv[l].double())
            q = qkv[:, :hq * d].reshape(bt, hq, d)
            lens[l] += 1
            kc = base[l].k.cpu().view(torch.int16).numpy()
            vc = base[l].v.cpu().view(torch.int16).numpy()
            row0 = base[l].host["seg_row0"]
            as_f = lambda a: torch.from_numpy(a.copy()).view(torch.bfloat16).double().numpy()  # noqa: E731
            ks, vs = [], []
            for bh in range(bt * hkv):
                n = int(lens[l][bh])
                ks.append(as_f(okv.unswizzle_rows(kc[row0[bh]:row0[bh] + n], row0[bh])))
                vs.append(as_f(okv.unswizzle_rows(vc[row0[bh]:row0[bh] + n], row0[bh])))
            # the appended row is the new token's k / v (bf16 GEMM output)
            knew = qkv[:, hq * d:(hq + hkv) * d].reshape(bt * hkv, d).numpy()
            vnew = qkv[:, (hq + hkv) * d:].reshape(bt * hkv, d).numpy()
            for bh in range(bt * hkv):
                np.testing.assert_allclose(ks[bh][-1], knew[bh], rtol=2e-2, atol=2e-2)
                np.testing.assert_allclose(vs[bh][-1], vnew[bh], rtol=2e-2, atol=2e-2)
            o_ref, _ = okv.decode_heads(q.numpy(), ks, vs, G)
            y_ref = _bf(o_ref).reshape(bt, hidden) @ w_o[l].double()
            torch.testing.assert_close(y.cpu().double(), y_ref, rtol=2e-2, atol=1e-2)
            x = y
    if grp:
        grp.close()
