"""One prefill compression of one layer (cfg2-like: Llama-3.1-8B shape, 16k context,
budget 256), for ncu: K1 score (2 tcgen05 passes + pool), A18+K2 ada_select, K3 compact."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2502_15804_b200 import ops
dev = torch.device('cuda:0')
bt, hq, hkv, T, w, B = 1, 32, 8, 16384, 32, 256
q = torch.randn(bt, hq, w, 128, device=dev).to(torch.bfloat16)
k = torch.randn(bt, hkv, T, 128, device=dev).to(torch.bfloat16)
v = torch.randn(bt, hkv, T, 128, device=dev).to(torch.bfloat16)
cache, hb, sc = ops.compress_layer(q, k, v, B, w)
torch.cuda.synchronize()
print("prefill ok", hb.sum().item())
