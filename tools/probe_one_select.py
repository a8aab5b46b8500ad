"""For ncu: the standalone grid-wide Ada split + top-k (grid_select_kernel)
over pooled scores of the cfg5 shape (70B, 128k context, B=1024) and of a
batch-32 8B prefill at 16k (the library's path when K1's grid cannot be
co-resident)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2502_15804_b200 import ops
dev = torch.device('cuda:0')
for bt, hq, T, B in ((1, 64, 131072, 1024), (32, 32, 16384, 256)):
    q = torch.randn(bt, hq, 32, 128, device=dev).to(torch.bfloat16)
    k = torch.randn(bt, 8, T, 128, device=dev).to(torch.bfloat16)
    sc = ops.score(q, k)
    del q, k
    hb, off, idx = ops.ada_select(sc, B, 32)
    torch.cuda.synchronize()
    print("select ok", bt, T, hb.sum().item())
