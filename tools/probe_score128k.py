"""One K1 launch at the cfg5 shape (70B heads, 128k context) for ncu."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2502_15804_b200 import ops
dev = torch.device('cuda')
q = torch.randn((1, 64, 32, 128), device=dev).to(torch.bfloat16)
k = torch.randn((1, 8, 131072, 128), device=dev).to(torch.bfloat16)
for _ in range(3):
    ops.score(q, k)
torch.cuda.synchronize()
