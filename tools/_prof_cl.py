import sys, cProfile, pstats
sys.path.insert(0, '.')
import torch
from paper_2502_15804_b200 import ops
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
q = (torch.randn((1, 64, 32, 128), generator=g, device=dev) * 2).to(torch.bfloat16)
k = torch.randn((1, 8, 32768, 128), generator=g, device=dev).to(torch.bfloat16)
v = torch.randn((1, 8, 32768, 128), generator=g, device=dev).to(torch.bfloat16)
for _ in range(3):
    ops.compress_layer(q, k, v, 1024)
torch.cuda.synchronize()
cProfile.run('for _ in range(20): ops.compress_layer(q, k, v, 1024)\ntorch.cuda.synchronize()', '/tmp/cl.out')
pstats.Stats('/tmp/cl.out').sort_stats('tottime').print_stats(25)
