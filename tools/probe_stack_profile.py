"""cProfile of ops.compress_stack's host side (L layers, 8B 16k batch 1):
where the host time per layer goes.  usage: python tools/probe_stack_profile.py [layers]"""
import cProfile
import pstats
import sys
sys.path.insert(0, '.')
import torch
from paper_2502_15804_b200 import ops

dev = torch.device("cuda:0")
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
g = torch.Generator(device=dev).manual_seed(0)
q = (torch.randn((1, 32, 32, 128), generator=g, device=dev) * 2).to(torch.bfloat16)
k = torch.randn((1, 8, 16384, 128), generator=g, device=dev).to(torch.bfloat16)
v = torch.randn((1, 8, 16384, 128), generator=g, device=dev).to(torch.bfloat16)
for _ in range(3):
    ops.compress_stack([q] * L, [k] * L, [v] * L, 256)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
ops.compress_stack([q] * L, [k] * L, [v] * L, 256)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
