"""Bounded single-GPU check of the fused exchange (loopback), with progress prints."""
import sys, time
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import torch
from test_exchange_gpu import _setup
from paper_2502_15804_b200 import ops
from paper_2502_15804_b200.exchange import P2PGroup
dev = torch.device('cuda:0')
base, per_rank, finals, bt, hq, G = _setup(2, "dp", dev)
grp = P2PGroup.loopback(2, max(f.slots for f in finals), G)
q = torch.randn(len(base), bt, hq, 128, device=dev).to(torch.bfloat16)
o = torch.zeros(bt, hq, 128, dtype=torch.bfloat16, device=dev)
for r in range(2):
    ops.decode_exchange(q[0], per_rank[r][0], grp.endpoints[r], 0)
torch.cuda.synchronize()
fl = [torch.empty(2, dtype=torch.int32) for _ in range(2)]
import ctypes
for r, ep in enumerate(grp.endpoints):
    buf = (ctypes.c_int32 * 4)()
    torch.cuda.synchronize()
    import numpy as np
    t = torch.empty(4, dtype=torch.int32, device=dev)
    print("rank", r, "flags ptr", hex(ep.flags.ptr))
print("decodes done")
f = finals[0]
tabs = [torch.as_tensor(x, device=dev) for x in (f.grp_ptr, f.src_idx, f.out_row)]
ops.merge_wait(grp.endpoints[0], 0, *tabs, G, out_bf16=o)
torch.cuda.synchronize()
print("merge done", float((o.float() - ops.decode(q[0], base[0])[0].float()).abs().max()))
