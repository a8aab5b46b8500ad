"""B3: the compressed-cache decode path as torch-facing ops over the C ABI.

Every op launches hand-written sm_100a kernels from libfairkv.so on the
current torch CUDA stream; nothing here computes on the CPU and there is no
fallback -- a CPU tensor or a missing library is an error.  Kernels never
allocate; these wrappers allocate outputs/workspaces with torch (the caching
allocator) or take caller-provided buffers (``out=`` / ``ws=``) so the whole
decode step can be captured in a CUDA graph.

    score(q_win, k, window, pool_k=7)   -> scores  f32 [Bt,Hkv,T-w]       (K1)
    budgets(scores, budget, window, alpha=0.2) -> int32 [Bt,Hkv]          (A18)
    select(scores, budgets, window)     -> (offsets, idx)                 (K2)
    compact(k, v, offsets, idx, ...)    -> LayerCache                     (K3)
    decode(q, cache)                    -> (o bf16 [Bt,Hq,d], lse f32)    (K4+K5)
    merge_lse(...)                      LSE merge of partials             (K5)
"""

from __future__ import annotations

import math

import torch

from . import _native
from .cache import HEAD_DIM, LayerCache
from .errors import NativeError

_lib = _native.lib


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise NativeError("fairkv ops run on CUDA tensors only (no CPU path)")


def _p(t):
    return None if t is None else t.data_ptr()


# -------------------------------------------------------------- decode ----
class DecodeWorkspace:
    """Persistent partial-output buffers for one cache (graph-capturable)."""

    def __init__(self, cache: LayerCache):
        dev = cache.k.device
        self.part_o = torch.empty((max(cache.n_items, 1), cache.group, HEAD_DIM), dtype=torch.float32,
                                  device=dev)
        self.part_lse = torch.empty((max(cache.n_items, 1), cache.group), dtype=torch.float32, device=dev)


def decode_partial(q: torch.Tensor, cache: LayerCache, ws: DecodeWorkspace | None = None,
                   sm_scale: float | None = None):
    """K4: per work item (o, lse) partials.  q: bf16 [..., 128] contiguous."""
    _need_cuda(q, cache.k)
    if q.dtype != torch.bfloat16 or q.shape[-1] != HEAD_DIM or not q.is_contiguous():
        raise NativeError("q must be contiguous bf16 [..., 128]")
    ws = ws or DecodeWorkspace(cache)
    scale = 1.0 / math.sqrt(HEAD_DIM) if sm_scale is None else sm_scale
    _native.check(_lib.fkv_decode_partial(
        q.data_ptr(), cache.k.data_ptr(), cache.v.data_ptr(), cache.seg_row0.data_ptr(),
        cache.seg_len.data_ptr(), cache.seg_qrow.data_ptr(), cache.item_seg.data_ptr(),
        cache.item_t0.data_ptr(), cache.item_t1.data_ptr(), cache.n_items, cache.group, scale,
        ws.part_o.data_ptr(), ws.part_lse.data_ptr(), _stream()))
    return ws.part_o, ws.part_lse


def merge_lse(part_o, part_lse, grp_ptr, src_idx, out_row, group: int, *, out_bf16=None,
              out_f32=None, out_lse=None):
    """K5: out rows out_row[g]..+group-1 <- LSE merge of partial rows
    src_idx[grp_ptr[g]:grp_ptr[g+1]]."""
    _need_cuda(part_o, part_lse, grp_ptr, src_idx, out_row)
    n_groups = int(out_row.shape[0])
    _native.check(_lib.fkv_merge_lse(
        part_o.data_ptr(), part_lse.data_ptr(), grp_ptr.data_ptr(), src_idx.data_ptr(),
        out_row.data_ptr(), n_groups, int(group), _p(out_bf16), _p(out_f32), _p(out_lse),
        _stream()))


def decode(q: torch.Tensor, cache: LayerCache, *, out: torch.Tensor | None = None,
           out_lse: torch.Tensor | None = None, ws: DecodeWorkspace | None = None):
    """Decode attention of one layer over a single-GPU cache.

    q [Bt, Hq, 128] bf16 -> o [Bt, Hq, 128] bf16 and lse [Bt, Hq] f32
    (rows not covered by any segment are left untouched)."""
    ws = ws or DecodeWorkspace(cache)
    if out is None:
        out = torch.empty_like(q)
    if out_lse is None:
        out_lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=q.device)
    part_o, part_lse = decode_partial(q, cache, ws)
    merge_lse(part_o, part_lse, cache.grp_ptr, cache.src_idx, cache.seg_out_row, cache.group,
              out_bf16=out, out_lse=out_lse)
    return out, out_lse
