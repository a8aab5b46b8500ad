"""B3: the compressed-cache decode path as torch-facing ops over the C ABI.

Every op launches hand-written sm_100a kernels from libfairkv.so on the
current torch CUDA stream; nothing here computes on the CPU and there is no
fallback -- a CPU tensor or a missing library is an error.  Kernels never
allocate; these wrappers allocate outputs/workspaces with torch (the caching
allocator) or take caller-provided buffers (``out=`` / ``ws=``) so the whole
decode step can be captured in a CUDA graph.

    score(q_win, k, window, pool_k=7)   -> scores  f32 [Bt,Hkv,T-w]       (K1)
    score_select(q_win, k, budget, ...) -> scores, budgets, offsets, idx  (K1+A18+K2, one launch)
    budgets(scores, budget, window, alpha=0.2) -> int32 [Bt,Hkv]          (A18)
    select(scores, budgets, window)     -> (offsets, idx)                 (K2)
    compact(k, v, offsets, idx, ...)    -> LayerCache                     (K3)
    decode(q, cache)                    -> (o bf16 [Bt,Hq,d], lse f32)    (K4+K5)
    merge_lse(...)                      LSE merge of partials             (K5)
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _native
from .cache import HEAD_DIM, LayerCache, to_device_async
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
REC = 132  # floats per partial record of a split segment (FKV_REC): o[128], lse, pad
XREC_ROW = HEAD_DIM * 2 + 4  # bytes per head of an exchange record: bf16 o[128] + f32 lse
XLL_ROW = 528  # FKV_XLL_ROW_BYTES: the same head row in the fused exchange's LL format


def xrec_bytes(slots: int, group: int) -> int:
    """FKV_XREC_BYTES: one block of exchange records (``slots`` segments of
    ``group`` heads): bf16 o [slots*group, 128] then f32 lse [slots*group]."""
    return int(slots) * int(group) * XREC_ROW


def xrec_empty(slots: int, group: int, device, ranks: int = 1) -> torch.Tensor:
    """uint8 [ranks, xrec_bytes]: a send block (ranks=1) or a receive area."""
    return torch.zeros((ranks, xrec_bytes(slots, group)), dtype=torch.uint8, device=device)


def xrec_view(buf: torch.Tensor, group: int):
    """(o bf16 [ranks, slots*group, 128], lse f32 [ranks, slots*group]) views
    of exchange-record blocks ``buf`` (uint8 [ranks, block])."""
    buf = buf.reshape(-1, buf.shape[-1])
    n = buf.shape[-1] // XREC_ROW  # rows = slots * group
    o = buf[:, :n * HEAD_DIM * 2].view(torch.bfloat16).view(-1, n, HEAD_DIM)
    lse = buf[:, n * HEAD_DIM * 2:].view(torch.float32)
    return o, lse


def _xrec_slots(buf: torch.Tensor, group: int) -> int:
    row = group * XREC_ROW
    if buf.dtype != torch.uint8 or buf.shape[-1] % row:
        raise NativeError(f"exchange records must be uint8 [..., slots * {row}]")
    return buf.shape[-1] // row


class DecodeWorkspace:
    """Persistent partial-record buffer for one cache (graph-capturable)."""

    def __init__(self, cache: LayerCache):
        self.part = torch.empty((max(cache.n_items, 1), cache.group, REC), dtype=torch.float32,
                                device=cache.k.device)


def _decode(q, cache: LayerCache, ws: DecodeWorkspace | None, sm_scale, out_bf16, out_rec, out_lse):
    _need_cuda(q, cache.k)
    if q.dtype != torch.bfloat16 or q.shape[-1] != HEAD_DIM or not q.is_contiguous():
        raise NativeError("q must be contiguous bf16 [..., 128]")
    ws = ws or DecodeWorkspace(cache)
    scale = 1.0 / math.sqrt(HEAD_DIM) if sm_scale is None else sm_scale
    slots = _xrec_slots(out_rec, cache.group) if out_rec is not None else 0
    _native.check(_lib.fkv_decode(
        q.data_ptr(), cache.k.data_ptr(), cache.v.data_ptr(), cache.work.data_ptr(), cache.work_k,
        cache.n_workers, cache.n_items, cache.group, cache.launch_flags, scale, ws.part.data_ptr(),
        cache.counters.data_ptr(), _p(out_bf16), _p(out_rec), slots, _p(out_lse), _stream()))
    return ws.part


def decode_partial(q: torch.Tensor, cache: LayerCache, ws: DecodeWorkspace | None = None,
                   sm_scale: float | None = None) -> torch.Tensor:
    """K4 alone: one (o, lse) record per (work item, head), no merge."""
    return _decode(q, cache, ws, sm_scale, None, None, None)


def decode_into(q: torch.Tensor, cache: LayerCache, ws: DecodeWorkspace | None = None, *,
                out_bf16=None, out_rec=None, out_lse=None, sm_scale: float | None = None):
    """K4 with the fused per-segment LSE merge: segment s writes rows
    seg_out_row[s] .. + G - 1 of the given outputs (one launch): ``out_bf16``
    bf16 [*, 128], ``out_lse`` f32 [*], ``out_rec`` one exchange-record block
    (``xrec_empty(slots, G, dev)``; the NCCL all-gather's send buffer)."""
    if out_bf16 is None and out_rec is None and out_lse is None:
        raise NativeError("decode_into needs at least one output")
    _decode(q, cache, ws, sm_scale, out_bf16, out_rec, out_lse)


def decode_exchange(q: torch.Tensor, cache: LayerCache, endpoint, parity: int,
                    ws: DecodeWorkspace | None = None, sm_scale: float | None = None):
    """K4 with the fused NVLink all-gather: every segment's final record goes
    to this rank's block of every peer's receive area ``parity`` as XLL units
    tagged with this layer's exchange epoch (16-byte P2P stores; no fence, no
    completion flag -- ``exchange.RankEndpoint``)."""
    import ctypes as C
    _need_cuda(q, cache.k)
    if q.dtype != torch.bfloat16 or q.shape[-1] != HEAD_DIM or not q.is_contiguous():
        raise NativeError("q must be contiguous bf16 [..., 128]")
    ws = ws or DecodeWorkspace(cache)
    scale = 1.0 / math.sqrt(HEAD_DIM) if sm_scale is None else sm_scale
    dests = endpoint.dest_records(parity)
    recs = (C.c_void_p * len(dests))(*dests)
    _native.check(_lib.fkv_decode_exchange(
        q.data_ptr(), cache.k.data_ptr(), cache.v.data_ptr(), cache.work.data_ptr(), cache.work_k,
        cache.n_workers, cache.n_items, cache.group, cache.launch_flags, scale, ws.part.data_ptr(),
        cache.counters.data_ptr(), None, recs, len(dests), endpoint.slots, None, endpoint.epoch,
        _stream()))


def merge_wait(endpoint, parity: int, grp_ptr, src_idx, out_row, group: int, *, out_bf16=None,
               out_lse=None):
    """K5 after the fused all-gather: every warp polls its records in
    receive area ``parity`` until they carry this layer's epoch, merges the
    DP copies of each head by LSE, and the last CTA advances the epoch."""
    _need_cuda(grp_ptr, src_idx, out_row)
    n_groups = int(out_row.shape[0])
    _native.check(_lib.fkv_merge_wait(
        endpoint.recv[parity].ptr, endpoint.slots, grp_ptr.data_ptr(), src_idx.data_ptr(),
        out_row.data_ptr(), n_groups, int(group), _p(out_bf16), _p(out_lse), endpoint.epoch,
        _stream()))


def merge_lse(xrec, grp_ptr, src_idx, out_row, group: int, *, out_bf16=None, out_lse=None):
    """K5: rows out_row[g] .. +group-1 <- LSE merge of the exchange records
    src_idx[grp_ptr[g]:grp_ptr[g+1]] of ``xrec`` (uint8 [ranks, block]; record
    i = rank * slots + slot)."""
    _need_cuda(xrec, grp_ptr, src_idx, out_row)
    if out_bf16 is None and out_lse is None:
        raise NativeError("merge_lse needs at least one output")
    n_groups = int(out_row.shape[0])
    _native.check(_lib.fkv_merge_lse(
        xrec.data_ptr(), _xrec_slots(xrec, group), grp_ptr.data_ptr(), src_idx.data_ptr(),
        out_row.data_ptr(), n_groups, int(group), _p(out_bf16), _p(out_lse), _stream()))


def decode(q: torch.Tensor, cache: LayerCache, *, out: torch.Tensor | None = None,
           out_lse: torch.Tensor | None = None, ws: DecodeWorkspace | None = None):
    """Decode attention of one layer over a single-GPU cache (one launch).

    q [Bt, Hq, 128] bf16 -> o [Bt, Hq, 128] bf16 and lse [Bt, Hq] f32
    (rows not covered by any segment are left untouched)."""
    if out is None:
        out = torch.empty_like(q)
    if out_lse is None:
        out_lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=q.device)
    decode_into(q, cache, ws, out_bf16=out, out_lse=out_lse)
    return out, out_lse


def append(cache: LayerCache, k_new: torch.Tensor, v_new: torch.Tensor):
    """Decode-time append of one token per (request, KV head): segment s takes
    row ``append_src[s]`` of k_new / v_new (bf16 [Bt, Hkv, 128]) into its
    reserved headroom; the work table's last piece grows on the device, so
    the next ``decode`` includes it.  Segments at capacity are skipped and
    counted in ``cache.host['overflow_t']`` (re-lay the cache out then)."""
    _need_cuda(k_new, v_new, cache.k)
    if k_new.dtype != torch.bfloat16 or k_new.shape != v_new.shape or k_new.shape[-1] != HEAD_DIM \
            or not (k_new.is_contiguous() and v_new.is_contiguous()):
        raise NativeError("k_new / v_new must be contiguous bf16 [..., 128] of one shape")
    h = cache.host
    h["written"] = True
    _native.check(_lib.fkv_append(k_new.data_ptr(), v_new.data_ptr(), cache.append_src_t.data_ptr(),
                                  cache.seg_row0.data_ptr(), cache.seg_len.data_ptr(),
                                  cache.seg_cap_t.data_ptr(), cache.work.data_ptr(),
                                  cache.last_piece_t.data_ptr(), cache.n_segments,
                                  cache.overflow_t.data_ptr(), cache.k.data_ptr(), cache.v.data_ptr(),
                                  _stream()))


# ------------------------------------------------- compression (prefill) ----
def score(q_win: torch.Tensor, k: torch.Tensor, window: int | None = None, pool_k: int = 7,
          sm_scale: float | None = None, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """K1: Ada-SnapKV observation-window scores (tcgen05 two-pass kernel).

    q_win bf16 [Bt, Hq, w, 128] (the last w query positions), k bf16
    [Bt, Hkv, T, 128] -> pooled scores f32 [Bt, Hkv, T - w]; G*w must be 128
    or 256 (Llama-3.1-8B: G=4, 70B: G=8, with w=32)."""
    _need_cuda(q_win, k)
    if q_win.dtype != torch.bfloat16 or k.dtype != torch.bfloat16 or q_win.shape[-1] != HEAD_DIM \
            or k.shape[-1] != HEAD_DIM or not (q_win.is_contiguous() and k.is_contiguous()):
        raise NativeError("q_win / k must be contiguous bf16 [..., 128]")
    bt, hq, w, _ = q_win.shape
    _, hkv, T, _ = k.shape
    if window is not None and window != w:
        raise NativeError(f"window {window} != q_win.shape[2] {w}")
    scale = 1.0 / math.sqrt(HEAD_DIM) if sm_scale is None else sm_scale
    out = torch.empty((bt, hkv, T - w), dtype=torch.float32, device=k.device)
    need = int(_lib.fkv_score_workspace_bytes(bt, hkv, T, w, hq // hkv))
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=k.device)
    _native.check(_lib.fkv_snapkv_score(q_win.data_ptr(), k.data_ptr(), bt, hq, hkv, T, w,
                                        int(pool_k), scale, out.data_ptr(), workspace.data_ptr(),
                                        _stream()))
    return out


def score_select(q_win: torch.Tensor, k: torch.Tensor, budget: int, window: int | None = None,
                 alpha: float = 0.2, pool_k: int = 7, sm_scale: float | None = None,
                 workspace: torch.Tensor | None = None):
    """K1 + A18 + K2 in one cooperative launch: Ada-SnapKV scores, the Ada
    budget split and the per-head top-k (tcgen05 scoring, grid-wide radix
    select).  -> (scores f32 [Bt,Hkv,T-w], budgets int32 [Bt,Hkv], offsets
    int64 [Bt*Hkv+1], idx int32 [Bt*Hkv*budget]); identical to ``score``
    followed by ``ada_select``.  Shapes whose grid cannot be co-resident fall
    back to those two launches inside the library."""
    _need_cuda(q_win, k)
    if q_win.dtype != torch.bfloat16 or k.dtype != torch.bfloat16 or q_win.shape[-1] != HEAD_DIM \
            or k.shape[-1] != HEAD_DIM or not (q_win.is_contiguous() and k.is_contiguous()):
        raise NativeError("q_win / k must be contiguous bf16 [..., 128]")
    bt, hq, w, _ = q_win.shape
    _, hkv, T, _ = k.shape
    if window is not None and window != w:
        raise NativeError(f"window {window} != q_win.shape[2] {w}")
    scale = 1.0 / math.sqrt(HEAD_DIM) if sm_scale is None else sm_scale
    dev = k.device
    sc = torch.empty((bt, hkv, T - w), dtype=torch.float32, device=dev)
    hb = torch.empty((bt, hkv), dtype=torch.int32, device=dev)
    offsets = torch.empty(bt * hkv + 1, dtype=torch.int64, device=dev)
    idx = torch.empty(max(bt * hkv * budget, 1), dtype=torch.int32, device=dev)
    need = int(_lib.fkv_score_workspace_bytes(bt, hkv, T, w, hq // hkv))
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    _native.check(_lib.fkv_snapkv_select(q_win.data_ptr(), k.data_ptr(), bt, hq, hkv, T, w, int(pool_k),
                                         scale, int(budget), ada_floor(budget, w, alpha), sc.data_ptr(),
                                         hb.data_ptr(), offsets.data_ptr(), idx.data_ptr(),
                                         workspace.data_ptr(), _stream()))
    return sc, hb, offsets, idx[:bt * hkv * budget]


def ada_floor(budget: int, window: int, alpha: float) -> int:
    """Per-head Ada safeguard floor floor(alpha * (B - w))."""
    return int(math.floor(alpha * (budget - window)))


def _select_workspace(bt: int, hkv: int, n: int, dev, workspace: torch.Tensor | None) -> torch.Tensor:
    need = int(_lib.fkv_ada_select_workspace_bytes(bt, hkv, n))
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    return workspace


def budgets(scores: torch.Tensor, budget: int, window: int = 32, alpha: float = 0.2,
            workspace: torch.Tensor | None = None) -> torch.Tensor:
    """A18: Ada cross-head split of Hkv*budget retained tokens per request.

    scores f32 [Bt, Hkv, T-w] (pooled Ada-SnapKV scores) -> int32 [Bt, Hkv],
    every row summing to Hkv*budget, every head >= window + floor."""
    _need_cuda(scores)
    if scores.dtype != torch.float32 or scores.dim() != 3 or not scores.is_contiguous():
        raise NativeError("scores must be contiguous f32 [Bt, Hkv, n]")
    bt, hkv, n = scores.shape
    out = torch.empty((bt, hkv), dtype=torch.int32, device=scores.device)
    ws = _select_workspace(bt, hkv, n, scores.device, workspace)
    _native.check(_lib.fkv_ada_budgets(scores.data_ptr(), bt, hkv, n, int(budget), int(window),
                                       ada_floor(budget, window, alpha), out.data_ptr(), ws.data_ptr(),
                                       _stream()))
    return out


def select(scores: torch.Tensor, head_budgets: torch.Tensor, window: int = 32,
           total: int | None = None, workspace: torch.Tensor | None = None):
    """K2: per-head top-(b_h - w) tokens by (score desc, token asc), ascending,
    then the window tokens.  Returns (offsets int64 [Bt*Hkv+1], idx int32).
    ``total`` = sum of budgets (Hkv*budget*Bt when they come from
    ``budgets``); if omitted it is read back (one device sync)."""
    _need_cuda(scores, head_budgets)
    bt, hkv, n = scores.shape
    if total is None:
        total = int(head_budgets.sum().item())
    offsets = torch.empty(bt * hkv + 1, dtype=torch.int64, device=scores.device)
    idx = torch.empty(max(total, 1), dtype=torch.int32, device=scores.device)
    ws = _select_workspace(bt, hkv, n, scores.device, workspace)
    _native.check(_lib.fkv_topk_select(scores.data_ptr(), head_budgets.data_ptr(), bt, hkv, n,
                                       int(window), offsets.data_ptr(), idx.data_ptr(), ws.data_ptr(),
                                       _stream()))
    return offsets, idx[:total]


def ada_select(scores: torch.Tensor, budget: int, window: int = 32, alpha: float = 0.2,
               workspace: torch.Tensor | None = None):
    """A18 + K2 in one cooperative grid-wide launch: -> (budgets int32
    [Bt, Hkv], offsets int64 [Bt*Hkv+1], idx int32 [Bt*Hkv*budget]);
    identical to ``budgets`` followed by ``select``."""
    _need_cuda(scores)
    if scores.dtype != torch.float32 or scores.dim() != 3 or not scores.is_contiguous():
        raise NativeError("scores must be contiguous f32 [Bt, Hkv, n]")
    bt, hkv, n = scores.shape
    dev = scores.device
    hb = torch.empty((bt, hkv), dtype=torch.int32, device=dev)
    offsets = torch.empty(bt * hkv + 1, dtype=torch.int64, device=dev)
    idx = torch.empty(max(bt * hkv * budget, 1), dtype=torch.int32, device=dev)
    workspace = _select_workspace(bt, hkv, n, dev, workspace)
    _native.check(_lib.fkv_ada_select(scores.data_ptr(), bt, hkv, n, int(budget), int(window),
                                      ada_floor(budget, window, alpha), hb.data_ptr(),
                                      offsets.data_ptr(), idx.data_ptr(), workspace.data_ptr(),
                                      _stream()))
    return hb, offsets, idx[:bt * hkv * budget]


def compact_into(cache: LayerCache, k: torch.Tensor, v: torch.Tensor, offsets: torch.Tensor,
                 idx: torch.Tensor, seg_bh: torch.Tensor, seg_lo: torch.Tensor,
                 seg_hi: torch.Tensor, max_tokens: int):
    """K3 alone into an existing cache (device int32 segment tables; one launch)."""
    _need_cuda(k, v, offsets, idx, seg_bh, seg_lo, seg_hi)
    cache.host["written"] = True
    _native.check(_lib.fkv_compact(k.data_ptr(), v.data_ptr(), k.shape[2], int(seg_bh.shape[0]),
                                   offsets.data_ptr(), idx.data_ptr(), seg_bh.data_ptr(),
                                   seg_lo.data_ptr(), seg_hi.data_ptr(), cache.seg_row0.data_ptr(),
                                   1, int(max_tokens), cache.k.data_ptr(), cache.v.data_ptr(),
                                   _stream()))


def compact(k: torch.Tensor, v: torch.Tensor, offsets: torch.Tensor, idx: torch.Tensor,
            seg_bh, seg_lo, seg_hi, seg_qrow, seg_out_row, group: int,
            chunk: int | None = None) -> LayerCache:
    """K3: gather selected rows of k/v [Bt, Hkv, T, 128] (bf16, contiguous)
    into a fresh page-aligned, swizzled LayerCache.  Segment i takes entries
    [seg_lo[i], seg_hi[i]) of head seg_bh[i]'s selection (host int arrays;
    one segment per head for TP=1, the owned copies for a sharded rank)."""
    import numpy as np
    _need_cuda(k, v, offsets, idx)
    if k.dtype != torch.bfloat16 or k.shape != v.shape or k.shape[-1] != HEAD_DIM \
            or not (k.is_contiguous() and v.is_contiguous()):
        raise NativeError("k/v must be contiguous bf16 [Bt, Hkv, T, 128]")
    seg_lo = np.asarray(seg_lo, dtype=np.int64)
    seg_hi = np.asarray(seg_hi, dtype=np.int64)
    cache = LayerCache.allocate(seg_hi - seg_lo, seg_qrow, seg_out_row, group, k.device, chunk=chunk)
    n = len(seg_lo)
    host = np.empty(3 * n, dtype=np.int32)  # the three segment tables in one host-to-device copy
    host[:n], host[n:2 * n], host[2 * n:] = seg_bh, seg_lo, seg_hi
    dev_tabs = to_device_async(host, k.device)
    tabs = (dev_tabs[:n], dev_tabs[n:2 * n], dev_tabs[2 * n:])
    compact_into(cache, k, v, offsets, idx, *tabs,
                 int((seg_hi - seg_lo).max()) if len(seg_lo) else 0)
    cache.host["compact_args"] = tabs  # keep alive until the stream consumes them
    return cache


def compress_layer(q_win: torch.Tensor, k: torch.Tensor, v: torch.Tensor, budget: int,
                   window: int = 32, alpha: float = 0.2, pool_k: int = 7):
    """Prefill of one layer on one GPU: K1 score + A18 budgets + K2 select
    (one cooperative launch) -> K3 compact (TP=1 layout).  Returns (cache,
    head_budgets, scores).  The host needs the budgets to lay out the ragged
    cache: the launch writes them to pinned host memory (compress_stack of
    one layer); the same result as score_select followed by compact."""
    caches, hbs, scs = compress_stack([q_win], [k], [v], budget, window, alpha, pool_k)
    return caches[0], hbs[0], scs[0]


def compress_stack(q_wins, ks, vs, budget: int, window: int | None = 32, alpha: float = 0.2, pool_k: int = 7):
    """Prefill compression of a whole layer stack on one GPU without
    stalling the stream per layer: every layer's fused K1 + A18 + K2 launch
    is queued first (outputs of all layers in one allocation each, workspace
    reused, stream ordered); each layer's budgets come back on a side stream
    as soon as its launch ends, and the host lays out that layer's ragged
    cache (schedule + tables, fkv_cache_tables) while the GPU scores the
    next ones; then one K/V allocation and one host-to-device copy for the
    whole stack and every layer's K3 compaction (compress_layer is the stack
    of one layer: the host waits for that layer's budgets before laying out
    its cache).  q_wins / ks / vs: one tensor per layer,
    shapes as compress_layer.  Returns ([cache], budgets int32 [L, Bt, Hkv]
    on the device, [scores])."""
    import numpy as np
    if not (len(q_wins) == len(ks) == len(vs)) or not ks:
        raise NativeError("compress_stack needs the same number (>= 1) of q_win, k and v tensors")
    L = len(ks)
    bt, hq, w = q_wins[0].shape[0], q_wins[0].shape[1], q_wins[0].shape[2]
    hkv, T = ks[0].shape[1], ks[0].shape[2]
    group = hq // hkv
    dev = ks[0].device
    if window is not None and window != w:
        raise NativeError(f"window {window} != q_win.shape[2] {w}")
    for q, k, v in zip(q_wins, ks, vs):
        _need_cuda(q, k, v)
        if q.dtype != torch.bfloat16 or k.dtype != torch.bfloat16 or v.dtype != torch.bfloat16 \
                or q.shape != q_wins[0].shape or k.shape != ks[0].shape or v.shape != k.shape \
                or k.shape[-1] != HEAD_DIM or q.shape[-1] != HEAD_DIM \
                or not (q.is_contiguous() and k.is_contiguous() and v.is_contiguous()):
            raise NativeError("compress_stack: every layer's q_win / k / v contiguous bf16 [..., 128], same shapes")
    BH = bt * hkv
    # every layer's outputs in one allocation each; the launches queued back to back
    need = int(_lib.fkv_score_workspace_bytes(bt, hkv, T, w, group))
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    sc = torch.empty((L, bt, hkv, T - w), dtype=torch.float32, device=dev)
    # the budgets are written by the kernels straight into pinned host memory
    # (at its device address, fkv_host_device_ptr), so the host lays out
    # layer l as soon as its launch ends, while the GPU scores the next ones
    hb_pin = torch.empty((L, BH), dtype=torch.int32, pin_memory=True)
    hb_np = hb_pin.numpy()
    offsets = torch.empty((L, BH + 1), dtype=torch.int64, device=dev)
    idx = torch.empty((L, max(BH * budget, 1)), dtype=torch.int32, device=dev)
    scale, floor, stream = 1.0 / math.sqrt(HEAD_DIM), ada_floor(budget, w, alpha), _stream()
    dptr = ctypes.c_void_p()
    _native.check(_lib.fkv_host_device_ptr(hb_pin.data_ptr(), ctypes.byref(dptr)))
    p_sc, p_hb, p_off, p_idx = sc.data_ptr(), dptr.value, offsets.data_ptr(), idx.data_ptr()
    s_sc, s_hb, s_off, s_idx = 4 * sc[0].numel(), 4 * BH, 8 * (BH + 1), 4 * idx.shape[1]
    ready = []
    for l, (q, k) in enumerate(zip(q_wins, ks)):
        _native.check(_lib.fkv_snapkv_select(q.data_ptr(), k.data_ptr(), bt, hq, hkv, T, w, int(pool_k), scale,
                                             int(budget), floor, p_sc + l * s_sc, p_hb + l * s_hb,
                                             p_off + l * s_off, p_idx + l * s_idx, ws.data_ptr(), stream))
        ev = torch.cuda.Event()
        ev.record()
        ready.append(ev)
    bh = np.arange(BH)
    qrow = (bh // hkv) * hq + (bh % hkv) * group

    def layers():
        for l in range(L):
            ready[l].synchronize()
            yield hb_np[l].astype(np.int64), qrow, qrow

    # every layer's cache laid out as its budgets arrive, then one K/V
    # allocation and ONE host-to-device copy for every plan, the
    # compactions' segment tables and the budgets' device copy
    try:
        caches, (seg_bh, seg_lo, seg_hi) = LayerCache.allocate_many(layers(), group, dev,
                                                                    extra=[bh, np.zeros(BH), hb_np])
    except BaseException:
        for ev in ready:  # the launches still write hb_pin: let them land before it is freed
            ev.synchronize()
        raise
    lens = hb_np
    hbs = seg_hi.view(L, bt, hkv)
    p_bh, p_lo, p_hi = seg_bh.data_ptr(), seg_lo.data_ptr(), seg_hi.data_ptr()
    for l, (k, v, cache) in enumerate(zip(ks, vs, caches)):
        cache.host["written"] = True
        _native.check(_lib.fkv_compact(k.data_ptr(), v.data_ptr(), T, BH, p_off + l * s_off, p_idx + l * s_idx,
                                       p_bh, p_lo, p_hi + 4 * l * BH, cache.ptr(16), 1,
                                       int(lens[l].max()), cache.k.data_ptr(), cache.v.data_ptr(), stream))
        # the compaction's segment tables (compact_into's arguments), and its
        # selection alive until the stream consumes it
        cache.host["compact_args"] = (seg_bh, seg_lo, seg_hi[l * BH:(l + 1) * BH])
        cache.host["selection"] = (offsets, idx)
    return caches, hbs, list(sc)
