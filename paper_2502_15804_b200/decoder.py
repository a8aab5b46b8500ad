"""Decode step of the attention sub-stack on one rank (SURVEY §8d metric).

For every layer: K4 over this rank's segments (its fused K5 merging chunks
straight into fixed send slots) ->
all-gather of the slot records across the TP group -> K5 over the DP copies
of each head -> o [Bt, Hq, 128] bf16 on every rank.  At tp == 1 K5 writes o
directly.  The per-layer order is the synchronous barrier model of the
reference simulator (reference simulate.py:118-136): the all-gather is the
layer barrier.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops
from .cache import LayerCache
from .exchange import exchange_buffer
from .sharding import FinalMerge, LayerShard


def rank_caches(shards: list[LayerShard], bt: int, hq: int, group: int, tp: int, device,
                *, base: list[LayerCache] | None = None, base_index=None, fill: str = "random",
                seed: int = 0, reserve: int = 0, head_len=None) -> list[LayerCache]:
    """Per-layer caches of one rank.  With ``base`` (full per-head caches, one
    segment per (b, h) in b-major order) the rank's segments are views into
    it (DP copies = 16-aligned sub-ranges); otherwise fresh storage filled
    with ``fill`` and ``reserve`` rows of append headroom per segment.

    Decode-time appends (``ops.append`` with the step's K/V [Bt, Hkv, 128]):
    only the segment that owns the end of its head's token axis (a whole
    head, or the last DP copy) takes the new token -- known from the base
    cache's lengths, or from ``head_len`` [L][Bt, Hkv] for fresh storage."""
    hkv = hq // group
    out = []
    gen = torch.Generator(device=device).manual_seed(seed)
    for l, sh in enumerate(shards):
        qrow = sh.seg_b * hq + sh.seg_h * group
        # tp > 1: segment i's record rows are slot i's G heads; tp == 1: o rows
        out_row = np.arange(sh.n_segments) * group if tp > 1 else qrow
        lens = sh.seg_hi - sh.seg_lo
        bh = sh.seg_b * hkv + sh.seg_h
        if base is not None:
            b0 = base[l].host["seg_row0"]
            full = base[l].host["seg_len"][bh]
            owns_end = sh.seg_hi >= full
            cap = np.where(owns_end, base[l].host["seg_cap"][bh] - sh.seg_lo, lens)
            src = np.where(owns_end, bh, -1)
            row0 = b0[bh] + sh.seg_lo
            out.append(LayerCache.view(base[l].k, base[l].v, row0, lens, qrow, out_row, group,
                                       seg_cap=cap, append_src=src))
        else:
            c = LayerCache.allocate(lens, qrow, out_row, group, device, fill=fill, generator=gen,
                                    reserve=reserve)
            if head_len is not None:
                owns_end = sh.seg_hi >= np.asarray(head_len[l]).reshape(-1)[bh]
                c.append_src_t.copy_(torch.as_tensor(np.where(owns_end, bh, -1).astype(np.int32)))
            else:
                c.append_src_t.copy_(torch.as_tensor(bh.astype(np.int32)))
            out.append(c)
    return out


class StackDecoder:
    """exchange = "p2p" (default for tp > 1): fused NVLink all-gather inside
    the decode kernel (exchange.P2PGroup, one endpoint = this rank);
    "nccl": K4 into local slots + torch.distributed all_gather_into_tensor."""

    def __init__(self, caches: list[LayerCache], finals: list[FinalMerge] | None, *, tp: int,
                 bt: int, hq: int, group: int, process_group=None, exchange: str = "nccl",
                 endpoint=None):
        self.caches = caches
        self.tp = tp
        self.exchange_mode = exchange
        self.endpoint = endpoint
        self.group = group
        self.bt, self.hq = bt, hq
        self.pg = process_group
        dev = caches[0].k.device
        self.ws = [ops.DecodeWorkspace(c) for c in caches]
        self.send, self.recv, self.final = [], [], []
        if tp > 1:
            for c, f in zip(caches, finals):
                if exchange != "p2p":  # NCCL: exchange-record send block + gathered blocks
                    self.send.append(ops.xrec_empty(f.slots, group, dev)[0])
                    self.recv.append(ops.xrec_empty(f.slots, group, dev, ranks=tp))
                self.final.append(tuple(torch.as_tensor(x, device=dev) for x in (f.grp_ptr, f.src_idx, f.out_row)))
        self.kernel_launches_per_step = len(caches) * (2 if tp > 1 else 1)

    def layer(self, l: int, q: torch.Tensor, out: torch.Tensor, out_lse: torch.Tensor | None = None):
        c = self.caches[l]
        if self.tp == 1:
            ops.decode_into(q, c, self.ws[l], out_bf16=out, out_lse=out_lse)
            return
        if self.exchange_mode == "p2p":
            ptr, src, row = self.final[l]
            buf = exchange_buffer(l, len(self.caches))
            ops.decode_exchange(q, c, self.endpoint, buf, self.ws[l])
            ops.merge_wait(self.endpoint, buf, ptr, src, row, self.group, out_bf16=out,
                           out_lse=out_lse)
            return
        self.produce(l, q)
        self.exchange(l)
        self.consume(l, out, out_lse)

    # The NCCL path in its three stream-ordered parts (tests drive them in
    # lockstep for several virtual ranks with a loopback all-gather).
    def produce(self, l: int, q: torch.Tensor):
        """K4 + fused segment merge -> this rank's exchange-record block."""
        ops.decode_into(q, self.caches[l], self.ws[l], out_rec=self.send[l])

    def exchange(self, l: int):
        """All-gather of the blocks: recv[l][r] = rank r's send block."""
        import torch.distributed as dist
        dist.all_gather_into_tensor(self.recv[l].view(-1), self.send[l], group=self.pg)

    def consume(self, l: int, out: torch.Tensor, out_lse: torch.Tensor | None = None):
        """K5: LSE merge of each head's DP copies -> o [Bt, Hq, 128]."""
        ptr, src, row = self.final[l]
        ops.merge_lse(self.recv[l], ptr, src, row, self.group, out_bf16=out, out_lse=out_lse)

    def step(self, q_layers: torch.Tensor, out_layers: torch.Tensor):
        """q_layers / out_layers: [L, Bt, Hq, 128] bf16."""
        for l in range(len(self.caches)):
            self.layer(l, q_layers[l], out_layers[l])

    def kv_bytes(self) -> int:
        return sum(c.kv_bytes() for c in self.caches)


class DecodeLayer:
    """One decode layer of the sharded model on one rank, with its weight
    GEMMs: for x [Bt, Hq*128] bf16 (the layer input, the
    same on every rank)

      qkv  = x @ W_qkv[:, this rank's heads]    cuBLAS bf16: q of every local
             KV-head copy's G query heads, k and v of its KV head (AHA-DP
             copies replicate these columns on every GPU holding the head)
      append the new k / v to the copies that own their head's token tail
             (ops.append: a DP copy's earlier token range does not grow)
      o    = K4 over the local copies + fused NVLink all-gather + K5 LSE merge
             (ops.decode_exchange / merge_wait; TP = 1: ops.decode_into)
             -> o [Bt, Hq, 128] on every rank
      y_g  = o @ W_o[:, g-th 1/tp of the columns]   cuBLAS bf16

    and returns y_g [Bt, Hq*128 / tp] (column-parallel o_proj: the caller
    all-gathers the y_g into the next layer's x).  The QKV and o_proj GEMMs
    are plain library GEMMs; the attention between them is this package's
    kernels.  ``w_qkv`` [Hq*128, (Hq + 2 Hkv)*128] in the usual
    [q heads | k heads | v heads] column order, ``w_o`` [Hq*128, Hq*128]."""

    def __init__(self, w_qkv: torch.Tensor, w_o: torch.Tensor, cache: LayerCache, shard: LayerShard,
                 final: FinalMerge | None, *, tp: int, rank: int, bt: int, hq: int, group: int,
                 endpoint=None, buf: int = 0):
        d = 128
        hkv = hq // group
        hidden = hq * d
        if w_qkv.shape != (hidden, (hq + 2 * hkv) * d) or w_o.shape != (hidden, hidden):
            raise ValueError("w_qkv must be [Hq*128, (Hq+2Hkv)*128] and w_o [Hq*128, Hq*128]")
        if hidden % tp:
            raise ValueError("Hq*128 must divide by tp (column-parallel o_proj)")
        if tp > 1 and (endpoint is None or final is None):
            raise ValueError("tp > 1 needs the exchange endpoint and the final merge tables")
        heads = np.unique(np.asarray(shard.seg_h, dtype=np.int64))
        qcols = [np.arange(h * group * d, (h + 1) * group * d) for h in heads]
        kcols = [hq * d + np.arange(h * d, (h + 1) * d) for h in heads]
        vcols = [(hq + hkv) * d + np.arange(h * d, (h + 1) * d) for h in heads]
        cols = np.concatenate(qcols + kcols + vcols) if len(heads) else np.zeros(0, np.int64)
        dev = cache.k.device
        self.w_qkv = w_qkv[:, torch.as_tensor(cols, device=w_qkv.device)].contiguous()
        oc = hidden // tp
        self.w_o = w_o[:, rank * oc:(rank + 1) * oc].contiguous()
        self.cache, self.tp, self.rank, self.endpoint, self.buf = cache, tp, rank, endpoint, buf
        self.bt, self.hq, self.hkv, self.group, self.nh = bt, hq, hkv, group, len(heads)
        self.heads = torch.as_tensor(heads, device=dev)
        self.ws = ops.DecodeWorkspace(cache)
        self.q = torch.zeros((bt, hkv, group, d), dtype=torch.bfloat16, device=dev)
        self.k_new = torch.zeros((bt, hkv, d), dtype=torch.bfloat16, device=dev)
        self.v_new = torch.zeros((bt, hkv, d), dtype=torch.bfloat16, device=dev)
        self.o = torch.empty((bt, hq, d), dtype=torch.bfloat16, device=dev)
        self.qkv = torch.empty((bt, self.w_qkv.shape[1]), dtype=torch.bfloat16, device=dev)
        self.y = torch.empty((bt, oc), dtype=torch.bfloat16, device=dev)
        self.final = None if final is None else tuple(
            torch.as_tensor(x, device=dev) for x in (final.grp_ptr, final.src_idx, final.out_row))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """One decode step of this layer on this rank -> y_g (a view of a
        buffer reused by the next call)."""
        self.produce(x)
        return self.consume()

    # forward() in its two stream-ordered halves: virtual ranks sharing one
    # GPU (loopback tests) must issue every rank's produce() before any
    # consume() polls for the peers' records.
    def produce(self, x: torch.Tensor):
        """QKV GEMM, append, K4 (+ the fused exchange stores at tp > 1)."""
        d, G, nh = 128, self.group, self.nh
        torch.mm(x, self.w_qkv, out=self.qkv)
        self.q.index_copy_(1, self.heads, self.qkv[:, :nh * G * d].view(self.bt, nh, G, d))
        self.k_new.index_copy_(1, self.heads, self.qkv[:, nh * G * d:nh * (G + 1) * d].view(self.bt, nh, d))
        self.v_new.index_copy_(1, self.heads, self.qkv[:, nh * (G + 1) * d:].view(self.bt, nh, d))
        ops.append(self.cache, self.k_new, self.v_new)
        q = self.q.view(self.bt, self.hq, d)
        if self.tp == 1:
            ops.decode_into(q, self.cache, self.ws, out_bf16=self.o)
        else:
            ops.decode_exchange(q, self.cache, self.endpoint, self.buf, self.ws)

    def consume(self) -> torch.Tensor:
        """K5 merge of the gathered records (tp > 1) and the o_proj GEMM."""
        if self.tp > 1:
            ops.merge_wait(self.endpoint, self.buf, *self.final, self.group, out_bf16=self.o)
        torch.mm(self.o.view(self.bt, self.hq * 128), self.w_o, out=self.y)
        return self.y
