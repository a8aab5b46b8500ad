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
                c.host["append_src_t"].copy_(torch.as_tensor(np.where(owns_end, bh, -1).astype(np.int32)))
            else:
                c.host["append_src_t"].copy_(torch.as_tensor(bh.astype(np.int32)))
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
