"""Fused NVLink all-gather for the sharded decode (replaces NCCL all_gather).

Each rank owns, in memory it allocated with ``fkv_dev_alloc`` and exported
with CUDA IPC, receive areas ``recv[buf]`` of tp exchange-record blocks in
the XLL format (include/fairkv.h: per head row 32 units {4 o bytes, epoch,
4 o bytes, epoch} + one {lse, epoch, 0, epoch} unit) and an epoch counter.
Per layer the decode kernel of rank r writes every segment's final (o, lse)
record straight into block r of ``recv[buf]`` of *every* rank (16-byte P2P
stores over NVLink, ``fkv_decode_exchange``), each unit tagged with the
layer's epoch (the rank's counter + 1).  The merge kernel on each rank
polls exactly the units it merges until they carry that epoch, merges the
DP copies and writes o (``fkv_merge_wait``); its last CTA advances the
counter.  The data carries its own completion flag (NCCL's LL idea), so
the producer needs no fence and no flag write: a system-scope release
(MEMBAR.SYS) measured ~10 us per launch on B200, as much as a TP=8 rank's
whole decode.  Epochs grow monotonically and every rank runs the same
layer sequence, so all ranks agree on them without communicating.
Receive areas rotate per layer (``exchange_buffer``): a rank can run at
most one layer ahead of any peer (its merge of layer s needs every peer's
decode of s, which follows that peer's merge of s-1 in stream order), so it
suffices that consecutive layers of the running sequence -- including the
wrap from the last layer of one step to layer 0 of the next -- use different
buffers.  Parity alone does that for an even layer count; an odd count
gives its last layer a third buffer.  The assignment is static, so the whole
step can be captured once in a CUDA graph and replayed.

``P2PGroup.connect`` maps peers via torch.distributed (one process per GPU);
``P2PGroup.loopback`` builds tp virtual ranks inside one process on one GPU
(all "peer" pointers local) -- the same kernels and protocol, used by the
single-GPU tests and the emulated-TP bench.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native

NBUF = 3  # receive areas per rank (see exchange_buffer)


def exchange_buffer(layer: int, num_layers: int) -> int:
    """Receive area of ``layer`` in a step of ``num_layers`` layers: layer
    parity, except the last layer of an odd-length step (its successor is
    layer 0 of the next step, also parity 0), which takes area 2."""
    if num_layers < 2:
        raise ValueError("the fused exchange needs >= 2 layers per step: consecutive steps of a "
                         "1-layer stack would reuse one receive area while a peer still reads it")
    if not 0 <= layer < num_layers:
        raise ValueError(f"layer {layer} outside 0..{num_layers - 1}")
    return 2 if num_layers % 2 and layer == num_layers - 1 else layer & 1


class _Buf:
    def __init__(self, nbytes: int):
        ptr = C.c_void_p()
        _native.check(_native.lib.fkv_dev_alloc(int(nbytes), C.byref(ptr)))
        self.ptr = ptr.value
        self.nbytes = nbytes

    def handle(self) -> bytes:
        h = (C.c_char * 64)()
        _native.check(_native.lib.fkv_ipc_get(self.ptr, h))
        return bytes(h)

    def free(self):
        if self.ptr:
            _native.check(_native.lib.fkv_dev_free(self.ptr))
            self.ptr = None


def _open(handle: bytes) -> int:
    ptr = C.c_void_p()
    buf = (C.c_char * 64).from_buffer_copy(handle)
    _native.check(_native.lib.fkv_ipc_open(buf, C.byref(ptr)))
    return ptr.value


class RankEndpoint:
    """One rank's view: its own buffers plus every peer's mapped addresses."""

    def __init__(self, rank: int, tp: int, slots: int, group: int):
        self.rank, self.tp, self.slots, self.group = rank, tp, slots, group
        self.block = slots * group * 528              # FKV_XLL_BYTES: one rank's block
        self.recv = [_Buf(tp * self.block) for _ in range(NBUF)]  # exchange_buffer()
        self.ctr = _Buf(16)                            # [0] epoch, [1] merge arrival counter
        self.peer_recv: list[list[int]] = [[] for _ in range(NBUF)]  # [buffer][peer] base

    # -- pointers handed to the kernels
    def dest_records(self, parity: int) -> list[int]:
        """Where this rank's records go: its block in every peer's receive area."""
        return [base + self.rank * self.block for base in self.peer_recv[parity]]

    def recv_tensor(self, buf: int) -> torch.Tensor:
        """uint8 [tp, block] view of receive area ``buf`` (XLL blocks)."""
        return _as_tensor(self.recv[buf].ptr, self.tp * self.block).view(self.tp, self.block)

    @property
    def epoch(self) -> int:
        """Device address of the epoch counter (int32[2])."""
        return self.ctr.ptr

    def free(self):
        for b in (*self.recv, self.ctr):
            b.free()


def _as_tensor(ptr: int, nbytes: int) -> torch.Tensor:
    """Zero-copy uint8 CUDA tensor over library-owned device memory."""
    class _Ifc:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_Ifc(), device="cuda")


class P2PGroup:
    def __init__(self, endpoints: list[RankEndpoint], owned_remote: list[int] | None = None):
        self.endpoints = endpoints
        self._remote = owned_remote or []

    @staticmethod
    def loopback(tp: int, slots: int, group: int) -> "P2PGroup":
        eps = [RankEndpoint(r, tp, slots, group) for r in range(tp)]
        for ep in eps:
            ep.peer_recv = [[e.recv[par].ptr for e in eps] for par in range(NBUF)]
        return P2PGroup(eps)

    @staticmethod
    def connect(rank: int, tp: int, slots: int, group: int, process_group=None) -> "P2PGroup":
        import torch.distributed as dist
        ep = RankEndpoint(rank, tp, slots, group)
        mine = {"recv": [b.handle() for b in ep.recv]}
        allh = [None] * tp
        dist.all_gather_object(allh, mine, group=process_group)
        opened = []
        for par in range(NBUF):
            row = []
            for r, h in enumerate(allh):
                if r == rank:
                    row.append(ep.recv[par].ptr)
                else:
                    row.append(_open(h["recv"][par]))
                    opened.append(row[-1])
            ep.peer_recv[par] = row
        return P2PGroup([ep], opened)

    def close(self):
        for p in self._remote:
            _native.check(_native.lib.fkv_ipc_close(p))
        for ep in self.endpoints:
            ep.free()
