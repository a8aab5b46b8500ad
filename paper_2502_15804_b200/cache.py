"""Ragged, page-aligned compressed KV cache of one layer on one GPU, and its
decode work plan.

HBM layout (include/fairkv.h):
  k, v       bf16 [rows, 128]; row r stores 16-byte chunk c at c ^ (r & 7)
  segment s  = retained tokens of one (request, KV-head copy), rows
             [seg_row0[s], seg_row0[s] + seg_len[s]), seg_row0 % PAGE == 0,
             padding rows up to the next page are zero
Work plan (built on the host once per cache, uploaded once):
  items      chunks [t0, t1) of segments, ~equal size, t0 % 16 == 0
  groups     one per segment: items of the segment are merged by LSE into the
             segment's output rows (o rows = seg_out_row .. + G - 1)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

HEAD_DIM = 128
PAGE = 64
CHUNK_QUANTUM = 16  # one 16-token tile
NUM_SMS = 148
WORKERS = NUM_SMS * 8  # persistent decode warps (2 CTAs x 4 warps per SM)


def page_rows(n_tok) -> np.ndarray:
    n = np.asarray(n_tok, dtype=np.int64)
    return (n + PAGE - 1) // PAGE * PAGE


def segment_offsets(seg_len) -> tuple[np.ndarray, int]:
    """Page-aligned first row of every segment, and the total row count."""
    rows = page_rows(seg_len)
    row0 = np.zeros(len(rows), dtype=np.int64)
    if len(rows):
        row0[1:] = np.cumsum(rows)[:-1]
    total = int(rows.sum()) if len(rows) else 0
    return row0, max(total, PAGE)


def choose_chunk(seg_len, target_items: int | None = None, max_chunk: int = 2048,
                 min_chunk: int = 128) -> int:
    """Tokens per work item for the warp-persistent decode kernel: about
    three items per worker warp (the longest-first queue then drains with a
    short tail), at least ``min_chunk`` tokens so the per-item record/merge
    overhead stays a few percent, multiple of the 16-token tile."""
    total = int(np.asarray(seg_len, dtype=np.int64).sum())
    target = target_items or WORKERS * 3
    c = -(-total // max(target, 1))
    c = -(-c // CHUNK_QUANTUM) * CHUNK_QUANTUM
    return int(min(max(c, min_chunk), max_chunk))


def longest_first(t0, t1) -> np.ndarray:
    """Item processing order for the persistent decode kernel: longest
    first (LPT), ties by item id, so the queue drains with a short tail."""
    n = np.asarray(t1, dtype=np.int64) - np.asarray(t0, dtype=np.int64)
    return np.lexsort((np.arange(len(n)), -n)).astype(np.int32)


def plan_items(seg_len, chunk: int) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """-> item_seg, item_t0, item_t1 (int32) and per-segment item CSR ptr."""
    seg_len = np.asarray(seg_len, dtype=np.int64)
    counts = np.maximum(1, -(-seg_len // chunk))  # an empty segment still gets one item
    ptr = np.zeros(len(seg_len) + 1, dtype=np.int32)
    ptr[1:] = np.cumsum(counts)
    item_seg = np.repeat(np.arange(len(seg_len), dtype=np.int32), counts)
    local = np.arange(ptr[-1], dtype=np.int64) - np.repeat(ptr[:-1], counts)
    t0 = (local * chunk).astype(np.int32)
    t1 = np.minimum(t0.astype(np.int64) + chunk, seg_len[item_seg]).astype(np.int32)
    return item_seg, t0, t1, ptr


@dataclass
class LayerCache:
    """Device-resident compressed cache + decode plan for one layer on one GPU."""

    k: torch.Tensor
    v: torch.Tensor
    group: int
    seg_row0: torch.Tensor
    seg_len: torch.Tensor
    seg_qrow: torch.Tensor
    seg_out_row: torch.Tensor
    item_seg: torch.Tensor
    item_t0: torch.Tensor
    item_t1: torch.Tensor
    grp_ptr: torch.Tensor
    src_idx: torch.Tensor
    item_order: torch.Tensor
    counters: torch.Tensor
    host: dict = field(default_factory=dict, repr=False)

    @property
    def n_items(self) -> int:
        return int(self.item_seg.shape[0])

    @property
    def n_segments(self) -> int:
        return int(self.seg_len.shape[0])

    @property
    def retained_tokens(self) -> int:
        return int(self.host["seg_len"].sum())

    def kv_bytes(self) -> int:
        """Algorithmic K+V bytes one decode step reads from this cache."""
        return self.retained_tokens * HEAD_DIM * 2 * 2

    @staticmethod
    def allocate(seg_len, seg_qrow, seg_out_row, group: int, device, chunk: int | None = None,
                 fill: str = "zeros", generator: torch.Generator | None = None) -> "LayerCache":
        """Lay out segments and build the work plan.  ``fill='zeros'`` leaves
        the storage for the compaction kernel; ``fill='random'`` writes N(0,1)
        bf16 into every retained row (synthetic benchmark caches; the swizzle
        is a permutation, so random data needs no packing) and keeps padding
        rows zero."""
        seg_len = np.asarray(seg_len, dtype=np.int64)
        row0, rows = segment_offsets(seg_len)
        chunk = chunk or choose_chunk(seg_len)
        item_seg, t0, t1, ptr = plan_items(seg_len, chunk)
        dev = torch.device(device)
        k = torch.zeros((rows, HEAD_DIM), dtype=torch.bfloat16, device=dev)
        v = torch.zeros((rows, HEAD_DIM), dtype=torch.bfloat16, device=dev)
        if fill == "random":
            k.normal_(generator=generator)
            v.normal_(generator=generator)
            valid = torch.zeros(rows, dtype=torch.bool, device=dev)
            live = np.zeros(rows, dtype=bool)
            for r0, n in zip(row0, seg_len):
                live[r0:r0 + n] = True
            valid.copy_(torch.from_numpy(live))
            k.mul_(valid[:, None])
            v.mul_(valid[:, None])

        def i32(a):
            return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=dev)

        return LayerCache(
            k=k, v=v, group=int(group),
            seg_row0=torch.as_tensor(row0, device=dev),
            seg_len=i32(seg_len), seg_qrow=i32(seg_qrow), seg_out_row=i32(seg_out_row),
            item_seg=i32(item_seg), item_t0=i32(t0), item_t1=i32(t1),
            grp_ptr=i32(ptr), src_idx=i32(np.arange(ptr[-1])),
            item_order=i32(longest_first(t0, t1)),
            counters=torch.zeros(len(seg_len) + 2, dtype=torch.int32, device=dev),
            host={"seg_len": seg_len, "seg_row0": row0, "chunk": chunk,
                  "seg_qrow": np.asarray(seg_qrow), "seg_out_row": np.asarray(seg_out_row)},
        )

    @staticmethod
    def view(k: torch.Tensor, v: torch.Tensor, seg_row0, seg_len, seg_qrow, seg_out_row,
             group: int, chunk: int | None = None) -> "LayerCache":
        """A segment table over existing storage (e.g. the DP copies / shards
        of a base cache: each copy is a 16-aligned sub-range of its head's
        rows).  No data moves."""
        seg_row0 = np.asarray(seg_row0, dtype=np.int64)
        seg_len = np.asarray(seg_len, dtype=np.int64)
        if np.any(seg_row0 % 16):
            raise ValueError("segment starts must be multiples of 16 rows")
        chunk = chunk or choose_chunk(seg_len)
        item_seg, t0, t1, ptr = plan_items(seg_len, chunk)
        dev = k.device

        def i32(a):
            return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=dev)

        return LayerCache(
            k=k, v=v, group=int(group), seg_row0=torch.as_tensor(seg_row0, device=dev),
            seg_len=i32(seg_len), seg_qrow=i32(seg_qrow), seg_out_row=i32(seg_out_row),
            item_seg=i32(item_seg), item_t0=i32(t0), item_t1=i32(t1), grp_ptr=i32(ptr),
            src_idx=i32(np.arange(ptr[-1])),
            item_order=i32(longest_first(t0, t1)),
            counters=torch.zeros(len(seg_len) + 2, dtype=torch.int32, device=dev),
            host={"seg_len": seg_len, "seg_row0": seg_row0, "chunk": chunk,
                  "seg_qrow": np.asarray(seg_qrow), "seg_out_row": np.asarray(seg_out_row)},
        )
