"""Ragged, page-aligned compressed KV cache of one layer on one GPU, and its
decode work plan.

HBM layout (include/fairkv.h):
  k, v       bf16 [rows, 128]; row r stores 16-byte chunk c at c ^ (r & 7)
  segment s  = retained tokens of one (request, KV-head copy), rows
             [seg_row0[s], seg_row0[s] + seg_len[s]), seg_row0 % PAGE == 0,
             padding rows up to the next page are zero
Work plan (built on the host once per cache, uploaded once):
  items      pieces [t0, t1) of segments, t0 % 16 == 0, dealt to the persistent
             decode warps so every warp streams the same number of tiles
  groups     one per segment: items of the segment are merged by LSE into the
             segment's output rows (o rows = seg_out_row .. + G - 1)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import os

import numpy as np
import torch

HEAD_DIM = 128
PAGE = 64
NUM_SMS = 148


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


MAX_ITEMS_PER_SEGMENT = 32  # FKV_MAX_PIECES (kMergeMax in decode.cu)
MAX_WORK_PER_WORKER = 32    # FKV_MAX_WORK: descriptor entries per worker
HYBRID_MIN_PIECE_TILES = 32  # whole-segment schedule: shortest piece a long segment is cut into
HYBRID_MIN_SAVING_US = 0.5   # ... and only when the modelled critical path shrinks by more than this
HYBRID_LONE_TILE_US = 0.045  # per-tile time of a lone streaming CTA (<= 32 segments busy)
LONE_PREFETCH_TILES = 28     # tiles a wide CTA's rings hold at once (7 streaming warps x 4 stages)
TILE = 16


def default_workers(device=None, flags: int = 0) -> int:
    """Persistent decode CTAs of a schedule (``flags``: FKV_DECODE_SOLO /
    FKV_DECODE_WIDE / 0): SMs x its co-resident CTAs per SM (libfairkv: 1 for
    the 8-warp cooperative CTA, 2 otherwise)."""
    try:
        sms = torch.cuda.get_device_properties(device).multi_processor_count
    except Exception:  # no device visible (host-side planning / CPU tests)
        sms = NUM_SMS
    from . import _native
    return sms * int(_native.lib.fkv_decode_ctas_per_sm(int(flags)))


MIN_TILES_PER_WORKER = 8  # floor on tiles per worker CTA (one 2-tile round per warp)
MAX_PIECES_PER_SEGMENT = 4  # typical split bound: merge cost grows with pieces per segment


def _cut_stream(seg_len, tiles, per: int, cap: int):
    """Cut the concatenated tile stream into worker ranges of ``per`` tiles and
    at most ``cap`` pieces (an empty segment is one piece with no tiles)."""
    seg_i, t0s, t1s, owner = [], [], [], []
    w, used, cnt = 0, 0, 0
    for s in range(len(seg_len)):
        n, t = int(tiles[s]), 0
        while True:
            if cnt >= cap or (used >= per and n > t):
                w, used, cnt = w + 1, 0, 0
            take = min(n - t, per - used)
            seg_i.append(s)
            t0s.append(t * TILE)
            t1s.append(min(int(seg_len[s]), (t + take) * TILE))
            owner.append(w)
            used += take
            cnt += 1
            t += take
            if t >= n:
                break
    return seg_i, t0s, t1s, np.asarray(owner, dtype=np.int64)


def _cut_stream_cost(seg_len, tiles, C: int, P: int, cap: int):
    """Cut the tile stream into worker ranges of estimated cost <= C, a
    worker's cost being sum over its pieces of (P + tiles): every piece pays
    a fixed epilogue (hand-over, combine, output or record + merge)."""
    seg_i, t0s, t1s, owner = [], [], [], []
    w, cost, cnt = 0, 0, 0
    for s in range(len(seg_len)):
        n, t = int(tiles[s]), 0
        while True:
            if cnt >= cap or (cnt > 0 and (C - cost - P < 1 or (n == t and C - cost - P < 0))):
                w, cost, cnt = w + 1, 0, 0
            take = min(n - t, max(C - cost - P, 1))
            seg_i.append(s)
            t0s.append(t * TILE)
            t1s.append(min(int(seg_len[s]), (t + take) * TILE))
            owner.append(w)
            cost += P + take
            cnt += 1
            t += take
            if t >= n:
                break
    return seg_i, t0s, t1s, np.asarray(owner, dtype=np.int64)


PIECE_COST_TILES = 48  # coop schedule: one piece's cost in tile-equivalents (plateau >= 32, probe_sched)


PAIR_PIECE_TILES = 12  # SM pairing: measured per-piece cost (~2.4 us vs ~0.21 us per tile per CTA)


def _pair_on_sms(owner, t0s, t1s, sms: int):
    """Relabel workers so that the two CTAs sharing an SM (CTA j and j + sms:
    the block scheduler places a fresh grid round robin over the SMs, second
    slots in the same order) carry similar work.  The per-CTA cut equalises
    tiles + P x pieces, so tile counts vary inversely with piece counts; two
    piece-heavy CTAs on one SM would leave it idle early while another SM
    streams two tile-heavy ones.  Heaviest CTAs (by tiles) get an SM to
    themselves when the grid has fewer than 2 x sms CTAs; the rest are paired
    heaviest with lightest."""
    owner = np.asarray(owner, dtype=np.int64)
    busy = int(owner.max()) + 1 if len(owner) else 0
    k = busy - sms  # number of SMs running two CTAs
    if k <= 0:
        return owner
    import os
    pw = float(os.environ.get("FKV_PAIR_PIECE", PAIR_PIECE_TILES))
    w_tiles = np.bincount(owner, weights=(np.asarray(t1s) - np.asarray(t0s) + TILE - 1) // TILE + pw,
                          minlength=busy)
    order = np.argsort(-w_tiles, kind="stable")
    new_id = np.empty(busy, dtype=np.int64)
    solo, paired = order[:sms - k], order[sms - k:]
    new_id[solo] = np.arange(k, sms)
    for j in range(k):  # heaviest remaining with lightest remaining
        new_id[paired[j]] = j
        new_id[paired[2 * k - 1 - j]] = j + sms
    return new_id[owner]


def plan_work(seg_len, n_workers: int, chunk: int | None = None,
              min_tiles: int = MIN_TILES_PER_WORKER, piece_cost: int | None = None,
              sms: int | None = None):
    """Static decode schedule for the warp-persistent K4 kernel.

    Default: the segments' 16-token tiles are laid end to end and the stream
    is cut into equal ranges of R = max(ceil(total_tiles / n_workers),
    min_tiles, ceil(mean_segment_tiles / 4)) tiles, one range per worker: every busy worker streams the
    same number of bytes and at most one segment per range boundary is split
    (and needs an LSE merge).  With ``chunk``, every segment is cut into
    ``chunk``-token pieces instead and consecutive pieces are dealt to
    workers by equal token count.  Every segment has at least one piece (an
    empty one still produces o = 0, lse = -inf), pieces of a segment are
    consecutive item ids and start on a 16-token tile.

    Returns item_seg, item_t0, item_t1 (int32 [n_items]), seg_item_ptr (int32
    [n_seg+1]), warp_ptr (int32 [busy+1], busy <= n_workers: only busy
    workers are launched, and fewer busy warps per CTA get deeper rings) and
    work_list (int32 [n_items], item ids grouped by worker).
    """
    seg_len = np.asarray(seg_len, dtype=np.int64)
    n_seg = len(seg_len)
    tiles = (seg_len + TILE - 1) // TILE
    W = max(1, int(n_workers))
    longest = int(tiles.max()) if n_seg else 0
    if chunk is None:
        per = max(-(-int(tiles.sum()) // W), int(min_tiles), 1)
        # keep the average segment within a few pieces: the last warp of a split
        # segment merges every piece's record, so many pieces lengthen the tail
        avg = int(tiles.sum()) // max(n_seg, 1)
        per = max(per, -(-avg // MAX_PIECES_PER_SEGMENT))
        per = max(per, -(-longest // (MAX_ITEMS_PER_SEGMENT - 1)))
        import os
        P = int(os.environ.get("FKV_PIECE_COST", PIECE_COST_TILES)) if piece_cost is None else piece_cost
        if P > 0 and n_seg:
            # equal estimated time per worker (tiles + P per piece): smallest C
            # whose greedy cut fits in W workers (binary search)
            # C >= per + P: a worker still takes >= per tiles in one piece
            # (min_tiles, and <= MAX_ITEMS_PER_SEGMENT pieces per segment)
            lo = max(per + P, -(-(int(tiles.sum()) + P * n_seg) // W))
            hi = max(lo, int(tiles.sum()) + P * (n_seg + 1))
            best = None
            while lo <= hi:
                C = (lo + hi) // 2
                cut = _cut_stream_cost(seg_len, tiles, C, P, MAX_WORK_PER_WORKER)
                if int(cut[3].max()) < W:
                    best, hi = cut, C - 1
                else:
                    lo = C + 1
            if best is None:
                raise ValueError(f"{n_seg} segments exceed one launch "
                                 f"({W} workers x {MAX_WORK_PER_WORKER} pieces)")
            seg_i, t0s, t1s, owner = best
        else:
            while True:
                seg_i, t0s, t1s, owner = _cut_stream(seg_len, tiles, per, MAX_WORK_PER_WORKER)
                if not len(owner) or int(owner.max()) < W:
                    break
                if per >= int(tiles.sum()):  # only the piece cap can bind: too many segments
                    raise ValueError(f"{n_seg} segments exceed one launch "
                                     f"({W} workers x {MAX_WORK_PER_WORKER} pieces)")
                per *= 2
    else:
        ch = max(1, -(-int(chunk) // TILE))
        ch = max(ch, -(-longest // MAX_ITEMS_PER_SEGMENT)) * TILE
        counts = np.maximum(1, -(-seg_len // ch))
        seg_i = np.repeat(np.arange(n_seg), counts)
        ptr0 = np.zeros(n_seg + 1, dtype=np.int64)
        ptr0[1:] = np.cumsum(counts)
        local = np.arange(ptr0[-1]) - np.repeat(ptr0[:-1], counts)
        t0s = local * ch
        t1s = np.minimum(t0s + ch, seg_len[seg_i])
        lens = np.maximum(t1s - t0s, 0)
        cum = np.concatenate([[0], np.cumsum(lens)[:-1]])
        per = max(1, -(-int(lens.sum()) // W))
        owner = np.minimum(cum // per, W - 1)
        if len(owner) and np.bincount(owner).max() > MAX_WORK_PER_WORKER:
            # piece cap binds: deal pieces in order, at most the cap per worker
            owner = np.zeros(len(lens), dtype=np.int64)
            w, used, cnt = 0, 0, 0
            for i, n in enumerate(lens):
                if cnt >= MAX_WORK_PER_WORKER or used >= per:
                    w, used, cnt = w + 1, 0, 0
                owner[i] = w
                used += int(n)
                cnt += 1
            if w >= W:
                raise ValueError(f"{len(lens)} pieces exceed one launch "
                                 f"({W} workers x {MAX_WORK_PER_WORKER} pieces)")
    import os
    if sms and os.environ.get("FKV_SM_PAIRING", "1") == "1":
        owner = _pair_on_sms(owner, t0s, t1s, int(sms))
    item_seg = np.asarray(seg_i, dtype=np.int32)
    t0 = np.asarray(t0s, dtype=np.int32)
    t1 = np.asarray(t1s, dtype=np.int32)
    owner = np.asarray(owner, dtype=np.int64)
    seg_item_ptr = np.zeros(n_seg + 1, dtype=np.int32)
    seg_item_ptr[1:] = np.cumsum(np.bincount(item_seg, minlength=n_seg))
    busy = int(owner.max()) + 1 if len(owner) else 1  # owners are 0..busy-1
    warp_ptr = np.zeros(busy + 1, dtype=np.int32)
    warp_ptr[1:] = np.cumsum(np.bincount(owner, minlength=busy))
    # Within a worker, pieces of split segments go first: their LSE merges
    # (done by whichever piece finishes last) then overlap the streaming of
    # whole segments instead of all landing in the kernel's tail.
    split = (np.diff(seg_item_ptr) > 1)[item_seg]
    work_list = np.lexsort((np.arange(len(item_seg)), ~split, owner)).astype(np.int32)
    return item_seg, t0, t1, seg_item_ptr, warp_ptr, work_list


def work_table(seg_row0, seg_len, seg_qrow, seg_out_row, item_seg, t0, t1, seg_item_ptr,
               warp_ptr, work_list, solo_ctas: int | None = None) -> np.ndarray:
    """The kernel-facing form of a schedule: fkv_work_t [rows, K, 8 x int32]
    (include/fairkv.h), zero-filled (n_it = 0) after each row's last piece,
    K = max pieces per row (<= FKV_MAX_WORK).  Coop schedule: row = worker
    = one CTA.  Solo schedule (``solo_ctas``): worker w is warp w // solo_ctas
    of CTA w % solo_ctas, tagged in the high half of n_it."""
    seg_row0 = np.asarray(seg_row0, dtype=np.int64)
    seg_len = np.asarray(seg_len, dtype=np.int64)
    busy = len(warp_ptr) - 1
    counts = np.diff(warp_ptr)
    n_it = np.diff(seg_item_ptr)
    w = np.repeat(np.arange(busy), counts)
    if solo_ctas:
        rows = min(solo_ctas, max(busy, 1))
        row_of, tag_of = w % rows, w // rows
    else:
        rows = max(busy, 1)
        row_of, tag_of = w, np.zeros_like(w)
    per_row = np.bincount(row_of, minlength=rows) if len(w) else np.zeros(rows, np.int64)
    K = max(1, int(per_row.max()) if len(per_row) else 1)
    if K > MAX_WORK_PER_WORKER:
        raise ValueError(f"{K} pieces on one CTA exceed FKV_MAX_WORK")
    tab = np.zeros((rows, K, 8), dtype=np.int32)
    if len(work_list):
        it = np.asarray(work_list, dtype=np.int64)
        order = np.argsort(row_of, kind="stable")  # pieces of a row in worker order
        j = np.empty(len(it), dtype=np.int64)
        starts = np.concatenate([[0], np.cumsum(per_row)[:-1]])
        j[order] = np.arange(len(it)) - np.repeat(starts, per_row)
        seg = np.asarray(item_seg, dtype=np.int64)[it]
        a = np.asarray(t0, dtype=np.int64)[it]
        b = np.minimum(np.asarray(t1, dtype=np.int64)[it], seg_len[seg])
        row0 = seg_row0[seg] + a
        tab[row_of, j, 0] = (row0 & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
        tab[row_of, j, 1] = (row0 >> 32).astype(np.int32)
        tab[row_of, j, 2] = np.maximum(b - a, 0)
        tab[row_of, j, 3] = np.asarray(seg_qrow, dtype=np.int64)[seg]
        tab[row_of, j, 4] = np.asarray(seg_out_row, dtype=np.int64)[seg]
        tab[row_of, j, 5] = it
        tab[row_of, j, 6] = np.asarray(seg_item_ptr, dtype=np.int64)[seg]
        tab[row_of, j, 7] = n_it[seg] | (tag_of << 16)
    return tab


def plan_work_solo(seg_len, n_workers: int, piece_tiles: int = 16, whole_tiles: int = 24):
    """Segment-aligned per-warp schedule for small caches: a segment of at
    most ``whole_tiles`` tiles stays one piece (no LSE merge); longer ones are
    cut into near-equal 16-token-aligned pieces of about
    max(piece_tiles, total / n_workers) tiles; pieces go to workers one each
    while they last, else largest-first onto the least-loaded worker.  Same
    return convention as ``plan_work``."""
    import heapq
    seg_len = np.asarray(seg_len, dtype=np.int64)
    n_seg = len(seg_len)
    tiles = (seg_len + TILE - 1) // TILE
    W = max(1, int(n_workers))
    total = int(tiles.sum())
    piece = max(int(piece_tiles), -(-total // W), 1)
    seg_i, t0s, t1s = [], [], []
    for s in range(n_seg):
        n = int(tiles[s])
        k = 1 if n <= whole_tiles else min(MAX_ITEMS_PER_SEGMENT, -(-n // piece))
        cuts = [round(j * n / k) for j in range(k + 1)]
        for j in range(k):
            seg_i.append(s)
            t0s.append(cuts[j] * TILE)
            t1s.append(min(int(seg_len[s]), cuts[j + 1] * TILE))
    item_seg = np.asarray(seg_i, dtype=np.int32)
    t0 = np.asarray(t0s, dtype=np.int32)
    t1 = np.asarray(t1s, dtype=np.int32)
    n_items = len(item_seg)
    if n_items <= W:
        owner = np.arange(n_items, dtype=np.int64)
    else:
        size = np.maximum(t1.astype(np.int64) - t0, 0)
        owner = np.empty(n_items, dtype=np.int64)
        heap = [(0, w) for w in range(W)]
        for i in np.lexsort((np.arange(n_items), -size)):
            load, w = heapq.heappop(heap)
            owner[i] = w
            heapq.heappush(heap, (load + int(size[i]) + 1, w))
        if np.bincount(owner, minlength=W).max() > MAX_WORK_PER_WORKER:
            raise ValueError("too many pieces for the per-warp schedule")
        # renumber workers by first piece so owners are 0..busy-1
        _, owner = np.unique(owner, return_inverse=True)
    seg_item_ptr = np.zeros(n_seg + 1, dtype=np.int32)
    seg_item_ptr[1:] = np.cumsum(np.bincount(item_seg, minlength=n_seg))
    busy = int(owner.max()) + 1 if n_items else 1
    warp_ptr = np.zeros(busy + 1, dtype=np.int32)
    warp_ptr[1:] = np.cumsum(np.bincount(owner, minlength=busy))
    split = (np.diff(seg_item_ptr) > 1)[item_seg]
    work_list = np.lexsort((np.arange(n_items), ~split, owner)).astype(np.int32)
    return item_seg, t0, t1, seg_item_ptr, warp_ptr, work_list


# K4 schedule choice: the per-warp ("solo") schedule when the cache is small
# enough that the CTA-cooperative one would give each CTA few tiles
# (FKV_K4_SCHEDULE = coop | solo | auto overrides, for measurements).
SOLO_MAX_TILES_PER_CTA = 19  # measured crossover (tools/probe_solo_params.py, probe_sched.py): ~5600 tiles per GPU-layer
FKV_DECODE_SOLO = 1
FKV_DECODE_WIDE = 2
FKV_DECODE_AFTER_WAIT = 4
WIDE_MAX_SEGMENTS = 128
WIDE_MIN_MEAN_TILES = 6  # probe_sched: wide wins from ~6 tiles per segment (TP=8 B=128 SHA), coop below (its AHA-DP copies, ~4)
# long segments (>= 40 tiles on average, up to 384 of them: TP=2/4 shards at
# B=1024) also stream faster on the wide shape, whole and packed
# longest-first (tools/probe_wide.py: TP=2 27.4 -> 24.7 us, TP=4 AHA-DP 17.1
# -> 15.8); a TP=1 layer (512 segments) stays on the 4-warp shape
WIDE_LONG_MAX_SEGMENTS = 384
WIDE_LONG_MIN_MEAN_TILES = 40


# Whole-segment schedule (one segment per CTA, no splits) vs the equal-cost
# split cut, by a linear model of the per-layer K4 time fitted on
# tools/probe_whole.py (the heaviest rank of TP=4/8 shards of the 70B
# workload, SHA / AHA-DP, B = 128..1024, 16 chained layers, profiles/):
#   split ~ S0 + 0.165 us per MB of the cache   (S0: launch, PDL release and
#           the split-segment merge tail -- record, acq_rel counter, L2 round
#           trips; larger for the 2-CTA-per-SM shape, more pieces)
#   whole ~ W0 + max(per-tile cost x the most loaded CTA's tiles (7
#           streaming warps ~0.1 us per 16-token tile, 3 ~0.285 us),
#           0.161 us per MB: HBM-bound once every SM is busy)
# The whole schedule also wins for a TP=1 layer of the bench workload (512
# segments, two per CTA longest-first: 47.1 -> 43.2 us, 6.2 TB/s): the
# split cut's merge tail costs more than the packing's imbalance.
#                        S0    W0   us per tile
WHOLE_MODEL = {"wide": (5.6, 3.3, 0.104), "coop": (7.6, 2.6, 0.285)}
SPLIT_US_PER_MB = 0.165
WHOLE_MARGIN_US = 0.5   # near a tie the split cut stays (TP=8 uniform TP, B=512: 8.7 vs 9.5 us)
WHOLE_US_PER_MB = 0.161  # the whole schedule is HBM-bound once every SM is busy (TP=1: 6.2 TB/s)
# at least two segments per CTA on average (a full grid of 4-warp CTAs, e.g.
# the Llama-3.1-8B shape at batch >= 128): every SM streams, the per-tile
# cost is the HBM share -- batch 128: whole 24.1 vs split 28.1 us per layer
WHOLE_FULL_PER_TILE_US = 0.20


def _whole_owners(seg_tiles, workers: int, sms: int) -> np.ndarray:
    """CTA id of each segment in the whole-segment schedule.  Up to `sms`
    segments: one per CTA, each on its own SM.  More: longest-first onto the
    least-loaded of `workers` CTAs (a CTA's load = its tiles + PAIR_PIECE_TILES
    per extra segment), then CTA ids relabelled so that CTA j and j + sms --
    which share an SM -- pair heavy with light (_pair_on_sms)."""
    import heapq
    seg_tiles = np.asarray(seg_tiles, dtype=np.int64)
    n = len(seg_tiles)
    if n <= sms:
        return np.arange(n, dtype=np.int64)
    owner = np.empty(n, dtype=np.int64)
    heap = [(0, w) for w in range(workers)]
    for s in np.lexsort((np.arange(n), -seg_tiles)):
        load, w = heapq.heappop(heap)
        owner[s] = w
        heapq.heappush(heap, (load + int(seg_tiles[s]) + (PAIR_PIECE_TILES if load else 0), w))
    _, owner = np.unique(owner, return_inverse=True)  # busy CTAs 0..k-1
    t1 = seg_tiles * TILE
    return _pair_on_sms(owner, np.zeros(n, dtype=np.int64), t1, sms)


def _whole_cta_tiles(seg_tiles, owner) -> np.ndarray:
    own = np.asarray(owner, dtype=np.int64)
    tiles = np.bincount(own, weights=np.asarray(seg_tiles, dtype=np.float64))
    extra = np.maximum(np.bincount(own) - 1, 0) * PAIR_PIECE_TILES
    return tiles + extra


def whole_segments_win(seg_tiles, workers: int, wide: bool, sms: int = NUM_SMS) -> bool:
    """Whole segments (one or a few per CTA) beat the split schedule (model
    above, with the most loaded CTA's tiles as the critical path)."""
    seg_tiles = np.asarray(seg_tiles, dtype=np.int64)
    n = len(seg_tiles)
    if not n or n > workers * MAX_WORK_PER_WORKER:
        return False
    s0, w0, per_tile = WHOLE_MODEL["wide" if wide else "coop"]
    if not wide and n >= 2 * workers:
        per_tile = WHOLE_FULL_PER_TILE_US
    if wide and n <= 32 and int(seg_tiles.max()) <= LONE_PREFETCH_TILES:
        # a few short segments: each CTA streams alone and its ring holds the
        # whole segment (Llama-3.1-8B shape at batch 1), tiles are cheap
        per_tile = HYBRID_LONE_TILE_US
    mb = float(seg_tiles.sum()) * TILE * HEAD_DIM * 4 / 1e6
    crit = float(_whole_cta_tiles(seg_tiles, _whole_owners(seg_tiles, workers, sms)).max())
    whole = w0 + max(per_tile * crit, WHOLE_US_PER_MB * mb)
    return whole + WHOLE_MARGIN_US <= s0 + SPLIT_US_PER_MB * mb


def plan_work_whole(seg_len, workers: int, sms: int):
    """Whole-segment schedule: every segment is one piece, on the CTA given
    by _whole_owners.  Same return convention as ``plan_work``."""
    seg_len = np.asarray(seg_len, dtype=np.int64)
    n = len(seg_len)
    owner = _whole_owners((seg_len + TILE - 1) // TILE, workers, sms)
    busy = int(owner.max()) + 1
    if np.bincount(owner).max() > MAX_WORK_PER_WORKER:
        raise ValueError("too many segments per CTA for the whole-segment schedule")
    item_seg = np.arange(n, dtype=np.int32)
    t0 = np.zeros(n, dtype=np.int32)
    t1 = seg_len.astype(np.int32)
    seg_item_ptr = np.arange(n + 1, dtype=np.int32)
    warp_ptr = np.zeros(busy + 1, dtype=np.int32)
    warp_ptr[1:] = np.cumsum(np.bincount(owner, minlength=busy))
    work_list = np.argsort(owner, kind="stable").astype(np.int32)
    return item_seg, t0, t1, seg_item_ptr, warp_ptr, work_list


def plan_work_hybrid(seg_len, workers: int, per_tile_us: float = 1.0, min_saving_us: float = 0.0):
    """Whole segments, except that the longest are cut into equal pieces so
    that no CTA streams more than T tiles, T the least (and >=
    HYBRID_MIN_PIECE_TILES) with sum_s ceil(tiles_s / T) <= workers, one
    piece per CTA: the longest segment no longer sets the launch's critical
    path (a lone CTA streams it at one SM's bandwidth), and only the cut
    segments need an LSE merge.  The cut is kept only if it shortens the
    critical path by more than ``min_saving_us`` at ``per_tile_us`` per tile
    (the merges' cost).  For at most `workers` segments (the SMs).  Same
    return convention as ``plan_work``."""
    seg_len = np.asarray(seg_len, dtype=np.int64)
    n = len(seg_len)
    tiles = np.maximum((seg_len + TILE - 1) // TILE, 1)
    hi = longest = int(tiles.max()) if n else 1
    lo = min(HYBRID_MIN_PIECE_TILES, hi)
    while lo < hi:
        T = (lo + hi) // 2
        if int((-(-tiles // T)).sum()) <= workers:
            hi = T
        else:
            lo = T + 1
    if per_tile_us * (longest - lo) <= min_saving_us:
        lo = longest  # the cut would not pay for its merges: whole segments
    k = np.minimum(-(-tiles // lo), MAX_ITEMS_PER_SEGMENT)
    item_seg = np.repeat(np.arange(n), k).astype(np.int32)
    ptr = np.zeros(n + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(k)
    j = np.arange(ptr[-1]) - np.repeat(ptr[:-1], k)
    kk = np.repeat(k, k)
    tt = np.repeat(tiles, k)
    t0 = (j * tt // kk) * TILE
    t1 = np.minimum(((j + 1) * tt // kk) * TILE, np.repeat(seg_len, k))
    t0 = np.minimum(t0, t1)
    n_items = len(item_seg)
    warp_ptr = np.arange(n_items + 1, dtype=np.int32)
    return (item_seg, t0.astype(np.int32), t1.astype(np.int32), ptr.astype(np.int32), warp_ptr,
            np.arange(n_items, dtype=np.int32))


_DEVICE_SHAPES: dict = {}  # device index -> (SMs, CTAs per SM of coop / wide / solo)
_PLAN_SCRATCH = __import__("threading").local()  # output buffers of fkv_plan_schedule, per thread


def _device_shapes(device):
    from . import _native
    try:
        idx = torch.device(device).index if device is not None else torch.cuda.current_device()
        idx = torch.cuda.current_device() if idx is None else idx
    except Exception:  # no device visible (host-side planning / CPU tests)
        idx = -1
    if idx not in _DEVICE_SHAPES:
        try:
            sms = torch.cuda.get_device_properties(idx).multi_processor_count
        except Exception:
            sms = NUM_SMS
        _DEVICE_SHAPES[idx] = (sms, *(int(_native.lib.fkv_decode_ctas_per_sm(f))
                                     for f in (0, FKV_DECODE_WIDE, FKV_DECODE_SOLO)))
    return _DEVICE_SHAPES[idx]


_SCHED_ENV = ("FKV_K4_SCHEDULE", "FKV_K4_WHOLE", "FKV_SOLO_SMALL", "FKV_SOLO_PIECE", "FKV_SOLO_WHOLE",
              "FKV_PIECE_COST", "FKV_SM_PAIRING", "FKV_PAIR_PIECE", "FKV_HYBRID_SAVING")
_SCHED_PARAMS: dict = {}  # (device, chunk, planner environment) -> (fkv_sched_params, SMs)


def _sched_params(device, chunk):
    """fkv_sched_params of the native planner: the device and the planner's
    environment knobs, as plan_schedule_py reads them (cached per device,
    chunk and environment: building it costs more than planning a small
    cache)."""
    import ctypes as C
    from . import _native
    env = os.environ
    key = (str(device), chunk, tuple(env.get(k) for k in _SCHED_ENV))
    hit = _SCHED_PARAMS.get(key)
    if hit is not None:
        return hit
    sms, c_coop, c_wide, c_solo = _device_shapes(device)
    mode = {"auto": 0, "coop": 1, "wide": 2, "solo": 3}.get(env.get("FKV_K4_SCHEDULE", "auto"), 0)
    whole = env.get("FKV_K4_WHOLE")
    prm = _native.SchedParams(
        sms=sms, ctas_coop=c_coop, ctas_wide=c_wide, ctas_solo=c_solo, mode=mode,
        whole=-1 if whole is None else (1 if whole == "1" else 0),
        solo_small=int(env.get("FKV_SOLO_SMALL") == "1"),
        solo_piece=int(env.get("FKV_SOLO_PIECE", -1)), solo_whole=int(env.get("FKV_SOLO_WHOLE", -1)),
        piece_cost=int(env.get("FKV_PIECE_COST", PIECE_COST_TILES)),
        sm_pairing=int(env.get("FKV_SM_PAIRING", "1") == "1"),
        chunk=-1 if chunk is None else int(chunk),
        pair_piece=float(env.get("FKV_PAIR_PIECE", PAIR_PIECE_TILES)),
        hybrid_saving_us=float(env.get("FKV_HYBRID_SAVING", HYBRID_MIN_SAVING_US)))
    if len(_SCHED_PARAMS) > 64:
        _SCHED_PARAMS.clear()
    _SCHED_PARAMS[key] = hit = (C.byref(prm), sms)
    return hit


def plan_schedule(seg_len, seg_row0, seg_qrow, seg_out_row, device=None, chunk: int | None = None):
    """Pick the K4 schedule for one cache and build its work table: the
    native planner (csrc/schedule.cpp, fkv_plan_schedule), bit-identical to
    ``plan_schedule_py`` below (tests/test_schedule_native.py), which
    FKV_PY_SCHEDULE=1 selects.  Same return value."""
    if os.environ.get("FKV_PY_SCHEDULE") == "1":
        return plan_schedule_py(seg_len, seg_row0, seg_qrow, seg_out_row, device, chunk)
    from . import _native
    i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731
    seg_len, seg_row0 = i64(seg_len), i64(seg_row0)
    seg_qrow, seg_out_row = i64(seg_qrow), i64(seg_out_row)
    n = len(seg_len)
    prm, sms = _sched_params(device, chunk)
    cap_items = max(1, n * MAX_ITEMS_PER_SEGMENT)
    cap_workers = max(1, 8 * sms)
    cap_table = cap_workers * MAX_WORK_PER_WORKER * 8
    sc = _PLAN_SCRATCH.__dict__  # reused across calls, one set per thread
    if sc.get("items", 0) < cap_items or sc.get("workers", 0) < cap_workers:
        sc.update(items=cap_items, workers=cap_workers,
                  out=[np.empty(cap_items, np.int32) for _ in range(4)],
                  wptr=np.empty(cap_workers + 1, np.int32), tab=np.empty(cap_table, np.int32))
    out, wptr, tab = sc["out"], sc["wptr"], sc["tab"]
    wlist = out[3]
    sptr = np.empty(n + 1, np.int32)
    sizes = np.zeros(5, np.int32)
    p = lambda a: a.ctypes.data  # noqa: E731
    rc = _native.lib.fkv_plan_schedule(
        p(seg_len), p(seg_row0), p(seg_qrow), p(seg_out_row), n, prm, cap_items, cap_workers, cap_table,
        p(out[0]), p(out[1]), p(out[2]), p(sptr), p(wptr), p(wlist), p(tab), p(sizes))
    if rc < 0:  # the same exception as the Python planner (e.g. too many segments for one launch)
        raise ValueError(_native.last_error())
    n_items, busy, rows, K, flags = (int(x) for x in sizes)
    return (out[0][:n_items].copy(), out[1][:n_items].copy(), out[2][:n_items].copy(), sptr,
            wptr[:busy + 1].copy(), wlist[:n_items].copy(), tab[:rows * K * 8].reshape(rows, K, 8).copy(), flags)


def plan_schedule_py(seg_len, seg_row0, seg_qrow, seg_out_row, device=None, chunk: int | None = None):
    """Pick the K4 schedule for one cache and build its work table.

    * default: the CTA-cooperative schedule, stream cut to equal *estimated
      time* per CTA (tiles + PIECE_COST_TILES per piece: a CTA with more,
      shorter pieces gets fewer tiles, and ranges prefer segment boundaries);
    * many short segments (at least one per warp and <= 24 tiles on average,
      or 0.4 per warp and <= 12 tiles): the per-warp ("solo") schedule,
      segments up to max(16, 2 x the per-warp share) kept whole and packed
      largest-first -- balanced with few LSE merges (Llama-3.1-8B shape at
      batch 256: 94 % of HBM);
    * FKV_SOLO_SMALL=1 additionally sends small caches (<= 19 tiles per CTA)
      to the solo schedule with 4-8-tile pieces (the choice before the
      piece-cost planner).
    * few segments of >= WIDE_MIN_MEAN_TILES tiles on average (<= WIDE_MAX_SEGMENTS, e.g. a TP=4/8
      rank's KV heads), or up to WIDE_LONG_MAX_SEGMENTS long ones (>=
      WIDE_LONG_MIN_MEAN_TILES, TP=2/4 shards at B=1024): the cooperative
      schedule with 8-warp CTAs (one per SM, seven streaming warps per piece).
    * cooperative schedules: one whole segment per CTA instead of the split
      cut when the model in ``whole_segments_win`` says the saved merge tail
      outweighs the longer critical segment (small TP shards).
    FKV_K4_SCHEDULE = coop | wide | solo | auto and FKV_K4_WHOLE = 0 | 1
    override (measurements).
    -> (item_seg, t0, t1, seg_item_ptr, warp_ptr, work_list, table, flags)."""
    import os
    seg_len = np.asarray(seg_len, dtype=np.int64)
    solo_ctas = default_workers(device, FKV_DECODE_SOLO)
    seg_tiles = (seg_len + TILE - 1) // TILE
    tiles = int(seg_tiles.sum())
    n_seg = len(seg_len)
    mode = os.environ.get("FKV_K4_SCHEDULE", "auto")
    small = tiles <= SOLO_MAX_TILES_PER_CTA * solo_ctas and os.environ.get("FKV_SOLO_SMALL") == "1"
    mean = tiles / n_seg if n_seg else 0
    warps = 4 * solo_ctas
    many_short = (n_seg >= warps and mean <= 24) or (n_seg >= 0.4 * warps and mean <= 12)
    solo = mode == "solo" or (mode == "auto" and chunk is None and (small or many_short))
    if solo:
        if small or mode == "solo" and not many_short:
            # piece / whole-segment thresholds grow with the cache: 4 tiles for a
            # few hundred tiles per GPU-layer, 8 near the crossover (probe_solo_params)
            pt = wt = int(np.clip(round(1.5 * tiles / warps), 4, 8))
        else:
            # pieces of at least 16 tiles, at least twice the per-warp share:
            # most segments stay whole, only the long tail is split
            pt = wt = max(16, -(-2 * tiles // warps))
        pt = int(os.environ.get("FKV_SOLO_PIECE", pt))
        wt = int(os.environ.get("FKV_SOLO_WHOLE", wt))
        try:
            plan = plan_work_solo(seg_len, warps, pt, wt)
            tab = work_table(seg_row0, seg_len, seg_qrow, seg_out_row, *plan, solo_ctas=solo_ctas)
            return (*plan, tab, FKV_DECODE_SOLO)
        except ValueError:
            pass  # too many pieces for the per-CTA tables: cooperative schedule
    # few segments (a TP-sharded rank's cache): 8-warp CTAs, seven streams per
    # piece; otherwise 4-warp CTAs, two per SM (tools/probe_sched.py)
    wide = mode == "wide" or (mode != "coop" and (
        (n_seg <= WIDE_MAX_SEGMENTS and mean >= WIDE_MIN_MEAN_TILES)
        or (n_seg <= WIDE_LONG_MAX_SEGMENTS and mean >= WIDE_LONG_MIN_MEAN_TILES)))
    flags = FKV_DECODE_WIDE if wide else 0
    workers = default_workers(device, flags)
    ctas_sm = max(1, workers // default_workers(device, FKV_DECODE_WIDE))
    whole = os.environ.get("FKV_K4_WHOLE")
    sms = workers // ctas_sm
    if chunk is None and 0 < n_seg <= workers * MAX_WORK_PER_WORKER and (
            whole == "1" or (whole is None and whole_segments_win(seg_tiles, workers, wide, sms))):
        # one whole segment per CTA: no split-segment LSE merges (their
        # record -> acq_rel counter -> L2 round trips sit in the launch's tail)
        if n_seg <= sms:  # one CTA per SM: the longest segments cut (few merges)
            per_tile = HYBRID_LONE_TILE_US if n_seg <= 32 else WHOLE_MODEL["wide" if wide else "coop"][2]
            plan = plan_work_hybrid(seg_len, sms, per_tile,
                                    float(os.environ.get("FKV_HYBRID_SAVING", HYBRID_MIN_SAVING_US)))
        else:
            plan = plan_work_whole(seg_len, workers, sms)
        tab = work_table(seg_row0, seg_len, seg_qrow, seg_out_row, *plan)
        return (*plan, tab, flags)
    plan = plan_work(seg_len, workers, chunk, sms=workers // ctas_sm if ctas_sm > 1 else None)
    tab = work_table(seg_row0, seg_len, seg_qrow, seg_out_row, *plan)
    return (*plan, tab, flags)


CT_PARTS = 17  # FKV_CT_PARTS: the parts of fkv_cache_tables' packed buffer, in its order


def _pack_tables_py(seg_len, seg_row0, seg_qrow, seg_out_row, seg_cap, append_src, device, chunk):
    """Python form of fkv_cache_tables (the checker; FKV_PY_SCHEDULE=1):
    plan_schedule_py plus the packing, same buffer, offsets and sizes."""
    seg_len = np.asarray(seg_len, dtype=np.int64)
    item_seg, t0, t1, ptr, wptr, wlist, tab, flags = plan_schedule_py(seg_len, seg_row0, seg_qrow,
                                                                      seg_out_row, device, chunk)
    # flat work-table index of every segment's last piece (append grows it)
    valid = (tab[:, :, 7] & 0xFFFF) != 0
    pos_of_item = np.zeros(max(len(item_seg), 1), dtype=np.int64)
    pos_of_item[tab[:, :, 5][valid]] = np.flatnonzero(valid.reshape(-1))
    last_piece = pos_of_item[np.asarray(ptr[1:], dtype=np.int64) - 1] if len(seg_len) else np.zeros(0)
    seg_cap = seg_len if seg_cap is None else np.asarray(seg_cap, dtype=np.int64)
    append_src = np.full(len(seg_len), -1) if append_src is None else np.asarray(append_src)
    parts = [np.ascontiguousarray(a, dtype=np.int32).reshape(-1) for a in (
        seg_len, seg_qrow, seg_out_row, item_seg, t0, t1, ptr, np.arange(ptr[-1]), wptr, wlist, tab,
        seg_cap, append_src, last_piece, np.zeros(max(len(item_seg), 1)), np.zeros(1),
        np.ascontiguousarray(seg_row0, dtype=np.int64).view(np.int32))]
    offs = np.cumsum([0] + [-(-len(a) // 4) * 4 for a in parts])
    host_buf = np.zeros(int(offs[-1]), dtype=np.int32)
    for a, o in zip(parts, offs[:-1]):
        host_buf[o:o + len(a)] = a
    return host_buf, offs, (len(item_seg), len(wptr) - 1, tab.shape[0], tab.shape[1], flags)


def cache_tables(seg_len, seg_row0, seg_qrow, seg_out_row, seg_cap=None, append_src=None, device=None,
                 chunk: int | None = None):
    """Plan one cache's K4 schedule and pack every int32 table it keeps on
    the device into one host buffer (fkv_cache_tables, csrc/schedule.cpp;
    ``_pack_tables_py`` is its Python form, FKV_PY_SCHEDULE=1).  Returns
    (int32 buffer, part offsets [CT_PARTS + 1] in words, (n_items, busy,
    rows, K, flags)).  The buffer is per-thread scratch, valid until the
    thread's next call."""
    if os.environ.get("FKV_PY_SCHEDULE") == "1":
        return _pack_tables_py(seg_len, seg_row0, seg_qrow, seg_out_row, seg_cap, append_src, device, chunk)
    from . import _native
    i64 = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731
    seg_len, seg_row0, seg_qrow, seg_out_row = i64(seg_len), i64(seg_row0), i64(seg_qrow), i64(seg_out_row)
    seg_cap, append_src = i64(seg_cap), i64(append_src)
    n = len(seg_len)
    prm, sms = _sched_params(device, chunk)
    items = max(1, n * MAX_ITEMS_PER_SEGMENT)
    words = 10 * n + 6 * items + 8 * sms + 8 * sms * MAX_WORK_PER_WORKER * 8 + 4 * (CT_PARTS + 2)
    sc = _PLAN_SCRATCH.__dict__
    if sc.get("ct_words", 0) < words:
        sc.update(ct_words=words, ct=np.empty(words, np.int32))
    buf = sc["ct"]
    offs = np.empty(CT_PARTS + 1, np.int64)
    sizes = np.zeros(5, np.int32)
    p = lambda a: None if a is None else a.ctypes.data  # noqa: E731
    rc = _native.lib.fkv_cache_tables(p(seg_len), p(seg_row0), p(seg_qrow), p(seg_out_row), p(seg_cap),
                                      p(append_src), n, prm, p(buf), len(buf), p(offs), p(sizes))
    if rc < 0:  # the same exception as the Python planner (e.g. too many segments for one launch)
        raise ValueError(_native.last_error())
    return buf[:int(offs[-1])], offs, tuple(int(x) for x in sizes)


def _part_lens(n: int, sizes) -> tuple:
    """Lengths of fkv_cache_tables' parts (FKV_CT_* order) for n segments."""
    n_items, busy, rows, K, _ = sizes
    return (n, n, n, n_items, n_items, n_items, n + 1, n_items, busy + 1, n_items, rows * K * 8,
            n, n, n, max(n_items, 1), 1, 2 * n)


def to_device_async(host: np.ndarray, device) -> torch.Tensor:
    """int32 host array -> device tensor with one host-to-device copy that does not stall the host: staged through
    torch's caching pinned-memory allocator (which keeps the staging block
    until the copy has run) and issued non-blocking on the current stream,
    so queuing a layer's tables never waits for the kernels before it."""
    device = torch.device(device)
    host = np.ascontiguousarray(host, dtype=np.int32)
    if device.type != "cuda":
        return torch.from_numpy(host.copy()).to(device)
    pin = torch.empty(host.shape, dtype=torch.int32, pin_memory=True)
    pin.numpy()[...] = host
    return pin.to(device, non_blocking=True)


_PART_NAMES = ("seg_len", "seg_qrow", "seg_out_row", "item_seg", "item_t0", "item_t1", "grp_ptr", "src_idx",
               "warp_ptr", "work_list", "work", "seg_cap_t", "append_src_t", "last_piece_t", "counters",
               "overflow_t", "seg_row0")  # FKV_CT_* order


class _Part:
    """A table of the cache's packed device buffer, viewed on first use (the
    kernels only need its address; building seventeen views per layer costs
    more host time than planning the layer)."""

    def __init__(self, i: int):
        self.i = i

    def __set_name__(self, owner, name):
        self.name = name

    def __get__(self, obj, owner=None):
        if obj is None:
            return self
        t = obj.tables[obj.offs[self.i]:obj.offs[self.i] + obj.lens[self.i]]
        if self.i == 16:        # SEG_ROW0: int64
            t = t.view(torch.int64)
        elif self.i == 10:      # WORK: fkv_work_t [workers, K, 8]
            t = t.view(obj.sizes[2], obj.sizes[3], 8)
        obj.__dict__[self.name] = t
        return t


@dataclass(eq=False)
class LayerCache:
    """Device-resident compressed cache + decode plan for one layer on one
    GPU: K/V storage plus every int32 table K3/K4/K5/append read, packed in
    one device buffer (fkv_cache_tables' layout) and exposed as views."""

    k: torch.Tensor
    v: torch.Tensor
    group: int
    tables: torch.Tensor      # int32, the packed parts
    offs: list                # word offset of each part
    lens: tuple               # length of each part (words; SEG_ROW0 counts int32 words)
    sizes: tuple              # (n_items, busy workers, work rows, K, schedule flags)
    host: dict = field(default_factory=dict, repr=False)

    seg_len = _Part(0)
    seg_qrow = _Part(1)
    seg_out_row = _Part(2)
    item_seg = _Part(3)
    item_t0 = _Part(4)
    item_t1 = _Part(5)
    grp_ptr = _Part(6)
    src_idx = _Part(7)
    warp_ptr = _Part(8)
    work_list = _Part(9)
    work = _Part(10)          # fkv_work_t [workers, K, 8] int32 (what K4 reads)
    seg_cap_t = _Part(11)
    append_src_t = _Part(12)
    last_piece_t = _Part(13)
    counters = _Part(14)      # int32 [n_items]
    overflow_t = _Part(15)
    seg_row0 = _Part(16)

    def ptr(self, part: int) -> int:
        """Device address of a part (FKV_CT_* index) without building its view."""
        return self.tables.data_ptr() + 4 * self.offs[part]

    @property
    def n_workers(self) -> int:
        return self.sizes[2]

    @property
    def flags(self) -> int:
        return self.sizes[4]

    @property
    def launch_flags(self) -> int:
        """Schedule flags plus FKV_DECODE_AFTER_WAIT once the cache has been
        written on the device (compaction, decode-time appends): the decode
        kernel then reads nothing before its programmatic-launch wait."""
        return self.sizes[4] | (FKV_DECODE_AFTER_WAIT if self.host.get("written") else 0)

    @property
    def work_k(self) -> int:
        return self.sizes[3]

    @property
    def n_items(self) -> int:
        return self.sizes[0]

    @property
    def n_segments(self) -> int:
        return self.lens[0]

    @property
    def retained_tokens(self) -> int:
        return int(self.host["seg_len"].sum())

    def kv_bytes(self) -> int:
        """Algorithmic K+V bytes one decode step reads from this cache."""
        return self.retained_tokens * HEAD_DIM * 2 * 2

    @staticmethod
    def allocate(seg_len, seg_qrow, seg_out_row, group: int, device, chunk: int | None = None,
                 fill: str = "zeros", generator: torch.Generator | None = None,
                 reserve: int = 0) -> "LayerCache":
        """Lay out segments and build the work plan.  ``fill='zeros'`` leaves
        the storage for the compaction kernel; ``fill='random'`` writes N(0,1)
        bf16 into every retained row (synthetic benchmark caches; the swizzle
        is a permutation, so random data needs no packing) and keeps padding
        rows zero.  ``reserve``: rows of headroom per segment for decode-time
        appends (``ops.append``; segment s receives row s of the step's
        [Bt, Hkv, 128] K/V)."""
        seg_len = np.asarray(seg_len, dtype=np.int64)
        cap = page_rows(seg_len + int(reserve))
        row0, rows = segment_offsets(seg_len + int(reserve))
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

        return LayerCache._build(k, v, row0, seg_len, seg_qrow, seg_out_row, group, chunk,
                                 seg_cap=cap, append_src=np.arange(len(seg_len)))

    @staticmethod
    def view(k: torch.Tensor, v: torch.Tensor, seg_row0, seg_len, seg_qrow, seg_out_row,
             group: int, chunk: int | None = None, seg_cap=None, append_src=None) -> "LayerCache":
        """A segment table over existing storage (e.g. the DP copies / shards
        of a base cache: each copy is a 16-aligned sub-range of its head's
        rows).  No data moves.  ``seg_cap`` / ``append_src``: append headroom
        and the K/V row each segment receives per decode step (-1: none, e.g.
        a DP copy that does not own the end of its head)."""
        seg_row0 = np.asarray(seg_row0, dtype=np.int64)
        seg_len = np.asarray(seg_len, dtype=np.int64)
        if np.any(seg_row0 % 16):
            raise ValueError("segment starts must be multiples of 16 rows")
        return LayerCache._build(k, v, seg_row0, seg_len, seg_qrow, seg_out_row, group, chunk,
                                 seg_cap=seg_cap, append_src=append_src)

    @staticmethod
    def allocate_many(layers, group: int, device, chunk: int | None = None, reserve: int = 0,
                      extra=None) -> "tuple[list[LayerCache], list[torch.Tensor]]":
        """``allocate`` (zero storage) for a stack of layers at once: one
        zero-filled K/V allocation for all of them, every layer's planned
        tables packed into one pinned buffer and sent in ONE host-to-device
        copy.  ``layers``: (seg_len, seg_qrow, seg_out_row) per layer.
        ``extra``: optional int32 host arrays that ride in the same copy (the
        compaction's segment tables); returned as device views."""
        dev = torch.device(device)
        plans, caps = [], []
        total_rows = 0
        if os.environ.get("FKV_PY_SCHEDULE") == "1":
            for seg_len, qrow, orow in layers:
                seg_len = np.asarray(seg_len, dtype=np.int64)
                row0, rows = segment_offsets(seg_len + int(reserve))  # rows of the layer's own K/V view
                caps.append((total_rows, rows))
                total_rows += rows
                plans.append(LayerCache._plan_host(row0, seg_len, qrow, orow, chunk, page_rows(seg_len + int(reserve)),
                                                   np.arange(len(seg_len)), dev, copy=True))
        else:  # the native planner straight into one scratch buffer, layer after layer
            from . import _native
            prm, _ = _sched_params(dev, chunk)
            fn = _native.lib.fkv_cache_tables
            sc = _PLAN_SCRATCH.__dict__
            scratch = sc.get("many")
            if scratch is None:
                scratch = sc["many"] = np.empty(1 << 20, np.int32)
            o = 0
            i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731
            for seg_len, qrow, orow in layers:
                seg_len, qrow, orow = i64(seg_len), i64(qrow), i64(orow)
                n = len(seg_len)
                cap = page_rows(seg_len + int(reserve))
                row0 = np.zeros(n, dtype=np.int64)
                if n:
                    np.cumsum(cap[:-1], out=row0[1:])
                rows = max(int(cap.sum()), PAGE)
                asrc = np.arange(n, dtype=np.int64)
                offs = np.zeros(CT_PARTS + 1, np.int64)  # a planning error leaves it zero
                sizes = np.zeros(5, np.int32)
                while True:
                    rc = fn(seg_len.ctypes.data, row0.ctypes.data, qrow.ctypes.data, orow.ctypes.data,
                            cap.ctypes.data, asrc.ctypes.data, n, prm, scratch.ctypes.data + 4 * o,
                            len(scratch) - o, offs.ctypes.data, sizes.ctypes.data)
                    if rc >= 0:
                        break
                    if offs[-1] + o <= len(scratch):  # not a buffer problem
                        raise ValueError(_native.last_error())
                    grown = np.empty(2 * (int(offs[-1]) + o), np.int32)
                    grown[:o] = scratch[:o]
                    scratch = sc["many"] = grown
                meta = {"seg_len": seg_len, "seg_row0": row0, "chunk": chunk, "seg_qrow": qrow,
                        "seg_out_row": orow, "seg_cap": cap}
                plans.append((o, offs, tuple(int(x) for x in sizes), meta))
                o += int(offs[-1])
                caps.append((total_rows, rows))
                total_rows += rows
        kv = torch.zeros((2, total_rows, HEAD_DIM), dtype=torch.bfloat16, device=dev)
        extra = [np.ascontiguousarray(e, dtype=np.int32).reshape(-1) for e in (extra or [])]
        words = [int(pl[1][-1]) for pl in plans] + [-(-len(e) // 4) * 4 for e in extra]
        host = np.zeros(sum(words), dtype=np.int32)
        o = 0
        for pl, w in zip(plans, words):
            host[o:o + w] = pl[0] if isinstance(pl[0], np.ndarray) else scratch[pl[0]:pl[0] + w]
            o += w
        for e, w in zip(extra, words[len(plans):]):
            host[o:o + len(e)] = e
            o += w
        buf = to_device_async(host, dev)
        caches = []
        o = 0
        for (_, offs, sz, meta), (r0, rows), w in zip(plans, caps, words):
            caches.append(LayerCache._assemble(kv[0, r0:r0 + rows], kv[1, r0:r0 + rows], group, buf, o, offs,
                                               sz, meta))
            o += w
        views = []
        for e, w in zip(extra, words[len(plans):]):
            views.append(buf[o:o + len(e)])
            o += w
        return caches, views

    @staticmethod
    def _plan_host(seg_row0, seg_len, seg_qrow, seg_out_row, chunk, seg_cap, append_src, dev, copy=False):
        seg_row0 = np.asarray(seg_row0, dtype=np.int64)
        seg_len = np.asarray(seg_len, dtype=np.int64)
        seg_cap = seg_len if seg_cap is None else np.asarray(seg_cap, dtype=np.int64)
        host_buf, offs, sizes = cache_tables(seg_len, seg_row0, seg_qrow, seg_out_row, seg_cap, append_src,
                                             dev, chunk)
        meta = {"seg_len": seg_len, "seg_row0": seg_row0, "chunk": chunk, "seg_qrow": np.asarray(seg_qrow),
                "seg_out_row": np.asarray(seg_out_row), "seg_cap": seg_cap}
        return (host_buf.copy() if copy else host_buf), offs, sizes, meta

    @staticmethod
    def _assemble(k, v, group, buf, base: int, offs, sizes, meta) -> "LayerCache":
        """The cache over its tables at word ``base`` of the device buffer."""
        return LayerCache(k=k, v=v, group=int(group), tables=buf, offs=[base + x for x in offs.tolist()],
                          lens=_part_lens(len(meta["seg_len"]), sizes), sizes=sizes,
                          host={**meta, "n_workers": sizes[1]})

    @staticmethod
    def _build(k, v, seg_row0, seg_len, seg_qrow, seg_out_row, group, chunk, seg_cap=None,
               append_src=None) -> "LayerCache":
        # every int32 table in one host buffer and one host-to-device copy
        # (fifteen small copies cost more than the planning itself)
        host_buf, offs, sizes, meta = LayerCache._plan_host(seg_row0, seg_len, seg_qrow, seg_out_row, chunk,
                                                            seg_cap, append_src, k.device)
        return LayerCache._assemble(k, v, group, to_device_async(host_buf, k.device), 0, offs, sizes, meta)

    def sync_lengths(self) -> np.ndarray:
        """Read the device segment lengths back (after appends) into host state."""
        self.host["seg_len"] = self.seg_len.cpu().numpy().astype(np.int64)
        return self.host["seg_len"]
