"""Host-side decode schedule (cache.plan_work) invariants -- CPU only."""

import numpy as np
import pytest

from paper_2502_15804_b200.cache import (MAX_ITEMS_PER_SEGMENT, MAX_WORK_PER_WORKER, plan_work,
                                         segment_offsets, work_table)


@pytest.mark.parametrize("chunk", [None, 64, 100, 512])
@pytest.mark.parametrize("workers", [300, 1184])
def test_plan_covers_each_segment_once(chunk, workers):
    _plan_covers(chunk, workers)


def test_tiny_plan_respects_piece_caps():
    # few tiles, many workers: pieces must not shrink below min_tiles / exceed
    # MAX_ITEMS_PER_SEGMENT per segment (the kernel's merge scratch)
    item_seg, t0, t1, sptr, wptr, wlist = plan_work([333, 1, 666], 296)
    assert np.diff(sptr).max() <= MAX_ITEMS_PER_SEGMENT
    for s in range(3):
        its = list(range(sptr[s], sptr[s + 1]))
        assert all(t1[i] - t0[i] >= 16 * 8 for i in its[:-1])  # only a segment's tail is short


def _plan_covers(chunk, workers):
    rng = np.random.default_rng(workers + (chunk or 0))
    seg_len = rng.integers(0, 3000, size=300)
    seg_len[:3] = [0, 1, 16]
    item_seg, t0, t1, sptr, wptr, wlist = plan_work(seg_len, workers, chunk)
    assert wptr[0] == 0 and wptr[-1] == len(item_seg) and (np.diff(wptr) >= 0).all()
    assert sorted(wlist.tolist()) == list(range(len(item_seg)))
    assert sptr[-1] == len(item_seg)
    assert (t0 % 16 == 0).all()
    for s in range(len(seg_len)):
        its = range(sptr[s], sptr[s + 1])
        assert len(its) >= 1 and len(its) <= MAX_ITEMS_PER_SEGMENT
        assert all(item_seg[i] == s for i in its)
        spans = [(t0[i], t1[i]) for i in its]
        assert spans[0][0] == 0 and spans[-1][1] == seg_len[s]
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert len(wptr) - 1 <= workers and np.diff(wptr).max() <= MAX_WORK_PER_WORKER


def test_piece_cap_and_infeasible_plans():
    # many tiny (and empty) segments next to one long one: the per-worker
    # piece cap (FKV_MAX_WORK) binds, not the tile count
    seg_len = np.concatenate([[40000], np.zeros(2000, dtype=np.int64), np.full(3000, 16)])
    item_seg, t0, t1, sptr, wptr, wlist = plan_work(seg_len, 1184)
    assert np.diff(wptr).max() <= MAX_WORK_PER_WORKER and len(wptr) - 1 <= 1184
    assert sorted(wlist.tolist()) == list(range(len(item_seg)))
    with pytest.raises(ValueError):
        plan_work(np.zeros(1184 * MAX_WORK_PER_WORKER + 1, dtype=np.int64), 1184)


def test_work_table_matches_plan():
    rng = np.random.default_rng(3)
    seg_len = rng.integers(0, 2000, size=200)
    row0, _ = segment_offsets(seg_len)
    qrow = np.arange(200) * 8
    orow = np.arange(200) * 8 + 1
    item_seg, t0, t1, sptr, wptr, wlist = plan_work(seg_len, 1184)
    tab = work_table(row0, seg_len, qrow, orow, item_seg, t0, t1, sptr, wptr, wlist)
    assert tab.shape == (len(wptr) - 1, np.diff(wptr).max(), 8)
    seen = []
    for w in range(tab.shape[0]):
        for j in range(tab.shape[1]):
            e = tab[w, j]
            if e[7] == 0:
                assert j >= wptr[w + 1] - wptr[w]
                continue
            it = wlist[wptr[w] + j]
            s = item_seg[it]
            r0 = int(np.uint32(e[0].view(np.uint32))) + (int(e[1]) << 32)
            assert r0 == row0[s] + t0[it] and e[2] == t1[it] - t0[it]
            assert (e[3], e[4], e[5], e[6], e[7]) == (qrow[s], orow[s], it, sptr[s], sptr[s + 1] - sptr[s])
            seen.append(it)
    assert sorted(seen) == list(range(len(item_seg)))


def test_balanced_plan_equalises_tiles_per_worker():
    rng = np.random.default_rng(0)
    seg_len = rng.integers(300, 3000, size=512)
    W = 1184
    item_seg, t0, t1, sptr, wptr, wlist = plan_work(seg_len, W, piece_cost=0)
    tiles = -(-(t1 - t0) // 16)
    assert len(wptr) - 1 <= W
    per = np.array([tiles[wlist[wptr[w]:wptr[w + 1]]].sum() for w in range(len(wptr) - 1)])
    assert per.max() <= -(-tiles.sum() // W) + 1


def test_piece_cost_plan_balances_estimated_time():
    """Default coop planner: equal (tiles + P * pieces) per worker -- a worker
    with more pieces gets fewer tiles; pieces prefer segment boundaries."""
    from paper_2502_15804_b200.cache import PIECE_COST_TILES as P
    rng = np.random.default_rng(1)
    seg_len = rng.integers(100, 3000, size=512)
    W = 296
    item_seg, t0, t1, sptr, wptr, wlist = plan_work(seg_len, W)
    tiles = -(-(t1 - t0) // 16)
    busy = len(wptr) - 1
    assert busy <= W and sorted(wlist.tolist()) == list(range(len(item_seg)))
    cost = np.array([tiles[wlist[wptr[w]:wptr[w + 1]]].sum() + P * (wptr[w + 1] - wptr[w])
                     for w in range(busy)])
    ideal = (tiles.sum() + P * len(item_seg)) / busy
    assert cost.max() <= 1.15 * ideal + P
    # fewer split segments than the equal-tiles cut
    eq = plan_work(seg_len, W, piece_cost=0)
    assert (np.diff(sptr) > 1).sum() <= (np.diff(eq[3]) > 1).sum()


def test_segment_offsets_page_aligned():
    row0, total = segment_offsets([0, 1, 64, 65])
    assert row0.tolist() == [0, 0, 64, 128] and total == 256


def _check_plan(seg_len, item_seg, t0, t1, sptr, wptr, wlist):
    assert sorted(wlist.tolist()) == list(range(len(item_seg)))
    assert (t0 % 16 == 0).all() and np.diff(wptr).max() <= MAX_WORK_PER_WORKER
    for s in range(len(seg_len)):
        its = range(sptr[s], sptr[s + 1])
        assert 1 <= len(its) <= MAX_ITEMS_PER_SEGMENT and all(item_seg[i] == s for i in its)
        spans = [(t0[i], t1[i]) for i in its]
        assert spans[0][0] == 0 and spans[-1][1] == seg_len[s]
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


@pytest.mark.parametrize("workers", [8, 64, 1184])
def test_solo_plan_segment_aligned(workers):
    """Per-warp planner: short segments stay whole (no merge), long ones are
    cut into near-equal pieces; every piece on one worker."""
    from paper_2502_15804_b200.cache import plan_work_solo
    rng = np.random.default_rng(workers)
    seg_len = np.concatenate([rng.integers(0, 384, size=200), rng.integers(2000, 9000, size=20)])
    item_seg, t0, t1, sptr, wptr, wlist = plan_work_solo(seg_len, workers)
    _check_plan(seg_len, item_seg, t0, t1, sptr, wptr, wlist)
    n_pieces = np.diff(sptr)
    assert (n_pieces[seg_len <= 24 * 16] == 1).all()
    if workers == 1184:  # enough workers: long segments are spread
        assert (n_pieces[seg_len >= 2000] > 1).all()
    assert len(wptr) - 1 <= workers


def test_solo_work_table_tags_warps():
    """Per-warp schedule: worker w -> warp w // ctas of CTA w % ctas, tagged
    in the high half of n_it; every piece appears once."""
    from paper_2502_15804_b200.cache import work_table
    rng = np.random.default_rng(4)
    seg_len = rng.integers(16, 300, size=64)
    row0, _ = segment_offsets(seg_len)
    qrow = np.arange(64) * 8
    ctas = 296
    item_seg, t0, t1, sptr, wptr, wlist = plan_work(seg_len, 4 * ctas, min_tiles=2)
    _check_plan(seg_len, item_seg, t0, t1, sptr, wptr, wlist)
    tab = work_table(row0, seg_len, qrow, qrow, item_seg, t0, t1, sptr, wptr, wlist, solo_ctas=ctas)
    busy = len(wptr) - 1
    assert tab.shape[0] == min(ctas, busy)
    seen = []
    for c in range(tab.shape[0]):
        for e in tab[c]:
            if e[7] == 0:
                continue
            w = (e[7] >> 16) * tab.shape[0] + c
            it = int(e[5])
            assert wptr[w] <= list(wlist).index(it) < wptr[w + 1]
            assert (e[7] & 0xffff) == sptr[item_seg[it] + 1] - sptr[item_seg[it]]
            seen.append(it)
    assert sorted(seen) == list(range(len(item_seg)))


def test_sm_pairing_is_a_permutation_that_balances_sms():
    """_pair_on_sms relabels workers (every piece kept, ids 0..busy-1) so the
    two CTAs sharing an SM (j, j + sms) carry similar work."""
    from paper_2502_15804_b200.cache import plan_work
    rng = np.random.default_rng(3)
    seg = rng.integers(200, 2000, 512)
    a = plan_work(seg, 296)
    b = plan_work(seg, 296, sms=148)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert len(b[4]) == len(a[4])
    def per_worker_tiles(plan):
        item_seg, t0, t1, _, wp, wl = plan
        return np.array([((t1[wl[wp[w]:wp[w + 1]]] - t0[wl[wp[w]:wp[w + 1]]] + 15) // 16).sum()
                         for w in range(len(wp) - 1)])
    ta, tb = per_worker_tiles(a), per_worker_tiles(b)
    assert sorted(ta) == sorted(tb)
    sm_a = ta[:148] + np.append(ta[148:], np.zeros(296 - len(ta)))[:148]
    sm_b = tb[:148] + np.append(tb[148:], np.zeros(296 - len(tb)))[:148]
    assert sm_b.max() - sm_b.min() <= sm_a.max() - sm_a.min()


def test_whole_segment_plan_and_choice():
    """plan_work_whole: every segment is exactly one piece; up to one segment
    per SM each gets its own CTA; with more, longest-first onto the least
    loaded of the CTAs and CTA j / j + sms (one SM) paired heavy with light.
    The choice model picks it for small TP shards and keeps the split cut for
    long segments and for a TP=1 layer."""
    from paper_2502_15804_b200.cache import (_whole_cta_tiles, _whole_owners, plan_work_whole,
                                             whole_segments_win, work_table)
    rng = np.random.default_rng(4)
    sms, workers = 148, 296
    for n in (100, 200, 400):
        seg_len = rng.integers(0, 2000, size=n)
        item_seg, t0, t1, ptr, warp_ptr, work_list = plan_work_whole(seg_len, workers, sms)
        assert np.array_equal(item_seg, np.arange(n)) and (t0 == 0).all() and np.array_equal(t1, seg_len)
        assert np.array_equal(ptr, np.arange(n + 1))
        tiles = (seg_len + 15) // 16
        own = _whole_owners(tiles, workers, sms)
        busy = int(own.max()) + 1
        assert busy <= workers and sorted(set(own.tolist())) == list(range(busy))
        cta = _whole_cta_tiles(tiles, own)
        if n <= sms:
            assert np.array_equal(own, np.arange(n))
        else:  # LPT bound: no CTA above the mean share + the longest segment (+ piece costs)
            assert cta.max() <= tiles.sum() / workers + tiles.max() + 12 * 2
        tab = work_table(np.arange(n) * 2048, seg_len, np.arange(n) * 8, np.arange(n) * 8,
                         item_seg, t0, t1, ptr, warp_ptr, work_list)
        assert tab.shape[0] == busy and (tab[:, :, 7][tab[:, :, 7] > 0] == 1).all()
        assert sorted(tab[:, :, 5][tab[:, :, 7] > 0].tolist()) == list(range(n))
    # TP=8 rank at B=256 (64 segments of ~18 tiles) and a TP=1 layer (512
    # segments, two per CTA): whole; one long segment among short ones, or 64
    # long segments on 148 SMs (uniform TP=8, B=1024): split
    assert whole_segments_win(np.full(64, 18), 148, True)
    assert whole_segments_win(np.full(512, 64), 296, False)
    assert not whole_segments_win(np.r_[np.full(63, 40), 200], 148, True)
    assert not whole_segments_win(np.full(64, 120), 148, True)
