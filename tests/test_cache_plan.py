"""Host-side decode schedule (cache.plan_work) invariants -- CPU only."""

import numpy as np
import pytest

from paper_2502_15804_b200.cache import MAX_ITEMS_PER_SEGMENT, plan_work, segment_offsets


@pytest.mark.parametrize("chunk", [None, 64, 100, 512])
@pytest.mark.parametrize("workers", [1, 7, 1184])
def test_plan_covers_each_segment_once(chunk, workers):
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


def test_balanced_plan_equalises_tiles_per_worker():
    rng = np.random.default_rng(0)
    seg_len = rng.integers(300, 3000, size=512)
    W = 1184
    item_seg, t0, t1, sptr, wptr, wlist = plan_work(seg_len, W)
    tiles = -(-(t1 - t0) // 16)
    assert len(wptr) - 1 <= W
    per = np.array([tiles[wlist[wptr[w]:wptr[w + 1]]].sum() for w in range(len(wptr) - 1)])
    assert per.max() <= -(-tiles.sum() // W) + 1


def test_segment_offsets_page_aligned():
    row0, total = segment_offsets([0, 1, 64, 65])
    assert row0.tolist() == [0, 0, 64, 128] and total == 256
