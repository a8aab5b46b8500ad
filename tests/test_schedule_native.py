"""The native K4 schedule planner (csrc/schedule.cpp, fkv_plan_schedule)
against its Python form (cache.plan_schedule_py): every output -- pieces,
pointers, work list, the fkv_work_t table and the chosen CTA shape -- equal,
on random caches across the size range (a TP=8 rank's few heads to a TP=1
batch-64 layer), skewed and empty segments, every schedule override and the
chunked path.  CPU only."""

import numpy as np
import pytest

from paper_2502_15804_b200 import cache as C


def _segments(rng, n, mean):
    kind = rng.integers(3)
    if kind == 0:
        lens = rng.integers(0, 2 * mean + 1, n)
    elif kind == 1:  # dirichlet-skewed, like Ada budgets
        lens = np.round(rng.dirichlet(np.full(n, 2.0)) * mean * n).astype(np.int64)
    else:  # a few very long segments among short ones
        lens = rng.integers(0, mean // 4 + 1, n)
        lens[rng.integers(0, n, max(1, n // 10))] = rng.integers(mean, 8 * mean + 1)
    return lens.astype(np.int64)


def _check(lens, chunk=None):
    row0, _ = C.segment_offsets(lens)
    qrow = np.arange(len(lens), dtype=np.int64) * 8
    orow = qrow[::-1].copy()
    got = C.plan_schedule(lens, row0, qrow, orow, None, chunk)
    want = C.plan_schedule_py(lens, row0, qrow, orow, None, chunk)
    names = ("item_seg", "t0", "t1", "seg_item_ptr", "warp_ptr", "work_list", "table")
    for nm, a, b in zip(names, got[:7], want[:7]):
        np.testing.assert_array_equal(np.asarray(a), np.asarray(b), err_msg=nm)
    assert got[7] == want[7], "flags"
    return got[7]


@pytest.mark.parametrize("seed", range(12))
def test_native_matches_python_random(seed):
    rng = np.random.default_rng(seed)
    seen = set()
    for n, mean in ((8, 1024), (16, 300), (64, 1024), (130, 700), (512, 1024), (1100, 120), (2048, 40),
                    (5, 3), (300, 2000)):
        seen.add(_check(_segments(rng, n, mean)))
    assert len(seen) >= 2  # several CTA shapes exercised


@pytest.mark.parametrize("env", [{"FKV_K4_SCHEDULE": "coop"}, {"FKV_K4_SCHEDULE": "wide"},
                                 {"FKV_K4_SCHEDULE": "solo"}, {"FKV_K4_WHOLE": "1"}, {"FKV_K4_WHOLE": "0"},
                                 {"FKV_SOLO_SMALL": "1"}, {"FKV_PIECE_COST": "0"}, {"FKV_SM_PAIRING": "0"},
                                 {"FKV_PAIR_PIECE": "7.5"}, {"FKV_SOLO_PIECE": "6", "FKV_SOLO_WHOLE": "9"}])
def test_native_matches_python_overrides(monkeypatch, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(99)
    for n, mean in ((8, 1024), (64, 500), (512, 1024), (1500, 60), (200, 5)):
        _check(_segments(rng, n, mean))


@pytest.mark.parametrize("chunk", [16, 100, 512, 4096])
def test_native_matches_python_chunked(chunk):
    rng = np.random.default_rng(chunk)
    for n, mean in ((8, 1024), (64, 3000), (300, 200)):
        _check(_segments(rng, n, mean), chunk)


def test_native_edge_cases():
    _check(np.zeros(0, dtype=np.int64))
    _check(np.zeros(7, dtype=np.int64))
    _check(np.array([1], dtype=np.int64))
    _check(np.array([100000], dtype=np.int64))  # one very long segment: many pieces
    _check(np.full(296 * 32, 1, dtype=np.int64))  # at the piece cap of a launch


def test_native_errors_match():
    # more segments than one launch can hold: both planners refuse
    lens = np.ones(148 * 8 * 32 + 5000, dtype=np.int64)
    row0, _ = C.segment_offsets(lens)
    q = np.zeros(len(lens), dtype=np.int64)
    with pytest.raises(ValueError):
        C.plan_schedule_py(lens, row0, q, q)
    from paper_2502_15804_b200.errors import NativeError
    with pytest.raises((ValueError, NativeError)):
        C.plan_schedule(lens, row0, q, q)


def _check_tables(lens, chunk=None, cap=None, asrc=None):
    row0, _ = C.segment_offsets(lens)
    qrow = np.arange(len(lens), dtype=np.int64) * 8
    orow = qrow[::-1].copy()
    got, goff, gsz = C.cache_tables(lens, row0, qrow, orow, cap, asrc, None, chunk)
    want, woff, wsz = C._pack_tables_py(lens, row0, qrow, orow, cap, asrc, None, chunk)
    assert gsz == wsz
    np.testing.assert_array_equal(goff, woff)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("seed", range(6))
def test_packed_tables_match_python(seed):
    """fkv_cache_tables (schedule + every device table of a LayerCache in one
    buffer) against the Python packing, with and without append headroom."""
    rng = np.random.default_rng(100 + seed)
    for n, mean in ((8, 1024), (64, 500), (512, 1024), (1100, 120), (5, 3)):
        lens = _segments(rng, n, mean)
        _check_tables(lens)
        _check_tables(lens, cap=C.page_rows(lens + 16), asrc=np.arange(n))
        src = rng.integers(-1, n, n)
        _check_tables(lens, chunk=256, cap=lens + rng.integers(0, 64, n), asrc=src)
    _check_tables(np.zeros(0, dtype=np.int64))
    _check_tables(np.zeros(9, dtype=np.int64))


def test_layer_cache_tables_on_cpu():
    """LayerCache built from the packed buffer: every view equals the Python
    planner's tables (CPU storage: the packing, not the kernels)."""
    rng = np.random.default_rng(7)
    lens = _segments(rng, 96, 700)
    qrow = np.arange(96, dtype=np.int64) * 8
    cache = C.LayerCache.allocate(lens, qrow, qrow, 8, "cpu", reserve=16)
    row0, _ = C.segment_offsets(lens + 16)
    item_seg, t0, t1, ptr, wptr, wlist, tab, flags = C.plan_schedule_py(lens, row0, qrow, qrow)
    for t, want in ((cache.item_seg, item_seg), (cache.item_t0, t0), (cache.item_t1, t1), (cache.grp_ptr, ptr),
                    (cache.warp_ptr, wptr), (cache.work_list, wlist), (cache.work, tab),
                    (cache.seg_len, lens), (cache.seg_row0, row0), (cache.src_idx, np.arange(len(item_seg)))):
        np.testing.assert_array_equal(t.numpy(), want)
    assert cache.flags == flags and cache.n_workers == len(wptr) - 1
    assert int(cache.counters.abs().sum()) == 0 and int(cache.overflow_t[0]) == 0
    np.testing.assert_array_equal(cache.seg_cap_t.numpy(), C.page_rows(lens + 16))


def test_allocate_many_matches_allocate():
    """LayerCache.allocate_many (one K/V allocation, every layer's tables in
    one copy, extra arrays riding along) == allocate per layer."""
    import torch
    rng = np.random.default_rng(11)
    layers = []
    for n, mean in ((8, 300), (40, 1000), (8, 3)):
        lens = _segments(rng, n, mean)
        q = np.arange(n, dtype=np.int64) * 4
        layers.append((lens, q, q[::-1].copy()))
    extra = [np.arange(5), np.full(3, 7)]
    caches, views = C.LayerCache.allocate_many(layers, 4, "cpu", reserve=32, extra=extra)
    for c, (lens, q, o) in zip(caches, layers):
        ref = C.LayerCache.allocate(lens, q, o, 4, "cpu", reserve=32)
        for name in ("seg_row0", "seg_len", "seg_qrow", "seg_out_row", "item_seg", "item_t0", "item_t1",
                     "grp_ptr", "src_idx", "warp_ptr", "work_list", "work", "counters"):
            assert torch.equal(getattr(c, name), getattr(ref, name)), name
        for name in ("seg_cap_t", "append_src_t", "last_piece_t", "overflow_t"):
            assert torch.equal(getattr(c, name), getattr(ref, name)), name
        assert c.k.shape == ref.k.shape and c.flags == ref.flags and c.n_workers == ref.n_workers
        assert c.k.is_contiguous() and int(c.k.abs().sum()) == 0
    for vw, e in zip(views, extra):
        np.testing.assert_array_equal(vw.numpy(), e)


def test_allocate_many_grows_scratch_and_reports_errors():
    """More tables than the planner scratch holds: it grows and the result is
    unchanged; a stack with an unplannable layer raises the planner's error."""
    import torch
    rng = np.random.default_rng(5)
    C._PLAN_SCRATCH.__dict__["many"] = np.empty(64, np.int32)  # force growth
    layers = [(lens, np.arange(len(lens)) * 8, np.arange(len(lens)) * 8)
              for lens in (_segments(rng, 300, 800) for _ in range(4))]
    caches, _ = C.LayerCache.allocate_many(layers, 8, "cpu")
    for c, (lens, q, o) in zip(caches, layers):
        ref = C.LayerCache.allocate(lens, q, o, 8, "cpu")
        assert torch.equal(c.work, ref.work) and torch.equal(c.grp_ptr, ref.grp_ptr)
    bad = np.ones(148 * 8 * 32 + 5000, dtype=np.int64)
    with pytest.raises(ValueError):
        C.LayerCache.allocate_many([layers[0], (bad, np.zeros_like(bad), np.zeros_like(bad))], 8, "cpu")


def test_schedule_shape_rules(monkeypatch):
    """The CTA-shape / whole-segment rules, identically in both planners:
    a few short segments that fit a wide CTA's rings -> wide, whole (8B
    batch 1); up to 384 long segments -> wide (TP=2/4 shards at B=1024); a
    TP=1 layer of 512 long segments -> the 4-warp shape; at most one
    segment per SM with a dominant one -> the long one is cut."""
    rng = np.random.default_rng(3)
    short = rng.integers(200, 300, 8)                 # 8 segments of ~16 tiles
    assert _check(short) == C.FKV_DECODE_WIDE
    row0, _ = C.segment_offsets(short)
    q = np.arange(8, dtype=np.int64)
    plan = C.plan_schedule(short, row0, q, q)
    assert len(plan[0]) == 8                          # whole: one piece per segment
    long_ = rng.integers(700, 1400, 256)              # 256 segments of ~65 tiles
    assert _check(long_) == C.FKV_DECODE_WIDE
    tp1 = rng.integers(700, 1400, 512)
    assert _check(tp1) == 0
    # whole-segment schedule, at most one segment per SM: the longest are cut
    # into equal pieces, one per SM, the dominant one most
    monkeypatch.setenv("FKV_K4_WHOLE", "1")
    cut = np.concatenate([rng.integers(600, 700, 120), [3000]])
    assert _check(cut) == C.FKV_DECODE_WIDE
    row0, _ = C.segment_offsets(cut)
    q = np.arange(len(cut), dtype=np.int64)
    item_seg, t0, t1, _, warp_ptr = C.plan_schedule(cut, row0, q, q)[:5]
    per_seg = np.bincount(item_seg)
    assert per_seg[-1] == per_seg.max() > 2 and len(item_seg) <= C.NUM_SMS
    assert (np.diff(warp_ptr) == 1).all()             # one piece per CTA
    assert (t1 - t0).max() <= 3000 // 2


def test_cache_tables_c_contract():
    """fkv_cache_tables through the C ABI: a short buffer is refused with the
    needed size in part_off[FKV_CT_PARTS] (and nothing written), a buffer of
    exactly that size is accepted; parts are 16-byte aligned and ordered."""
    from paper_2502_15804_b200 import _native
    lens = np.array([100, 0, 2000, 33], dtype=np.int64)
    row0, _ = C.segment_offsets(lens)
    q = np.arange(4, dtype=np.int64) * 8
    prm, _ = C._sched_params(None, None)
    offs = np.zeros(C.CT_PARTS + 1, np.int64)
    sizes = np.zeros(5, np.int32)
    small = np.full(8, -7, np.int32)
    p = lambda a: a.ctypes.data  # noqa: E731
    rc = _native.lib.fkv_cache_tables(p(lens), p(row0), p(q), p(q), None, None, 4, prm, p(small), len(small),
                                      p(offs), p(sizes))
    assert rc == -1 and offs[-1] > len(small) and (small == -7).all()
    buf = np.empty(int(offs[-1]), np.int32)
    rc = _native.lib.fkv_cache_tables(p(lens), p(row0), p(q), p(q), None, None, 4, prm, p(buf), len(buf),
                                      p(offs), p(sizes))
    assert rc == 0 and (offs % 4 == 0).all() and (np.diff(offs) >= 0).all()
    np.testing.assert_array_equal(buf[offs[0]:offs[0] + 4], lens)                 # SEG_LEN
    np.testing.assert_array_equal(buf[offs[11]:offs[11] + 4], lens)               # SEG_CAP defaults to seg_len
    np.testing.assert_array_equal(buf[offs[12]:offs[12] + 4], [-1] * 4)           # APPEND_SRC defaults to -1
    np.testing.assert_array_equal(buf[offs[16]:offs[16] + 8].view(np.int64), row0)  # SEG_ROW0 as int64
