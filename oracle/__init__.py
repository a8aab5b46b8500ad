"""CPU oracle for the FairKV hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import anything under ``oracle/``, and only as
the checker or the timed CPU reference, never as the product path.

Contents
--------
planner.py   float64 restatement of the reference AHA search
             (pkg/src/headbalance/_kernel/reference.py, allocate.py).
             PINNED: golden vectors produced by the reference itself
             (tests/golden/planner_golden.json, tests/golden/make_golden.py) and,
             where /root/reference exists, live comparison with it.
kv.py        numpy float64 restatement of Ada-SnapKV scoring, the Ada
             cross-head budget split, per-head top-k, page-aligned compaction,
             decode attention and the LSE merge.  PARITY UNPINNED against the
             reference: the reference contains none of these and
             its paper's dependency (KVPress AdaKV) is neither
             vendored nor pinned.  The restatement follows the published
             SnapKV / Ada-KV algorithms with the parameters fixed in DESIGN.md
             and is cross-checked against an independent implementation
             (torch scaled_dot_product_attention in float64) in the tests.
_ref/        (git-ignored) the reference's own compiled search kernel,
             built from /root/reference by oracle/Makefile.
"""
