"""B1 drop-in: the reference's search-kernel module interface
(``solve_equal_split`` / ``solve_free_split`` with the argument meaning and
return shape of pkg/src/headbalance/_kernel/reference.py:80-100) served by the
C++ planner in libfairkv.so.

Returns ``((spread, rgs_list), nodes)`` or ``(None, nodes)``; never raises
for infeasibility, exactly like the reference.  Inputs are copied into
contiguous buffers owned by this call (the reference copies into malloc'd
scratch, _fastpath.pyx:150-226); the GIL is released while the search runs.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .. import _native

DEFAULT_NODE_BUDGET = 200_000


def _call(fn, weights, heads, tp, cutoff, node_budget, hint):
    w = np.ascontiguousarray(weights, dtype=np.float64)
    h = np.ascontiguousarray(heads, dtype=np.int32)
    m = int(w.shape[0])
    if h.shape[0] != m:
        raise ValueError(f"{m} weights but {h.shape[0]} head ids")
    out_rgs = np.zeros(max(m, 1), dtype=np.int32)
    out_spread = C.c_double(0.0)
    out_nodes = C.c_int64(0)
    if hint is not None:
        hs = C.c_double(float(hint[0]))
        hr = np.ascontiguousarray(hint[1], dtype=np.int32)
        if hr.shape[0] != m:
            raise ValueError("hint assignment length differs from the copy count")
        hint_args = (C.addressof(hs), hr.ctypes.data)
    else:
        hint_args = (None, None)
    rc = _native.check(fn(w.ctypes.data, h.ctypes.data, m, int(tp), float(cutoff),
                          int(node_budget), *hint_args, C.addressof(out_spread),
                          out_rgs.ctypes.data, C.addressof(out_nodes)))
    nodes = int(out_nodes.value)
    if rc == 0:
        return None, nodes
    return (float(out_spread.value), [int(x) for x in out_rgs[:m]]), nodes


def solve_equal_split(weights, heads, tp, cutoff, node_budget=DEFAULT_NODE_BUDGET, hint=None):
    """Equal-cardinality B&B (reference _kernel/reference.py:80-235)."""
    return _call(_native.lib.fkv_solve_equal_split, weights, heads, tp, cutoff, node_budget, hint)


def solve_free_split(weights, heads, tp, cutoff, node_budget=DEFAULT_NODE_BUDGET, hint=None):
    """Nonempty-groups B&B (reference _kernel/reference.py:238-340)."""
    return _call(_native.lib.fkv_solve_free_split, weights, heads, tp, cutoff, node_budget, hint)
