"""ctypes binding of libfairkv.so (the C ABI in include/fairkv.h).

The library is loaded eagerly and must be present: there is no Python or
CPU fallback for anything behind this module.  A missing library raises
``ImportError`` naming the build command.  Failing calls raise the
``errors`` class matching the C return code, with ``fkv_last_error()`` as
message.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import errors

LIB_PATH = Path(os.environ.get("FAIRKV_LIB", Path(__file__).resolve().parent / "libfairkv.so"))

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2502_15804_b200/csrc/build.py` "
        "(or __graft_entry__.build()); this package has no fallback path"
    )

def _check_fresh() -> None:
    """Refuse a library built from other sources than the ones next to it
    (a stale prebuilt binary in a snapshot): its embedded source hash must
    equal the hash of csrc/ + include/ (csrc/build.py).  Skipped when the
    sources are not shipped, or FAIRKV_LIB points elsewhere on purpose."""
    if "FAIRKV_LIB" in os.environ:
        return
    from .csrc import build as _build
    if not all((_build.CSRC / n).exists() for n in _build.CU_SOURCES + _build.CXX_SOURCES):
        return
    have, want = _build.embedded_hash(LIB_PATH), _build.source_hash()
    if have != want:
        raise ImportError(
            f"{LIB_PATH} was built from different sources (embedded hash {have}, sources {want}); "
            "rebuild with `python paper_2502_15804_b200/csrc/build.py` (or __graft_entry__.build())")


_check_fresh()
lib = C.CDLL(str(LIB_PATH))  # CDLL releases the GIL for the duration of each call

_i32, _i64, _f32, _f64, _vp = C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_void_p


class SchedParams(C.Structure):
    """fkv_sched_params (include/fairkv.h)."""
    _fields_ = [(n, C.c_int32) for n in ("sms", "ctas_coop", "ctas_wide", "ctas_solo", "mode", "whole",
                                         "solo_small", "solo_piece", "solo_whole", "piece_cost",
                                         "sm_pairing", "chunk")] + [("pair_piece", C.c_double), ("hybrid_saving_us", C.c_double)]
_pi32, _pi64, _pf64 = C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_f64)

_SIGS = {
    "fkv_last_error": (C.c_char_p, []),
    "fkv_version": (C.c_int, []),
    "fkv_source_hash": (C.c_char_p, []),
    "fkv_solve_equal_split": (C.c_int, [_vp, _vp, _i32, _i32, _f64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "fkv_solve_free_split": (C.c_int, [_vp, _vp, _i32, _i32, _f64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "fkv_select_best": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i64, _i64,
                                  _vp, _vp, _vp, _vp, _vp]),
    "fkv_optimize_plan": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _i64, _i64, _i32,
                                    _vp, _vp, _vp, _vp, _vp]),
    "fkv_decode_ctas_per_sm": (C.c_int, [_i32]),
    "fkv_plan_schedule": (C.c_int, [_vp, _vp, _vp, _vp, _i32, _vp, _i32, _i32, _i32,
                                    _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fkv_cache_tables": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _i64, _vp, _vp]),
    "fkv_decode": (C.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _f32, _vp, _vp,
                             _vp, _vp, _i32, _vp, _vp]),
    "fkv_merge_lse": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp]),
    "fkv_decode_exchange": (C.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _f32,
                                      _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp]),
    "fkv_merge_wait": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "fkv_dev_alloc": (C.c_int, [_i64, _vp]),
    "fkv_dev_free": (C.c_int, [_vp]),
    "fkv_ipc_get": (C.c_int, [_vp, _vp]),
    "fkv_ipc_open": (C.c_int, [_vp, _vp]),
    "fkv_ipc_close": (C.c_int, [_vp]),
    "fkv_host_device_ptr": (C.c_int, [_vp, _vp]),
    "fkv_snapkv_score": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _f32, _vp, _vp,
                                   _vp]),
    "fkv_score_workspace_bytes": (C.c_int64, [_i32, _i32, _i32, _i32, _i32]),
    "fkv_snapkv_select": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _f32, _i32, _i32,
                                    _vp, _vp, _vp, _vp, _vp, _vp]),
    "fkv_ada_budgets": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "fkv_ada_select_workspace_bytes": (C.c_int64, [_i32, _i32, _i32]),
    "fkv_ada_select": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "fkv_topk_select": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "fkv_append": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp]),
    "fkv_compact": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp,
                              _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    fn = getattr(lib, _name, None)
    if fn is None:
        continue  # entry points of later kernels; absence is reported by `missing_symbols`
    fn.restype = _res
    fn.argtypes = _args

_CODE_TO_EXC = {
    -1: errors.NativeError,
    -2: errors.NativeError,
    -3: errors.ValidationError,
    -4: errors.InfeasibleError,
    -5: errors.SearchSpaceError,
}


def missing_symbols() -> list[str]:
    return [n for n in EXPORTED if getattr(lib, n, None) is None]


def last_error() -> str:
    msg = lib.fkv_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> int:
    """Raise the mapped error for a negative return code, else pass rc through."""
    if rc < 0:
        raise _CODE_TO_EXC.get(rc, errors.NativeError)(last_error() or f"fairkv error {rc}")
    return rc


def ptr(x) -> int | None:
    """Device/host address of a torch tensor or numpy array (None passes NULL)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data
