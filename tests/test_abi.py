"""The C-ABI library loads on a CPU-only host and exports exactly what
include/fairkv.h declares; errors map onto the reference's exception
classes.  (No compute calls here -- those need the GPU.)"""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "fairkv.h").read_text()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(fkv_\w+)\(", text, re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for name in ("fkv_solve_equal_split", "fkv_solve_free_split", "fkv_select_best",
                 "fkv_optimize_plan", "fkv_decode", "fkv_decode_exchange", "fkv_merge_lse",
                 "fkv_merge_wait", "fkv_snapkv_score", "fkv_snapkv_select",
                 "fkv_ada_budgets", "fkv_topk_select", "fkv_compact", "fkv_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2502_15804_b200 import _native
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert not _native.missing_symbols()
    assert lib.fkv_version() >= 1


def test_error_codes_map_to_reference_exceptions():
    import paper_2502_15804_b200 as fk
    from paper_2502_15804_b200 import _native
    with pytest.raises(fk.NativeError):
        _native.check(-1)
    with pytest.raises(fk.InfeasibleError):
        _native.check(-4)
    with pytest.raises(fk.SearchSpaceError):
        _native.check(-5)
    # a real failing call: tp that does not divide the copy count
    rc = _native.lib.fkv_solve_equal_split(None, None, 3, 2, 1.0, 10, None, None, None, None, None)
    assert rc < 0 and "null" in _native.last_error()


def test_ops_refuse_cpu_tensors():
    import torch
    from paper_2502_15804_b200 import ops
    from paper_2502_15804_b200.errors import NativeError
    with pytest.raises(NativeError):
        ops.budgets(torch.zeros(1, 8, 100), 64, 32)


def _prototypes():
    """name -> parameter count of every function fairkv.h declares."""
    text = (ROOT / "include" / "fairkv.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"^(?:int|int64_t|const char\*)\s+(fkv_\w+)\(([^;]*?)\);", text, re.M | re.S):
        params = m.group(2).strip()
        out[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_ctypes_signatures_match_the_header():
    """Every function the Python binding declares has the header's argument
    count (a drifted prototype would pass garbage through ctypes)."""
    from paper_2502_15804_b200 import _native
    protos = _prototypes()
    for name, (_res, args) in _native._SIGS.items():
        assert name in protos, f"{name} bound in _native.py but not declared in fairkv.h"
        assert len(args) == protos[name], f"{name}: {len(args)} ctypes args vs {protos[name]} in fairkv.h"
