"""Search-kernel plugin registry (drop-in for pkg/src/headbalance/_kernel/__init__.py:1-57).

One backend, reported as ``"compiled"`` like the reference's compiled
kernel: the C++ planner inside libfairkv.so.  The
reference's pure-Python kernel is not part of this product; its CPU
restatement lives in ``oracle/`` and is used only by the tests as the
checker.  ``HEADBALANCE_KERNEL`` keeps the reference's spelling: unset /
"auto" / "native" / "compiled" / "c" / "ext" select the native kernel; asking
for the Python kernel ("python", "py", "pure", "reference") fails loudly
instead of silently running something else; any other value is a
``ValueError`` as in the reference (_kernel/__init__.py:28-29).
"""

import os

from . import native
from .native import DEFAULT_NODE_BUDGET

_NATIVE_NAMES = {"", "auto", "native", "compiled", "c", "ext"}
_PY_NAMES = {"python", "py", "pure", "reference"}

_choice = os.environ.get("HEADBALANCE_KERNEL", "").strip().lower()
if _choice in _PY_NAMES:
    raise ImportError(
        "HEADBALANCE_KERNEL selects the pure-Python kernel, which this B200 build does not ship; "
        "unset it (the native C++ kernel is bit-identical, including node counts)"
    )
if _choice not in _NATIVE_NAMES:
    raise ValueError(f"unrecognized HEADBALANCE_KERNEL value: {_choice!r}")


def backend() -> str:
    """Name of the active kernel backend: "compiled", as the reference names
    its compiled kernel (_kernel/__init__.py:32-34) -- this one is the C++
    planner in libfairkv.so."""
    return "compiled"


def implementations() -> dict:
    """All kernel implementations shipped, for parity tests and benchmarks
    (reference _kernel/__init__.py:37-46; the pure-Python kernel is not
    shipped -- tests bring it as the checker)."""
    return {"compiled": native}


def solve_equal_split(weights, heads, tp, cutoff, node_budget=DEFAULT_NODE_BUDGET, hint=None):
    return native.solve_equal_split(weights, heads, tp, cutoff, node_budget, hint)


def solve_free_split(weights, heads, tp, cutoff, node_budget=DEFAULT_NODE_BUDGET, hint=None):
    return native.solve_free_split(weights, heads, tp, cutoff, node_budget, hint)
