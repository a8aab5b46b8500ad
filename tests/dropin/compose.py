"""Compose the reference's off-hot-path modules over this package -- TEST
INFRASTRUCTURE ONLY.

The reference package ``headbalance`` (pkg/src/headbalance) is, by module:

* on the hot path, rebuilt here: ``errors``, ``profiles``,
  ``schemes``, ``allocate`` and the ``_kernel`` plugin (the C++ planner);
* off it (OUT OF SCOPE): the analytic latency law (``latency``),
  the decode simulator (``simulate``), ``manifest`` and the ``cli``.

A user switching to this package keeps the second group as it is.  This
module shows that works: it loads the reference's own source files of the
second group *as submodules of this package*, so their relative imports
(``from .allocate import ...``) resolve to the rebuilt modules, and
``alias_as_headbalance`` registers the result under the name ``headbalance``
so the reference's unmodified test suite can import it.  Nothing here is
copied: the files are read from the installed reference (baseline/_ref) or
from /root/reference at test time.
"""

from __future__ import annotations

import importlib
import importlib.util
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
SOURCES = (ROOT / "baseline" / "_ref" / "headbalance", Path("/root/reference/pkg/src/headbalance"))
PKG = "paper_2502_15804_b200"
HOT = ("errors", "profiles", "schemes", "allocate", "_kernel")
OFF = ("latency", "manifest", "simulate", "cli")
_DEPS = {"simulate": ("latency",), "cli": ("latency", "manifest", "simulate")}


def reference_file(name: str) -> Path | None:
    for d in SOURCES:
        if (d / f"{name}.py").exists():
            return d / f"{name}.py"
    return None


def available() -> bool:
    return all(reference_file(n) is not None for n in OFF)


def off_path_module(name: str):
    """The reference's module ``name`` (one of OFF) loaded as
    ``paper_2502_15804_b200.<name>`` over the rebuilt hot-path modules."""
    full = f"{PKG}.{name}"
    if full in sys.modules:
        return sys.modules[full]
    for dep in _DEPS.get(name, ()):
        off_path_module(dep)
    if name == "simulate":
        # simulate.compare reads DEFAULT_NODE_BUDGET from _kernel.reference
        # (pkg/src/headbalance/simulate.py:193); the product's value is the same
        py = reference_python_kernel()
        kern = importlib.import_module(f"{PKG}._kernel")
        assert py is not None and py.DEFAULT_NODE_BUDGET == kern.DEFAULT_NODE_BUDGET
        sys.modules.setdefault(f"{PKG}._kernel.reference", py)
    src = reference_file(name)
    if src is None:
        raise ImportError(f"reference module {name}.py not found in {[str(s) for s in SOURCES]}")
    pkg = importlib.import_module(PKG)
    spec = importlib.util.spec_from_file_location(full, src)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[full] = mod
    spec.loader.exec_module(mod)
    setattr(pkg, name, mod)
    return mod


def reference_python_kernel():
    """The reference's pure-Python search kernel (_kernel/reference.py), the
    checker the reference's backend-parity tests compare against."""
    for d in SOURCES:
        f = d / "_kernel" / "reference.py"
        if f.exists():
            spec = importlib.util.spec_from_file_location("_headbalance_python_kernel", f)
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    return None


def alias_as_headbalance():
    """Register this package (+ the reference's off-path modules) as
    ``headbalance``.  The kernel registry keeps the product's single
    "compiled" backend and gains the reference's Python kernel as "python"
    for the parity tests (the reference ships both, _kernel/__init__.py:37-46)."""
    pkg = importlib.import_module(PKG)
    sys.modules["headbalance"] = pkg
    for name in HOT:
        sys.modules[f"headbalance.{name}"] = importlib.import_module(f"{PKG}.{name}")
    for name in OFF:
        sys.modules[f"headbalance.{name}"] = off_path_module(name)
    kern = sys.modules["headbalance._kernel"]
    py = reference_python_kernel()
    if py is not None:
        impls = dict(kern.implementations())
        impls["python"] = py
        kern.implementations = lambda: dict(impls)
    # the reference's package-level re-exports of the off-path modules
    # (pkg/src/headbalance/__init__.py:8-70)
    for name in OFF:
        mod = sys.modules[f"headbalance.{name}"]
        for sym, obj in list(vars(mod).items()):
            if not sym.startswith("_") and getattr(obj, "__module__", None) == mod.__name__ \
                    and not hasattr(pkg, sym):
                setattr(pkg, sym, obj)
    return pkg
