"""Error hierarchy of the drop-in planning API.

Names and inheritance follow the reference package so callers that catch
``HeadBalanceError`` subclasses keep working unchanged
(reference: pkg/src/headbalance/errors.py:4-29).  The native library reports
failures through negative return codes plus ``fkv_last_error()``; the ctypes
shim in ``_native.py`` maps those codes onto these classes.
"""

__all__ = [
    "HeadBalanceError",
    "ParseError",
    "ValidationError",
    "InfeasibleError",
    "SearchSpaceError",
    "CalibrationError",
    "SimulationError",
    "NativeError",
]


class HeadBalanceError(Exception):
    """Root of every domain error raised by this package."""


class ParseError(HeadBalanceError):
    """A profile / plan / model / sample file is not parseable at all."""


class ValidationError(HeadBalanceError):
    """A value parsed fine but breaks a structural invariant."""


class InfeasibleError(HeadBalanceError):
    """The requested placement cannot exist (too few copies, too many GPUs...)."""


class SearchSpaceError(HeadBalanceError):
    """Replication-scheme enumeration would exceed its cap."""


class CalibrationError(HeadBalanceError):
    """The latency-law least-squares fit cannot be made or is degenerate."""


class SimulationError(HeadBalanceError):
    """Inputs to the synchronous decode walk disagree with each other."""


class NativeError(HeadBalanceError):
    """The CUDA / C++ library rejected a call (bad shape, launch failure...)."""
