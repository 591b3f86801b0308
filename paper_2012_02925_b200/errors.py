"""Exception taxonomy of the drop-in.

Mirrors blockflow/errors.py:4-45 so callers written against the reference
catch the same names.  When the reference package is already loaded in the
process (``blockflow.errors`` in ``sys.modules``), :func:`raise_as` raises an
exception that is an instance of BOTH the local class and the reference's
class of the same name, so ``pytest.raises(blockflow.errors.X)`` written for
the CPU path also catches the GPU path.
"""

from __future__ import annotations

import sys


class BlockflowError(Exception):
    """Base class (errors.py:4)."""


class GridFormatError(BlockflowError):
    """Malformed grid input (errors.py:8)."""


class MetricError(BlockflowError):
    """Inverted cell / bad metrics (errors.py:12)."""


class NonPhysicalStateError(BlockflowError):
    """rho <= 0 or p <= 0 in a face state or an update (errors.py:16)."""


class DecompositionError(BlockflowError):
    """Decomposition constraints cannot be met (errors.py:20)."""


class TopologyError(BlockflowError):
    """Inconsistent connectivity (errors.py:24)."""


class DeadlockError(BlockflowError):
    """Exchange made no progress (errors.py:28-37)."""

    def __init__(self, message, blocked=None):
        super().__init__(message)
        self.blocked = tuple(blocked or ())


class DivergenceError(BlockflowError):
    """Residual blew up (errors.py:40)."""


class ConfigError(BlockflowError):
    """Invalid configuration (errors.py:44)."""


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or failed; there is no CPU fallback."""


_BRIDGED = {}


def bridged(cls):
    """The class to raise for `cls`: itself, or a subclass that also derives
    from the reference's class of the same name when the reference is loaded."""
    ref = sys.modules.get("blockflow.errors")
    ref_cls = getattr(ref, cls.__name__, None) if ref is not None else None
    if ref_cls is None or not isinstance(ref_cls, type) or issubclass(cls, ref_cls):
        return cls
    key = (cls, ref_cls)
    if key not in _BRIDGED:
        _BRIDGED[key] = type(cls.__name__, (cls, ref_cls), {"__module__": cls.__module__})
    return _BRIDGED[key]


def raise_as(cls, message):
    raise bridged(cls)(message)


__all__ = ["BlockflowError", "GridFormatError", "MetricError", "NonPhysicalStateError",
           "DecompositionError", "TopologyError", "DeadlockError", "DivergenceError",
           "ConfigError", "NativeLibraryError", "bridged", "raise_as"]
