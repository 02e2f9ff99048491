"""Error types of the engine, named after the reference hierarchy
(reference ``pkg/src/gradflow/errors.py:11-132``) so callers can catch the
same conditions by the same names.

When the reference package is importable in the host process, every class
here also derives from its reference counterpart, so ``except
gradflow.errors.DomainError`` keeps working for code that switches to this
engine. The reference is never imported on its own initiative: only if a
``gradflow`` package is already installed.
"""
from __future__ import annotations

import importlib.util

_ref = None
if importlib.util.find_spec("gradflow") is not None:  # pragma: no cover - environment dependent
    try:
        import gradflow.errors as _ref  # type: ignore
    except Exception:
        _ref = None


def _bases(name: str, *local):
    ref = getattr(_ref, name, None) if _ref is not None else None
    if ref is None or any(issubclass(b, ref) for b in local):
        return local
    # a local base that the reference class already derives from (Exception)
    # is replaced by the reference class to keep the MRO consistent
    kept = tuple(b for b in local if not issubclass(ref, b))
    return kept + (ref,)


class GradflowError(*_bases("GradflowError", Exception)):
    """Base class of every engine error."""


def _mk(name: str, doc: str, base=GradflowError):
    cls = type(name, _bases(name, base), {"__doc__": doc, "__module__": __name__})
    globals()[name] = cls
    return cls


ProgramSyntaxError = _mk("ProgramSyntaxError", "Malformed program text or expression.")
UnboundName = _mk("UnboundName", "A name was referenced with no binding in scope.")
DomainError = _mk("DomainError", "Arithmetic outside an operation's domain; raised eagerly, never a silent NaN.")
ShapeMismatch = _mk("ShapeMismatch", "Concrete array shapes incompatible with an operation.")
OutOfBounds = _mk("OutOfBounds", "A subset expression evaluated outside the array's extent.")
NonTermination = _mk("NonTermination", "A loop exceeded the trip guard (GRADFLOW_TRIP_LIMIT).")
MissingTapeValue = _mk("MissingTapeValue", "The reverse pass needed a recorded value the tape does not hold.")
UnresolvableTripCount = _mk("UnresolvableTripCount", "A trip count was required statically but is data dependent.")
UnsupportedLoop = _mk("UnsupportedLoop", "Loop shape outside the supported reversal classes.")
UnsupportedConstruct = _mk("UnsupportedConstruct", "A recognized construct this engine deliberately rejects.")
MissingInverse = _mk("MissingInverse", "A non-affine loop reversal required a declared inverse or a tape.")
BatchDivergence = _mk("BatchDivergence", "A branch condition disagreed across the batch axis.")
PathExplosion = _mk("PathExplosion", "Control-flow path enumeration exceeded its cap.")


class Infeasible(*_bases("Infeasible", GradflowError)):
    """No store/recompute assignment satisfies the memory limit."""

    def __init__(self, message: str, min_peak_bytes: int | None = None):
        self.min_peak_bytes = min_peak_bytes
        super().__init__(message)


class EngineError(GradflowError):
    """The CUDA engine failed (missing extension, launch error)."""


__all__ = [
    "GradflowError", "ProgramSyntaxError", "UnboundName", "DomainError", "ShapeMismatch", "OutOfBounds",
    "NonTermination", "MissingTapeValue", "UnresolvableTripCount", "UnsupportedLoop",
    "UnsupportedConstruct", "MissingInverse", "BatchDivergence", "PathExplosion", "Infeasible",
    "EngineError",
]
