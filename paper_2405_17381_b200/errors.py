"""Exception classes of the reference API (matrixops.py:28-33), kept by name.

Both subclass ValueError, as in the reference, so callers that catch the
reference's errors keep working after switching to this package.
"""


class ShapeError(ValueError):
    """Operands have incompatible or malformed shapes."""


class DomainError(ValueError):
    """A scalar argument or result lies outside its legal domain."""


def check_decay(lam: float) -> float:
    """Reject decay rates outside (0, 1] (matrixops.py:72-77)."""
    lam = float(lam)
    if not (0.0 < lam <= 1.0):
        raise DomainError(f"decay rate must lie in (0, 1], got {lam}")
    return lam
