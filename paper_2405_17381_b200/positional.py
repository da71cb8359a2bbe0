"""Per-head decay schedule -- the source of lam for every call (positional.py:39-84).

lam[h][l] = exp(-(8h/H)(1 - l/L)), 1-indexed head h and layer l; frozen.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import DomainError


def decay_rate(h: int, l: int, H: int, L: int, temperature: bool = True) -> float:
    """positional.py:39-50."""
    if not (1 <= h <= H):
        raise DomainError(f"head index {h} outside 1..{H}")
    if not (1 <= l <= L):
        raise DomainError(f"layer index {l} outside 1..{L}")
    scale = (1.0 - l / L) if temperature else 1.0
    return math.exp(-(8.0 * h / H) * scale)


@dataclass(frozen=True)
class DecaySchedule:
    """Frozen (H, L) table of decay rates (positional.py:53-84)."""

    H: int
    L: int
    temperature: bool = True
    table: np.ndarray = field(default=None, repr=False)

    @classmethod
    def build(cls, H: int, L: int, temperature: bool = True) -> "DecaySchedule":
        if H < 1 or L < 1:
            raise DomainError(f"need H >= 1 and L >= 1, got H={H}, L={L}")
        t = np.array([[decay_rate(h, l, H, L, temperature) for l in range(1, L + 1)] for h in range(1, H + 1)],
                     dtype=np.float64)
        t.setflags(write=False)
        return cls(H=H, L=L, temperature=temperature, table=t)

    def rate(self, h: int, l: int) -> float:
        if not (1 <= h <= self.H and 1 <= l <= self.L):
            raise DomainError(f"(h={h}, l={l}) outside 1..{self.H} x 1..{self.L}")
        return float(self.table[h - 1, l - 1])

    def layer(self, l: int) -> np.ndarray:
        """All heads' decays for layer l -- the ``lam`` vector one batched call takes."""
        if not (1 <= l <= self.L):
            raise DomainError(f"layer index {l} outside 1..{self.L}")
        return self.table[:, l - 1].copy()
