"""Prior parameter object (reference model.py:33-54).

Only the parameter validation lives on the host; every density evaluation
on the hot path runs in libspa_b200 (K2 prior/reweight kernels).
`a = math.inf` selects the double-exponential (Bayesian-lasso) limit
explicitly (the reference evaluates inf*log1p(0) = nan there).
"""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class GtPrior:
    """Centred L1 generalised-t prior with degrees of freedom a and scale c."""

    a: float
    c: float

    def __post_init__(self):
        if not self.a > 0:
            raise ValueError(f"degrees of freedom must be positive, got a={self.a}")
        if not self.c > 0 or math.isinf(self.c):
            raise ValueError(f"scale must be positive, got c={self.c}")

    @property
    def b(self) -> float:
        return self.a * self.c

    @property
    def lambda_de(self) -> float:
        return 1.0 / self.c
