"""Input side of the hot path: the `Dataset` type and the synthetic generator.

`run_sampler` accepts any object with `X` [n x p] float64, `y` [n] in {0,1}
and `names` (duck-typed, so the reference's own `spa.data.Dataset` objects
are accepted unchanged).  The generator below restates the reference's
synthetic LD-blocked genotype recipe (reference data.py:113-174) so that the
bench can build the named configurations (BASELINE.json configs C1-C5)
without the reference installed; bit-identity with the reference generator
is pinned by a golden hash (tests/golden/make_golden.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


class DataError(ValueError):
    """Malformed dataset or simulation spec (reference data.py:22-23)."""


@dataclass
class Dataset:
    """Standardised design matrix with a binary response (reference
    data.py:26-66; the same validation rules and error type)."""

    X: np.ndarray
    y: np.ndarray
    names: list

    def __post_init__(self):
        self.X = np.asarray(self.X, dtype=np.float64)
        self.y = np.asarray(self.y, dtype=np.float64)
        if self.X.ndim != 2:
            raise DataError(f"X must be 2-d, got shape {self.X.shape}")
        n, p = self.X.shape
        if self.y.shape != (n,):
            raise DataError(f"y has shape {self.y.shape}, expected ({n},)")
        if len(self.names) != p:
            raise DataError(f"{len(self.names)} names for {p} columns")
        if not np.all((self.y == 0.0) | (self.y == 1.0)):
            raise DataError("response values must all be 0 or 1")
        mu = self.X.mean(axis=0)
        sd = self.X.std(axis=0, ddof=1) if n > 1 else np.ones(p)
        bad = np.flatnonzero((np.abs(mu) > 1e-10) | (np.abs(sd - 1.0) > 1e-10))
        if bad.size:
            j = bad[0]
            raise DataError(f"column {self.names[j]} is not standardized (mean {mu[j]:.3e}, sd {sd[j]:.6f})")

    @property
    def n(self) -> int:
        return self.X.shape[0]

    @property
    def p(self) -> int:
        return self.X.shape[1]


@dataclass
class SimSpec:
    """Recipe for one simulated dataset (reference data.py:69-105)."""

    n: int
    p: int
    block_size: int = 10
    within_block_corr: float = 0.0
    nonzero: list = field(default_factory=list)
    seed: int = 0

    def __post_init__(self):
        if self.n < 1 or self.p < 1:
            raise DataError(f"need n >= 1 and p >= 1, got n={self.n}, p={self.p}")
        if not 1 <= self.block_size <= self.p:
            raise DataError(f"block_size must lie in [1, p], got {self.block_size}")
        if not 0.0 <= self.within_block_corr < 1.0:
            raise DataError(f"within-block correlation must lie in [0, 1), got {self.within_block_corr}")
        idx = [i for i, _ in self.nonzero]
        if len(set(idx)) != len(idx) or any(not 1 <= i <= self.p for i in idx):
            raise DataError("nonzero indices must be unique and within [1, p]")


def marker_names(p: int) -> list:
    w = max(3, len(str(p)))
    return [f"snp_{j + 1:0{w}d}" for j in range(p)]


def genotype_counts(spec: SimSpec) -> np.ndarray:
    """Minor-allele counts in {0,1,2}: a shared latent Gaussian per LD block
    cut at Hardy-Weinberg thresholds (reference data.py:113-128)."""
    from scipy.special import ndtri

    rng = np.random.default_rng([spec.seed, 0])
    f = rng.uniform(0.1, 0.5, size=spec.p)
    nblk = -(-spec.p // spec.block_size)
    shared = rng.standard_normal((spec.n, nblk))
    own = rng.standard_normal((spec.n, spec.p))
    r = spec.within_block_corr
    latent = math.sqrt(r) * shared[:, np.arange(spec.p) // spec.block_size] + math.sqrt(1.0 - r) * own
    hom_major = (1.0 - f) ** 2
    cut1 = ndtri(hom_major)
    cut2 = ndtri(hom_major + 2.0 * f * (1.0 - f))
    return (latent > cut1).astype(np.float64) + (latent > cut2)


def standardize(G: np.ndarray) -> np.ndarray:
    """Column centring and unit sample-sd scaling (reference data.py:131-140)."""
    G = np.asarray(G, dtype=np.float64)
    sd = G.std(axis=0, ddof=1)
    if np.any(sd == 0.0):
        raise DataError(f"column {int(np.flatnonzero(sd == 0.0)[0])} is constant and cannot be standardized")
    return (G - G.mean(axis=0)) / sd


def simulate_dataset(spec: SimSpec):
    """Genotypes -> standardise -> phenotypes y ~ Bernoulli(expit(X beta*))
    (reference data.py:143-174).  Returns (Dataset, beta_true)."""
    from scipy.special import expit

    X = standardize(genotype_counts(spec))
    beta = np.zeros(spec.p)
    for idx, v in spec.nonzero:
        beta[idx - 1] = v
    rng = np.random.default_rng([spec.seed, 2])
    y = (rng.random(spec.n) < expit(X @ beta)).astype(np.float64)
    return Dataset(X, y, marker_names(spec.p)), beta


_EFFECTS = (-0.2538, 0.4578, -0.1873, -0.1498, 0.0996)  # paper's five signals


def named_spec(name: str) -> SimSpec:
    """The BASELINE.json configurations (SURVEY.md section 8(d) recipes)."""
    name = name.lower()
    if name == "c1":
        return SimSpec(500, 20, 5, 0.3, [(2, 0.45), (8, -0.4), (14, 0.35)], seed=101)
    if name == "c2":
        return SimSpec(2000, 200, 8, 0.6, list(zip((108, 22, 5, 117, 162), _EFFECTS)), seed=18)
    if name in ("c3", "c4"):
        return SimSpec(5000, 500, 10, 0.6, list(zip((10, 14, 24, 31, 37), _EFFECTS)), seed=18)
    if name == "c5":
        return SimSpec(10000, 1000, 10, 0.6, list(zip((10, 14, 24, 31, 37), _EFFECTS)), seed=18)
    if name == "a_small":
        return SimSpec(200, 10, 5, 0.3, [(3, 0.4578), (7, -0.2538)], seed=18)
    if name == "a":
        return SimSpec(500, 50, 10, 0.45, list(zip((10, 14, 24, 31, 37), _EFFECTS)), seed=18)
    raise KeyError(name)
