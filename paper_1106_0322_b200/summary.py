"""Path summaries from the device marginal summaries (reference summary.py).

`run_sampler` with `SmcConfig(summary_levels=..., summary_deltas=...)` stores
per-step weighted marginals computed on the GPU in `StepRecord.summary`
(`smc.marginal_summaries`), for every step whether or not its particles are
retained.  These functions assemble the reference's path views from them,
with the reference's names and shapes (summary.py:64-94, 113-122):

    mean_path(out)              -> [T][q]   (summary.py:83-85)
    quantile_path(out, q)       -> [T][q]   (summary.py:64-74), q one of the levels
    abs_median_path(out)        -> [T][q]   (summary.py:77-79)
    concentration_path(out, d)  -> [T][q]   (summary.py:88-97), d one of the deltas
    c_posterior(out)            -> CPosterior (summary.py:113-122)
    pooled_posterior(out)       -> PooledPosterior from snapshots (summary.py:126-140)
    pooled_marginals(out)       -> the pooled posterior's mean / quantiles / V(delta)
                                   computed on the device (SmcConfig.summary_pooled)

Quantiles follow summary.py:36-45 exactly (smallest value whose cumulative
weight reaches the level), the mean and V(delta) to float64 rounding.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class SummaryError(ValueError):
    """The run did not compute the requested device summary."""


def _summaries(output):
    recs = output.steps
    if not recs or any(r.summary is None for r in recs):
        raise SummaryError("no device summaries: run with SmcConfig(summary_levels=..., summary_deltas=...)")
    return recs


def mean_path(output) -> np.ndarray:
    return np.stack([r.summary["mean"] for r in _summaries(output)])


def quantile_path(output, q: float) -> np.ndarray:
    recs = _summaries(output)
    levels = recs[0].summary["levels"]
    hits = [i for i, v in enumerate(levels) if abs(v - q) < 1e-12]
    if not hits:
        raise SummaryError(f"quantile level {q} was not computed (levels {levels})")
    return np.stack([r.summary["quantiles"][hits[0]] for r in recs])


def abs_median_path(output) -> np.ndarray:
    return np.abs(quantile_path(output, 0.5))


def concentration_path(output, delta: float) -> np.ndarray:
    recs = _summaries(output)
    deltas = recs[0].summary["deltas"]
    hits = [i for i, v in enumerate(deltas) if abs(v - delta) < 1e-12]
    if not hits:
        raise SummaryError(f"delta {delta} was not computed (deltas {deltas})")
    return np.stack([r.summary["concentration"][hits[0]] for r in recs])


@dataclass
class CPosterior:
    """Discrete posterior over the scale grid {c_t = b_t / a} (summary.py:98-110)."""

    c: np.ndarray
    mass: np.ndarray

    @property
    def mode_index(self) -> int:
        return int(np.argmax(self.mass))

    @property
    def mode(self) -> float:
        return float(self.c[self.mode_index])


def _require_validated_evidence(output, allow_unvalidated: bool):
    if not allow_unvalidated and not getattr(output, "evidence_validated", True):
        raise SummaryError("the evidence of a move_kernel='rw' run is outside the validated envelope (finite-N mixing "
                           "bias, DESIGN.md section 4): use move_kernel='mwg' for c-posterior / pooled summaries, or "
                           "pass allow_unvalidated=True")


def c_posterior(output, allow_unvalidated: bool = False) -> CPosterior:
    """Evidence ratios normalised over the scale grid (summary.py:113-122)."""
    _require_validated_evidence(output, allow_unvalidated)
    log_z = np.array([s.log_z_ratio_cum for s in output.steps])
    mass = np.exp(log_z - log_z.max())
    mass /= mass.sum()
    return CPosterior(output.c_values[: len(output.steps)], mass)


@dataclass
class PooledPosterior:
    """All particles from all steps, weighted by evidence and local weight (summary.py:126-130)."""

    samples: np.ndarray
    weights: np.ndarray


def pooled_posterior(output, allow_unvalidated: bool = False) -> PooledPosterior:
    """summary.py:133-140 on retained snapshots (every step must be kept)."""
    _require_validated_evidence(output, allow_unvalidated)
    if any(s.particles is None for s in output.steps):
        raise SummaryError("pooled_posterior needs every step's particles (snapshot_thin=1); "
                           "use SmcConfig(summary_pooled=True) and pooled_marginals for the device version")
    mass = c_posterior(output, allow_unvalidated).mass
    samples = np.concatenate([s.particles for s in output.steps], axis=0)
    weights = np.concatenate([m * s.weights for m, s in zip(mass, output.steps)])
    return PooledPosterior(samples, weights / weights.sum())


def pooled_marginals(output, allow_unvalidated: bool = False) -> dict:
    """Weighted mean, quantiles at the configured levels and V(delta) of the
    pooled posterior (summary.py:126-140 marginals), computed on the device
    over every step's particles: {"mean": [q], "quantiles": [L][q],
    "concentration": [D][q], "levels", "deltas", "mass"}."""
    _require_validated_evidence(output, allow_unvalidated)
    if getattr(output, "pooled", None) is None:
        raise SummaryError("no pooled summaries: run with SmcConfig(summary_pooled=True, summary_levels=...)")
    return output.pooled
