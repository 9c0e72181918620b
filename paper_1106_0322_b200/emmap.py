"""Batched EM MAP on the GPU (reference emmap.py:117-165) and the MAP path
along the schedule (reference summary.py:173-211).

`em_map_batch` solves many independent local-mode searches in one launch of
`spa_em_map` (one CTA per problem, float64).  `map_path` follows the
reference: at every step EM runs from the particle with the highest
posterior density and from the previous step's MAP, keeping the better mode
(ties to the previous-MAP branch).  The particle-seeded runs of all steps are
batched; the previous-MAP chain is sequential, as in the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import _lib
from .design import DeviceDesign
from .model import GtPrior


class EmBatch(NamedTuple):
    betas: np.ndarray  # [P][q]
    log_posts: np.ndarray  # [P]
    converged: np.ndarray  # [P] bool (EM)
    inner_converged: np.ndarray  # [P] bool (every inner solve)
    iterations: np.ndarray  # [P]


@dataclass
class EmState:
    """The final point of an EM run (the reference keeps every iterate)."""

    beta: np.ndarray
    log_post: float
    iter: int


class EmMapResult(NamedTuple):
    beta: np.ndarray
    trace: list
    converged: bool
    inner_converged: bool


def _design_x(data, intercept: bool) -> np.ndarray:
    X = np.asarray(data.X, dtype=np.float64)
    return np.column_stack([np.ones(X.shape[0]), X]) if intercept else X


def em_map_batch(data, a, c, seeds, intercept: bool = False, tol: float = 1e-6, max_iter: int = 500,
                 inner_tol: float = 1e-8, inner_max_sweeps: int = 10_000, design: DeviceDesign | None = None,
                 curv: torch.Tensor | None = None) -> EmBatch:
    """Local posterior modes for seeds[k] (float64 [P][q]) under
    GtPrior(a[k], c[k]) (scalars broadcast), emmap.py:117-165 semantics."""
    if design is None:
        design = DeviceDesign.build(data.X, data.y, intercept)
    dev = design.tensors["sy"].device
    seeds = np.atleast_2d(np.asarray(seeds, dtype=np.float64))
    P, q = seeds.shape
    if q != design.q:
        raise ValueError(f"seeds have {q} columns, the design {design.q}")
    a = np.broadcast_to(np.asarray(a, dtype=np.float64), (P,)).copy()
    c = np.broadcast_to(np.asarray(c, dtype=np.float64), (P,)).copy()
    if not (np.all(np.isfinite(a)) and np.all(a > 0) and np.all(c > 0)):
        raise ValueError("EM MAP needs finite a > 0 and c > 0")
    if curv is None:
        X = _design_x(data, intercept)
        curv = torch.from_numpy(0.25 * np.einsum("ij,ij->j", X, X)).to(dev)
    f64 = dict(dtype=torch.float64, device=dev)
    s_d, a_d, c_d = (torch.from_numpy(v).to(dev) for v in (seeds, a, c))
    beta = torch.empty((P, q), **f64)
    lp = torch.empty(P, **f64)
    info = torch.empty(P, dtype=torch.int32, device=dev)
    iters = torch.empty(P, dtype=torch.int32, device=dev)
    p = ctypes.c_void_p
    _lib.call("spa_em_map", ctypes.byref(design.struct), P, p(s_d.data_ptr()), p(a_d.data_ptr()), p(c_d.data_ptr()),
              p(curv.data_ptr()), float(tol), int(max_iter), float(inner_tol), int(inner_max_sweeps),
              p(beta.data_ptr()), p(lp.data_ptr()), p(info.data_ptr()), p(iters.data_ptr()),
              p(torch.cuda.current_stream().cuda_stream))
    inf = info.cpu().numpy()
    return EmBatch(beta.cpu().numpy(), lp.cpu().numpy(), (inf & 1) != 0, (inf & 2) != 0, iters.cpu().numpy())


def em_map(data, prior: GtPrior, beta_init=None, tol: float = 1e-6, max_iter: int = 500, inner_tol: float = 1e-8,
           inner_max_sweeps: int = 10_000, intercept: bool = False) -> EmMapResult:
    """Single-problem form of the reference's em_map (emmap.py:117-165)."""
    q = np.asarray(data.X).shape[1] + (1 if intercept else 0)
    seed = np.zeros(q) if beta_init is None else np.asarray(beta_init, dtype=np.float64)
    if seed.shape != (q,):
        raise ValueError(f"beta_init has shape {seed.shape}, expected ({q},)")
    r = em_map_batch(data, prior.a, prior.c, seed[None, :], intercept, tol, max_iter, inner_tol, inner_max_sweeps)
    return EmMapResult(r.betas[0], [EmState(r.betas[0], float(r.log_posts[0]), int(r.iterations[0]))],
                       bool(r.converged[0]), bool(r.inner_converged[0]))


@dataclass
class MapPath:
    """EM MAP estimates along the schedule (summary.py:140-149)."""

    betas: np.ndarray
    log_posts: np.ndarray
    log_posts_particle_seed: np.ndarray
    log_posts_previous_seed: np.ndarray
    converged: np.ndarray


def map_path(output, data, a: float | None = None, **em_kwargs) -> MapPath:
    """MAP estimate per step seeded twice, keeping the better mode
    (summary.py:173-211).  Needs every step's particle snapshot."""
    from .smc import _p, _round_up, _stream, prior_scale

    missing = [s.t for s in output.steps if s.particles is None]
    if missing:
        raise ValueError(f"steps {missing[:5]} have no particle snapshots; rerun without snapshot thinning")
    a = output.a if a is None else a
    design = DeviceDesign.build(data.X, data.y, output.intercept)
    dev = design.tensors["sy"].device
    X = _design_x(data, output.intercept)
    curv = torch.from_numpy(0.25 * np.einsum("ij,ij->j", X, X)).to(dev)
    q = design.q
    ldb = _round_up(q, 16)
    # particle seeds: argmax over particles of loglik + sum_pen gt (GPU prior kernel)
    seeds, priors = [], []
    for rec in output.steps:
        c = prior_scale(a, rec.b)
        N = rec.particles.shape[0]
        beta = torch.zeros((N, ldb), dtype=torch.float32, device=dev)
        beta[:, :q] = torch.from_numpy(rec.particles).to(dev, torch.float32)
        lp = torch.empty(N, dtype=torch.float64, device=dev)
        _lib.call("spa_prior_rows", ctypes.byref(design.struct), _p(beta), N, ldb, float(a), float(c), float(c), 0,
                  _p(lp), _stream())
        dens = lp.cpu().numpy() + np.asarray(rec.logliks, dtype=np.float64)
        seeds.append(rec.particles[int(np.argmax(dens))])
        priors.append(c)
    T = len(output.steps)
    c_arr = np.array(priors)
    cand1 = em_map_batch(data, a, c_arr, np.stack(seeds), output.intercept, design=design, curv=curv, **em_kwargs)
    betas, chosen_lp, lp2s, conv = [], [], [], []
    prev = None
    for k in range(T):
        b1, lp1 = cand1.betas[k], float(cand1.log_posts[k])
        ok1 = bool(cand1.converged[k] and cand1.inner_converged[k])
        if prev is None:
            chosen, lp, lp2, ok = b1, lp1, -np.inf, ok1
        else:
            r2 = em_map_batch(data, a, c_arr[k], prev[None, :], output.intercept, design=design, curv=curv,
                              **em_kwargs)
            lp2 = float(r2.log_posts[0])
            if lp2 >= lp1:
                chosen, ok = r2.betas[0], bool(r2.converged[0] and r2.inner_converged[0])
            else:
                chosen, ok = b1, ok1
            lp = max(lp1, lp2)
        prev = chosen
        betas.append(chosen)
        chosen_lp.append(lp)
        lp2s.append(lp2)
        conv.append(ok)
    return MapPath(np.stack(betas), np.array(chosen_lp), cand1.log_posts.copy(), np.array(lp2s), np.array(conv))
