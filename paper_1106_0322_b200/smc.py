"""Drop-in replacement for the reference sampler surface (`spa.smc`).

Public API mirrors reference pkg/src/spa/smc.py:
    Schedule, make_schedule, SmcConfig, StepRecord, SmcOutput, DegeneracyError,
    ParticleSystem, init_particles, reweight, ess, systematic_resample_indices,
    systematic_resample, smc_step, run_sampler, fixed_b_mcmc, save_run, load_run
with the same argument meanings, output layout and error behaviour.  All
arithmetic on particles runs in libspa_b200 (hand-written sm_100a kernels)
through the C ABI; the host only orders launches, makes the ESS branch and
copies snapshots out.

Extra SmcConfig fields (defaults keep the reference's behaviour):
    move_kernel  "mwg" (reference Metropolis-within-Gibbs, default) or "rw"
                 (north-star population-covariance random walk on tcgen05)
    moves        RW moves per step
    rw_scale     RW proposal scale numerator (scale = rw_scale / sqrt(q))
    init_chains  parallel MwG chains for initialisation (0 = auto)
    init_forks   thinning chains forked from each burned-in chain (0 = auto:
                 1 when init_chains is pinned, else auto_chains' choice)
    summary_levels / summary_deltas
                 per-step weighted marginal summaries computed on the device
                 (StepRecord.summary; see marginal_summaries)
    summary_pooled
                 also the pooled posterior's marginals over all steps
                 (summary.py:126-140; SmcOutput.pooled), from every step's
                 particles kept on the device -- no snapshots needed
    rw_factor_lag
                 RW covariance factor pipelining: 0 = every move of step t
                 uses the factor of step t's population (computed before the
                 first move); 1 = the first move uses the previous step's
                 factor while the new one is computed on a side stream;
                 2 (default) = every move of step t uses the factor of step
                 t-1's population, computed on the side stream during step
                 t-1's moves (never on the critical path)
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._philox_host import first_uniform
from .design import DeviceDesign
from .model import GtPrior

TAG_INIT, TAG_MOVE, TAG_RESAMPLE, TAG_RWMOVE, TAG_INIT_FORK = 0, 1, 2, 3, 4

# Optional CUDA-event timer around the dominant kernel (bench.py sets it;
# events are recorded on the launching stream).
KERNEL_TIMER = None


def _nvtx_push(name: str) -> None:
    """NVTX range around a phase of the lambda step (reweight, resample,
    cov, move, snapshot) for timelines / `ncu --nvtx`."""
    torch.cuda.nvtx.range_push(name)


def _nvtx_pop() -> None:
    torch.cuda.nvtx.range_pop()
_CHUNK = 4096
TRACE_COLUMNS = ("t", "b", "ess", "log_z_ratio_cum", "acceptance_rate")


class DegeneracyError(RuntimeError):
    """All particle weights collapsed to zero mass (reference smc.py:31-32)."""


@dataclass(frozen=True)
class Schedule:
    """Geometric scale sequence b_t = b1 * rho^(t-1), t = 1..T (smc.py:46-64)."""

    b1: float
    rho: float
    T: int

    def __post_init__(self):
        if not self.b1 > 0:
            raise ValueError(f"b1 must be positive, got {self.b1}")
        if not 0.0 < self.rho < 1.0:
            raise ValueError(f"rho must lie in (0, 1) for a decreasing schedule, got {self.rho}")
        if self.T < 1:
            raise ValueError(f"T must be >= 1, got {self.T}")

    @property
    def bs(self) -> np.ndarray:
        return self.b1 * self.rho ** np.arange(self.T)


def make_schedule(b1: float, rho: float, T: int) -> Schedule:
    return Schedule(b1, rho, T)


def prior_scale(a: float, b: float) -> float:
    """Prior scale c_t = b_t / a (reference smc.py:410-411).  In the
    double-exponential limit a = inf the schedule is read as c_t = b_t (the
    reference would evaluate GtPrior(inf, 0) -> nan)."""
    return float(b) if math.isinf(a) else float(b) / a


@dataclass
class SmcConfig:
    """Sampler knobs (smc.py:71-103) plus the B200 extensions above."""

    N: int = 8192
    cycles: int = 5
    step_sd: float = 0.5
    ess_threshold_frac: float = 0.75
    seed: int = 0
    init_burn: int = 2000
    init_thin: int = 5
    snapshot_thin: int = 1
    threads: int = 1
    move_kernel: str = "mwg"
    moves: int = 5
    rw_scale: float = 2.38
    init_chains: int = 0
    init_forks: int = 0
    summary_levels: tuple = ()
    summary_deltas: tuple = ()
    rw_factor_lag: int = 2
    summary_pooled: bool = False

    def __post_init__(self):
        if self.N < 2:
            raise ValueError(f"need at least 2 particles, got N={self.N}")
        if self.cycles < 1:
            raise ValueError(f"cycles must be >= 1, got {self.cycles}")
        if not self.step_sd > 0:
            raise ValueError(f"step_sd must be positive, got {self.step_sd}")
        if not 0.0 < self.ess_threshold_frac <= 1.0:
            raise ValueError(f"ESS threshold fraction must lie in (0, 1], got {self.ess_threshold_frac}")
        if self.seed < 0:
            raise ValueError(f"seed must be nonnegative, got {self.seed}")
        if self.init_burn < 0 or self.init_thin < 1 or self.snapshot_thin < 1 or self.threads < 1:
            raise ValueError("init_burn >= 0, init_thin >= 1, snapshot_thin >= 1, threads >= 1 required")
        if self.move_kernel not in ("mwg", "rw"):
            raise ValueError(f"move_kernel must be 'mwg' or 'rw', got {self.move_kernel!r}")
        if self.rw_factor_lag not in (0, 1, 2):
            raise ValueError(f"rw_factor_lag must be 0, 1 or 2, got {self.rw_factor_lag!r}")
        if self.moves < 1 or self.init_chains < 0 or self.init_forks < 0 or not self.rw_scale > 0:
            raise ValueError("moves >= 1, init_chains >= 0, init_forks >= 0, rw_scale > 0 required")
        if len(self.summary_levels) > 4 or not all(0.0 < float(v) < 1.0 for v in self.summary_levels):
            raise ValueError("summary_levels: at most 4 quantile levels in (0, 1)")
        if len(self.summary_deltas) > 4 or not all(float(v) > 0.0 for v in self.summary_deltas):
            raise ValueError("summary_deltas: at most 4 positive deltas")
        if self.summary_pooled and not (self.summary_levels or self.summary_deltas):
            raise ValueError("summary_pooled needs summary_levels and/or summary_deltas")


@dataclass
class StepRecord:
    """Per-step trace entry with the particle snapshot when retained (smc.py:362-374)."""

    t: int
    b: float
    ess: float
    log_z_ratio_cum: float
    acceptance: float
    resampled: bool
    weights: np.ndarray | None = None
    particles: np.ndarray | None = None
    logliks: np.ndarray | None = None
    summary: dict | None = None  # device marginal summaries (SmcConfig.summary_levels/deltas)


@dataclass
class SmcOutput:
    """Configuration echo and per-step records (smc.py:377-394)."""

    a: float
    schedule: Schedule
    config: SmcConfig
    intercept: bool
    names: list
    steps: list
    init_acceptance: float
    timings: dict = field(default_factory=dict)
    pooled: dict | None = None  # SmcConfig.summary_pooled: pooled-posterior marginals (summary.pooled_marginals)

    @property
    def c_values(self) -> np.ndarray:
        return self.schedule.bs if math.isinf(self.a) else self.schedule.bs / self.a

    @property
    def evidence_validated(self) -> bool:
        """Whether log_z_ratio_cum is inside the validated envelope.  The
        reference's MwG kernel: yes.  The RW population-covariance move
        (north-star throughput kernel): its marginal posteriors pass the
        reference's fixed-b criterion at C3, but its
        evidence carries a finite-N mixing bias (+1.4 nats at C3 with
        N=65536 and 5 moves, SD 0.5; MwG 0.014), so evidence-derived
        summaries (summary.c_posterior, pooled posterior) refuse RW runs
        unless asked explicitly."""
        return self.config.move_kernel == "mwg"

    def step(self, t: int) -> StepRecord:
        return self.steps[t - 1]


# ---------------------------------------------------------------------------
# device plumbing


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    """The current CUDA stream as a raw handle (the C ABI's `stream`).  Read
    through torch's C accessors: torch.cuda.current_stream() builds a Stream
    object per call, which was ~40% of the host time of a launch-bound step
    (C2)."""
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


def _require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1106_0322_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    _lib.load()


def _round_up(x, m):
    return -(-x // m) * m


class ParticleSystem:
    """Device-resident particle state (reference smc.py:126-168).

    beta [N][ldb] float32, loglik / logprior / log_weights [N] float64.
    The reference's fp64 eta cache is not kept: the kernels rematerialise
    eta (MwG) or never form it in HBM (tensor-core likelihood).
    """

    def __init__(self, design: DeviceDesign, N: int, prior_a: float, intercept: bool = False,
                 rank_offset: int = 0, N_total: int | None = None):
        self.design = design
        self.N = int(N)
        self.N_total = int(N_total if N_total is not None else N)
        self.i0 = int(rank_offset)
        self.q = design.q
        self.ldb = _round_up(self.q, 16)  # 64 B (float32) / 32 B (bf16 eps) aligned rows
        self.prior_a = float(prior_a)
        self.intercept = bool(intercept)
        self.t = 1
        self.log_z_cum = 0.0
        dev = design.tensors["sy"].device
        self.device = dev
        f64 = dict(dtype=torch.float64, device=dev)
        self.beta = torch.zeros((self.N, self.ldb), dtype=torch.float32, device=dev)
        self.beta_alt = torch.empty_like(self.beta)
        self.ll = torch.zeros(self.N, **f64)
        self.lp = torch.zeros(self.N, **f64)
        self.ll_alt = torch.empty_like(self.ll)
        self.lp_alt = torch.empty_like(self.lp)
        self.logw = torch.full((self.N,), -math.log(self.N_total), **f64)
        self.lw = torch.empty(self.N, **f64)
        self.w = torch.empty(self.N, **f64)
        self.nchunks = -(-self.N // _CHUNK)
        self.stats = torch.empty((self.nchunks, 3), **f64)
        self.stats_rwf = torch.empty((2 * self.nchunks, 3), **f64)  # spa_reweight_finish: two sets
        self.res = torch.empty(3, **f64)
        self.counter = torch.zeros(1, dtype=torch.int64, device=dev)
        self._rw = None
        self._ll_ws = None

    # --- reference-compatible host views -------------------------------
    @property
    def betas(self) -> np.ndarray:
        return self.beta[:, : self.q].double().cpu().numpy()

    @property
    def logliks(self) -> np.ndarray:
        return self.ll.cpu().numpy()

    @property
    def log_weights(self) -> np.ndarray:
        return self.logw.cpu().numpy()

    @log_weights.setter
    def log_weights(self, v):
        self.logw.copy_(torch.as_tensor(np.asarray(v, dtype=np.float64)))

    @property
    def weights(self) -> np.ndarray:
        return self.device_weights().cpu().numpy()

    def ess(self) -> float:
        _lse(self, None)
        return float(self.res[1].item())

    def device_weights(self) -> torch.Tensor:
        """Normalised weights exp(logw - lse(logw)) (smc.py:151-154), on device."""
        _lse(self, None)
        _lib.call("spa_logw_apply", _p(self.logw), None, self.N, _p(self.res), _p(self.w), _stream())
        return self.w

    def load_betas(self, B: np.ndarray):
        B = np.asarray(B, dtype=np.float64)
        self.beta.zero_()
        self.beta[:, : self.q] = torch.from_numpy(B).to(self.beta.device, torch.float32)

    # --- work buffers -----------------------------------------------------
    def ll_workspace(self):
        if self._ll_ws is None:
            d = self.design
            lib = _lib.load()
            a_bytes = lib.spa_k1_operand_bytes(ctypes.byref(d.struct), self.N)
            nbytes = lib.spa_loglik_workspace_bytes(self.N, d.n)
            self._ll_ws = dict(
                A=torch.empty(max(a_bytes, 8), dtype=torch.uint8, device=self.device),  # K1 operand
                ylin=torch.empty(self.N, dtype=torch.float64, device=self.device),
                sp=torch.empty(self.N, dtype=torch.float64, device=self.device),
                ws=torch.empty(max(nbytes, 8), dtype=torch.uint8, device=self.device),
            )
        return self._ll_ws

    def rw_workspace(self):
        if self._rw is None:
            q = self.q
            kq = _round_up(q, 64)
            dev = self.device
            self._rw = dict(
                prop=torch.zeros((self.N, self.ldb), dtype=torch.bfloat16, device=dev),  # eps = L z
                lp_p=torch.empty(self.N, dtype=torch.float64, device=dev),
                acc=torch.zeros(q + q * q, dtype=torch.int64, device=dev),
                L=torch.empty((q, q), dtype=torch.float32, device=dev),
                fws=torch.empty((_round_up(8 * q * q, 256) + _round_up(2 * q * kq, 256) + 8192) // 8,
                                dtype=torch.float64, device=dev),
                fws2=torch.empty((_round_up(8 * q * q, 256) + _round_up(2 * q * kq, 256) + 8192) // 8,
                                 dtype=torch.float64, device=dev),
                info=torch.zeros(1, dtype=torch.int32, device=dev),
                ctr=torch.zeros(q, dtype=torch.float32, device=dev),  # centring point (previous mean)
                wf=torch.empty(self.N, dtype=torch.float64, device=dev),  # the factor's normalised weights
                statsf=torch.empty((self.nchunks, 3), dtype=torch.float64, device=dev),
                resf=torch.empty(3, dtype=torch.float64, device=dev),
                mws=torch.empty(max(_lib.load().spa_rw_moments_workspace_bytes(self.N, q), 8), dtype=torch.uint8,
                                device=dev),
            )
        return self._rw

    def resample_buffers(self):
        """(exact-scan workspace for the global N, this shard's ancestor slots)."""
        if getattr(self, "_rs_ws", None) is None:
            self._rs_ws = torch.empty(_lib.load().spa_resample_workspace_bytes(self.N_total), dtype=torch.uint8,
                                      device=self.device)
            self._anc = torch.empty(self.N, dtype=torch.int64, device=self.device)
        return self._rs_ws, self._anc

    def gate_one(self):
        if getattr(self, "_one", None) is None:
            self._one = torch.ones(1, dtype=torch.float64, device=self.device)
        return self._one

    def side_stream(self):
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.device)
        return self._side

    def z_buffers(self, moves: int):
        kq = _round_up(self.q, 64)
        zs = getattr(self, "_zs", None)
        if zs is None or len(zs) < moves:
            self._zs = zs = [torch.empty((self.N, kq), dtype=torch.bfloat16, device=self.device) for _ in range(moves)]
            self._z_pending = None  # normals drawn ahead went to the old buffers
        return zs

    def factor_operand(self, buf: int | None = None):
        """bf16 operand of factor buffer `buf` (default: the current one)."""
        rw = self.rw_workspace()
        buf = getattr(self, "_fcur", 0) if buf is None else buf
        return ctypes.c_void_p(rw["fws" if buf == 0 else "fws2"].data_ptr() + _round_up(8 * self.q * self.q, 256))

    def factor_stream(self):
        if getattr(self, "_fstream", None) is None:
            self._fstream = torch.cuda.Stream(self.device)
        return self._fstream


_REWEIGHT_FINISH_LIMIT = None


def _reweight_finish_limit() -> int:
    """Particles spa_reweight_finish handles (its chunks must be co-resident)."""
    global _REWEIGHT_FINISH_LIMIT
    if _REWEIGHT_FINISH_LIMIT is None:
        _REWEIGHT_FINISH_LIMIT = int(_lib.load().spa_reweight_finish_max_particles())
    return _REWEIGHT_FINISH_LIMIT


def _lse(system: ParticleSystem, lw):
    _lib.call("spa_lse_chunk_stats", _p(system.logw), _p(lw), system.N, _p(system.stats), _stream())
    _lib.call("spa_lse_combine", _p(system.stats), system.nchunks, _p(system.res), _stream())


# ---------------------------------------------------------------------------
# reference building blocks


def ess(weights) -> float:
    """Effective sample size 1 / sum(W^2) of normalised weights (smc.py:171-174),
    computed by the K3 chunk kernels: ESS = (sum w)^2 / sum w^2."""
    _require_cuda()
    w = torch.as_tensor(np.asarray(weights, dtype=np.float64)).cuda()
    with np.errstate(divide="ignore"):
        logw = torch.log(w)
    m = w.numel()
    nch = -(-m // _CHUNK)
    stats = torch.empty((nch, 3), dtype=torch.float64, device=w.device)
    res = torch.empty(3, dtype=torch.float64, device=w.device)
    _lib.call("spa_lse_chunk_stats", _p(logw), None, m, _p(stats), _stream())
    _lib.call("spa_lse_combine", _p(stats), nch, _p(res), _stream())
    return float(res[1].item())


def systematic_resample_indices(weights, u: float) -> np.ndarray:
    """Ancestor indices for one systematic draw u in [0, 1/N) (smc.py:273-281),
    bit-exact (K4: np.cumsum's sequential float64 sums by a parallel exact
    scan, csrc/resample.cu, + parallel search)."""
    _require_cuda()
    w = torch.as_tensor(np.ascontiguousarray(weights, dtype=np.float64)).cuda()
    N = w.numel()
    anc = torch.empty(N, dtype=torch.int64, device=w.device)
    ws = torch.empty(_lib.load().spa_resample_workspace_bytes(N), dtype=torch.uint8, device=w.device)
    _lib.call("spa_systematic_ancestors", _p(w), N, float(u), 0, N, _p(anc), _p(ws), ws.numel(), _stream())
    return anc.cpu().numpy()


def _penalized_count(system):
    return int(system.design.penalized.sum())


def reweight(system: ParticleSystem, prior_t: GtPrior, prior_prev: GtPrior):
    """Reweight toward the new scale; the likelihood cancels (smc.py:248-263).

    Returns (incremental log-weights, log Z_t/Z_{t-1}) and leaves the
    system's log-weights renormalised."""
    if prior_t.a != prior_prev.a:
        raise ValueError("consecutive targets must share the degrees of freedom")
    inc = _reweight_device(system, prior_t, prior_prev)
    return system.lw.cpu().numpy(), inc


def _reweight_device(system: ParticleSystem, prior_t: GtPrior, prior_prev: GtPrior, group=None) -> float:
    d = system.design
    # one pass: increments lw and the log-prior lp at the new scale (the moves' lp)
    _lib.call("spa_prior_reweight", ctypes.byref(d.struct), _p(system.beta), system.N, system.ldb,
              float(prior_t.a), float(prior_t.c), float(prior_prev.c), _p(system.lw), _p(system.lp), _stream())
    _lib.call("spa_lse_chunk_stats", _p(system.logw), _p(system.lw), system.N, _p(system.stats), _stream())
    stats = system.stats
    nch = system.nchunks
    if group is not None:
        stats = group.all_gather_cat(system.stats)
        nch = stats.shape[0]
    _lib.call("spa_lse_combine", _p(stats), nch, _p(system.res), _stream())
    # apply before the host read so the device is not idle across the sync
    _lib.call("spa_logw_apply", _p(system.logw), _p(system.lw), system.N, _p(system.res), None, _stream())
    res = system.res.cpu()
    inc = float(res[0])
    if not math.isfinite(inc):
        raise DegeneracyError("all incremental weights vanished")
    system._ess_after_reweight = float(res[1])
    return inc


def systematic_resample(system: ParticleSystem, rng_or_u, group=None) -> np.ndarray:
    """Resample in place with one uniform; weights reset to 1/N (smc.py:284-295).
    `rng_or_u` is a float u in [0, 1) (the reference passes a Generator whose
    first draw is u; pass `first_uniform(seed, 2, t)` to reproduce it)."""
    u = float(rng_or_u.random()) if hasattr(rng_or_u, "random") else float(rng_or_u)
    u = u / system.N_total
    d_anc = _resample_device(system, u, group)
    return d_anc.cpu().numpy()


def _resample_device(system: ParticleSystem, u: float, group=None) -> torch.Tensor:
    """Systematic resampling now (host-decided).  Sharded: the ancestors of
    this rank's slots (global indices), rows fetched from their owners over
    peer memory, buffers updated in place."""
    N = system.N_total
    if group is not None:
        _global_weights(system, group)
        ws, anc = system.resample_buffers()
        one = system.gate_one()
        group.resample(system, ctypes.c_void_p(one.data_ptr()), u, ws, anc)
        return anc
    # normalised weights (smc.py:151-154)
    w = system.device_weights()
    anc = torch.empty(N, dtype=torch.int64, device=system.device)
    ws = torch.empty(_lib.load().spa_resample_workspace_bytes(N), dtype=torch.uint8, device=system.device)
    _lib.call("spa_systematic_ancestors", _p(w), N, u, 0, N, _p(anc), _p(ws), ws.numel(), _stream())
    _lib.call("spa_gather_rows", _p(system.beta), system.ldb, _p(system.beta_alt), system.ldb, system.q, _p(anc),
              0, system.N, _p(system.ll), _p(system.ll_alt), _p(system.lp), _p(system.lp_alt), _stream())
    system.beta, system.beta_alt = system.beta_alt, system.beta
    system.ll, system.ll_alt = system.ll_alt, system.ll
    system.lp, system.lp_alt = system.lp_alt, system.lp
    system.logw.fill_(-math.log(N))
    return anc


# ---------------------------------------------------------------------------
# moves


def _mwg(system: ParticleSystem, prior: GtPrior, sd: float, cycles: int, seed: int, tag: int, t: int,
         sweep0: int = 0, counts: torch.Tensor | None = None):
    """`cycles` MwG sweeps; returns the accepted count (host int), or, given
    a per-particle int64 `counts` tensor, adds each particle's count to it
    on the device (no sync)."""
    d = system.design
    if counts is None:
        system.counter.zero_()
    _lib.call("spa_mwg_move", ctypes.byref(d.struct), _p(system.beta), system.N, system.ldb, float(prior.a),
              float(prior.c), float(sd), int(cycles), int(seed), int(tag), int(t), int(system.i0), int(sweep0),
              _p(system.ll), _p(system.lp), _p(system.counter if counts is None else counts),
              0 if counts is None else 1, _stream())
    return None if counts is not None else int(system.counter.item())


def _loglik_device(system: ParticleSystem, out: torch.Tensor):
    d = system.design
    ws = system.ll_workspace()
    _lib.call("spa_loglik_rows", ctypes.byref(d.struct), _p(system.beta), system.N, system.ldb, _p(ws["A"]),
              _p(ws["ylin"]), _p(out), _p(ws["ws"]), ws["ws"].numel(), _stream())


def _rw_factor(system: ParticleSystem, scale: float, group=None, buf: int = 0, centred=None):
    """Population covariance (fixed-point moments, tcgen05 SYRK) and its
    Cholesky factor into factor buffer `buf`, on the current stream.  The
    particles are read once, centred on the previous population mean (the
    exact covariance is recovered as M - delta delta^T); the first call
    seeds that centre with a mean pass.  `centred` (optional event) is
    recorded once the particles have been read for the last time."""
    rw = system.rw_workspace()
    # normalised weights into the factor's own buffers (this may run on a
    # side stream beside the main stream's use of system.w / stats / res)
    w = _normalised_weights(system, group, (rw["wf"], rw["statsf"], rw["resf"]))
    rw["acc"].zero_()
    if not getattr(system, "_ctr_ready", False):
        _lib.call("spa_rw_moments", _p(system.beta), system.N, system.ldb, system.q, _p(w), None, 0, _p(rw["acc"]),
                  None, 0, _stream())
        if group is not None:
            group.all_reduce_sum(rw["acc"][: system.q])
        rw["ctr"].copy_(rw["acc"][: system.q].double() * 2.0**-48)
        rw["acc"][: system.q].zero_()
        system._ctr_ready = True
    _lib.call("spa_rw_moments", _p(system.beta), system.N, system.ldb, system.q, _p(w), _p(rw["ctr"]), 2,
              _p(rw["acc"]), _p(rw["mws"]), rw["mws"].numel(), _stream())
    if centred is not None:
        centred.record()
    _lib.call("spa_rw_moments", _p(system.beta), system.N, system.ldb, system.q, _p(w), None, 3, _p(rw["acc"]),
              _p(rw["mws"]), rw["mws"].numel(), _stream())
    _lib.add_launches(1)  # phase 3 = tcgen05 SYRK + split reduce
    if group is not None:
        group.all_reduce_sum(rw["acc"])
    _lib.call("spa_rw_factor", _p(rw["acc"]), system.q, float(scale), 1e-6, _p(rw["L"]),
              _p(rw["fws" if buf == 0 else "fws2"]), _p(rw["info"]), _p(rw["ctr"]), _stream())
    panels = -(-system.q // 32)
    _lib.add_launches(2 + 2 * panels - 1)  # cov + graph of panel kernels + emit


def _normalised_weights(system, group=None, out=None):
    """Normalised weights exp(logw - lse(logw)) (smc.py:151-154) into
    out = (w, stats, res) (default: the system's buffers); sharded, the LSE
    runs over ALL shards with the same fixed-chunk combine as one process
    (identical bits)."""
    w, stats, res = out if out is not None else (system.w, system.stats, system.res)
    _lib.call("spa_lse_chunk_stats", _p(system.logw), None, system.N, _p(stats), _stream())
    allst = stats if group is None else group.all_gather_cat(stats)
    _lib.call("spa_lse_combine", _p(allst), allst.shape[0], _p(res), _stream())
    _lib.call("spa_logw_apply", _p(system.logw), None, system.N, _p(res), _p(w), _stream())
    return w


def _global_weights(system, group):
    """system.w = the globally normalised weights of this shard."""
    return _normalised_weights(system, group)


def _launch_normals(system: ParticleSystem, config: SmcConfig, t: int, mv: int):
    """Proposal normals of (step t, move mv) into z buffer mv, on the side
    stream after everything enqueued on the current stream so far (so the
    buffer's previous reader is done).  Returns the ready event."""
    main = torch.cuda.current_stream()
    side = system.side_stream()
    zs = system.z_buffers(config.moves)
    side.wait_stream(main)
    _lib.call("spa_rw_normals", system.N, system.q, int(config.seed), int(t), int(system.i0), mv, _p(zs[mv]),
              ctypes.c_void_p(side.cuda_stream))
    ev = torch.cuda.Event()
    ev.record(side)
    return ev


_NORMALS_AHEAD = 2  # moves between a move's normals being drawn and used
_NORMALS_AFTER_K1 = os.environ.get("SPA_NORMALS_AFTER_K1", "0") == "1"  # A/B knob


def _normals_key(system: ParticleSystem, config: SmcConfig, t: int, mv: int):
    return (int(config.seed), int(t), int(mv), int(system.i0), system.N, system.q)


def _normals_event(system: ParticleSystem, config: SmcConfig, t: int, mv: int):
    """Ready event of the normals of (t, mv): drawn ahead by an earlier move,
    else now."""
    pending = getattr(system, "_z_pending", None)
    ev = pending.pop(_normals_key(system, config, t, mv), None) if pending else None
    return ev if ev is not None else _launch_normals(system, config, t, mv)


def _normals_ahead(system: ParticleSystem, config: SmcConfig, t: int, mv: int):
    """After move mv's accept: draw the normals _NORMALS_AHEAD moves ahead (of
    this step or the next), on the side stream beside the following moves'
    proposal GEMM and pack -- not beside K1, whose tensor-pipe time they
    would stretch."""
    g = mv + _NORMALS_AHEAD
    tt, mm = (t, g) if g < config.moves else (t + 1, g - config.moves)
    if mm >= config.moves:
        return
    if getattr(system, "_z_pending", None) is None:
        system._z_pending = {}
    system._z_pending[_normals_key(system, config, tt, mm)] = _launch_normals(system, config, tt, mm)


def _rw_normals_async(system: ParticleSystem, config: SmcConfig, t: int):
    """The proposal normals depend only on (seed, t, move, particle), so they
    are drawn ahead on a side stream (see _normals_ahead); returns move 0's
    ready event, drawing them now if no earlier move did."""
    pending = getattr(system, "_z_pending", None)
    if pending:  # drop draws for other steps / seeds (a step sequence changed)
        for k in [k for k in pending if k[1] < t or k[0] != int(config.seed)]:
            pending.pop(k)
    return _normals_event(system, config, t, 0)


def _rw_moves(system: ParticleSystem, prior: GtPrior, config: SmcConfig, t: int, group=None, z_ready=None):
    d = system.design
    ws = system.ll_workspace()
    rw = system.rw_workspace()
    if z_ready is None:
        z_ready = _rw_normals_async(system, config, t)
    zs = system.z_buffers(config.moves)
    main = torch.cuda.current_stream()
    cur = getattr(system, "_fcur", 0)
    lag = int(config.rw_factor_lag) if getattr(system, "_factor_ready", False) else 0
    if lag == 1 and config.moves == 1:
        lag = 2  # the new factor would only serve the next step anyway
    centred = factored = None
    if lag:
        # the new factor is built on a side stream from the current particles
        # while the moves propose with the previous one; only move 0's accept
        # (the first write of beta) waits for the centring pass.  Lag 1
        # switches to the new factor at move 1, lag 2 at the next step.
        nxt = 1 - cur
        fs = system.factor_stream()
        centred, factored = torch.cuda.Event(), torch.cuda.Event()
        fs.wait_stream(main)
        with torch.cuda.stream(fs):
            _nvtx_push("cov")
            _rw_factor(system, config.rw_scale, None if group is None else group.side, buf=nxt, centred=centred)
            _nvtx_pop()
            factored.record()
    else:
        _rw_factor(system, config.rw_scale, group, buf=cur)
        nxt = cur
        system._factor_ready = True
    pending = getattr(system, "_factored", None)
    if pending is not None:  # lag 2: the previous step's factor (normally long finished)
        main.wait_event(pending)
        system._factored = None
    # system.lp already holds the log-prior at the new scale (fused reweight pass)
    system.counter.zero_()
    Lb = system.factor_operand(cur)
    for mv in range(config.moves):
        if lag == 1 and mv == 1:
            main.wait_event(factored)
            Lb = system.factor_operand(nxt)
        main.wait_event(z_ready if mv == 0 else _normals_event(system, config, t, mv))
        _lib.call("spa_rw_propose", ctypes.byref(d.struct), _p(system.beta), system.N, system.ldb, Lb,
                  int(config.seed), int(t), int(system.i0), mv, _p(zs[mv]), _p(rw["prop"]), _p(ws["A"]),
                  _p(ws["ylin"]), float(prior.a), float(prior.c), _p(rw["lp_p"]), _stream())
        if mv == 0 and config.moves > 1:  # first step of a run: move 1's normals were not drawn ahead
            pend = system._z_pending = getattr(system, "_z_pending", None) or {}
            if _normals_key(system, config, t, 1) not in pend:
                pend[_normals_key(system, config, t, 1)] = _launch_normals(system, config, t, 1)
        fused = d.coded  # K1 without its row reduction; the accept sums the partial rows itself
        if KERNEL_TIMER is not None:
            KERNEL_TIMER.start("loglik")
        if fused:
            _lib.call("spa_loglik_partials", ctypes.byref(d.struct), _p(ws["A"]), system.N, _p(ws["ws"]),
                      ws["ws"].numel(), _stream())
        else:
            _lib.call("spa_loglik_softplus", ctypes.byref(d.struct), _p(ws["A"]), system.N, _p(ws["sp"]),
                      _p(ws["ws"]), ws["ws"].numel(), _stream())
        if KERNEL_TIMER is not None:
            KERNEL_TIMER.stop("loglik")
        if _NORMALS_AFTER_K1:
            _normals_ahead(system, config, t, mv)
        if lag and mv == 0:
            main.wait_event(centred)  # the factor stream has read the particles
        if fused:
            _lib.call("spa_rw_accept_k1", _p(system.beta), system.ldb, _p(rw["prop"]), system.q, system.N,
                      ctypes.byref(d.struct), _p(ws["A"]), _p(ws["ylin"]), _p(ws["ws"]), _p(rw["lp_p"]),
                      _p(system.ll), _p(system.lp), int(config.seed), int(t), int(system.i0), mv,
                      _p(system.counter), _stream())
        else:
            _lib.call("spa_rw_accept", _p(system.beta), system.ldb, _p(rw["prop"]), system.q, system.N,
                      _p(ws["ylin"]), _p(ws["sp"]), _p(rw["lp_p"]), _p(system.ll), _p(system.lp), int(config.seed),
                      int(t), int(system.i0), mv, _p(system.counter), _stream())
        if not _NORMALS_AFTER_K1:
            _normals_ahead(system, config, t, mv)
    if lag == 2:
        system._factored = factored
    system._fcur = nxt
    acc = system.counter.clone() if group is None else group.all_reduce_sum(system.counter.clone())
    return acc  # device tensor: read lazily (no host sync inside the step)


# ---------------------------------------------------------------------------
# initialisation (reference smc.py:202-245, as parallel chains)


def _prepare_for_path(system: ParticleSystem, config: SmcConfig) -> None:
    """One-time host work of the first lambda step, done while the GPU runs
    the initialisation chains: load all kernels, allocate the step
    workspaces and record the Cholesky's CUDA graph (a factor of the zeroed
    moments, queued behind the chains; its result is discarded)."""
    _lib.call("spa_prepare")
    system.ll_workspace()
    if config.move_kernel == "rw":
        rw = system.rw_workspace()
        system.z_buffers(config.moves)
        system.side_stream()
        for buf in ("fws", "fws2"):  # both factor buffers (the lagged factor alternates them)
            _lib.call("spa_rw_factor", _p(rw["acc"]), system.q, float(config.rw_scale), 1e-6, _p(rw["L"]),
                      _p(rw[buf]), _p(rw["info"]), None, _stream())


def resident_chains(design: DeviceDesign) -> int:
    """MwG chains (one CTA each) resident at once on this GPU for `design`."""
    out = ctypes.c_int64(0)
    _lib.call("spa_mwg_resident_chains", ctypes.byref(design.struct), ctypes.byref(out))
    return int(out.value)


# Sequential sweep time of one chain with c chains resident per SM, relative
# to one chain per SM: measured 1.43 at c = 2 (C3 chain layout) -- the
# chains are latency-bound, so a second one per SM costs less than 2x.
_CHAIN_SHARE_EXP = 0.52


def auto_chains(design: DeviceDesign, N: int, burn: int, thin: int, forks: int = 0) -> tuple[int, int]:
    """Parallel initialisation chains per GPU and thinning forks per chain:
    c burn-in chains per SM, each forked into F thinning chains (c F per SM
    within the resident wave), minimising the sequential sweep time
        burn * c^0.52 + (N thin / (SMs c F)) * (c F)^0.52
    (a sweep at k chains per SM takes ~k^0.52 of one chain's).  forks > 0
    pins F.  C3 with 2000 burn sweeps: c = 1, F = 3 (init 1.37 -> 1.16 s vs
    one unforked chain per SM); with 200: c = 1, F = 3."""
    resident = resident_chains(design)
    sms = torch.cuda.get_device_properties(design.tensors["sy"].device).multi_processor_count
    occ = max(1, resident // max(sms, 1))
    best, plan = None, (1, 1)
    for c in range(1, occ + 1):
        for f in ([forks] if forks else range(1, occ // c + 1)):
            k = c * f
            cost = (burn * c**_CHAIN_SHARE_EXP if burn > 0 else 0.0) + (N * thin / (sms * k)) * k**_CHAIN_SHARE_EXP
            if best is None or cost < best - 1e-9:
                best, plan = cost, (c, f)
    return plan[0] * sms, plan[1]


def init_plan(N_total: int, init_chains: int, chains_auto: int) -> tuple[int, int]:
    """(K chains, R slots per chain): chain c fills the contiguous slots
    [c R, min((c+1) R, N)).  K = init_chains, else one resident wave per GPU
    (`chains_auto`); R = ceil(N / K), then K = ceil(N / R)."""
    K = max(1, min(N_total, init_chains or chains_auto))
    R = -(-N_total // K)
    return -(-N_total // R), R


def init_particles(data, prior_at_b1: GtPrior, config: SmcConfig, intercept: bool = False, design=None,
                   group=None):
    """Seed the particles from MwG chains targeting the first posterior.

    The reference runs ONE chain (init_burn sweeps, then every init_thin-th
    state; smc.py:202-245).  Here K1 independent chains run in parallel, chain
    c keyed (seed, 0, 0, c), each burning init_burn sweeps; each burned-in
    chain is then forked into F thinning chains (fork f of chain c is chain
    k = c F + f, keyed (seed, TAG_INIT_FORK, 0, k); F = 1 keeps chain c's own
    stream), and chain k's state after every further init_thin sweeps fills
    its next slot of the contiguous block [k R, (k+1) R).  Every thinning
    chain is a Markov chain started from a burned-in state, as in the
    reference, and F only changes which chain a slot comes from.  K1 defaults
    to whole waves of chains per GPU (auto_chains x ranks: one or more per
    SM) and F jointly minimise the wall time of these latency-bound sweeps
    (auto_chains).  A rank
    simulates only the chains whose blocks meet its shard (and their
    parents), so for given K1 and F the particles are identical for any
    number of GPUs.  Returns (system, acceptance_rate)."""
    _require_cuda()
    if design is None:
        design = DeviceDesign.build(data.X, data.y, intercept)
    N_total = config.N
    world = 1 if group is None else group.world
    shard, offset = (N_total, 0) if group is None else group.shard(N_total)
    system = ParticleSystem(design, shard, prior_at_b1.a, intercept, rank_offset=offset, N_total=N_total)
    auto, F = 0, 1
    if not config.init_chains:
        auto, F = auto_chains(design, N_total // world, config.init_burn, config.init_thin, config.init_forks)
        auto *= world
    elif config.init_forks:
        F = config.init_forks
    if config.init_burn <= 0:
        F = 1
    K1, _ = init_plan(N_total, config.init_chains, auto)  # burn-in chains
    # thinning chains: fork f of burned chain c is chain c F + f (keyed (seed, TAG_INIT_FORK, 0, c F + f);
    # F = 1 keeps the single-chain keys), each filling R slots
    K, R = init_plan(N_total, K1 * F, 0)
    lo, hi = offset, offset + shard
    c0, c1 = lo // R, min(K, -(-hi // R))  # thinning chains whose slot blocks meet [lo, hi)
    p0, p1 = c0 // F, -(-c1 // F)  # their burned-in parents
    chains = ParticleSystem(design, c1 - c0, prior_at_b1.a, intercept, rank_offset=c0)
    Kl = c1 - c0
    counts = torch.zeros(Kl, dtype=torch.int64, device=system.device)  # per chain, read once at the end
    d = chains.design
    if config.init_burn > 0:  # the burn-in: one chain-slot block of init_burn sweeps (the chains' layout)
        parents = chains if F == 1 else ParticleSystem(design, p1 - p0, prior_at_b1.a, intercept, rank_offset=p0)
        pcounts = counts if F == 1 else torch.zeros(p1 - p0, dtype=torch.int64, device=system.device)
        bb = torch.empty((parents.N, system.ldb), dtype=torch.float32, device=system.device)
        bl = torch.empty(parents.N, dtype=torch.float64, device=system.device)
        bp = torch.empty(parents.N, dtype=torch.float64, device=system.device)
        _lib.call("spa_mwg_chain_slots", ctypes.byref(d.struct), _p(parents.beta), parents.N, parents.ldb,
                  float(prior_at_b1.a), float(prior_at_b1.c), float(config.step_sd), int(config.init_burn), 1,
                  int(config.seed), TAG_INIT, 0, int(parents.i0), 0, _p(parents.ll), _p(parents.lp), _p(bb), _p(bl),
                  _p(bp), _p(pcounts), 1, 0, _stream())  # layout 0: one latency-bound chain per SM
        del bb, bl, bp
        if F > 1:  # fork: thinning chain k starts from its parent's burned-in state
            par = torch.arange(c0, c1, device=system.device) // F - p0
            chains.beta.copy_(parents.beta.index_select(0, par))
            counts.copy_(pcounts.index_select(0, par) * (par * F + p0 * F == torch.arange(c0, c1, device=system.device)))
            del parents, pcounts
    _prepare_for_path(system, config)  # host work while the chains run
    stage_b = torch.empty((Kl, R, system.ldb), dtype=torch.float32, device=system.device)
    stage_l = torch.empty((Kl, R), dtype=torch.float64, device=system.device)
    stage_p = torch.empty((Kl, R), dtype=torch.float64, device=system.device)
    # all R thinning blocks in one launch (slot j = the state after init_burn
    # + (j+1)*init_thin sweeps; bit-identical to one chain-slot call per slot)
    _lib.call("spa_mwg_chain_slots", ctypes.byref(d.struct), _p(chains.beta), chains.N, chains.ldb,
              float(prior_at_b1.a), float(prior_at_b1.c), float(config.step_sd), int(config.init_thin), int(R),
              int(config.seed), TAG_INIT if F == 1 else TAG_INIT_FORK, 0, int(chains.i0), int(config.init_burn),
              _p(chains.ll), _p(chains.lp), _p(stage_b), _p(stage_l), _p(stage_p), _p(counts), 1, 1,
              _stream())  # layout 1: the thinning chains' resident wave
    a, b = lo - c0 * R, hi - c0 * R  # this shard inside the staged slots [c0 R, c1 R)
    system.beta.copy_(stage_b.view(Kl * R, system.ldb)[a:b])
    system.ll.copy_(stage_l.view(-1)[a:b])
    system.lp.copy_(stage_p.view(-1)[a:b])
    del stage_b, stage_l, stage_p
    # acceptance over the chains this rank owns (first slot in its shard), so
    # every chain counts once for any number of ranks
    own = torch.arange(c0, c1, device=system.device) * R >= lo
    # (a fork's burn-in sweeps are its parent's: counted with the parent's first fork only)
    first = torch.arange(c0, c1, device=system.device) % F == 0
    tally = torch.stack([counts[own].sum(),
                         (own.sum() * R * config.init_thin + (own & first).sum() * config.init_burn) * design.q])
    if group is not None:
        tally = group.all_reduce_sum(tally)
    acc, total = (int(v) for v in tally.tolist())
    if group is not None:
        group.setup_peers(system)  # map the peers' particle buffers (the resampling exchange reads them)
    return system, acc / max(total, 1)


# ---------------------------------------------------------------------------
# one lambda step (reference smc.py:397-424)


class _LazyRate:
    """Acceptance rate whose device-side counter is read on first use."""

    def __init__(self, counter: torch.Tensor, denom: int):
        self.counter, self.denom = counter, denom

    def __float__(self):
        return int(self.counter.item()) / self.denom


class _Pending:
    """A StepRecord field held in the device step records (rec[t][col]),
    filled in by resolve_records after the step loop."""

    def __init__(self, t: int, col: int):
        self.t, self.col = t, col


def resolve_records(system: ParticleSystem, steps: list) -> None:
    """Read the device step records once and fill the deferred StepRecord
    fields (ESS, log Z_t/Z_1, resampled, acceptance).  Raises
    DegeneracyError for the first step whose weights vanished, as the
    host-decided path would have at that step."""
    rec = system._records.cpu().numpy() if getattr(system, "_records", None) is not None else None
    for s in steps:
        for name in ("ess", "log_z_ratio_cum", "resampled"):
            v = getattr(s, name)
            if isinstance(v, _Pending):
                if not math.isfinite(rec[v.t, 0]):
                    raise DegeneracyError(f"step {v.t}: all incremental weights vanished")
                val = rec[v.t, v.col]
                setattr(s, name, bool(val != 0.0) if name == "resampled" else float(val))
        if not isinstance(s.acceptance, float):
            s.acceptance = float(s.acceptance)
    if rec is not None and steps:
        system.log_z_cum = float(rec[steps[-1].t, 3])


def _smc_step_async(system: ParticleSystem, schedule: Schedule, t: int, config: SmcConfig,
                    group=None) -> StepRecord:
    """One lambda step with no host synchronisation: the ESS test runs on
    the device (spa_step_record) and resampling is gated on its flag
    (spa_resample_gated; sharded: group.resample, peer-memory exchange), so
    the host only enqueues launches and fixed-size collectives.  The
    arithmetic is the host-decided path's (bit-identical particles, weights
    and evidence); the record's ESS / evidence / resampled / acceptance are
    resolved after the loop by resolve_records."""
    a = system.prior_a
    bs = schedule.bs
    prior_prev = GtPrior(a, prior_scale(a, bs[t - 2]))
    prior_t = GtPrior(a, prior_scale(a, bs[t - 1]))
    z_ready = _rw_normals_async(system, config, t) if config.move_kernel == "rw" else None
    d = system.design
    N = system.N_total
    if getattr(system, "_records", None) is None or system._records.shape[0] < schedule.T + 1:
        system._records = torch.zeros((schedule.T + 1, 4), dtype=torch.float64, device=system.device)
        system._records[:, 3] = system.log_z_cum
    rec = system._records
    ws, anc = system.resample_buffers()
    _nvtx_push("reweight")
    _lib.call("spa_prior_reweight", ctypes.byref(d.struct), _p(system.beta), system.N, system.ldb,
              float(prior_t.a), float(prior_t.c), float(prior_prev.c), _p(system.lw), _p(system.lp), _stream())
    fused = group is None and system.N <= _reweight_finish_limit()
    if fused:  # the weight update, step record and normalised weights in one cooperative launch
        _lib.call("spa_reweight_finish", _p(system.logw), _p(system.lw), system.N, _p(system.stats_rwf), _p(system.res),
                  _p(rec), t, float(config.ess_threshold_frac * N), _p(system.w), _stream())
    else:
        _lib.call("spa_lse_chunk_stats", _p(system.logw), _p(system.lw), system.N, _p(system.stats), _stream())
        stats = system.stats if group is None else group.all_gather_cat(system.stats)
        _lib.call("spa_lse_combine", _p(stats), stats.shape[0], _p(system.res), _stream())
        _lib.call("spa_logw_apply", _p(system.logw), _p(system.lw), system.N, _p(system.res), None, _stream())
        _lib.call("spa_step_record", _p(system.res), _p(rec), t, float(config.ess_threshold_frac * N), _stream())
    _nvtx_pop()
    _nvtx_push("resample")
    u = first_uniform(config.seed, TAG_RESAMPLE, t) / N
    gate = ctypes.c_void_p(rec.data_ptr() + (4 * t + 2) * 8)
    if group is None:
        w = system.w if fused else system.device_weights()
        _lib.call("spa_resample_gated", gate, _p(w), system.N, u, _p(system.beta), _p(system.beta_alt), system.ldb,
                  system.q, _p(system.ll), _p(system.ll_alt), _p(system.lp), _p(system.lp_alt), _p(system.logw),
                  _p(anc), _p(ws), ws.numel(), _stream())
    else:
        _global_weights(system, group)
        group.resample(system, gate, u, ws, anc)
    _nvtx_pop()
    _nvtx_push("move")
    if config.move_kernel == "mwg":
        cnt = torch.zeros(1, dtype=torch.int64, device=system.device)
        _lib.call("spa_mwg_move", ctypes.byref(d.struct), _p(system.beta), system.N, system.ldb, float(prior_t.a),
                  float(prior_t.c), float(config.step_sd), int(config.cycles), int(config.seed), TAG_MOVE, int(t),
                  int(system.i0), 0, _p(system.ll), _p(system.lp), _p(cnt), 0, _stream())
        if group is not None:
            group.all_reduce_sum(cnt)
        acceptance = _LazyRate(cnt, N * config.cycles * system.q)
    else:
        if t == 2 or not getattr(system, "_ll_from_k1", False):
            _loglik_device(system, system.ll)
            system._ll_from_k1 = True
        acc = _rw_moves(system, prior_t, config, t, group, z_ready)
        acceptance = _LazyRate(acc, N * config.moves)
    _nvtx_pop()
    system.t = t
    return StepRecord(t, float(bs[t - 1]), _Pending(t, 1), _Pending(t, 3), acceptance, _Pending(t, 2))


def smc_step(system: ParticleSystem, data, schedule: Schedule, t: int, config: SmcConfig, group=None,
             _defer: bool = False) -> StepRecord:
    """Advance from step t-1 to t: reweight -> accumulate evidence -> ESS ->
    resample if ESS < frac*N -> move with the invariant kernel at prior_t.

    _defer (internal; run_sampler and the bench): steps run without host
    synchronisation (also sharded) and return records with pending fields,
    resolved by resolve_records."""
    if not 2 <= t <= schedule.T:
        raise ValueError(f"step index {t} outside [2, {schedule.T}]")
    if system.t != t - 1:
        raise ValueError(f"system is at step {system.t}, cannot advance to {t}")
    if _defer:
        return _smc_step_async(system, schedule, t, config, group)
    a = system.prior_a
    bs = schedule.bs
    prior_prev = GtPrior(a, prior_scale(a, bs[t - 2]))
    prior_t = GtPrior(a, prior_scale(a, bs[t - 1]))
    # move 0's normals (normally drawn during the previous step)
    z_ready = _rw_normals_async(system, config, t) if config.move_kernel == "rw" else None
    try:
        inc = _reweight_device(system, prior_t, prior_prev, group)
    except DegeneracyError as exc:
        raise DegeneracyError(f"step {t}: {exc}") from None
    system.log_z_cum += inc
    step_ess = system._ess_after_reweight
    resampled = step_ess < config.ess_threshold_frac * system.N_total
    if resampled:
        u = first_uniform(config.seed, TAG_RESAMPLE, t) / system.N_total
        _resample_device(system, u, group)
    if config.move_kernel == "mwg":
        acc = _mwg(system, prior_t, config.step_sd, config.cycles, config.seed, TAG_MOVE, t, 0)
        if group is not None:
            acc = int(group.all_reduce_sum(torch.tensor([acc], dtype=torch.int64, device=system.device)).item())
        acceptance = acc / (system.N_total * config.cycles * system.q)
    else:
        if t == 2 or not getattr(system, "_ll_from_k1", False):
            _loglik_device(system, system.ll)  # keep ll on the K1 arithmetic the MH ratio uses
            system._ll_from_k1 = True
        acc = _rw_moves(system, prior_t, config, t, group, z_ready)
        acceptance = _LazyRate(acc, system.N_total * config.moves)
    system.t = t
    rec = StepRecord(t, float(bs[t - 1]), float(step_ess), system.log_z_cum, acceptance, bool(resampled))
    if not _defer:
        rec.acceptance = float(rec.acceptance)
    return rec


def marginal_summaries(system: ParticleSystem, levels=(0.05, 0.5, 0.95), deltas=(0.05, 0.1), group=None,
                       out=None):
    """Per-coordinate weighted marginals of the current weighted particle set
    on the device (reference summary.py:36-61): weighted mean, weighted
    quantiles at `levels` (smallest value whose cumulative weight reaches the
    level; exact radix select) and concentration V(delta) = mass outside
    (-delta, delta).  Sums are exact integers, so sharded runs all-reduce them
    and get the same result for any number of GPUs.  Returns device float64
    tensors {"mean": [q], "quantiles": [len(levels)][q], "concentration":
    [len(deltas)][q]} (written into `out` when given)."""
    w = system.device_weights() if group is None else _global_weights(system, group)
    return _weighted_marginals(system.beta, system.N, system.ldb, system.q, w, levels, deltas, group, out)


def _weighted_marginals(beta, m, ldb, q, w, levels, deltas, group=None, out=None):
    """The summary kernels on rows beta[m][ldb] (float32) with weights w[m]."""
    dev = beta.device
    lv = (ctypes.c_double * max(1, len(levels)))(*[float(v) for v in levels])
    dl = (ctypes.c_double * max(1, len(deltas)))(*[float(v) for v in deltas])
    nl, nd = len(levels), len(deltas)
    u64 = dict(dtype=torch.int64, device=dev)
    hist = torch.zeros((max(1, nl), q, 256), **u64)
    acc_mean = torch.zeros(q, **u64)
    acc_in = torch.zeros((max(1, nd), q), **u64)
    total = torch.zeros(1, **u64)
    prefix = torch.zeros((max(1, nl), q), dtype=torch.int32, device=dev)
    below = torch.zeros((max(1, nl), q), **u64)
    if out is None:
        f64 = dict(dtype=torch.float64, device=dev)
        out = {"mean": torch.empty(q, **f64), "quantiles": torch.empty((nl, q), **f64),
               "concentration": torch.empty((nd, q), **f64)}
    for ps in range(4 if nl else 1):
        if ps:
            hist.zero_()
        _lib.call("spa_summary_pass", _p(beta), m, ldb, q, _p(w), nl, lv, nd, dl, ps,
                  _p(prefix), _p(hist), _p(acc_mean), _p(acc_in), _p(total), _stream())
        if group is not None:
            group.all_reduce_sum(hist)
            if ps == 0:
                for t_ in (acc_mean, acc_in, total):
                    group.all_reduce_sum(t_)
        if nl:
            _lib.call("spa_summary_select", _p(hist), q, nl, lv, ps, _p(total), _p(prefix), _p(below), _stream())
    _lib.call("spa_summary_finish", q, nl, nd, _p(prefix), _p(acc_mean), _p(acc_in), _p(total), _p(out["mean"]),
              _p(out["quantiles"]) if nl else None, _p(out["concentration"]) if nd else None, _stream())
    return out


class _PooledStore:
    """Every step's particles and normalised weights kept on the device
    (SmcConfig.summary_pooled) for the pooled posterior of
    summary.py:126-140: all particles of all steps, particle k of step t
    weighted by the c-posterior mass of t (Z_t/Z_1 normalised over the
    grid, summary.py:113-122) times its normalised weight.  The pooled
    marginals run the same exact-sum summary kernels over the T*N rows."""

    def __init__(self, system: ParticleSystem, T: int):
        self.beta = torch.empty((T, system.N, system.ldb), dtype=torch.float32, device=system.device)
        self.w = torch.empty((T, system.N), dtype=torch.float64, device=system.device)
        self.system = system

    def add(self, t: int, group=None):
        s = self.system
        w = s.device_weights() if group is None else _global_weights(s, group)
        self.w[t - 1].copy_(w)
        self.beta[t - 1].copy_(s.beta)

    def summarise(self, steps, levels, deltas, group=None):
        log_z = np.array([st.log_z_ratio_cum for st in steps])
        mass = np.exp(log_z - log_z.max())
        mass /= mass.sum()
        T = len(steps)
        s = self.system
        wp = (torch.from_numpy(mass).to(s.device)[:, None] * self.w[:T]).reshape(-1)
        out = _weighted_marginals(self.beta[:T].reshape(T * s.N, s.ldb), T * s.N, s.ldb, s.q, wp, levels, deltas,
                                  group)
        res = {k: v.cpu().numpy() for k, v in out.items()}
        res.update(levels=tuple(float(v) for v in levels), deltas=tuple(float(v) for v in deltas), mass=mass)
        return res


class _SnapshotWriter:
    """Copies retained steps out without stalling the step loop.

    At snapshot time only device-side clones are taken (weights, float32
    particles, log-likelihoods; ~0.1 ms) and an event is recorded; a
    background thread then copies them through a reused pinned staging buffer
    and widens to the reference's float64 NumPy layout on host threads."""

    def __init__(self):
        from concurrent.futures import ThreadPoolExecutor

        import threading

        # two host workers, each with its own side stream and pinned staging
        # buffer: a snapshot's float64 widening (page-faulting a fresh 262 MB
        # array at C3) can take longer than the 10 steps between snapshots
        self.pool = ThreadPoolExecutor(max_workers=2)
        self.jobs = []
        self.local = threading.local()
        self.wait_s = 0.0

    def submit(self, system: ParticleSystem, record: StepRecord, group=None):
        if group is None:
            w = system.device_weights()
            clones = (w.clone(), system.beta[:, : system.q].clone(), system.ll.clone())
        else:  # rank 0 assembles the global arrays from the peers' buffers; the others keep none
            got = group.snapshot_to_rank0(system, _global_weights(system, group))
            if got is None:
                return record
            clones = (got[0], got[1].contiguous(), got[2])
        ev = torch.cuda.Event()
        ev.record()
        dev = system.device
        while len(self.jobs) > 16 or (self.jobs and self.jobs[0].done()):
            # bound the device memory held by pending clones (16 x 131 MB at C3)
            t = time.perf_counter()
            self.jobs.pop(0).result()
            self.wait_s += time.perf_counter() - t
        self.jobs.append(self.pool.submit(self._finish, record, clones, ev, dev))
        return record

    def _finish(self, record, clones, ev, dev):
        w, beta, ll = clones
        with torch.cuda.device(dev):
            loc = self.local
            if getattr(loc, "stream", None) is None:
                loc.stream = torch.cuda.Stream(dev)
                loc.stage = None
            if loc.stage is None or loc.stage.numel() < beta.numel():
                loc.stage = torch.empty(beta.numel(), dtype=torch.float32, pin_memory=True)
            st = loc.stage[: beta.numel()].view(beta.shape)
            loc.stream.wait_event(ev)
            with torch.cuda.stream(loc.stream):
                st.copy_(beta, non_blocking=True)
                wh = w.to("cpu", non_blocking=False)
                llh = ll.to("cpu", non_blocking=False)
            loc.stream.synchronize()
        part = torch.empty(beta.shape, dtype=torch.float64)
        part.copy_(st)  # float32 -> float64 on host threads
        weights = wh.numpy().copy()
        weights /= weights.sum()
        record.weights = weights
        record.particles = part.numpy()
        record.logliks = llh.numpy().copy()
        del clones

    def close(self):
        for j in self.jobs:
            j.result()
        self.jobs.clear()
        self.pool.shutdown(wait=True)


def _snapshot(system: ParticleSystem, record: StepRecord, group=None):
    """Synchronous snapshot (reference layout: float64 NumPy arrays)."""
    writer = _SnapshotWriter()
    try:
        writer.submit(system, record, group)
    finally:
        writer.close()
    return record


_SAMPLER_STREAMS = {}


def sampler_stream(device=None) -> torch.cuda.Stream:
    """The high-priority stream the sampler's main work runs on (run_sampler
    uses it internally; per-step callers may enter it).  The covariance
    factor and the proposal normals run on default-priority side streams, so
    when a persistent K1 launch waits for SMs, its CTAs are scheduled ahead of
    pending side-stream blocks (C3: 2.27 -> 2.22 ms per step)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    s = _SAMPLER_STREAMS.get(dev.index)
    if s is None:
        s = _SAMPLER_STREAMS[dev.index] = torch.cuda.Stream(dev, priority=-1)
    return s


def run_sampler(data, a: float, schedule: Schedule, config: SmcConfig, intercept: bool = False,
                group=None) -> SmcOutput:
    """Initialise at the most diffuse scale and sweep the whole schedule
    (reference smc.py:427-449).  `group` (optional) is a
    `paper_1106_0322_b200.dist.ParticleGroup` sharding particles over GPUs.
    Runs on sampler_stream(), ordered after the caller's current stream."""
    _require_cuda()
    caller = torch.cuda.current_stream()
    stream = sampler_stream()
    stream.wait_stream(caller)
    with torch.cuda.stream(stream):
        out = _run_sampler(data, a, schedule, config, intercept, group)
    caller.wait_stream(stream)
    return out


def _run_sampler(data, a: float, schedule: Schedule, config: SmcConfig, intercept: bool, group) -> SmcOutput:
    timings = {}
    t0 = time.perf_counter()
    design = DeviceDesign.build(data.X, data.y, intercept)
    timings["design_s"] = time.perf_counter() - t0
    prior1 = GtPrior(a, prior_scale(a, schedule.bs[0]))
    system, init_acc = init_particles(data, prior1, config, intercept, design=design, group=group)
    torch.cuda.synchronize()
    timings["init_s"] = time.perf_counter() - t0
    names = (["intercept"] if intercept else []) + list(data.names)

    def retained(t):
        return t == 1 or t == schedule.T or (t - 1) % config.snapshot_thin == 0

    timings["snapshot_s"] = 0.0
    writer = _SnapshotWriter()

    summ = None
    if config.summary_levels or config.summary_deltas:
        f64 = dict(dtype=torch.float64, device=system.device)
        q, T = system.q, schedule.T
        summ = {"mean": torch.empty((T, q), **f64),
                "quantiles": torch.empty((T, len(config.summary_levels), q), **f64),
                "concentration": torch.empty((T, len(config.summary_deltas), q), **f64)}

    pool = _PooledStore(system, schedule.T) if config.summary_pooled else None

    def snap(rec):
        if pool is not None:
            pool.add(rec.t, group)
        if summ is not None:  # every step, retained or not (no host sync)
            marginal_summaries(system, config.summary_levels, config.summary_deltas, group,
                               out={k: v[rec.t - 1] for k, v in summ.items()})
        if not retained(rec.t):
            return rec
        ts = time.perf_counter()
        writer.submit(system, rec, group)
        timings["snapshot_s"] += time.perf_counter() - ts
        return rec

    try:
        steps = [snap(StepRecord(1, float(schedule.bs[0]), float(config.N), 0.0, init_acc, False))]
        t1 = time.perf_counter()
        for t in range(2, schedule.T + 1):
            steps.append(snap(smc_step(system, data, schedule, t, config, group, _defer=True)))
        resolve_records(system, steps)  # one read of the deferred step records
        if summ is not None:
            host = {k: v.cpu().numpy() for k, v in summ.items()}
            names_k = {"levels": tuple(float(v) for v in config.summary_levels),
                       "deltas": tuple(float(v) for v in config.summary_deltas)}
            for s in steps:
                s.summary = {"mean": host["mean"][s.t - 1], "quantiles": host["quantiles"][s.t - 1],
                             "concentration": host["concentration"][s.t - 1], **names_k}
        pooled = None
        if pool is not None:
            pooled = pool.summarise(steps, config.summary_levels, config.summary_deltas, group)
            del pool
        torch.cuda.synchronize()
        timings["path_s"] = time.perf_counter() - t1
        ts = time.perf_counter()
    finally:
        writer.close()
    timings["snapshot_drain_s"] = time.perf_counter() - ts
    timings["snapshot_wait_s"] = writer.wait_s
    timings["resampling_steps"] = sum(1 for s in steps if s.resampled)
    return SmcOutput(float(a), schedule, config, intercept, names, steps, init_acc, timings, pooled)


def fixed_b_mcmc(data, prior: GtPrior, n_samples: int, burn: int = 2000, thin: int = 5, seed: int = 0,
                 step_sd: float = 0.5, intercept: bool = False):
    """Fixed-prior MwG validation chains (reference smc.py:452-476): the
    reference's one chain (burn, then every thin-th state) run as parallel
    chains on the GPU (init_particles: one resident wave of chains, each
    filling a contiguous block of the n_samples slots)."""
    cfg = SmcConfig(N=max(2, n_samples), step_sd=step_sd, seed=seed, init_burn=burn, init_thin=thin)
    system, acc = init_particles(data, prior, cfg, intercept)
    return FixedBResult(system.betas[:n_samples], acc)


@dataclass
class FixedBResult:
    samples: np.ndarray
    acceptance: float


# ---------------------------------------------------------------------------
# run-directory persistence (reference smc.py:479-592, same files and format)


def _fmt(v: float) -> str:
    return f"{v:.17g}"


def manifest_entries(output: SmcOutput) -> dict:
    from . import __version__

    cfg = output.config
    return {
        "a": _fmt(output.a), "b1": _fmt(output.schedule.b1), "rho": _fmt(output.schedule.rho),
        "T": output.schedule.T, "N": cfg.N, "cycles": cfg.cycles, "step_sd": _fmt(cfg.step_sd),
        "ess_frac": _fmt(cfg.ess_threshold_frac), "seed": cfg.seed, "init_burn": cfg.init_burn,
        "init_thin": cfg.init_thin, "snapshot_thin": cfg.snapshot_thin, "threads": cfg.threads,
        "intercept": str(output.intercept).lower(), "spa_version": __version__,
        "numpy_version": np.__version__, "move_kernel": cfg.move_kernel, "moves": cfg.moves,
    }


def save_run(output: SmcOutput, outdir, extra: dict | None = None) -> None:
    os.makedirs(outdir, exist_ok=True)
    entries = manifest_entries(output)
    if extra:
        entries.update(extra)
    with open(os.path.join(outdir, "manifest.txt"), "w") as fh:
        for k, v in entries.items():
            fh.write(f"{k} = {v}\n")
    with open(os.path.join(outdir, "trace.csv"), "w") as fh:
        fh.write(",".join(TRACE_COLUMNS) + "\n")
        for s in output.steps:
            fh.write(f"{s.t},{_fmt(s.b)},{_fmt(s.ess)},{_fmt(s.log_z_ratio_cum)},{_fmt(s.acceptance)}\n")
    for s in output.steps:
        if s.particles is None:
            continue
        write_particles_csv(os.path.join(outdir, f"particles_t{s.t:04d}.csv"), output.names, s.weights, s.particles)


def write_particles_csv(path, names, weights, particles, threads: int = 0, chunk: int = 16384) -> None:
    """particles_tNNNN.csv of the reference run directory (smc.py:543-549),
    byte-identical (every value as f"{v:.17g}"), formatted by
    spa_format_particle_rows on host threads (the reference writer formats
    ~1.5 M values/s in one Python loop)."""
    P = np.ascontiguousarray(particles, dtype=np.float64)
    W = np.ascontiguousarray(weights, dtype=np.float64)
    n, q = P.shape
    threads = threads or (os.cpu_count() or 1)
    cap = chunk * (25 * (q + 1) + 24) + 64
    buf = ctypes.create_string_buffer(cap)
    view = memoryview(buf)
    used = ctypes.c_size_t(0)
    with open(path, "wb") as fh:
        fh.write(("particle_index,weight," + ",".join(names) + "\n").encode())
        for r0 in range(0, n, chunk):
            m = min(chunk, n - r0)
            _lib.call("spa_format_particle_rows", ctypes.c_void_p(W.ctypes.data + 8 * r0),
                      ctypes.c_void_p(P.ctypes.data + 8 * r0 * q), m, q, r0, buf, cap, ctypes.byref(used), threads)
            fh.write(view[:used.value])


def load_run(outdir) -> SmcOutput:
    kv = {}
    with open(os.path.join(outdir, "manifest.txt")) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                k, _, v = line.partition("=")
                kv[k.strip()] = v.strip()
    config = SmcConfig(N=int(kv["N"]), cycles=int(kv["cycles"]), step_sd=float(kv["step_sd"]),
                       ess_threshold_frac=float(kv["ess_frac"]), seed=int(kv["seed"]),
                       init_burn=int(kv["init_burn"]), init_thin=int(kv["init_thin"]),
                       snapshot_thin=int(kv["snapshot_thin"]), threads=int(kv["threads"]),
                       move_kernel=kv.get("move_kernel", "mwg"), moves=int(kv.get("moves", 5)))
    schedule = Schedule(float(kv["b1"]), float(kv["rho"]), int(kv["T"]))
    steps, names = [], []
    with open(os.path.join(outdir, "trace.csv")) as fh:
        header = fh.readline().strip().split(",")
        if tuple(header) != TRACE_COLUMNS:
            raise ValueError(f"{outdir}/trace.csv: unexpected columns {header}")
        for line in fh:
            t_s, b_s, e_s, z_s, a_s = line.strip().split(",")
            e = float(e_s)
            steps.append(StepRecord(int(t_s), float(b_s), e, float(z_s), float(a_s),
                                    int(t_s) > 1 and e < config.ess_threshold_frac * config.N))
    for rec in steps:
        path = os.path.join(outdir, f"particles_t{rec.t:04d}.csv")
        if not os.path.exists(path):
            continue
        with open(path) as fh:
            names = fh.readline().strip().split(",")[2:]
            block = np.loadtxt(fh, delimiter=",", ndmin=2)
        rec.weights = block[:, 1]
        rec.particles = block[:, 2:]
    return SmcOutput(float(kv["a"]), schedule, config, kv.get("intercept", "false") == "true", names, steps,
                     steps[0].acceptance if steps else 0.0)
