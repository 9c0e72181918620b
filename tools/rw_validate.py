"""Validity evidence for the north-star RW population-covariance move.

  c1     reference C1 (n=500, p=20, N=1024, T=50, a=1): log Z_T/Z_1 of 8 RW
         replicates per move count vs the reference's own 8 runs
         (tests/golden/path_c1.npz) and vs 8 GPU MwG replicates
  crit8  C3 (n=5000, p=500, N=65536, a=1, 5 moves, T=100): weighted 5/50/95%
         quantiles of every coordinate at t=50 and t=100 vs 1e5-sample
         fixed-b MwG chains (reference acceptance criterion 8,
         pkg/tests/test_acceptance.py:187-216: worst median diff < 0.05,
         worst 90%-endpoint diff < 0.1)
  c3z    C3 at N=8192: 6 RW (5 moves) vs 6 MwG (5 cycles) replicates, z of
         the weighted means, medians and log Z_t/Z_1 along the path
  c3n    C3: RW replicates at N in {8192, 65536} x moves in {5, 10, 20} vs 6
         MwG replicates at N=8192 (device marginal summaries, so it is fast):
         log Z_T mean / SD and the z of the means / medians along the path

    python tools/rw_validate.py [c1] [crit8] [c3z]   (JSON lines on stdout)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from helpers import summarize, weighted_quantile  # noqa: E402
from paper_1106_0322_b200 import GtPrior, SmcConfig, make_schedule, run_sampler  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.smc import fixed_b_mcmc  # noqa: E402


def emit(**kw):
    print(json.dumps(kw), flush=True)


def reps(data, a, sched, seeds, **kw):
    out = []
    for s in seeds:
        out.append(summarize(run_sampler(data, a, sched, SmcConfig(seed=s, **kw))))
    return {k: np.stack([r[k] for r in out]) for k in out[0]}


def z(ref, new, floor=1e-4):
    se = np.sqrt(ref.var(0, ddof=1) / ref.shape[0] + new.var(0, ddof=1) / new.shape[0] + floor**2)
    return (new.mean(0) - ref.mean(0)) / se


def c1():
    g = np.load(os.path.join(ROOT, "tests", "golden", "path_c1.npz"))
    data, _ = simulate_dataset(named_spec("c1"))
    a, b1, rho, T, N, cycles = g["params"]
    sched = make_schedule(float(b1), float(rho), int(T))
    ref = g["logz"][:, -1]
    emit(study="c1", kernel="reference-mwg", logz_mean=float(ref.mean()), logz_sd=float(ref.std(ddof=1)))
    seeds = range(201, 209)
    r = reps(data, float(a), sched, seeds, N=int(N), cycles=int(cycles), move_kernel="mwg")
    emit(study="c1", kernel="mwg", logz_mean=float(r["logz"][:, -1].mean()), logz_sd=float(r["logz"][:, -1].std(ddof=1)),
         z_logz_max=float(np.abs(z(g["logz"], r["logz"])).max()))
    for moves in (5, 10, 20, 40):
        for lag in (1, 0):
            t0 = time.time()
            r = reps(data, float(a), sched, seeds, N=int(N), move_kernel="rw", moves=moves, rw_factor_lag=lag)
            emit(study="c1", kernel="rw", moves=moves, lag=lag, logz_mean=float(r["logz"][:, -1].mean()),
                 logz_sd=float(r["logz"][:, -1].std(ddof=1)), z_logz_max=float(np.abs(z(g["logz"], r["logz"])).max()),
                 z_mean_max=float(np.abs(z(g["mean"], r["mean"])).max()),
                 acc_mean=float(r["acc"][:, 1:].mean()), wall=time.time() - t0)
    # larger N: does the gap shrink?
    r = reps(data, float(a), sched, seeds, N=8192, move_kernel="rw", moves=5)
    emit(study="c1", kernel="rw", moves=5, N=8192, logz_mean=float(r["logz"][:, -1].mean()),
         logz_sd=float(r["logz"][:, -1].std(ddof=1)))
    r = reps(data, float(a), sched, seeds, N=8192, cycles=int(cycles), move_kernel="mwg")
    emit(study="c1", kernel="mwg", N=8192, logz_mean=float(r["logz"][:, -1].mean()),
         logz_sd=float(r["logz"][:, -1].std(ddof=1)))


def crit8(moves=5):
    data, _ = simulate_dataset(named_spec("c3"))
    sched = make_schedule(2.0, 0.98, 100)
    t0 = time.time()
    cfg = SmcConfig(N=65536, move_kernel="rw", moves=moves, seed=17, snapshot_thin=49)
    out = run_sampler(data, 1.0, sched, cfg)
    t_smc = time.time() - t0
    res = {}
    for t in (50, 100):
        rec = out.step(t)
        t1 = time.time()
        chain = fixed_b_mcmc(data, GtPrior(1.0, rec.b / 1.0), 100_000, burn=2000, thin=5, seed=18)
        u = np.full(chain.samples.shape[0], 1.0 / chain.samples.shape[0])
        worst_med = worst_end = 0.0
        for j in range(data.p):
            for q in (0.05, 0.5, 0.95):
                d = abs(weighted_quantile(chain.samples[:, j], u, q) - weighted_quantile(rec.particles[:, j],
                                                                                         rec.weights, q))
                if q == 0.5:
                    worst_med = max(worst_med, d)
                else:
                    worst_end = max(worst_end, d)
        res[t] = (worst_med, worst_end)
        emit(study="crit8", moves=moves, t=t, b=rec.b, worst_median_diff=worst_med, worst_endpoint_diff=worst_end,
             pass_=bool(worst_med < 0.05 and worst_end < 0.1), chain_acceptance=chain.acceptance,
             chain_s=time.time() - t1, smc_s=t_smc, ess=rec.ess, acceptance=out.step(t).acceptance)
    return res


def c3z(N=8192, R=6):
    data, _ = simulate_dataset(named_spec("c3"))
    sched = make_schedule(2.0, 0.98, 100)
    t0 = time.time()
    mw = reps(data, 1.0, sched, range(301, 301 + R), N=N, cycles=5, move_kernel="mwg")
    t1 = time.time()
    rw = reps(data, 1.0, sched, range(401, 401 + R), N=N, move_kernel="rw", moves=5)
    t2 = time.time()
    zm, zq, zl = z(mw["mean"], rw["mean"]), z(mw["quant"][:, :, 1, :], rw["quant"][:, :, 1, :]), z(mw["logz"], rw["logz"])
    emit(study="c3z", N=N, R=R, z_mean_frac_gt3=float(np.mean(np.abs(zm) > 3)), z_mean_max=float(np.abs(zm).max()),
         z_median_frac_gt3=float(np.mean(np.abs(zq) > 3)), z_median_max=float(np.abs(zq).max()),
         z_logz_max=float(np.abs(zl).max()), logz_T_mwg=float(mw["logz"][:, -1].mean()),
         logz_T_rw=float(rw["logz"][:, -1].mean()), logz_T_sd_mwg=float(mw["logz"][:, -1].std(ddof=1)),
         logz_T_sd_rw=float(rw["logz"][:, -1].std(ddof=1)), mwg_s=t1 - t0, rw_s=t2 - t1)


def dev_reps(data, a, sched, seeds, **kw):
    """Replicates summarised by the device marginal summaries (mean, median)."""
    outs = []
    for s in seeds:
        o = run_sampler(data, a, sched, SmcConfig(seed=s, snapshot_thin=10**6, summary_levels=(0.5,), **kw))
        outs.append(dict(mean=np.stack([r.summary["mean"] for r in o.steps]),
                         med=np.stack([r.summary["quantiles"][0] for r in o.steps]),
                         logz=np.array([r.log_z_ratio_cum for r in o.steps]),
                         ess=np.array([r.ess for r in o.steps]), acc=np.array([float(r.acceptance) for r in o.steps])))
    return {k: np.stack([o[k] for o in outs]) for k in outs[0]}


def c3n(R=6):
    data, _ = simulate_dataset(named_spec("c3"))
    sched = make_schedule(2.0, 0.98, 100)
    t0 = time.time()
    mw = dev_reps(data, 1.0, sched, range(301, 301 + R), N=8192, cycles=5, move_kernel="mwg")
    emit(study="c3n", kernel="mwg", N=8192, logz_T=float(mw["logz"][:, -1].mean()),
         logz_T_sd=float(mw["logz"][:, -1].std(ddof=1)), min_ess_frac=float(mw["ess"][:, 1:].min() / 8192),
         wall=time.time() - t0)
    for N in (8192, 65536):
        for moves in (5, 10, 20):
            t0 = time.time()
            rw = dev_reps(data, 1.0, sched, range(401, 401 + R), N=N, move_kernel="rw", moves=moves)
            zm, zq, zl = z(mw["mean"], rw["mean"]), z(mw["med"], rw["med"]), z(mw["logz"], rw["logz"])
            emit(study="c3n", kernel="rw", N=N, moves=moves, logz_T=float(rw["logz"][:, -1].mean()),
                 logz_T_sd=float(rw["logz"][:, -1].std(ddof=1)), z_logz_max=float(np.abs(zl).max()),
                 z_mean_frac_gt3=float(np.mean(np.abs(zm) > 3)), z_mean_max=float(np.abs(zm).max()),
                 z_median_frac_gt3=float(np.mean(np.abs(zq) > 3)), z_median_max=float(np.abs(zq).max()),
                 max_abs_mean_diff=float(np.abs(rw["mean"].mean(0) - mw["mean"].mean(0)).max()),
                 max_abs_median_diff=float(np.abs(rw["med"].mean(0) - mw["med"].mean(0)).max()),
                 min_ess_frac=float(rw["ess"][:, 1:].min() / N), acc=float(rw["acc"][:, 1:].mean()),
                 wall=time.time() - t0)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "crit8", "c3z"]
    for w in which:
        globals()[w]()
