"""Generate the golden fixtures that pin the oracle and the CUDA path.

Runs the REFERENCE implementation (`spa` 0.1.0 at /root/reference/pkg/src)
in the build container and writes small .npz files next to this script.
The reference cannot travel to the GPU box, so the outputs are committed
together with this script; nothing at test/bench run time reads
/root/reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--skip-paths]
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from spa import data as rdata  # noqa: E402
from spa import model as rmodel  # noqa: E402
from spa import smc as rsmc  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_spec(name):
    eff = (-0.2538, 0.4578, -0.1873, -0.1498, 0.0996)
    if name == "c1":
        return rdata.SimSpec(n=500, p=20, block_size=5, within_block_corr=0.3,
                             nonzero=[(2, 0.45), (8, -0.4), (14, 0.35)], seed=101)
    if name == "c2":
        return rdata.SimSpec(n=2000, p=200, block_size=8, within_block_corr=0.6,
                             nonzero=list(zip((108, 22, 5, 117, 162), eff)), seed=18)
    if name == "c3":
        return rdata.SimSpec(n=5000, p=500, block_size=10, within_block_corr=0.6,
                             nonzero=list(zip((10, 14, 24, 31, 37), eff)), seed=18)
    if name == "c5":
        return rdata.SimSpec(n=10000, p=1000, block_size=10, within_block_corr=0.6,
                             nonzero=list(zip((10, 14, 24, 31, 37), eff)), seed=18)
    if name == "a_small":
        return rdata.scenario_a_small()
    if name == "a":
        return rdata.scenario_a()
    raise KeyError(name)


def gen_philox():
    out = {}
    keys = [(0, 0, 0, 0), (7, 1, 5, 3), (123456789, 2, 77, 0), (2**40 + 5, 1, 16777215, 2**34 - 1), (13, 3, 2, 4095)]
    raws, unis = [], []
    for (seed, tag, t, i) in keys:
        k = np.array([seed, (tag << 58) | (t << 34) | i], dtype=np.uint64)
        raws.append(np.random.Philox(key=k).random_raw(16))
        unis.append(rsmc._stream(seed, tag, t, i).random(9))
    out["keys"] = np.array(keys, dtype=np.uint64)
    out["raw"] = np.array(raws, dtype=np.uint64)
    out["uniform"] = np.array(unis)
    np.savez_compressed(os.path.join(HERE, "philox.npz"), **out)


def gen_data_hashes():
    out = {}
    for name in ("c1", "c2", "c3", "a_small", "a", "c5"):
        d, beta = rdata.simulate_dataset(ref_spec(name))
        out[f"{name}_X"] = sha(d.X)
        out[f"{name}_y"] = sha(d.y)
        out[f"{name}_ysum"] = float(d.y.sum())
    np.savez(os.path.join(HERE, "data_hashes.npz"), **{k: np.array(v) for k, v in out.items()})


def gen_loglik_prior():
    out = {}
    d, _ = rdata.simulate_dataset(ref_spec("c1"))
    out["c1_X"], out["c1_y"] = d.X, d.y
    rng = np.random.default_rng(0)
    for s in (0.02, 0.1, 0.5):
        B = rng.normal(0.0, s, size=(64, d.p))
        out[f"c1_B_{s}"] = B
        out[f"c1_ll_{s}"] = np.array([rmodel.log_likelihood(d, b)[0] for b in B])
        for (a, c) in ((1.0, 2.0), (4.0, 0.3), (0.5, 0.05)):
            out[f"c1_lp_{s}_{a}_{c}"] = rmodel.gt_log_density(B, rmodel.GtPrior(a, c)).sum(axis=1)
    # intercept design (smc.py:116-123)
    des = rsmc.make_design(d, True)
    Bi = np.random.default_rng(5).normal(0.0, 0.3, size=(32, d.p + 1))
    out["c1_Bi"] = Bi
    out["c1_lli"] = np.array([rmodel.log_likelihood(des, b)[0] for b in Bi])
    # larger shapes: regenerate the dataset from its spec in the test, store values only
    for name, N in (("c2", 16), ("c3", 8)):
        dd, _ = rdata.simulate_dataset(ref_spec(name))
        r = np.random.default_rng(1)
        for s in (0.02, 0.1):
            B = r.normal(0.0, s, size=(N, dd.p))
            out[f"{name}_B_{s}"] = B
            out[f"{name}_ll_{s}"] = np.array([rmodel.log_likelihood(dd, b)[0] for b in B])
            out[f"{name}_lp_{s}"] = rmodel.gt_log_density(B, rmodel.GtPrior(1.0, 2.0)).sum(axis=1)
    # non-integer (Gaussian) design, test_model.py:30-33 style
    r = np.random.default_rng(2)
    Xg = r.standard_normal((60, 7))
    yg = (r.random(60) < 0.5).astype(float)
    Bg = r.normal(0.0, 0.7, size=(40, 7))
    g = type("D", (), {})()
    g.X, g.y = Xg, yg
    out["g_X"], out["g_y"], out["g_B"] = Xg, yg, Bg
    out["g_ll"] = np.array([rmodel.log_likelihood(g, b)[0] for b in Bg])
    # known answers (test_model.py:131-154)
    out["ka_scalar"] = np.array(rmodel.log_likelihood(type("D", (), {"X": np.array([[1.0]]), "y": np.array([1.0])})(), [0.4578])[0])
    np.savez_compressed(os.path.join(HERE, "loglik_prior.npz"), **out)


def gen_loglik_c5():
    """C5 shapes (n=10000, p=1000; BASELINE configs[4]): reference
    log_likelihood (model.py:131-145) and prior sums for a in {0.5, 1, 4}
    plus the double-exponential limit de_log_density (model.py:84-88), on a
    few particles (the dataset is regenerated from its spec in the test)."""
    out = {}
    dd, _ = rdata.simulate_dataset(ref_spec("c5"))
    r = np.random.default_rng(55)
    for s in (0.02, 0.1):
        B = r.normal(0.0, s, size=(6, dd.p))
        out[f"c5_B_{s}"] = B
        out[f"c5_ll_{s}"] = np.array([rmodel.log_likelihood(dd, b)[0] for b in B])
        for a in (0.5, 1.0, 4.0):
            out[f"c5_lp_{s}_{a}"] = rmodel.gt_log_density(B, rmodel.GtPrior(a, 0.3)).sum(axis=1)
        out[f"c5_lp_{s}_de"] = rmodel.de_log_density(B, 0.3).sum(axis=1)
    np.savez_compressed(os.path.join(HERE, "loglik_c5.npz"), **out)


def gen_reweight():
    out = {}
    d, _ = rdata.simulate_dataset(ref_spec("c1"))
    rng = np.random.default_rng(3)
    for tag, (a, c_prev, c_t, N) in {"a4": (4.0, 0.5, 0.45, 128), "a1": (1.0, 2.0, 1.96, 256),
                                     "a05": (0.5, 0.2, 0.18, 64)}.items():
        B = rng.normal(0.0, 0.3, size=(N, d.p))
        lw0 = np.log(rng.dirichlet(np.ones(N)))
        sys_ = rsmc.ParticleSystem(B, np.zeros((N, d.n)), np.zeros(N), lw0.copy(), a)
        lw, inc = rsmc.reweight(sys_, rmodel.GtPrior(a, c_t), rmodel.GtPrior(a, c_prev))
        out[f"{tag}_B"], out[f"{tag}_lw0"] = B, lw0
        out[f"{tag}_params"] = np.array([a, c_prev, c_t])
        out[f"{tag}_lw"], out[f"{tag}_inc"] = lw, np.array(inc)
        out[f"{tag}_logw"] = sys_.log_weights
        out[f"{tag}_w"] = sys_.weights
        out[f"{tag}_ess"] = np.array(sys_.ess())
    np.savez_compressed(os.path.join(HERE, "reweight.npz"), **out)


def gen_resample():
    out = {}
    cases = []
    k = 0
    for N in (8, 1024, 4096, 65536):
        for alpha in (0.05, 0.3, 1.0, 2.0):
            rng = np.random.default_rng(1000 + k)
            w = rng.dirichlet(np.full(N, alpha))
            u = rng.random() / N
            idx = rsmc.systematic_resample_indices(w, u)
            if N <= 4096:
                out[f"w_{k}"] = w
            out[f"wsha_{k}"] = np.array(sha(w))  # N > 4096: regenerated in the test, pinned by hash
            out[f"u_{k}"] = np.array(u)
            out[f"idx_{k}"] = idx.astype(np.int32)
            cases.append((N, alpha))
            k += 1
    # edge cases (test_smc.py:212-222)
    edges = [np.array([0.5, 0.5]), np.array([0.3, 0.0, 0.7]), np.eye(1, 16, 5).ravel(),
             np.r_[np.zeros(100), 1.0, np.zeros(27)]]
    for e, w in enumerate(edges):
        for j, u in enumerate((0.0, 0.37 / w.size, 0.999999 / w.size)):
            out[f"ew_{e}_{j}"] = w
            out[f"eu_{e}_{j}"] = np.array(u)
            out[f"eidx_{e}_{j}"] = rsmc.systematic_resample_indices(w, u).astype(np.int32)
    out["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "resample.npz"), **out)


def weighted_quantile(x, w, q):
    o = np.argsort(x, kind="stable")
    cw = np.cumsum(w[o])
    cw /= cw[-1]
    return x[o][np.minimum(np.searchsorted(cw, q, side="left"), x.size - 1)]


def summarize(out, quantiles=(0.05, 0.5, 0.95)):
    T = len(out.steps)
    q = out.steps[0].particles.shape[1]
    mean = np.empty((T, q))
    quant = np.empty((T, len(quantiles), q))
    for k, s in enumerate(out.steps):
        w = s.weights
        mean[k] = w @ s.particles
        for j in range(q):
            quant[k, :, j] = [weighted_quantile(s.particles[:, j], w, qq) for qq in quantiles]
    return dict(
        ess=np.array([s.ess for s in out.steps]),
        logz=np.array([s.log_z_ratio_cum for s in out.steps]),
        acc=np.array([s.acceptance for s in out.steps]),
        resampled=np.array([s.resampled for s in out.steps]),
        mean=mean, quant=quant,
    )


def _one_path(args):
    name, a, b1, rho, T, N, cycles, seed = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    d, _ = rdata.simulate_dataset(ref_spec(name))
    cfg = rsmc.SmcConfig(N=N, cycles=cycles, seed=seed)
    t0 = time.time()
    out = rsmc.run_sampler(d, a, rsmc.make_schedule(b1, rho, T), cfg)
    res = summarize(out)
    res["wall"] = np.array(time.time() - t0)
    return res


def gen_paths(name, a, b1, rho, T, N, cycles, seeds, fname):
    jobs = [(name, a, b1, rho, T, N, cycles, s) for s in seeds]
    with Pool(min(8, len(jobs))) as pool:
        res = pool.map(_one_path, jobs)
    out = {k: np.stack([r[k] for r in res]) for k in res[0]}
    out["params"] = np.array([a, b1, rho, T, N, cycles])
    out["seeds"] = np.array(seeds)
    np.savez_compressed(os.path.join(HERE, fname), **out)
    print(fname, "mean wall per path", float(out["wall"].mean()))


def gen_summaries():
    """Per-coordinate weighted mean / quantiles / concentration with the
    reference's summary.py (36-61) on float32-representable particles (the
    device keeps float32 particles): ties, zero weights, ragged N."""
    from spa import summary as rsum

    rng = np.random.default_rng(2024)
    levels = np.array([0.05, 0.25, 0.5, 0.95])
    deltas = np.array([0.05, 0.1])
    cases = {
        "normal": (rng.normal(0.0, 0.3, size=(1000, 13)), rng.dirichlet(np.ones(1000) * 0.7)),
        "ties": (np.round(rng.normal(0.0, 0.3, size=(600, 7)), 1), rng.dirichlet(np.ones(600) * 0.3)),
        "ragged": (rng.standard_t(3.0, size=(4097, 3)) * 0.1, rng.dirichlet(np.ones(4097))),
        "equal": (rng.normal(0.0, 0.05, size=(512, 5)), np.full(512, 1.0 / 512)),
    }
    out = {"levels": levels, "deltas": deltas}
    for name, (B, w) in cases.items():
        B = B.astype(np.float32).astype(np.float64)
        if name == "ties":
            w[::7] = 0.0
            w /= w.sum()
        out[f"{name}_B"], out[f"{name}_w"] = B, w
        out[f"{name}_mean"] = np.array([rsum.weighted_mean(B[:, j], w) for j in range(B.shape[1])])
        out[f"{name}_quant"] = np.array([[rsum.weighted_quantile(B[:, j], w, q) for j in range(B.shape[1])]
                                         for q in levels])
        out[f"{name}_conc"] = np.array([[rsum.concentration(B[:, j], w, d) for j in range(B.shape[1])]
                                        for d in deltas])
    np.savez_compressed(os.path.join(HERE, "summaries.npz"), **out)


def gen_emmap():
    """Reference em_map (emmap.py:117-165) on the C1 and C2 shapes from zero
    and from perturbed seeds, several priors (with and without intercept)."""
    from spa import emmap as rem

    rng = np.random.default_rng(77)
    out = {}
    cases = [("c1", 1.0, 0.5, False), ("c1", 4.0, 0.05, True), ("c2", 1.0, 0.5, False), ("c2", 0.5, 0.2, False)]
    for k, (name, a, c, icpt) in enumerate(cases):
        ds = rdata.simulate_dataset(ref_spec(name))[0]
        q = ds.X.shape[1] + (1 if icpt else 0)
        seeds = [np.zeros(q), rng.normal(0, 0.2, size=q)]
        for s, seed in enumerate(seeds):
            r = rem.em_map(ds, rmodel.GtPrior(a, c), beta_init=seed, intercept=icpt)
            key = f"{k}_{s}"
            out[f"case_{key}"] = np.array([a, c, float(icpt)])
            out[f"name_{key}"] = np.array(name)
            out[f"seed_{key}"] = seed
            out[f"beta_{key}"] = r.beta
            out[f"lp_{key}"] = np.array(r.trace[-1].log_post)
            out[f"conv_{key}"] = np.array([r.converged, r.inner_converged])
            out[f"iters_{key}"] = np.array(len(r.trace) - 1)
    np.savez_compressed(os.path.join(HERE, "emmap.npz"), **out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-paths", action="store_true")
    ap.add_argument("--only", default=None, help="generate one fixture group (e.g. summaries)")
    args = ap.parse_args()
    if args.only:
        globals()[f"gen_{args.only}"]()
        sys.exit(0)
    gen_summaries()
    gen_emmap()
    gen_philox()
    gen_data_hashes()
    gen_loglik_prior()
    gen_loglik_c5()
    gen_reweight()
    gen_resample()
    if not args.skip_paths:
        # scenario-A-small path, a=4 (fast statistical path check)
        gen_paths("a_small", 4.0, 2.0, 0.95, 30, 1024, 5, list(range(1, 17)), "path_a_small.npz")
        # C1: the reference's own CPU run (BASELINE.json configs[0])
        gen_paths("c1", 1.0, 2.0, 0.98, 50, 1024, 5, list(range(1, 9)), "path_c1.npz")
