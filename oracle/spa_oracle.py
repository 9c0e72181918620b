"""CPU oracle for the SMC lambda-path hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference algorithm
(`spa` 0.1.0, /root/reference/pkg/src/spa) used as the *checker* for the
CUDA path.  Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline`
/ `--impl reference` legs of `bench.py` may import it.  The product package
(`paper_1106_0322_b200`) never imports anything from `oracle/`; if the CUDA
library is missing the product raises instead of falling back here.

Parity pinning: every function below is checked in
`tests/test_oracle_golden.py` against golden vectors produced by running the
reference itself in the build container (`tests/golden/make_golden.py`).

Each function cites the reference file:line it restates.
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# Philox4x64-10 counter RNG (reference: smc.py:40-43 builds
# np.random.Philox(key=[seed, tag<<58 | t<<34 | i]); NumPy's Philox4x64-10
# emits block b (0-based) from counter value b+1, words in order 0..3).

_PHILOX_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
_PHILOX_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)
_U32 = np.uint64(0xFFFFFFFF)
TAG_INIT, TAG_MOVE, TAG_RESAMPLE, TAG_RWMOVE = 0, 1, 2, 3


def _mulhilo64(a: np.ndarray, b: int):
    """Full 64x64->128 product of uint64 arrays by a constant, as (hi, lo)."""
    a = a.astype(np.uint64)
    b_lo, b_hi = np.uint64(b & 0xFFFFFFFF), np.uint64(b >> 32)
    a_lo, a_hi = a & _U32, a >> np.uint64(32)
    ll = a_lo * b_lo
    lh = a_lo * b_hi
    hl = a_hi * b_lo
    hh = a_hi * b_hi
    mid = (ll >> np.uint64(32)) + (lh & _U32) + (hl & _U32)
    lo = (ll & _U32) | ((mid & _U32) << np.uint64(32))
    hi = hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))
    return hi, lo


def philox4x64_10(counters: np.ndarray, key) -> np.ndarray:
    """Vectorised Philox4x64-10 bijection; counters [M,4] uint64 -> [M,4]."""
    c = np.array(counters, dtype=np.uint64).reshape(-1, 4).T.copy()
    k0, k1 = np.uint64(int(key[0]) & (2**64 - 1)), np.uint64(int(key[1]) & (2**64 - 1))
    with np.errstate(over="ignore"):
        for _ in range(10):
            hi0, lo0 = _mulhilo64(c[0], _PHILOX_M[0])
            hi1, lo1 = _mulhilo64(c[2], _PHILOX_M[1])
            c = np.stack([hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0])
            k0 = k0 + np.uint64(_PHILOX_W[0])
            k1 = k1 + np.uint64(_PHILOX_W[1])
    return c.T


def stream_key(seed: int, tag: int, t: int = 0, i: int = 0):
    """Key layout of smc.py:40-43: (seed, tag<<58 | t<<34 | i)."""
    return (int(seed), (int(tag) << 58) | (int(t) << 34) | int(i))


def stream_blocks(key, first_block: int, count: int) -> np.ndarray:
    """Raw Philox blocks first_block..first_block+count-1 ([count,4] uint64)."""
    ctr = np.zeros((count, 4), dtype=np.uint64)
    ctr[:, 0] = np.arange(first_block + 1, first_block + 1 + count, dtype=np.uint64)
    return philox4x64_10(ctr, key)


def stream_raw(key, count: int) -> np.ndarray:
    """The first `count` 64-bit draws of the stream, in NumPy's order."""
    nb = -(-count // 4)
    return stream_blocks(key, 0, nb).reshape(-1)[:count]


def u53(raw) -> np.ndarray:
    """NumPy's next_double: (raw >> 11) * 2^-53 (uniform in [0, 1))."""
    return (np.asarray(raw, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0**-53


def box_muller(w0, w1):
    """Device normal generator restated (csrc/philox.cuh): one N(0,1) from
    two raw words, u1 in (0,1], u2 in [0,1)."""
    u1 = ((np.asarray(w0, np.uint64) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53
    u2 = u53(w1)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def philox4x32_10(counters: np.ndarray, k0: int, k1: int) -> np.ndarray:
    """Philox4x32-10 bijection (the RW proposal stream, csrc/philox.cuh)."""
    c = np.array(counters, dtype=np.uint64).reshape(-1, 4).T.copy() & np.uint64(0xFFFFFFFF)
    k0, k1 = np.uint64(k0 & 0xFFFFFFFF), np.uint64(k1 & 0xFFFFFFFF)
    M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    W0, W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
    m32 = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = np.stack([((p1 >> np.uint64(32)) ^ c[1] ^ k0) & m32, p1 & m32, ((p0 >> np.uint64(32)) ^ c[3] ^ k1) & m32,
                      p0 & m32])
        k0 = (k0 + W0) & m32
        k1 = (k1 + W1) & m32
    return c.T


def rw_normals(seed: int, t: int, k: int, move: int, q: int) -> np.ndarray:
    """Proposal normals of the RW-cov move (csrc/spa_core.cu rw_normals8):
    Philox4x32-10, key = seed, counter (j/8, k, t, move | 3<<24); each 32-bit
    word w gives one sign-symmetric Box-Muller pair from two 15-bit uniforms,
    u1 = (w>>1 & 0x7fff) + 1, u2 = w>>17 & 0x7fff (x 2^-15), signs = bits 0 and
    16: z = (+-|r cos(pi/2 u2)|, +-|r sin(pi/2 u2)|).  Float32 math; the device
    uses fast intrinsics, so agreement is to ~1e-6."""
    nb = -(-q // 8)
    ctr = np.zeros((nb, 4), np.uint64)
    ctr[:, 0] = np.arange(nb)
    ctr[:, 1] = k
    ctr[:, 2] = t
    ctr[:, 3] = move | (3 << 24)
    w = philox4x32_10(ctr, seed & 0xFFFFFFFF, seed >> 32)
    out = np.empty((nb, 8))
    for h in range(4):
        a = w[:, h]
        u1 = (((a >> np.uint64(1)) & np.uint64(0x7FFF)).astype(np.float64) + 1.0) * 2.0**-15
        u2 = ((a >> np.uint64(17)) & np.uint64(0x7FFF)).astype(np.float64) * 2.0**-15
        r = np.sqrt(-2.0 * np.log(u1))
        m0, m1 = np.abs(r * np.cos(np.pi / 2 * u2)), np.abs(r * np.sin(np.pi / 2 * u2))
        out[:, 2 * h] = np.where(a & np.uint64(1), -m0, m0)
        out[:, 2 * h + 1] = np.where((a >> np.uint64(16)) & np.uint64(1), -m1, m1)
    return out.reshape(-1)[:q]


def rw_accept_uniform(seed: int, t: int, k: int, move: int) -> float:
    w = philox4x32_10(np.array([[0xFFFFFFFF, k, t, move | (3 << 24)]], np.uint64), seed & 0xFFFFFFFF, seed >> 32)[0]
    return float(((int(w[0]) << 21) | (int(w[1]) >> 11)) * 2.0**-53)


def box_muller_pair(w0, w1):
    u1 = ((np.asarray(w0, np.uint64) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53
    u2 = u53(w1)
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2.0 * np.pi * u2), r * np.sin(2.0 * np.pi * u2)


# ---------------------------------------------------------------------------
# Model (reference model.py)


def gt_log_density(beta, a: float, c: float):
    """model.py:78-81: -log(2c) - (a+1) log1p(|beta|/(a c))."""
    x = np.abs(np.asarray(beta, dtype=np.float64))
    return -math.log(2.0 * c) - (a + 1.0) * np.log1p(x / (a * c))


def de_log_density(beta, c: float):
    """model.py:84-88 (the a -> infinity limit)."""
    return -math.log(2.0 * c) - np.abs(np.asarray(beta, dtype=np.float64)) / c


def log_prior_rows(B, a: float, c: float, penalized=None):
    """Per-particle sum of the log-prior over penalized coordinates
    (model.py:166-169 prior part; smc.py:256, 266-270 for the mask)."""
    B = np.asarray(B, dtype=np.float64)
    dens = gt_log_density(B, a, c) if np.isfinite(a) else de_log_density(B, c)
    if penalized is not None:
        dens = dens[:, np.asarray(penalized, bool)]
    return dens.sum(axis=1)


def loglik_rows(X, y, B, block: int = 256):
    """Per-particle Bernoulli-logit log-likelihood (model.py:131-145, batched
    as in summary.py:154-170): sum_i y_i eta_i - logaddexp(0, eta_i)."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    B = np.atleast_2d(np.asarray(B, dtype=np.float64))
    out = np.empty(B.shape[0])
    for s in range(0, B.shape[0], block):
        eta = B[s:s + block] @ X.T
        out[s:s + block] = (eta * y).sum(axis=1) - np.logaddexp(0.0, eta).sum(axis=1)
    return out


# ---------------------------------------------------------------------------
# Sampler building blocks (reference smc.py)


def schedule_bs(b1: float, rho: float, T: int) -> np.ndarray:
    """smc.py:62-64."""
    return b1 * rho ** np.arange(T)


def reweight_increments(B, a: float, c_t: float, c_prev: float, penalized=None):
    """smc.py:248-263 incremental log-weights lw (before normalisation)."""
    return log_prior_rows(B, a, c_t, penalized) - log_prior_rows(B, a, c_prev, penalized)


def logsumexp(v) -> float:
    v = np.asarray(v, dtype=np.float64)
    m = np.max(v)
    if not np.isfinite(m):
        return float(m)
    return float(m + np.log(np.sum(np.exp(v - m))))


def normalise_log_weights(log_w, lw):
    """smc.py:258-262: unnorm = logW + lw; inc = lse(unnorm); logW' = unnorm - inc."""
    unnorm = np.asarray(log_w, np.float64) + np.asarray(lw, np.float64)
    inc = logsumexp(unnorm)
    return unnorm - inc, inc


def weights_from_log(log_w):
    """smc.py:151-154."""
    w = np.exp(log_w - logsumexp(log_w))
    return w / w.sum()


def ess(w) -> float:
    """smc.py:171-174."""
    w = np.asarray(w, dtype=np.float64)
    return float(1.0 / (w @ w))


def systematic_ancestors(w, u: float) -> np.ndarray:
    """smc.py:273-281: sequential cumsum, normalise by the last entry, pin it
    to 1, positions u + k/N, searchsorted(side='right')."""
    w = np.asarray(w, dtype=np.float64)
    n = w.size
    cum = np.cumsum(w)
    cum = cum / cum[-1]
    cum[-1] = 1.0
    pos = u + np.arange(n) / n
    return np.searchsorted(cum, pos, side="right")


def resample_uniform(seed: int, t: int, n: int) -> float:
    """smc.py:289 + smc.py:421: first uniform of stream (seed, 2, t) over N."""
    return float(u53(stream_raw(stream_key(seed, TAG_RESAMPLE, t), 1))[0]) / n


# ---------------------------------------------------------------------------
# Move kernels


def mwg_move_rows(B, eta, ll, X, y, a, c, sd, Z, U, penalized=None):
    """Vectorised Metropolis-within-Gibbs cycles (smc.py:298-332 restated).

    Z, U: [N, cycles, q] proposal normals / uniforms.  Mutates and returns
    (B, eta, ll, accepted).  Used as the statistical checker of the GPU
    coordinate kernel (which draws its own device-side normals)."""
    B = np.array(B, dtype=np.float64)
    eta = np.array(eta, dtype=np.float64)
    ll = np.array(ll, dtype=np.float64)
    N, cycles, q = Z.shape
    pen = np.ones(q, bool) if penalized is None else np.asarray(penalized, bool)
    acc_total = 0
    with np.errstate(divide="ignore"):
        for cyc in range(cycles):
            for j in range(q):
                old = B[:, j]
                new = old + sd * Z[:, cyc, j]
                eta_p = eta + np.outer(new - old, X[:, j])
                ll_p = (eta_p * y).sum(axis=1) - np.logaddexp(0.0, eta_p).sum(axis=1)
                d = ll_p - ll
                if pen[j]:
                    d = d + gt_log_density(new, a, c) - gt_log_density(old, a, c)
                ok = (d >= 0.0) | (np.log(U[:, cyc, j]) < d)
                B[ok, j] = new[ok]
                eta[ok] = eta_p[ok]
                ll[ok] = ll_p[ok]
                acc_total += int(ok.sum())
    return B, eta, ll, acc_total


def rw_cov_factor(B, w, scale_const: float = 2.38, jitter: float = 1e-6):
    """Population random-walk proposal factor for the north-star RW-cov move
    (no reference counterpart; BASELINE.json north_star item 4): weighted
    covariance of the particle cloud, Cholesky factor, scaled by 2.38/sqrt(q).
    Restates the K8 factor path (csrc/spa_core.cu: rw_center_kernel, the split-K
    SYRK, rw_cov_kernel, rw_chol_panel_kernel, rw_emit_kernel) in float64."""
    B = np.asarray(B, np.float64)
    w = np.asarray(w, np.float64)
    mu = w @ B
    D = B - mu
    S = (D * w[:, None]).T @ D
    q = B.shape[1]
    S = S + jitter * (np.trace(S) / q + 1e-300) * np.eye(q)
    L = np.linalg.cholesky(S)
    return L * (scale_const / math.sqrt(q)), mu, S


def rw_move_rows(B, ll, lp, X, y, a, c, Ls, Z, U, penalized=None):
    """One RW-cov Metropolis move for every row (float64 checker):
    beta' = beta + Ls z; accept if log u < (ll'+lp') - (ll+lp)."""
    B = np.asarray(B, np.float64)
    prop = B + np.asarray(Z, np.float64) @ np.asarray(Ls, np.float64).T
    ll_p = loglik_rows(X, y, prop)
    lp_p = log_prior_rows(prop, a, c, penalized)
    d = (ll_p + lp_p) - (ll + lp)
    with np.errstate(divide="ignore"):
        ok = (d >= 0.0) | (np.log(U) < d)
    B2 = np.where(ok[:, None], prop, B)
    return B2, np.where(ok, ll_p, ll), np.where(ok, lp_p, lp), ok


# ---------------------------------------------------------------------------
# Path summaries (reference summary.py:36-61) -- the per-step marginals the
# device summary kernels (spa_summary_*) compute.


def weighted_quantile(values, weights, q: float) -> float:
    """summary.py:36-45: smallest value whose cumulative weight reaches q
    (stable sort, sequential float64 cumsum, searchsorted left)."""
    values = np.asarray(values, dtype=float)
    weights = np.asarray(weights, dtype=float)
    order = np.argsort(values, kind="stable")
    cum = np.cumsum(weights[order])
    idx = int(np.searchsorted(cum, q * cum[-1], side="left"))
    return float(values[order][min(idx, values.size - 1)])


def weighted_mean(values, weights) -> float:
    """summary.py:48-51."""
    values = np.asarray(values, dtype=float)
    weights = np.asarray(weights, dtype=float)
    return float(values @ weights / weights.sum())


def concentration(samples, weights, delta: float) -> float:
    """summary.py:54-61: weighted mass outside the open interval (-delta, delta)."""
    samples = np.asarray(samples, dtype=float)
    weights = np.asarray(weights, dtype=float)
    return 1.0 - float(weights[np.abs(samples) < delta].sum() / weights.sum())


# ---------------------------------------------------------------------------
# EM MAP (reference emmap.py:48-165) -- the oracle of spa_em_map.


def em_l1_weights(beta, a: float, c: float, penalized):
    """emmap.py:48-56 adaptive L1 weights, zero for unpenalised coordinates."""
    w = (a + 1.0) / (a * c + np.abs(np.asarray(beta, dtype=float)))
    return np.where(penalized, w, 0.0)


def kkt_violation(grad, beta, w) -> float:
    """emmap.py:59-66: |grad| <= w at zero, grad = sign(beta) w elsewhere."""
    v = np.where(beta == 0.0, np.maximum(np.abs(grad) - w, 0.0), np.abs(grad - np.sign(beta) * w))
    return float(v.max()) if v.size else 0.0


def weighted_l1_cd(X, y, w, beta, tol=1e-8, max_sweeps=10_000):
    """emmap.py:69-108: cyclic coordinate descent on the quadratic majorisation
    (curvature 0.25 sum_i x_ij^2) with soft thresholding; returns
    (beta, converged, sweeps)."""
    X = np.asarray(X, dtype=float)
    beta = np.array(beta, dtype=float)
    curv = 0.25 * np.einsum("ij,ij->j", X, X)
    eta = X @ beta
    for sweep in range(1, max_sweeps + 1):
        mu = 1.0 / (1.0 + np.exp(-eta))
        for j in range(X.shape[1]):
            g = X[:, j] @ (y - mu)
            z = beta[j] + g / curv[j]
            new = np.sign(z) * max(abs(z) - w[j] / curv[j], 0.0)
            if new != beta[j]:
                eta += X[:, j] * (new - beta[j])
                mu = 1.0 / (1.0 + np.exp(-eta))
                beta[j] = new
        if kkt_violation(X.T @ (y - 1.0 / (1.0 + np.exp(-eta))), beta, w) < tol:
            return beta, True, sweep
    return beta, False, max_sweeps


def em_map(X, y, a: float, c: float, beta_init, penalized, tol=1e-6, max_iter=500, inner_tol=1e-8,
           inner_max_sweeps=10_000):
    """emmap.py:117-165 with X already augmented; returns (beta, log_post,
    converged, inner_converged, iterations)."""
    X = np.asarray(X, dtype=float)
    y = np.asarray(y, dtype=float)
    penalized = np.asarray(penalized, bool)
    beta = np.array(beta_init, dtype=float)
    w = em_l1_weights(beta, a, c, penalized)
    converged, inner_ok, it = False, True, 0
    for it in range(1, max_iter + 1):
        new, ok, _ = weighted_l1_cd(X, y, w, beta, inner_tol, inner_max_sweeps)
        inner_ok = inner_ok and ok
        move = float(np.max(np.abs(new - beta))) if beta.size else 0.0
        beta = new
        w = em_l1_weights(beta, a, c, penalized)
        if move < tol:
            converged = True
            break
    eta = X @ beta
    lp = float(eta @ y - np.logaddexp(0.0, eta).sum() + gt_log_density(beta[penalized], a, c).sum())
    return beta, lp, converged, inner_ok, it


# ---------------------------------------------------------------------------
# Whole-path timing baseline


def run_sampler_port(X, y, a: float, b1: float, rho: float, T: int, N: int, cycles: int = 5, step_sd: float = 0.5,
                     init_burn: int = 2000, init_thin: int = 5, seed: int = 0, threads: int = 1,
                     ess_frac: float = 0.75):
    """The reference's run_sampler (smc.py:427-449) restated for the CPU
    timing baseline of bench.py: ONE Metropolis-within-Gibbs chain from the
    origin, init_burn sweeps, then every init_thin-th state (init_particles /
    _run_chain, smc.py:202-245); then T-1 lambda steps of reweight -> ESS ->
    systematic resampling -> `cycles` MwG sweeps over particle blocks on
    `threads` workers (smc_step, smc.py:397-424; _move_particles,
    smc.py:335-359), with the vectorised arithmetic of _move_block
    (smc.py:298-332).  NumPy's default generator replaces the reference's
    Philox streams (same work, different draws).  Returns log Z_T / Z_1."""
    from concurrent.futures import ThreadPoolExecutor

    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    rng = np.random.default_rng(seed)
    q = X.shape[1]
    bs = schedule_bs(b1, rho, T)
    cs = bs / a if math.isfinite(a) else bs
    beta = np.zeros((1, q))
    eta = beta @ X.T
    ll = loglik_rows(X, y, beta)

    def sweep(b, e, l, c):
        return mwg_move_rows(b, e, l, X, y, a, c, step_sd, rng.standard_normal((b.shape[0], 1, q)),
                             rng.random((b.shape[0], 1, q)))[:3]

    for _ in range(init_burn):
        beta, eta, ll = sweep(beta, eta, ll, cs[0])
    B = np.empty((N, q))
    E = np.empty((N, X.shape[0]))
    L = np.empty(N)
    for k in range(N):
        for _ in range(init_thin):
            beta, eta, ll = sweep(beta, eta, ll, cs[0])
        B[k], E[k], L[k] = beta[0], eta[0], ll[0]
    logw = np.full(N, -math.log(N))
    log_z = 0.0
    bounds = np.linspace(0, N, threads + 1, dtype=int)
    with ThreadPoolExecutor(max_workers=threads) as pool:
        for t in range(1, T):
            lw = reweight_increments(B, a, cs[t], cs[t - 1])
            logw, inc = normalise_log_weights(logw, lw)
            log_z += inc
            w = weights_from_log(logw)
            if ess(w) < ess_frac * N:
                idx = systematic_ancestors(w, rng.random() / N)
                B, E, L = B[idx], E[idx], L[idx]
                logw = np.full(N, -math.log(N))
            Z = rng.standard_normal((N, cycles, q))
            U = rng.random((N, cycles, q))
            parts = list(pool.map(lambda lh: mwg_move_rows(B[lh[0]:lh[1]], E[lh[0]:lh[1]], L[lh[0]:lh[1]], X, y, a,
                                                           cs[t], step_sd, Z[lh[0]:lh[1]], U[lh[0]:lh[1]]),
                                  [(lo, hi) for lo, hi in zip(bounds[:-1], bounds[1:]) if hi > lo]))
            B = np.concatenate([p[0] for p in parts])
            E = np.concatenate([p[1] for p in parts])
            L = np.concatenate([p[2] for p in parts])
    return log_z
