"""Independent test oracles (dense 1-d quadrature), restating the reference
test helpers (pkg/tests/helpers.py:13-88) -- test infrastructure only."""

import numpy as np


def loglik_grid_1d(x, y, grid, chunk=20_000):
    x = np.asarray(x, float).ravel()
    y = np.asarray(y, float)
    out = np.empty(grid.size)
    for s in range(0, grid.size, chunk):
        g = grid[s:s + chunk]
        eta = np.outer(x, g)
        out[s:s + chunk] = y @ eta - np.logaddexp(0.0, eta).sum(axis=0)
    return out


class PosteriorGrid1d:
    """Trapezoid-grid view of a one-coefficient posterior (helpers.py:54-88)."""

    def __init__(self, x, y, a, c, lo=-8.0, hi=8.0, n=40_001):
        from oracle.spa_oracle import gt_log_density

        self.grid = np.linspace(lo, hi, n)
        lu = loglik_grid_1d(x, y, self.grid) + gt_log_density(self.grid, a, c)
        shift = lu.max()
        dens = np.exp(lu - shift)
        h = self.grid[1] - self.grid[0]
        w = np.full(n, h)
        w[0] = w[-1] = h / 2
        mass = float(w @ dens)
        self.log_z = shift + np.log(mass)
        cdf = np.concatenate([[0.0], np.cumsum((dens[1:] + dens[:-1]) * h / 2)]) / mass
        self.cdf_values = np.clip(cdf, 0.0, 1.0)
        self.cdf_values[-1] = 1.0

    def cdf(self, x):
        return np.interp(x, self.grid, self.cdf_values)

    def quantile(self, q):
        return float(np.interp(q, self.cdf_values, self.grid))

    def sample(self, n, rng):
        return np.interp(rng.random(n), self.cdf_values, self.grid)


def weighted_quantile(x, w, q):
    """Same definition as tests/golden/make_golden.py::weighted_quantile."""
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
    return dict(ess=np.array([s.ess for s in out.steps]), logz=np.array([s.log_z_ratio_cum for s in out.steps]),
                acc=np.array([s.acceptance for s in out.steps]), mean=mean, quant=quant)
