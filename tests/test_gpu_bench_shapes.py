"""Parity at the launch geometries the benchmark actually runs.

The headline configurations put many work items on every persistent CTA
(K1 at C3 with N=65536: 2,560 items over 148 CTAs; C4 N=2^20: ~41k items;
C5 kp=1024), carry the smem-ring / TMEM phases across items, and run the
grid-stride bookkeeping kernels over several passes.  These tests check
those exact shapes against the float64 oracle / torch float64 on a strided
subset of rows (every row of the tail tile included), plus the C5 golden
values produced by the reference (tests/golden/loglik_c5.npz).

Tolerances: log-likelihood 1e-5 relative (north_star); float64 prior /
reweight kernels 1e-12 relative against the oracle on the float32-stored
particles; the L z proposal GEMM and SYRK to their bf16 operand rounding.
"""

import ctypes
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from conftest import golden  # noqa: E402
from oracle import spa_oracle as orc  # noqa: E402
from paper_1106_0322_b200 import _lib  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.design import DeviceDesign  # noqa: E402
from paper_1106_0322_b200.smc import ParticleSystem, _p, _round_up, _stream  # noqa: E402

LL_RTOL = 1e-5
_DATA = {}


def dataset(name):
    if name not in _DATA:
        _DATA[name] = simulate_dataset(named_spec(name))[0]
    return _DATA[name]


def random_system(name, N, seed=0, a=1.0):
    """N particles drawn on the device, rows with scales cycling through
    0.02 / 0.1 / 0.3 (posterior-like to diffuse), stored float32."""
    data = dataset(name)
    d = DeviceDesign.build(data.X, data.y, False)
    s = ParticleSystem(d, N, a, False)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    scale = torch.tensor([0.02, 0.1, 0.3], device="cuda", dtype=torch.float32)[torch.arange(N, device="cuda") % 3]
    s.beta[:, : s.q] = torch.randn((N, s.q), generator=g, device="cuda", dtype=torch.float32) * scale[:, None]
    return data, d, s


def check_rows(N, count=512):
    """A strided subset of row indices plus the whole last 128-row tile."""
    rows = np.unique(np.concatenate([np.linspace(0, N - 1, count).astype(np.int64),
                                     np.arange(max(0, N - 128), N)]))
    return rows


def k1_loglik(d, s):
    ws = s.ll_workspace()
    out = torch.empty(s.N, dtype=torch.float64, device="cuda")
    _lib.call("spa_loglik_rows", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, _p(ws["A"]), _p(ws["ylin"]),
              _p(out), _p(ws["ws"]), ws["ws"].numel(), _stream())
    return out


@pytest.mark.parametrize("name,N", [("c3", 65536), ("c3", 65536 + 77), ("c5", 131072), ("c4", 1 << 20)])
def test_loglik_benchmark_geometry_vs_oracle(name, N):
    """K1 at the benched shapes (many work items per persistent CTA, TMEM /
    smem-ring phases carried across items; ragged last tile) vs float64."""
    data, d, s = random_system(name, N, seed=N)
    out = k1_loglik(d, s)
    assert bool(torch.isfinite(out).all())
    rows = check_rows(N)
    B = s.beta[rows, : s.q].double().cpu().numpy()
    ref = orc.loglik_rows(data.X, data.y, B)
    got = out[torch.from_numpy(rows).cuda()].cpu().numpy()
    np.testing.assert_allclose(got, ref, rtol=LL_RTOL)
    # position independence: the same particles evaluated as a short batch
    # (one work item per CTA) give the same bits as inside the long launch
    sub = ParticleSystem(d, rows.size, 1.0, False)
    sub.beta.copy_(s.beta[torch.from_numpy(rows).cuda()])
    out2 = k1_loglik(d, sub)
    np.testing.assert_allclose(out2.cpu().numpy(), got, rtol=1e-12)


def test_loglik_c5_golden_values():
    """Reference float64 log-likelihoods at n=10000, p=1000 (kp=1024)."""
    g = golden("loglik_c5.npz")
    data = dataset("c5")
    for sc in (0.02, 0.1):
        B = g[f"c5_B_{sc}"]
        d = DeviceDesign.build(data.X, data.y, False)
        s = ParticleSystem(d, B.shape[0], 1.0, False)
        s.load_betas(B)
        np.testing.assert_allclose(k1_loglik(d, s).cpu().numpy(), g[f"c5_ll_{sc}"], rtol=LL_RTOL)


@pytest.mark.parametrize("a", [0.5, 1.0, 4.0, float("inf")])
def test_prior_reweight_c5_geometry(a):
    """The q=1000 reweight kernel (prior_reweight_lean_kernel<16,16>) at
    N=131072 for every prior shape of the C5 sweep, vs the oracle on the
    float32-stored particles, and the C5 golden log-prior sums."""
    data, d, s = random_system("c5", 131072, seed=5, a=a)
    c_prev, c = 0.31, 0.3
    lw = torch.empty(s.N, dtype=torch.float64, device="cuda")
    lp = torch.empty_like(lw)
    _lib.call("spa_prior_reweight", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, a, c, c_prev, _p(lw), _p(lp),
              _stream())
    rows = check_rows(s.N)
    Bf = s.beta[rows, : s.q].double().cpu().numpy()
    idx = torch.from_numpy(rows).cuda()
    np.testing.assert_allclose(lw[idx].cpu().numpy(), orc.reweight_increments(Bf, a, c, c_prev), rtol=1e-11,
                               atol=1e-9)
    np.testing.assert_allclose(lp[idx].cpu().numpy(), orc.log_prior_rows(Bf, a, c), rtol=1e-12)
    g = golden("loglik_c5.npz")
    tag = "de" if math.isinf(a) else str(a)
    for sc in (0.02, 0.1):
        B = g[f"c5_B_{sc}"]
        s2 = ParticleSystem(d, B.shape[0], a, False)
        s2.load_betas(B)
        out = torch.empty(B.shape[0], dtype=torch.float64, device="cuda")
        lw2 = torch.empty_like(out)
        _lib.call("spa_prior_reweight", ctypes.byref(d.struct), _p(s2.beta), s2.N, s2.ldb, a, 0.3, 0.3, _p(lw2),
                  _p(out), _stream())
        np.testing.assert_allclose(out.cpu().numpy(), g[f"c5_lp_{sc}_{tag}"], rtol=1e-6)


def test_rw_propose_eps_benchmark_geometry():
    """eps = L z at C3 with N=65536 (512 particle tiles x 2 column tiles over
    148 persistent CTAs, lower-triangular k-block skipping) vs torch on the
    same bf16 operands, every row."""
    from paper_1106_0322_b200.smc import _rw_factor

    data, d, s = random_system("c3", 65536, seed=9)
    s.log_weights = np.full(s.N, -math.log(s.N))
    _rw_factor(s, 2.38)
    rw, ws = s.rw_workspace(), s.ll_workspace()
    assert int(rw["info"].item()) == 0
    zb = s.z_buffers(1)[0]
    _lib.call("spa_rw_normals", s.N, s.q, 3, 5, 0, 1, _p(zb), _stream())
    _lib.call("spa_rw_propose", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, s.factor_operand(), 3, 5, 0, 1,
              _p(zb), _p(rw["prop"]), _p(ws["A"]), _p(ws["ylin"]), 1.0, 0.9, _p(rw["lp_p"]), _stream())
    q, kq = s.q, _round_up(s.q, 64)
    off = _round_up(8 * q * q, 256)
    L = rw["fws"].view(torch.uint8)[off: off + 2 * q * kq].view(torch.bfloat16).view(q, kq).float()
    ref = zb.float() @ L.T
    got = rw["prop"][:, :q].float()
    err = (got - ref).abs() - (1e-2 * ref.abs() + 2e-3 * ref.abs().max())
    assert float(err.max()) <= 0.0
    assert not rw["prop"][:, q:].float().any()
    # the fused pack of the same proposals: ylin and the K1 operand's log-lik
    rows = check_rows(s.N)
    idx = torch.from_numpy(rows).cuda()
    prop = (s.beta[idx, :q] + rw["prop"][idx, :q].float()).double().cpu().numpy()
    np.testing.assert_allclose(ws["ylin"][idx].cpu().numpy(), prop @ (data.X.T @ data.y), rtol=1e-5, atol=1e-6)
    _lib.call("spa_loglik_softplus", ctypes.byref(d.struct), _p(ws["A"]), s.N, _p(ws["sp"]), _p(ws["ws"]),
              ws["ws"].numel(), _stream())
    ll_p = (ws["ylin"] - ws["sp"])[idx].cpu().numpy()
    np.testing.assert_allclose(ll_p, orc.loglik_rows(data.X, data.y, prop), rtol=LL_RTOL)


def test_rw_moments_benchmark_geometry():
    """Fixed-point weighted moments through the split-K tcgen05 SYRK at C3
    with N=65536 (one wave of 148 split units) vs torch float64 on the same
    float32 particles and weights."""
    from paper_1106_0322_b200.smc import _rw_factor

    data, d, s = random_system("c3", 65536, seed=10)
    w = torch.distributions.Dirichlet(torch.full((s.N,), 2.0, dtype=torch.float64)).sample().cuda()
    s.logw.copy_(torch.log(w))
    rw = s.rw_workspace()
    for shift in (0.0, 0.2):  # first call: exact mean centre; then the previous mean
        if shift:
            s.beta[:, : s.q] += shift * torch.linspace(-1, 1, s.q, device="cuda")
        _rw_factor(s, 2.38)
        assert int(rw["info"].item()) == 0
        B = s.beta[:, : s.q].double()
        wn = s.device_weights()
        mu = wn @ B
        S = (B - mu).T @ ((B - mu) * wn[:, None])
        np.testing.assert_allclose(rw["ctr"].double().cpu().numpy(), mu.cpu().numpy(), rtol=1e-6, atol=1e-7)
        L = rw["L"].double()
        LLt = (L @ L.T) * (s.q / 2.38**2)
        Sj = S + torch.eye(s.q, dtype=torch.float64, device="cuda") * (1e-6 * torch.trace(S) / s.q)
        tol = 2e-3 * Sj.abs() + 1e-3 * Sj.abs().max()
        assert bool(((LLt - Sj).abs() <= tol).all())


def test_resample_gated_multi_pass_vs_oracle():
    """spa_resample_gated (device-decided path) at N=32768 (> 9472 rows: the
    capped-grid gather / commit kernels take several grid-stride passes)
    against the oracle ancestors applied to the pre-resampling state."""
    data, d, s = random_system("a_small", 32768, seed=12)
    N = s.N
    rng = np.random.default_rng(4)
    w = rng.dirichlet(np.full(N, 0.3))
    s.logw.copy_(torch.from_numpy(np.log(w)))
    s.ll.copy_(torch.arange(N, dtype=torch.float64, device="cuda") * 0.5)
    s.lp.copy_(-torch.arange(N, dtype=torch.float64, device="cuda"))
    before = s.beta.clone()
    wd = s.device_weights().clone()
    u = 0.6180339887 / N
    anc_ref = orc.systematic_ancestors(wd.cpu().numpy(), u)
    gate = torch.ones(1, dtype=torch.float64, device="cuda")
    anc = torch.empty(N, dtype=torch.int64, device="cuda")
    wsb = torch.empty(_lib.load().spa_resample_workspace_bytes(N), dtype=torch.uint8, device="cuda")
    _lib.call("spa_resample_gated", _p(gate), _p(wd), N, u, _p(s.beta), _p(s.beta_alt), s.ldb, s.q, _p(s.ll),
              _p(s.ll_alt), _p(s.lp), _p(s.lp_alt), _p(s.logw), _p(anc), _p(wsb), wsb.numel(), _stream())
    assert np.array_equal(anc.cpu().numpy(), anc_ref)
    a = torch.from_numpy(anc_ref).cuda()
    assert torch.equal(s.beta[:, : s.q], before[a, : s.q])
    assert torch.equal(s.ll, a.double() * 0.5) and torch.equal(s.lp, -a.double())
    assert bool((s.logw == -math.log(N)).all())
    # gate off: nothing moves
    gate.zero_()
    snap = s.beta.clone()
    _lib.call("spa_resample_gated", _p(gate), _p(wd), N, u, _p(s.beta), _p(s.beta_alt), s.ldb, s.q, _p(s.ll),
              _p(s.ll_alt), _p(s.lp), _p(s.lp_alt), _p(s.logw), _p(anc), _p(wsb), wsb.numel(), _stream())
    assert torch.equal(s.beta, snap)


@pytest.mark.parametrize("kernel", ["mwg", "rw"])
def test_device_decided_resampling_every_step_large_n(small_data, kernel):
    """ess_threshold_frac = 1: every step resamples; N = 32768 particles (the
    gated gather / commit take several grid-stride passes); device-decided
    steps must reproduce host-decided steps bit for bit."""
    from paper_1106_0322_b200 import GtPrior, SmcConfig, init_particles, make_schedule, smc_step
    from paper_1106_0322_b200.smc import resolve_records

    cfg = SmcConfig(N=32768, cycles=1, moves=2, seed=17, init_burn=20, init_thin=1, move_kernel=kernel,
                    ess_threshold_frac=1.0)
    sched = make_schedule(2.0, 0.8, 5)
    prior1 = GtPrior(4.0, sched.bs[0] / 4.0)
    s1, _ = init_particles(small_data, prior1, cfg)
    s2, _ = init_particles(small_data, prior1, cfg)
    r1 = [smc_step(s1, small_data, sched, t, cfg) for t in range(2, sched.T + 1)]
    r2 = [smc_step(s2, small_data, sched, t, cfg, _defer=True) for t in range(2, sched.T + 1)]
    resolve_records(s2, r2)
    assert all(r.resampled for r in r1)
    for a, b in zip(r1, r2):
        assert (a.ess, a.log_z_ratio_cum, a.resampled, a.acceptance) == (b.ess, b.log_z_ratio_cum, b.resampled,
                                                                          b.acceptance)
    q = s1.q  # the padding columns of the swapped host-path buffer are not part of the state
    assert torch.equal(s1.beta[:, :q], s2.beta[:, :q])
    for name in ("logw", "ll", "lp"):
        assert torch.equal(getattr(s1, name), getattr(s2, name)), name


@pytest.mark.parametrize("name,N", [("c3", 65536), ("c5", 131072), ("c2", 8192 + 77)])
def test_accept_reducing_k1_partials_matches_two_step_path(name, N):
    """spa_loglik_partials + spa_rw_accept_k1 (the accept sums K1's partial
    rows itself) against spa_loglik_softplus + spa_rw_accept, bit for bit:
    the resident (contiguous ranges) and streamed (C5, round-robin items) K1
    schedules and a ragged N."""
    from paper_1106_0322_b200.smc import _rw_factor

    data, d, s = random_system(name, N, seed=3)
    s.log_weights = np.full(s.N, -math.log(s.N))
    _rw_factor(s, 2.38)
    rw, ws = s.rw_workspace(), s.ll_workspace()
    _lib.call("spa_loglik_rows", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, _p(ws["A"]), _p(ws["ylin"]),
              _p(s.ll), _p(ws["ws"]), ws["ws"].numel(), _stream())
    _lib.call("spa_prior_rows", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, 1.0, 0.9, 0.9, 2, _p(s.lp), _stream())
    zb = s.z_buffers(1)[0]
    _lib.call("spa_rw_normals", s.N, s.q, 3, 5, 0, 1, _p(zb), _stream())
    _lib.call("spa_rw_propose", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, s.factor_operand(), 3, 5, 0, 1,
              _p(zb), _p(rw["prop"]), _p(ws["A"]), _p(ws["ylin"]), 1.0, 0.9, _p(rw["lp_p"]), _stream())
    outs = []
    for fused in (False, True):
        beta, ll, lp = s.beta.clone(), s.ll.clone(), s.lp.clone()
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        if fused:
            _lib.call("spa_loglik_partials", ctypes.byref(d.struct), _p(ws["A"]), s.N, _p(ws["ws"]),
                      ws["ws"].numel(), _stream())
            _lib.call("spa_rw_accept_k1", _p(beta), s.ldb, _p(rw["prop"]), s.q, s.N, ctypes.byref(d.struct),
                      _p(ws["A"]), _p(ws["ylin"]), _p(ws["ws"]), _p(rw["lp_p"]), _p(ll), _p(lp), 3, 5, 0, 1, _p(cnt),
                      _stream())
        else:
            _lib.call("spa_loglik_softplus", ctypes.byref(d.struct), _p(ws["A"]), s.N, _p(ws["sp"]), _p(ws["ws"]),
                      ws["ws"].numel(), _stream())
            _lib.call("spa_rw_accept", _p(beta), s.ldb, _p(rw["prop"]), s.q, s.N, _p(ws["ylin"]), _p(ws["sp"]),
                      _p(rw["lp_p"]), _p(ll), _p(lp), 3, 5, 0, 1, _p(cnt), _stream())
        outs.append((beta, ll, lp, cnt))
    torch.cuda.synchronize()
    assert 0 < int(outs[0][3].item()) < s.N
    for a, b in zip(*outs):
        assert torch.equal(a, b)
