"""Per-kernel parity of the CUDA path against the golden vectors / oracle.

Tolerances:
  * Philox words, resampling ancestors: bit-exact;
  * per-particle log-likelihood (K1, bf16 hi/lo split on tcgen05, fp32
    accumulate): <= 1e-5 relative to the reference float64 values;
  * log-prior / reweight increments (float64 kernels): <= 1e-12 relative;
  * LSE / ESS: <= 1e-12 relative.
"""

import ctypes
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import spa_oracle as orc  # noqa: E402
from paper_1106_0322_b200 import _lib  # noqa: E402
from paper_1106_0322_b200.design import DeviceDesign  # noqa: E402
from paper_1106_0322_b200.smc import ParticleSystem, _p, _stream  # noqa: E402

LL_RTOL = 1e-5


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def system_from(X, y, B, intercept=False, a=1.0):
    d = DeviceDesign.build(X, y, intercept)
    s = ParticleSystem(d, B.shape[0], a, intercept)
    s.load_betas(B)
    return d, s


def gpu_loglik(X, y, B, intercept=False):
    d, s = system_from(X, y, B, intercept)
    out = torch.empty(s.N, dtype=torch.float64, device="cuda")
    ws = s.ll_workspace()
    _lib.call("spa_loglik_rows", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, _p(ws["A"]), _p(ws["ylin"]),
              _p(out), _p(ws["ws"]), ws["ws"].numel(), _stream())
    return out.cpu().numpy()


def test_philox_bits(gold_philox):
    for key, raw in zip(gold_philox["keys"], gold_philox["raw"]):
        k0, k1 = orc.stream_key(*(int(v) for v in key))
        out = torch.empty(16, dtype=torch.int64, device="cuda")
        _lib.call("spa_philox_blocks", k0, k1, 0, 4, _p(out), _stream())
        assert np.array_equal(out.cpu().numpy().view(np.uint64), raw)
    # far counters agree with the oracle too
    k = orc.stream_key(3, 1, 77, 12345)
    out = torch.empty(4 * 64, dtype=torch.int64, device="cuda")
    _lib.call("spa_philox_blocks", k[0], k[1], 10**9, 64, _p(out), _stream())
    assert np.array_equal(out.cpu().numpy().view(np.uint64).reshape(64, 4), orc.stream_blocks(k, 10**9, 64))


@pytest.mark.parametrize("s", [0.02, 0.1, 0.5])
def test_loglik_c1_vs_reference(gold_loglik, s):
    got = gpu_loglik(gold_loglik["c1_X"], gold_loglik["c1_y"], gold_loglik[f"c1_B_{s}"])
    ref = gold_loglik[f"c1_ll_{s}"]
    np.testing.assert_allclose(got, ref, rtol=LL_RTOL)


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_loglik_large_shapes_vs_reference(gold_loglik, name):
    from paper_1106_0322_b200.data import named_spec, simulate_dataset

    d, _ = simulate_dataset(named_spec(name))
    for s in (0.02, 0.1):
        got = gpu_loglik(d.X, d.y, gold_loglik[f"{name}_B_{s}"])
        np.testing.assert_allclose(got, gold_loglik[f"{name}_ll_{s}"], rtol=LL_RTOL)


def test_loglik_intercept_design(gold_loglik):
    got = gpu_loglik(gold_loglik["c1_X"], gold_loglik["c1_y"], gold_loglik["c1_Bi"], intercept=True)
    np.testing.assert_allclose(got, gold_loglik["c1_lli"], rtol=LL_RTOL)


def test_loglik_general_design(gold_loglik):
    """Non-integer (Gaussian) X takes the 3-product split path."""
    got = gpu_loglik(gold_loglik["g_X"], gold_loglik["g_y"], gold_loglik["g_B"])
    np.testing.assert_allclose(got, gold_loglik["g_ll"], rtol=LL_RTOL)


def test_loglik_many_particles_ragged_vs_oracle(gold_loglik):
    """Ragged particle count (not a multiple of the 128-row tile), several
    tiles and work units, against the float64 oracle."""
    X, y = gold_loglik["c1_X"], gold_loglik["c1_y"]
    B = np.random.default_rng(7).normal(0, 0.3, size=(1000 + 37, X.shape[1]))
    np.testing.assert_allclose(gpu_loglik(X, y, B), orc.loglik_rows(X, y, B), rtol=LL_RTOL)


@pytest.mark.parametrize("N", [1, 129, 255, 256, 257, 300, 513])
def test_loglik_int8_ragged_pair_tiles(gold_loglik, N):
    """The int8 CTA-pair kernel covers 256 particles per pair tile: particle
    counts below, at and across the pair boundary (the second CTA's rows
    partially or wholly beyond N), against the float64 oracle."""
    X, y = gold_loglik["c1_X"], gold_loglik["c1_y"]
    B = np.random.default_rng(N).normal(0, 0.3, size=(N, X.shape[1]))
    np.testing.assert_allclose(gpu_loglik(X, y, B), orc.loglik_rows(X, y, B), rtol=LL_RTOL)


def test_loglik_int8_row_scales():
    """Per-row fixed point: all-zero rows, a row dominated by one huge
    coefficient, rows far outside fp16's range (finite and correct here, the
    fp16 operand gave NaN from |alpha beta| >= 65504), tiny rows, and
    non-finite rows (NaN log-likelihood)."""
    from paper_1106_0322_b200.data import named_spec, simulate_dataset

    data, _ = simulate_dataset(named_spec("c2"))
    X, y = data.X, data.y
    q = X.shape[1]
    rng = np.random.default_rng(11)
    B = rng.normal(0, 0.05, size=(8, q))
    B[0] = 0.0                          # beta = 0: n log(1/2)
    B[1, 7] = 6.0                       # one dominant coefficient
    B[2] *= 1e5                         # |alpha beta| ~ 1e5: beyond fp16
    B[3] *= 1e-9                        # tiny but nonzero
    B[4, :] = 0.0
    B[4, q - 1] = -3.0                  # only the last (tail) column
    B[6, 3] = np.nan
    B[7, 5] = np.inf
    got = gpu_loglik(X, y, B)
    ref = orc.loglik_rows(X, y, np.nan_to_num(B[:6], posinf=0.0))
    np.testing.assert_allclose(got[:6], ref, rtol=LL_RTOL)
    assert np.isnan(got[6]) and np.isnan(got[7])


def test_loglik_known_answers():
    # beta = 0 -> n log(1/2) (test_model.py:131-136)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((40, 3))
    y = (rng.random(40) < 0.5).astype(float)
    got = gpu_loglik(X, y, np.zeros((2, 3)))
    np.testing.assert_allclose(got, 40 * np.log(0.5), rtol=1e-6)  # MUFU ex2/lg2


@pytest.mark.parametrize("s", [0.02, 0.5])
def test_log_prior_rows(gold_loglik, s):
    X, y, B = gold_loglik["c1_X"], gold_loglik["c1_y"], gold_loglik[f"c1_B_{s}"]
    d, sysm = system_from(X, y, B)
    out = torch.empty(sysm.N, dtype=torch.float64, device="cuda")
    for (a, c) in ((1.0, 2.0), (4.0, 0.3), (0.5, 0.05)):
        _lib.call("spa_prior_rows", ctypes.byref(d.struct), _p(sysm.beta), sysm.N, sysm.ldb, a, c, c, 0, _p(out),
                  _stream())
        # float32 particle storage: compare against the oracle on the stored values
        Bf = B.astype(np.float32).astype(np.float64)
        np.testing.assert_allclose(out.cpu().numpy(), orc.log_prior_rows(Bf, a, c), rtol=1e-12)
        np.testing.assert_allclose(out.cpu().numpy(), gold_loglik[f"c1_lp_{s}_{a}_{c}"], rtol=1e-6)


@pytest.mark.parametrize("a", [4.0, 1.0, 0.5, float("inf")])
def test_prior_reweight_fused(gold_loglik, a):
    """spa_prior_reweight = prior mode 1 (increments) + mode 2 (lp at the new
    scale; the fused pass groups columns per lane differently, so agreement
    is to float64 rounding)."""
    X, y, B = gold_loglik["c1_X"], gold_loglik["c1_y"], gold_loglik["c1_B_0.5"]
    d, s = system_from(X, y, B, a=a)
    c_prev, c = 0.9, 0.75
    lw = torch.empty(s.N, dtype=torch.float64, device="cuda")
    lp = torch.empty_like(lw)
    m1, m2 = torch.empty_like(lw), torch.empty_like(lw)
    _lib.call("spa_prior_reweight", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, a, c, c_prev, _p(lw), _p(lp),
              _stream())
    _lib.call("spa_prior_rows", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, a, c, c_prev, 1, _p(m1), _stream())
    _lib.call("spa_prior_rows", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, a, c, c, 2, _p(m2), _stream())
    np.testing.assert_allclose(lp.cpu().numpy(), m2.cpu().numpy(), rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(lw.cpu().numpy(), m1.cpu().numpy(), rtol=1e-12, atol=1e-12)
    Bf = B.astype(np.float32).astype(np.float64)
    np.testing.assert_allclose(lw.cpu().numpy(), orc.reweight_increments(Bf, a, c, c_prev), rtol=1e-9, atol=1e-10)


@pytest.mark.parametrize("q", [20, 200, 500, 1000])
def test_prior_reweight_wide_and_huge(q):
    """The vector-layout reweight kernels (one per q band) against the oracle,
    with rows of huge |beta| whose per-lane float64 product overflows and
    takes the sum-of-logs path (smc.py:248-263 semantics either way)."""
    from paper_1106_0322_b200.design import DeviceDesign
    from paper_1106_0322_b200.smc import ParticleSystem

    rng = np.random.default_rng(q)
    n, N, a, c, c_prev = 64, 96, 1.0, 0.6, 0.7
    X = rng.integers(0, 3, size=(n, q)).astype(np.float64)
    X = (X - X.mean(0)) / np.where(X.std(0) > 0, X.std(0), 1.0)
    y = (rng.random(n) < 0.5).astype(np.float64)
    B = rng.normal(0.0, 0.3, size=(N, q))
    B[::7] *= 1e12  # factors ~1e12: a lane's product overflows past 1e200
    B[3, :5] = 3e38
    d = DeviceDesign.build(X, y, False)
    s = ParticleSystem(d, N, a, False)
    s.load_betas(B)
    lw = torch.empty(N, dtype=torch.float64, device="cuda")
    lp = torch.empty_like(lw)
    _lib.call("spa_prior_reweight", ctypes.byref(d.struct), _p(s.beta), N, s.ldb, a, c, c_prev, _p(lw), _p(lp),
              _stream())
    Bf = B.astype(np.float32).astype(np.float64)
    np.testing.assert_allclose(lw.cpu().numpy(), orc.reweight_increments(Bf, a, c, c_prev), rtol=1e-11, atol=1e-9)
    np.testing.assert_allclose(lp.cpu().numpy(), orc.log_prior_rows(Bf, a, c), rtol=1e-12)


def test_reweight_and_ess(gold_reweight, gold_loglik):
    from paper_1106_0322_b200 import GtPrior, ess, reweight

    X, y = gold_loglik["c1_X"], gold_loglik["c1_y"]
    for tag in ("a4", "a1", "a05"):
        a, c_prev, c_t = (float(v) for v in gold_reweight[f"{tag}_params"])
        B = gold_reweight[f"{tag}_B"]
        d, s = system_from(X, y, B, a=a)
        s.log_weights = gold_reweight[f"{tag}_lw0"]
        lw, inc = reweight(s, GtPrior(a, c_t), GtPrior(a, c_prev))
        Bf = B.astype(np.float32).astype(np.float64)
        lw_ref = orc.reweight_increments(Bf, a, c_t, c_prev)
        np.testing.assert_allclose(lw, lw_ref, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(lw, gold_reweight[f"{tag}_lw"], rtol=1e-6, atol=1e-7)
        _, inc_ref = orc.normalise_log_weights(gold_reweight[f"{tag}_lw0"], lw_ref)
        assert inc == pytest.approx(inc_ref, abs=1e-12)
        w_ref = orc.weights_from_log(s.log_weights)
        np.testing.assert_allclose(s.weights, w_ref, rtol=1e-12)
        assert s.ess() == pytest.approx(orc.ess(w_ref), rel=1e-12)
        assert ess(gold_reweight[f"{tag}_w"]) == pytest.approx(float(gold_reweight[f"{tag}_ess"]), rel=1e-12)


def test_equal_scales_are_neutral(gold_loglik):
    from paper_1106_0322_b200 import GtPrior, reweight

    d, s = system_from(gold_loglik["c1_X"], gold_loglik["c1_y"], gold_loglik["c1_B_0.1"], a=4.0)
    before = s.log_weights.copy()
    lw, inc = reweight(s, GtPrior(4.0, 0.5), GtPrior(4.0, 0.5))
    assert np.array_equal(lw, np.zeros(s.N))
    assert inc == pytest.approx(0.0, abs=1e-12)
    np.testing.assert_allclose(s.log_weights, before, atol=1e-12)


def test_degenerate_weights_raise(gold_loglik):
    from paper_1106_0322_b200 import DegeneracyError, GtPrior, reweight

    d, s = system_from(gold_loglik["c1_X"], gold_loglik["c1_y"], gold_loglik["c1_B_0.1"], a=4.0)
    s.log_weights = np.full(s.N, -np.inf)
    with pytest.raises(DegeneracyError):
        reweight(s, GtPrior(4.0, 0.4), GtPrior(4.0, 0.5))
    with pytest.raises(ValueError):
        reweight(s, GtPrior(3.0, 0.4), GtPrior(4.0, 0.5))


def test_resample_ancestors_bit_exact(gold_resample):
    from paper_1106_0322_b200 import systematic_resample_indices

    for k, (N, alpha) in enumerate(gold_resample["cases"]):
        N = int(N)
        w = gold_resample[f"w_{k}"] if f"w_{k}" in gold_resample else \
            np.random.default_rng(1000 + k).dirichlet(np.full(N, alpha))
        assert sha(w) == str(gold_resample[f"wsha_{k}"])
        got = systematic_resample_indices(w, float(gold_resample[f"u_{k}"]))
        assert np.array_equal(got, gold_resample[f"idx_{k}"]), (N, alpha)


def test_resample_edge_cases(gold_resample):
    from paper_1106_0322_b200 import systematic_resample_indices

    for e in range(4):
        for j in range(3):
            w, u = gold_resample[f"ew_{e}_{j}"], float(gold_resample[f"eu_{e}_{j}"])
            assert np.array_equal(systematic_resample_indices(w, u), gold_resample[f"eidx_{e}_{j}"])


def test_resample_many_random_trials_bit_exact():
    """>= 1000 Dirichlet trials, alpha in [0.05, 2], N up to 2^16 (SURVEY 8(c) iii)."""
    from paper_1106_0322_b200 import systematic_resample_indices

    rng = np.random.default_rng(2024)
    for trial in range(1000):
        N = int(rng.choice([7, 100, 1024, 5000, 65536]) if trial % 50 else 65536)
        alpha = float(rng.uniform(0.05, 2.0))
        w = rng.dirichlet(np.full(N, alpha))
        u = rng.random() / N
        assert np.array_equal(systematic_resample_indices(w, u), orc.systematic_ancestors(w, u)), (trial, N, alpha)


def test_resample_large_n_bit_exact():
    from paper_1106_0322_b200 import systematic_resample_indices

    rng = np.random.default_rng(5)
    for N in (2**20,):
        w = rng.dirichlet(np.full(N, 0.5))
        u = rng.random() / N
        assert np.array_equal(systematic_resample_indices(w, u), orc.systematic_ancestors(w, u))


def _exact_cumsum(w):
    wd = torch.from_numpy(np.ascontiguousarray(w, dtype=np.float64)).cuda()
    N = wd.numel()
    cum = torch.empty(N, dtype=torch.float64, device="cuda")
    mode = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    ws = torch.empty(_lib.load().spa_resample_workspace_bytes(N), dtype=torch.uint8, device="cuda")
    _lib.call("spa_exact_cumsum", _p(wd), N, _p(cum), _p(mode), _p(ws), ws.numel(), _stream())
    return cum.cpu().numpy(), int(mode.item())


def _cumsum_families():
    """(name, weights, fast-path expected) covering ties, zeros, ragged
    tiles, many binade changes per tile and the fallback triggers."""
    rng = np.random.default_rng(99)
    out = []
    for N in (1, 2, 7, 2047, 2048, 2049, 65536, 65539, 1 << 20):
        for alpha in (0.3, 1.0, 2.0):
            out.append((f"dirichlet{alpha}_{N}", rng.dirichlet(np.full(N, alpha)), True))
    N = 65536
    out.append(("uniform", np.full(N, 1.0 / N), True))                      # every add a power-of-two pattern
    out.append(("uniform_3", np.full(N, 1.0 / 3.0), True))                  # sums > 1
    out.append(("exact_ints", rng.integers(0, 4, N) * 2.0**-20, True))      # exactly representable sums
    w = rng.choice([1.0, 3.0, 5.0], N) * 2.0**-53
    w[0] = 1.5
    out.append(("ties", w, True))                                           # every add an exact half-ulp tie
    w = w.copy()
    w[0] = 1.0
    out.append(("ties_at_power_of_two", w, False))                          # all prefixes ambiguous: fallback
    # multiples of 1e-3 land within rounding distance of 4: the float64 chain
    # sits below 4 where the fixed-point prefix is above, with nonzero weights
    # following -> the verified fallback (either path must give np.cumsum)
    out.append(("half_ulps", (rng.integers(1, 3, N) * 2.0**-60) + np.where(np.arange(N) % 5 == 0, 1e-3, 0.0), None))
    w = rng.random(N)
    w[:100] = 0.0
    out.append(("leading_zeros", w / w.sum(), True))
    w = rng.random(N)
    w[::3] = 0.0
    out.append(("interior_zeros", w, True))
    out.append(("single_one", np.eye(1, N, 4321).ravel(), True))
    out.append(("geometric_heads", np.geomspace(1e-28, 1.0, 4096), True))   # a binade change every ~30 elements
    out.append(("dense_heads", 2.0 ** np.arange(-90, -90 + 2048 * 3) .clip(-90, 20), False))  # > kHMax per tile
    w = rng.dirichlet(np.full(N, 0.05))
    out.append(("dirichlet0.05", w, None))                                   # tiny leading prefixes: either path
    w = rng.random(N)
    w[0] = 1e-310                                                            # denormal first prefix: fallback
    out.append(("denormal_start", w, False))
    out.append(("huge", rng.random(N) * 1e30, False))                        # >= 2^27: fallback
    w = rng.random(N)
    w[17] = np.nan
    out.append(("nan", w, False))
    return out


def test_exact_cumsum_matches_numpy_bit_for_bit():
    """The parallel binade-segmented scan equals np.cumsum (the reference's
    strictly sequential float64 chain, smc.py:276) on every element, and the
    realistic weight vectors take the parallel fast path."""
    for name, w, fast in _cumsum_families():
        cum, mode = _exact_cumsum(w)
        ref = np.cumsum(w)
        same = (cum == ref) | (np.isnan(cum) & np.isnan(ref))
        assert same.all(), (name, int(np.argmin(same)))
        if fast is not None:  # mode: 0 = parallel fast path, > 0 = the fallback's reason code
            assert (mode == 0) == fast, (name, mode)


def test_gather_rows_and_system_resample(gold_loglik):
    from paper_1106_0322_b200 import systematic_resample

    X, y, B = gold_loglik["c1_X"], gold_loglik["c1_y"], gold_loglik["c1_B_0.5"]
    d, s = system_from(X, y, B)
    rng = np.random.default_rng(33)
    s.log_weights = np.log(rng.dirichlet(np.ones(s.N)))
    s.ll.copy_(torch.arange(s.N, dtype=torch.float64))
    original = s.betas.copy()
    idx = systematic_resample(s, 0.37)
    np.testing.assert_allclose(s.weights, 1.0 / s.N)
    np.testing.assert_array_equal(s.betas, original[idx])
    np.testing.assert_array_equal(s.logliks, idx.astype(float))


def _tc_gemm(A, B, terms=1):
    m = A.shape[0]
    rows, kp = B.shape
    At = torch.from_numpy(np.ascontiguousarray(A, np.float32)).cuda().to(torch.bfloat16).contiguous()
    Bt = torch.from_numpy(np.ascontiguousarray(B, np.float32)).cuda().to(torch.bfloat16).contiguous()
    C = torch.zeros((m, rows), dtype=torch.float32, device="cuda")
    _lib.call("spa_tc_gemm_f32", _p(At), m, terms, _p(Bt), rows, kp, _p(C), rows, _stream())
    return C.cpu().numpy()


@pytest.mark.parametrize("m,rows,kp", [(128, 256, 64), (128, 256, 128), (300, 300, 192), (1, 20, 64)])
def test_tc_gemm_exact_integers(m, rows, kp):
    """The raw tcgen05 engine (TMA SW128 -> UMMA -> TMEM -> epilogue) on
    exactly representable integer inputs: results must be exact."""
    rng = np.random.default_rng(m + rows + kp)
    A = np.zeros((m, kp), np.float32)
    B = np.zeros((rows, kp), np.float32)
    A[np.arange(m), np.arange(m) % kp] = 1
    B[np.arange(rows), np.arange(rows) % kp] = 1
    np.testing.assert_array_equal(_tc_gemm(A, B), A @ B.T)
    A = rng.integers(-3, 4, (m, kp)).astype(np.float32)
    B = rng.integers(0, 3, (rows, kp)).astype(np.float32)
    np.testing.assert_array_equal(_tc_gemm(A, B), A @ B.T)
    A2 = np.concatenate([A, rng.integers(-3, 4, (m, kp)).astype(np.float32)], 1)
    np.testing.assert_array_equal(_tc_gemm(A2, B, 2), A2[:, :kp] @ B.T + A2[:, kp:] @ B.T)


def _rw_setup(name="c1", N=1000, seed=3):
    from paper_1106_0322_b200.data import named_spec, simulate_dataset

    data, _ = simulate_dataset(named_spec(name))
    rng = np.random.default_rng(seed)
    C = rng.normal(size=(data.p, data.p)) * 0.05
    B = rng.normal(size=(N, data.p)) @ C + rng.normal(0, 0.1, size=data.p)
    d, s = system_from(data.X, data.y, B)
    return data, d, s, B


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_rw_moments_and_factor(name):
    """Fixed-point moments (tcgen05 SYRK) and the blocked Cholesky factor vs
    the float64 oracle (weighted covariance, numpy Cholesky)."""
    from paper_1106_0322_b200.smc import _rw_factor

    data, d, s, B = _rw_setup(name)
    s.log_weights = np.log(np.random.default_rng(1).dirichlet(np.ones(s.N) * 2.0))
    rw = s.rw_workspace()
    # first call: centred on the exact mean; second: on the previous mean
    # after the population moved (covariance recovered as M - delta delta^T)
    for shift in (0.0, 0.3):
        B = B + shift * np.linspace(-1.0, 1.0, s.q)
        s.load_betas(B)
        _rw_factor(s, 2.38)
        assert int(rw["info"].item()) == 0
        w = s.weights
        Bf = B.astype(np.float32).astype(np.float64)
        Ls_ref, mu_ref, S_ref = orc.rw_cov_factor(Bf, w)
        np.testing.assert_allclose(rw["ctr"].cpu().numpy(), mu_ref, rtol=1e-6, atol=1e-7)
        L = rw["L"].cpu().numpy().astype(np.float64)
        # bf16 SYRK operands (2^-9 relative per element): entries within
        # 1e-3 of the largest variance
        np.testing.assert_allclose(L @ L.T, Ls_ref @ Ls_ref.T, rtol=2e-3,
                                   atol=1e-3 * np.abs(Ls_ref @ Ls_ref.T).max())
        assert np.allclose(np.triu(L, 1), 0.0)


@pytest.mark.parametrize("q", [5, 33, 100, 500, 512, 520, 700])
def test_rw_factor_paths(q):
    """spa_rw_factor (blocked Cholesky, graph of panel kernels) on a
    fixed-point SPD matrix vs numpy, including partial panels and q > 512;
    the scaled bf16 operand is L * scale/sqrt(q) with zero padding columns."""
    from paper_1106_0322_b200.smc import _round_up

    rng = np.random.default_rng(q)
    G = rng.normal(size=(q, q + 8)) / np.sqrt(q)
    S = G @ G.T + 0.05 * np.eye(q)
    Sfix = np.rint(np.tril(S) * 2.0**48).astype(np.int64)
    acc = torch.zeros(q + q * q, dtype=torch.int64)
    acc[q:] = torch.from_numpy(Sfix.reshape(-1))
    acc = acc.cuda()
    kq = _round_up(q, 64)
    L = torch.zeros((q, q), dtype=torch.float32, device="cuda")
    fws = torch.zeros((_round_up(8 * q * q, 256) + _round_up(2 * q * kq, 256) + 8192) // 8 + 1, dtype=torch.float64,
                      device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    jitter, scale = 1e-6, 2.38
    _lib.call("spa_rw_factor", _p(acc), q, scale, jitter, _p(L), _p(fws), _p(info), None, _stream())
    assert int(info.item()) == 0
    Sref = np.tril(Sfix).astype(np.float64) / 2.0**48
    Sref = Sref + np.tril(Sref, -1).T
    Sref[np.diag_indices(q)] += jitter * np.trace(Sref) / q
    Lref = np.linalg.cholesky(Sref) * (scale / np.sqrt(q))
    Lg = L.cpu().numpy().astype(np.float64)
    assert np.allclose(np.triu(Lg, 1), 0.0)
    np.testing.assert_allclose(Lg, Lref, rtol=0, atol=2e-5 * np.abs(Lref).max())
    off = _round_up(8 * q * q, 256)
    Lb = fws.view(torch.uint8)[off: off + 2 * q * kq].view(torch.bfloat16).view(q, kq).float().cpu().numpy()
    np.testing.assert_array_equal(Lb[:, :q], torch.from_numpy(L.cpu().numpy()).to(torch.bfloat16).float().numpy())
    assert not Lb[:, q:].any()


def test_rw_factor_under_contention():
    """The panel kernels' CTAs are not co-scheduled when other streams hold
    SMs: the factor must be bit-identical to the idle-device result while
    matmuls run on another stream (regression: the diagonal block used to be
    overwritten in place by CTA 0 before the other CTAs had read it)."""
    from paper_1106_0322_b200.smc import _round_up

    q = 500
    rng = np.random.default_rng(5)
    G = rng.normal(size=(q, q + 8)) / np.sqrt(q)
    S = G @ G.T + 0.05 * np.eye(q)
    acc = torch.zeros(q + q * q, dtype=torch.int64)
    acc[q:] = torch.from_numpy(np.rint(np.tril(S) * 2.0**48).astype(np.int64).reshape(-1))
    acc = acc.cuda()
    kq = _round_up(q, 64)
    nws = (_round_up(8 * q * q, 256) + _round_up(2 * q * kq, 256) + 8192) // 8 + 1

    def factor(stream):
        L = torch.zeros((q, q), dtype=torch.float32, device="cuda")
        fws = torch.zeros(nws, dtype=torch.float64, device="cuda")
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("spa_rw_factor", _p(acc), q, 2.38, 1e-6, _p(L), _p(fws), _p(info), None,
                  ctypes.c_void_p(stream.cuda_stream))
        return L, info

    main = torch.cuda.current_stream()
    L0, info0 = factor(main)
    torch.cuda.synchronize()
    ref = L0.cpu()
    busy, side = torch.cuda.Stream(), torch.cuda.Stream()
    X = torch.randn(4096, 4096, device="cuda")
    outs = []
    for _ in range(6):
        with torch.cuda.stream(busy):
            for _ in range(4):
                X = (X @ X).clamp_(-1, 1)
        with torch.cuda.stream(side):
            outs.append(factor(side))
    torch.cuda.synchronize()
    assert int(info0.item()) == 0
    for L, info in outs:
        assert int(info.item()) == 0
        assert torch.equal(L.cpu(), ref)


@pytest.mark.parametrize("name,N", [("c1", 1536 + 77), ("c2", 1536), ("c3", 1536), ("c5", 1536 + 77)])
def test_rw_propose_eps_multi_tile(name, N):
    """eps = L z of spa_rw_propose at q = 20 / 200 / 500 / 1000 (one to four
    256-coordinate tiles of the CTA-pair kernel, several K blocks, a ragged
    last pair of particle tiles) equals the float32 product of the same bf16
    operands to bf16 output rounding."""
    from paper_1106_0322_b200.smc import _round_up

    data, d, s, B = _rw_setup(name, N=N)
    from paper_1106_0322_b200.smc import _rw_factor

    _rw_factor(s, 2.38)
    rw, ws = s.rw_workspace(), s.ll_workspace()
    zb = s.z_buffers(1)[0]
    _lib.call("spa_rw_normals", s.N, s.q, 3, 5, 0, 1, _p(zb), _stream())
    _lib.call("spa_rw_propose", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, s.factor_operand(), 3, 5, 0, 1,
              _p(zb), _p(rw["prop"]), _p(ws["A"]), _p(ws["ylin"]), 1.0, 0.9, _p(rw["lp_p"]), _stream())
    q, kq = s.q, _round_up(s.q, 64)
    off = _round_up(8 * q * q, 256)
    L = rw["fws"].view(torch.uint8)[off: off + 2 * q * kq].view(torch.bfloat16).view(q, kq).float()
    ref = zb.float() @ L.T
    got = rw["prop"][:, :q].float()
    np.testing.assert_allclose(got.cpu().numpy(), ref.cpu().numpy(), rtol=1e-2, atol=2e-3 * ref.abs().max().item())
    assert not rw["prop"][:, q:].float().any()


def test_rw_propose_and_accept_vs_oracle():
    """One RW move: proposal (Philox normals, L z on tcgen05, fused pack),
    K1 likelihood of the proposal and the MH decision vs the oracle."""
    from paper_1106_0322_b200 import GtPrior
    from paper_1106_0322_b200.smc import _loglik_device, _rw_factor

    data, d, s, B = _rw_setup("c1", N=777)
    _rw_factor(s, 2.38)
    rw, ws = s.rw_workspace(), s.ll_workspace()
    a, c, seed, t, move = 1.0, 0.8, 11, 7, 2
    _loglik_device(s, s.ll)
    _lib.call("spa_prior_rows", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, a, c, c, 2, _p(s.lp), _stream())
    beta0, ll0, lp0 = s.betas.copy(), s.logliks.copy(), s.lp.cpu().numpy().copy()
    np.testing.assert_allclose(lp0, orc.log_prior_rows(beta0, a, c), rtol=1e-6)
    zb = s.z_buffers(1)[0]
    _lib.call("spa_rw_normals", s.N, s.q, seed, t, 0, move, _p(zb), _stream())
    _lib.call("spa_rw_propose", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, s.factor_operand(), seed, t, 0, move,
              _p(zb), _p(rw["prop"]), _p(ws["A"]), _p(ws["ylin"]), a, c, _p(rw["lp_p"]), _stream())
    eps = rw["prop"][:, : s.q].float().cpu().numpy()  # eps = L z (bf16)
    prop = (s.beta[:, : s.q].cpu().numpy() + eps).astype(np.float64)
    Lbf = torch.from_numpy(rw["L"].cpu().numpy()).to(torch.bfloat16).double().numpy()
    Z = np.stack([orc.rw_normals(seed, t, k, move, s.q) for k in range(s.N)])
    Zb = torch.from_numpy(Z).to(torch.bfloat16).double().numpy()
    # device normals use fast intrinsics (~1e-6); a z within that of a bf16
    # rounding boundary rounds the other way (one bf16 ulp): allow rare flips
    diff = np.abs(prop - (beta0 + Zb @ Lbf.T))
    # eps is stored in bf16: compare with the oracle increment rounded to bf16
    eps_ref = torch.from_numpy(Zb @ Lbf.T).to(torch.bfloat16).double().numpy()
    assert np.mean(np.abs(eps - eps_ref) > 2.0**-8 * np.abs(eps_ref) + 1e-12) < 0.005
    assert diff.max() < 2.0**-7 * np.abs(Zb).max() * np.abs(Lbf).max() * 4
    np.testing.assert_allclose(ws["ylin"].cpu().numpy(), prop @ (data.X.T @ data.y), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(rw["lp_p"].cpu().numpy(), orc.log_prior_rows(prop, a, c), rtol=1e-6)
    _lib.call("spa_loglik_softplus", ctypes.byref(d.struct), _p(ws["A"]), s.N, _p(ws["sp"]), _p(ws["ws"]),
              ws["ws"].numel(), _stream())
    ll_p = ws["ylin"].cpu().numpy() - ws["sp"].cpu().numpy()
    np.testing.assert_allclose(ll_p, orc.loglik_rows(data.X, data.y, prop), rtol=1e-5)
    s.counter.zero_()
    _lib.call("spa_rw_accept", _p(s.beta), s.ldb, _p(rw["prop"]), s.q, s.N, _p(ws["ylin"]), _p(ws["sp"]),
              _p(rw["lp_p"]), _p(s.ll), _p(s.lp), seed, t, 0, move, _p(s.counter), _stream())
    u = np.array([orc.rw_accept_uniform(seed, t, k, move) for k in range(s.N)])
    dlt = (ll_p + rw["lp_p"].cpu().numpy()) - (ll0 + lp0)
    with np.errstate(divide="ignore"):
        ok = (dlt >= 0) | (np.log(u) < dlt)
    assert int(s.counter.item()) == int(ok.sum()) and 0 < ok.sum() < s.N
    np.testing.assert_array_equal(s.betas, np.where(ok[:, None], prop, beta0))


def test_code_columns_on_device_match_host():
    """The device column coder (used by DeviceDesign.build) reproduces the
    host _code_column exactly: constant, 2-level, 3-level and continuous
    columns, including standardised genotypes."""
    from paper_1106_0322_b200.data import named_spec, simulate_dataset
    from paper_1106_0322_b200.design import _code_column, _code_columns

    data, _ = simulate_dataset(named_spec("c2"))
    X = np.asarray(data.X, dtype=np.float64)
    rng = np.random.default_rng(0)
    X = np.column_stack([np.ones(X.shape[0]), X, rng.normal(size=X.shape[0]),
                         np.where(X[:, 0] > X[:, 0].min(), 1.5, -0.25), np.full(X.shape[0], -3.0),
                         rng.integers(0, 3, X.shape[0]) * 0.7 - 0.1])
    host = [_code_column(X[:, j]) for j in range(X.shape[1])]
    dev = _code_columns(X, torch.device("cuda"))
    assert sum(h is None for h in host) == 1
    for h, d in zip(host, dev):
        assert (h is None) == (d is None)
        if h is not None:
            assert np.array_equal(h[0], d[0]) and h[1] == d[1] and h[2] == d[2] and np.array_equal(h[3], d[3])


@pytest.mark.parametrize("m", [1000, 8192, 65536 + 77])
def test_reweight_finish_matches_kernel_sequence(m):
    """spa_reweight_finish (one cooperative launch) against the sequence it
    replaces -- chunk statistics of logw + lw, combine, apply, step record,
    statistics and combine of the new logw, normalised weights -- bit for bit
    in every output (logw, chunk statistics, lse / ESS, step record, w)."""
    from paper_1106_0322_b200.smc import _p, _stream

    g = torch.Generator(device="cuda")
    g.manual_seed(m)
    logw0 = torch.randn(m, device="cuda", dtype=torch.float64, generator=g) * 2
    lw = torch.randn(m, device="cuda", dtype=torch.float64, generator=g) * 3
    nch = -(-m // 4096)
    outs = []
    for fused in (False, True):
        logw = logw0.clone()
        stats = torch.zeros((2 * nch if fused else nch, 3), dtype=torch.float64, device="cuda")
        res = torch.zeros(3, dtype=torch.float64, device="cuda")
        rec = torch.zeros((10, 4), dtype=torch.float64, device="cuda")
        rec[2, 3] = 1.25
        w = torch.zeros(m, dtype=torch.float64, device="cuda")
        if fused:  # stats: the final chunk statistics, then a scratch set
            _lib.call("spa_reweight_finish", _p(logw), _p(lw), m, _p(stats), _p(res), _p(rec), 3, 0.75 * m, _p(w),
                      _stream())
            stats = stats[:nch]
        else:
            _lib.call("spa_lse_chunk_stats", _p(logw), _p(lw), m, _p(stats), _stream())
            _lib.call("spa_lse_combine", _p(stats), nch, _p(res), _stream())
            _lib.call("spa_logw_apply", _p(logw), _p(lw), m, _p(res), None, _stream())
            _lib.call("spa_step_record", _p(res), _p(rec), 3, 0.75 * m, _stream())
            _lib.call("spa_lse_chunk_stats", _p(logw), None, m, _p(stats), _stream())
            _lib.call("spa_lse_combine", _p(stats), nch, _p(res), _stream())
            _lib.call("spa_logw_apply", _p(logw), None, m, _p(res), _p(w), _stream())
        outs.append((logw, stats, res, rec, w))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    assert abs(float(outs[1][4].sum()) - 1.0) < 1e-12
