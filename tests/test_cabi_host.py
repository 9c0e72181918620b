"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares, and the host-side logic (config validation, design coding,
persistence format) behaves like the reference."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "spa_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(spa_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    import ctypes

    from paper_1106_0322_b200 import _lib

    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    # the ctypes binding declares exactly the header's functions
    assert sorted(_lib.exported_symbols()) == names


def test_library_reports_version_and_errors_without_gpu():
    from paper_1106_0322_b200 import _lib

    lib = _lib.load()
    assert lib.spa_version() >= 1
    # argument validation runs before any device work
    rc = lib.spa_philox_blocks(0, 0, 0, -1, None, None)
    assert rc == 1001
    assert b"bad arguments" in lib.spa_last_error()


def test_sass_contains_tcgen05_and_tma():
    """The likelihood kernel is tcgen05/TMA code (B200_PROFILING.md mnemonics)."""
    import shutil
    import subprocess

    so = os.path.join(ROOT, "paper_1106_0322_b200", "libspa_b200.so")
    if shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("cuobjdump unavailable")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([exe, "-sass", so], capture_output=True, text=True, check=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert "HMMA" not in sass.replace("UTCHMMA", "")
    # the int8 likelihood kernel: CTA-pair integer MMAs and pair-scoped TMA loads
    assert "UTCIMMA.2CTA" in sass and "UTMALDG.2D.2CTA" in sass
    assert "IMMA" not in sass.replace("UTCIMMA", "")
    # the proposal increments L z: CTA-pair bf16 MMAs in lz_pair_kernel
    i = sass.index("lz_pair_kernel")
    body = sass[i: sass.find("Function :", i + 1)]
    assert "UTCHMMA.2CTA" in body and "UTMALDG.2D.2CTA" in body and "UTMASTG" in body


class TestConfig:
    @pytest.mark.parametrize("b1,rho,T", [(2.0, 1.0, 10), (2.0, 1.2, 10), (0.0, 0.9, 10), (2.0, 0.9, 0)])
    def test_invalid_schedule(self, b1, rho, T):
        from paper_1106_0322_b200 import make_schedule

        with pytest.raises(ValueError):
            make_schedule(b1, rho, T)

    def test_schedule_values(self):
        from paper_1106_0322_b200 import make_schedule

        s = make_schedule(2.0, 0.98, 450)
        assert s.bs[0] == pytest.approx(2.0) and s.bs[449] == pytest.approx(2.0 * 0.98**449)

    @pytest.mark.parametrize("kw", [dict(N=1), dict(cycles=0), dict(step_sd=0), dict(ess_threshold_frac=0),
                                    dict(seed=-1), dict(init_thin=0), dict(move_kernel="hmc"), dict(moves=0)])
    def test_invalid_config(self, kw):
        from paper_1106_0322_b200 import SmcConfig

        with pytest.raises(ValueError):
            SmcConfig(**kw)

    def test_prior_validation(self):
        import math

        from paper_1106_0322_b200 import GtPrior

        for a, c in [(0, 1), (-1, 1), (1, 0), (1, -0.5)]:
            with pytest.raises(ValueError):
                GtPrior(a, c)
        assert GtPrior(math.inf, 0.5).lambda_de == 2.0


class TestDesignCoding:
    def test_standardised_genotypes_are_coded(self, small_data):
        from paper_1106_0322_b200.design import _code_column

        for j in range(small_data.p):
            x = small_data.X[:, j]
            codes, alpha, gamma, lev = _code_column(x)
            np.testing.assert_allclose(alpha * codes + gamma, x, rtol=0, atol=1e-12)
            assert set(np.unique(codes)) <= {0, 1, 2}
            np.testing.assert_array_equal(lev[codes], x)

    def test_gaussian_column_is_not_coded(self):
        from paper_1106_0322_b200.design import _code_column

        assert _code_column(np.random.default_rng(0).standard_normal(40)) is None

    def test_intercept_column(self):
        from paper_1106_0322_b200.design import _code_column

        codes, alpha, gamma, lev = _code_column(np.ones(10))
        assert alpha == 0.0 and gamma == 1.0 and np.all(codes == 0)


def test_persistence_round_trip(tmp_path):
    """save_run/load_run keep the reference's files and format (smc.py:532-592)."""
    from paper_1106_0322_b200.smc import SmcConfig, SmcOutput, StepRecord, load_run, make_schedule, save_run

    rng = np.random.default_rng(0)
    steps = []
    for t in range(1, 4):
        w = rng.dirichlet(np.ones(8))
        steps.append(StepRecord(t, 2.0 * 0.9 ** (t - 1), float(1 / (w @ w)), -0.1 * t, 0.3, t == 2, w,
                                rng.standard_normal((8, 3)), rng.standard_normal(8)))
    out = SmcOutput(4.0, make_schedule(2.0, 0.9, 3), SmcConfig(N=8), False, ["a", "b", "c"], steps, 0.3)
    save_run(out, tmp_path / "run")
    back = load_run(tmp_path / "run")
    assert back.names == out.names and back.a == out.a and back.config.N == 8
    for s1, s2 in zip(out.steps, back.steps):
        assert s1.log_z_ratio_cum == s2.log_z_ratio_cum
        np.testing.assert_array_equal(s1.particles, s2.particles)
        np.testing.assert_array_equal(s1.weights, s2.weights)
    assert (tmp_path / "run" / "trace.csv").read_text().splitlines()[0] == "t,b,ess,log_z_ratio_cum,acceptance_rate"


def test_init_plan_covers_slots_once():
    """Chain c fills slots [c R, (c+1) R): every slot exactly once, K * R >= N,
    and a rank's chain range covers its shard for any world size."""
    from paper_1106_0322_b200.smc import init_plan

    for N, chains, auto in [(65536, 0, 444), (8192, 300, 0), (1000, 0, 4096), (7, 0, 3), (1, 0, 5)]:
        K, R = init_plan(N, chains, auto)
        assert K * R >= N > (K - 1) * R
        for world in (1, 2, 4):
            if N % world:
                continue
            M = N // world
            for r in range(world):
                lo, hi = r * M, (r + 1) * M
                c0, c1 = lo // R, min(K, -(-hi // R))
                assert c0 * R <= lo and hi <= c1 * R


def _py_rows(W, P, index0=0):
    """The reference writer's row format (smc.py:546-549)."""
    return "".join(f"{index0 + i},{W[i]:.17g}," + ",".join(f"{v:.17g}" for v in P[i]) + "\n"
                   for i in range(P.shape[0]))


def test_format_particle_rows_matches_python():
    """f2 fast writer: byte-identical to f"{v:.17g}" rows, edge values included."""
    import ctypes

    from paper_1106_0322_b200 import _lib

    rng = np.random.default_rng(9)
    P = rng.normal(0, 0.3, size=(1500, 7)).astype(np.float32).astype(np.float64)
    edge = [0.0, -0.0, 1e-300, -1e300, 5e-324, 2.2250738585072014e-308, 1 / 3, 0.1, 123456789.0, 1e16, 1e17,
            -1e-5, 1e-4, 9.999999999999999e22, float("inf"), float("-inf"), float("nan")]
    P[:3, :] = np.resize(np.array(edge), (3, 7))
    W = rng.dirichlet(np.ones(P.shape[0]))
    W[5] = 0.0
    cap = 4 << 20
    buf = ctypes.create_string_buffer(cap)
    used = ctypes.c_size_t(0)
    for threads in (1, 8):
        _lib.call("spa_format_particle_rows", W.ctypes.data, P.ctypes.data, P.shape[0], P.shape[1], 10, buf, cap,
                  ctypes.byref(used), threads)
        assert buf.raw[:used.value].decode() == _py_rows(W, P, 10)


def test_save_run_particles_byte_identical(tmp_path):
    from paper_1106_0322_b200.smc import write_particles_csv

    rng = np.random.default_rng(3)
    P = rng.standard_t(2.0, size=(40000, 5)) * 0.1
    W = rng.dirichlet(np.ones(P.shape[0]) * 0.5)
    names = [f"snp{j}" for j in range(5)]
    write_particles_csv(tmp_path / "p.csv", names, W, P, chunk=7000)
    expect = "particle_index,weight," + ",".join(names) + "\n" + _py_rows(W, P)
    assert (tmp_path / "p.csv").read_text() == expect
