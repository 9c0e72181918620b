"""Pin the CPU oracle (oracle/spa_oracle.py) against golden vectors produced
by running the reference implementation (tests/golden/make_golden.py).
CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import golden
from oracle import spa_oracle as orc


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class TestPhilox:
    def test_raw_words_match_numpy_philox(self, gold_philox):
        for key, raw in zip(gold_philox["keys"], gold_philox["raw"]):
            seed, tag, t, i = (int(v) for v in key)
            got = orc.stream_raw(orc.stream_key(seed, tag, t, i), 16)
            assert np.array_equal(got, raw)

    def test_uniforms_match_reference_stream(self, gold_philox):
        for key, uni in zip(gold_philox["keys"], gold_philox["uniform"]):
            seed, tag, t, i = (int(v) for v in key)
            got = orc.u53(orc.stream_raw(orc.stream_key(seed, tag, t, i), 9))
            assert np.array_equal(got, uni)

    def test_host_philox_matches_oracle(self, gold_philox):
        from paper_1106_0322_b200._philox_host import philox_block, stream_key

        for key, raw in zip(gold_philox["keys"], gold_philox["raw"]):
            k0, k1 = stream_key(*(int(v) for v in key))
            blocks = [philox_block(k0, k1, b) for b in range(4)]
            assert np.array_equal(np.array(blocks, dtype=np.uint64).ravel(), raw)


class TestModel:
    def test_loglik_rows(self, gold_loglik):
        X, y = gold_loglik["c1_X"], gold_loglik["c1_y"]
        for s in (0.02, 0.1, 0.5):
            got = orc.loglik_rows(X, y, gold_loglik[f"c1_B_{s}"])
            np.testing.assert_allclose(got, gold_loglik[f"c1_ll_{s}"], rtol=1e-12)

    def test_log_prior_rows(self, gold_loglik):
        for s in (0.02, 0.1, 0.5):
            B = gold_loglik[f"c1_B_{s}"]
            for (a, c) in ((1.0, 2.0), (4.0, 0.3), (0.5, 0.05)):
                np.testing.assert_allclose(orc.log_prior_rows(B, a, c), gold_loglik[f"c1_lp_{s}_{a}_{c}"], rtol=1e-13)

    def test_c5_shapes(self):
        """n=10000, p=1000 (BASELINE configs[4]): log-lik and the prior sums
        for a in {0.5, 1, 4} and the double-exponential limit."""
        from paper_1106_0322_b200.data import named_spec, simulate_dataset

        g = golden("loglik_c5.npz")
        d, _ = simulate_dataset(named_spec("c5"))
        for s in (0.02, 0.1):
            B = g[f"c5_B_{s}"]
            np.testing.assert_allclose(orc.loglik_rows(d.X, d.y, B), g[f"c5_ll_{s}"], rtol=1e-12)
            for a in (0.5, 1.0, 4.0):
                np.testing.assert_allclose(orc.log_prior_rows(B, a, 0.3), g[f"c5_lp_{s}_{a}"], rtol=1e-13)
            np.testing.assert_allclose(orc.log_prior_rows(B, float("inf"), 0.3), g[f"c5_lp_{s}_de"], rtol=1e-13)

    def test_gaussian_design(self, gold_loglik):
        got = orc.loglik_rows(gold_loglik["g_X"], gold_loglik["g_y"], gold_loglik["g_B"])
        np.testing.assert_allclose(got, gold_loglik["g_ll"], rtol=1e-12)

    def test_known_answers(self, gold_loglik):
        # test_model.py:131-154 and :36-41
        assert orc.loglik_rows(np.array([[1.0]]), np.array([1.0]), np.array([[0.4578]]))[0] == pytest.approx(
            float(gold_loglik["ka_scalar"]), abs=1e-15)
        assert orc.loglik_rows(np.array([[1.0], [-1.0]]), np.array([1.0, 0.0]), np.array([[800.0]]))[0] == \
            pytest.approx(0.0, abs=1e-12)
        assert orc.gt_log_density(0.0, 4.0, 0.1) == pytest.approx(np.log(5.0), abs=1e-12)
        assert orc.gt_log_density(1.0, 1.0, 1.0) == pytest.approx(-3 * np.log(2), abs=1e-12)


class TestReweightResample:
    def test_reweight(self, gold_reweight):
        for tag in ("a4", "a1", "a05"):
            a, c_prev, c_t = gold_reweight[f"{tag}_params"]
            B = gold_reweight[f"{tag}_B"]
            lw = orc.reweight_increments(B, a, c_t, c_prev)
            np.testing.assert_allclose(lw, gold_reweight[f"{tag}_lw"], rtol=1e-12, atol=1e-13)
            logw, inc = orc.normalise_log_weights(gold_reweight[f"{tag}_lw0"], lw)
            assert inc == pytest.approx(float(gold_reweight[f"{tag}_inc"]), abs=1e-12)
            w = orc.weights_from_log(logw)
            np.testing.assert_allclose(w, gold_reweight[f"{tag}_w"], rtol=1e-12)
            assert orc.ess(w) == pytest.approx(float(gold_reweight[f"{tag}_ess"]), rel=1e-12)

    def test_systematic_ancestors_bit_exact(self, gold_resample):
        cases = gold_resample["cases"]
        for k, (N, alpha) in enumerate(cases):
            N = int(N)
            if f"w_{k}" in gold_resample:
                w = gold_resample[f"w_{k}"]
            else:
                w = np.random.default_rng(1000 + k).dirichlet(np.full(N, alpha))
            assert sha(w) == str(gold_resample[f"wsha_{k}"])
            u = float(gold_resample[f"u_{k}"])
            assert np.array_equal(orc.systematic_ancestors(w, u), gold_resample[f"idx_{k}"])

    def test_edge_cases(self, gold_resample):
        for e in range(4):
            for j in range(3):
                w, u = gold_resample[f"ew_{e}_{j}"], float(gold_resample[f"eu_{e}_{j}"])
                assert np.array_equal(orc.systematic_ancestors(w, u), gold_resample[f"eidx_{e}_{j}"])

    def test_resample_uniform_matches_stream(self, gold_philox):
        # u = _stream(seed, 2, t).random() / N (smc.py:289, 421)
        keys = gold_philox["keys"]
        seed, tag, t, i = (int(v) for v in keys[2])
        assert tag == 2 and i == 0
        assert orc.resample_uniform(seed, t, 1) == float(gold_philox["uniform"][2][0])


class TestDataGenerator:
    @pytest.mark.parametrize("name", ["c1", "a_small", "a", "c2", "c3"])
    def test_generator_matches_reference(self, name):
        from paper_1106_0322_b200.data import named_spec, simulate_dataset

        hashes = golden("data_hashes.npz")
        d, _ = simulate_dataset(named_spec(name))
        assert sha(d.X) == str(hashes[f"{name}_X"])
        assert sha(d.y) == str(hashes[f"{name}_y"])


class TestSummaries:
    @pytest.mark.parametrize("name", ["normal", "ties", "ragged", "equal"])
    def test_marginal_summaries_match_reference(self, name):
        """summary.py:36-61 weighted mean / quantile / concentration."""
        g = golden("summaries.npz")
        B, w = g[f"{name}_B"], g[f"{name}_w"]
        q = B.shape[1]
        assert np.array_equal([orc.weighted_mean(B[:, j], w) for j in range(q)], g[f"{name}_mean"])
        assert np.array_equal([[orc.weighted_quantile(B[:, j], w, lv) for j in range(q)] for lv in g["levels"]],
                              g[f"{name}_quant"])
        assert np.array_equal([[orc.concentration(B[:, j], w, d) for j in range(q)] for d in g["deltas"]],
                              g[f"{name}_conc"])


class TestEmMap:
    @pytest.mark.parametrize("key", ["0_0", "0_1", "1_0", "1_1"])
    def test_em_map_matches_reference(self, key):
        """emmap.py:117-165 on C1 (C2 cases run in the GPU tests: slow in NumPy)."""
        from paper_1106_0322_b200.data import named_spec, simulate_dataset

        g = golden("emmap.npz")
        a, c, icpt = (float(v) for v in g[f"case_{key}"])
        d, _ = simulate_dataset(named_spec(str(g[f"name_{key}"])))
        X = np.column_stack([np.ones(d.X.shape[0]), d.X]) if icpt else d.X
        pen = np.ones(X.shape[1], bool)
        if icpt:
            pen[0] = False
        beta, lp, conv, inner, iters = orc.em_map(X, d.y, a, c, g[f"seed_{key}"], pen)
        np.testing.assert_allclose(beta, g[f"beta_{key}"], rtol=0, atol=1e-12)
        assert abs(lp - float(g[f"lp_{key}"])) < 1e-9
        assert [conv, inner] == list(g[f"conv_{key}"]) and iters == int(g[f"iters_{key}"])
