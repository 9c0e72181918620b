"""Float64 emulation of K1's operand splits on diffuse C3 particles (sigma =
0.3; CPU only): the relative log-likelihood error of the bf16 hi/lo split
(round 1) and of the fp16 hi/lo split (round 2), both with the centring
offset in three limbs, against the exact float64 log-likelihood.

    python tools/k1_precision.py      # bf16 ~6.7e-6, fp16 ~2.4e-7 (tolerance 1e-5)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import spa_oracle as orc  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.design import _code_column  # noqa: E402

d, _ = simulate_dataset(named_spec("c3"))
X, y = d.X, d.y
codes = [_code_column(X[:, j]) for j in range(X.shape[1])]
G = np.stack([c[0] for c in codes], 1).astype(np.float64)
alpha = np.array([c[1] for c in codes])
gamma = np.array([c[2] for c in codes])
B = (np.random.default_rng(0).standard_normal((40, X.shape[1])) * 0.3).astype(np.float32)
ref = orc.loglik_rows(X, y, B.astype(np.float64))
bs = (alpha.astype(np.float32)[None, :] * B).astype(np.float32)
off = B.astype(np.float64) @ gamma
ylin = B.astype(np.float64) @ (X.T @ y)


def rel_err(cast):
    hi = cast(bs)
    lo = cast(bs.astype(np.float64) - hi)
    o1 = cast(off)
    o2 = cast(off - o1)
    o3 = cast(off - o1 - o2)
    eta = G @ (hi + lo).T + (o1 + o2 + o3)[None, :]
    ll = ylin - np.logaddexp(0, eta).sum(0)
    return float(np.max(np.abs(ll - ref) / np.abs(ref)))


def bf16(x):
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def fp16(x):
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float64)


print(f"bf16 hi/lo: max relative log-lik error {rel_err(bf16):.2e}")
print(f"fp16 hi/lo: max relative log-lik error {rel_err(fp16):.2e}")


def fixed_point_rel_err(bits):
    """Per-row fixed point with `bits` significant bits relative to the row's
    max |alpha_j beta_j| (the int8 three-product scheme: bits = 20 for s8
    pieces hi*2^12 + mid*2^6 + lo), offset in float32, exact integer sums."""
    amax = np.abs(bs).max(axis=1, keepdims=True).astype(np.float64)
    scale = amax / (2.0 ** (bits - 1) - 1)
    Q = np.rint(bs.astype(np.float64) / scale)
    eta = G @ (Q * scale).T + off.astype(np.float32).astype(np.float64)[None, :]
    ll = ylin - np.logaddexp(0, eta).sum(0)
    return float(np.max(np.abs(ll - ref) / np.abs(ref)))


for b in (16, 20, 22):
    print(f"fixed point {b} bits (row max): max relative log-lik error {fixed_point_rel_err(b):.2e}")
