"""Time the GPU EM MAP: one problem at C2 / C3 and a batch of 100 at C3."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.emmap import em_map, em_map_batch  # noqa: E402
from paper_1106_0322_b200.model import GtPrior  # noqa: E402

for name in ("c2", "c3"):
    d, _ = simulate_dataset(named_spec(name))
    em_map(d, GtPrior(1.0, 0.5))  # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = em_map(d, GtPrior(1.0, 0.5))
    dt = time.perf_counter() - t
    print(f"{name}: one em_map {dt:.3f} s, EM iters {r.trace[-1].iter}, converged {r.converged}/{r.inner_converged}")
d, _ = simulate_dataset(named_spec("c3"))
rng = np.random.default_rng(0)
seeds = rng.normal(0, 0.05, size=(100, d.X.shape[1]))
c = 2.0 * 0.98 ** np.arange(100)
t = time.perf_counter()
r = em_map_batch(d, 1.0, c, seeds)
dt = time.perf_counter() - t
print(f"c3: batch of 100 em_map {dt:.3f} s, all converged {bool(r.converged.all() and r.inner_converged.all())}")
