"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family of the library at C1-like shapes
-- K1 (tcgen05 ring + TMEM), pack / propose / accept, the Cholesky panel
graph, MwG chains and moves, the exact resampling scan (fast path and
fallback), gather / commit, the summary histograms, EM MAP.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1106_0322_b200 import SmcConfig, make_schedule, run_sampler, systematic_resample_indices  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

data, _ = simulate_dataset(named_spec("c1"))
for kernel in ("rw", "mwg"):
    cfg = SmcConfig(N=1024, cycles=1, moves=2, seed=3, init_burn=5, init_thin=1, move_kernel=kernel,
                    ess_threshold_frac=0.99, snapshot_thin=2, summary_levels=(0.05, 0.5, 0.95),
                    summary_deltas=(0.1,), summary_pooled=True)
    out = run_sampler(data, 1.0, make_schedule(2.0, 0.9, 4), cfg)
    print(kernel, [s.resampled for s in out.steps], flush=True)
rng = np.random.default_rng(0)
for w in (rng.dirichlet(np.ones(5000)), np.r_[1e-310, rng.random(3000)]):  # fast path, fallback
    systematic_resample_indices(w, 0.3 / w.size)
from paper_1106_0322_b200 import emmap  # noqa: E402
from paper_1106_0322_b200.model import GtPrior  # noqa: E402

emmap.em_map(data, GtPrior(1.0, 0.5), beta_init=np.zeros(data.p))
torch.cuda.synchronize()
print("sanitize run ok", flush=True)
