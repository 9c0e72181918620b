"""run_sampler at C3 end to end (as bench.py's e2e: burn 2000, snapshots every
10th step), several runs: wall and the run's own phase timings, to find the
run-to-run spread.  E2E_RUNS (default 4), E2E_BURN (default 2000)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

data, _ = simulate_dataset(named_spec("c3"))
S.run_sampler(data, 1.0, S.make_schedule(2.0, 0.98, 3),
              S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=2, init_burn=1, init_thin=1, snapshot_thin=1))
torch.cuda.synchronize()
burn = int(os.environ.get("E2E_BURN", "2000"))
for r in range(int(os.environ.get("E2E_RUNS", "4"))):
    cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=1 + 2 * r, init_burn=burn, init_thin=5, snapshot_thin=10)
    t0 = time.perf_counter()
    out = S.run_sampler(data, 1.0, S.make_schedule(2.0, 0.98, 100), cfg)
    torch.cuda.synchronize()
    w = time.perf_counter() - t0
    tm = {k: round(v, 4) if isinstance(v, float) else v for k, v in out.timings.items()}
    print(f"run {r} wall {w:.4f}", tm, flush=True)
