"""Mean lambda-step GPU time at C3 for rw_factor_lag 0 / 1 / 2 (device-decided steps, 40 steps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

data, _ = simulate_dataset(named_spec("c3"))
sched = S.make_schedule(2.0, 0.98, 100)
for rep in range(2):
    for lag in (0, 1, 2):
        cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=1, init_burn=20, init_thin=1,
                          init_chains=1024, rw_factor_lag=lag)
        s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
        recs = [S.smc_step(s, data, sched, t, cfg, _defer=True) for t in (2, 3, 4)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for t in range(5, 45):
            recs.append(S.smc_step(s, data, sched, t, cfg, _defer=True))
        e1.record()
        torch.cuda.synchronize()
        S.resolve_records(s, recs)
        res = sum(r.resampled for r in recs[3:])
        print(f"lag {lag}: {e0.elapsed_time(e1) / 40:.3f} ms/step ({res} resampling steps), "
              f"final acc {recs[-1].acceptance:.3f}")
