"""Mean C3 lambda-step time when every step resamples (ESS threshold 1.0) vs
when none does (threshold tiny): the cost of a resampling step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

data, _ = simulate_dataset(named_spec("c3"))
sched = S.make_schedule(2.0, 0.98, 100)
for rep in range(2):
    for frac in (1e-9, 1.0):
        cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=1, init_burn=20, init_thin=1,
                          init_chains=1024, ess_threshold_frac=frac)
        s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
        recs = [S.smc_step(s, data, sched, t, cfg, _defer=True) for t in (2, 3, 4)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for t in range(5, 25):
            recs.append(S.smc_step(s, data, sched, t, cfg, _defer=True))
        e1.record()
        torch.cuda.synchronize()
        S.resolve_records(s, recs)
        print(f"ess threshold {frac:g}: {e0.elapsed_time(e1) / 20:.3f} ms/step "
              f"({sum(r.resampled for r in recs[3:])} of 20 resampled)", flush=True)
