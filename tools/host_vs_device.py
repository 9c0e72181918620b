"""Mean C3 lambda-step time: device-decided steps (_defer=True, the single-
process path) vs host-decided steps (the sharded path's structure), 40 steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

data, _ = simulate_dataset(named_spec("c3"))
sched = S.make_schedule(2.0, 0.98, 100)
for rep in range(2):
    for defer in (True, False):
        cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=1, init_burn=20, init_thin=1, init_chains=1024)
        s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
        recs = [S.smc_step(s, data, sched, t, cfg, _defer=defer) for t in (2, 3, 4)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for t in range(5, 45):
            recs.append(S.smc_step(s, data, sched, t, cfg, _defer=defer))
        e1.record()
        torch.cuda.synchronize()
        if defer:
            S.resolve_records(s, recs)
        print(f"{'device' if defer else 'host  '}-decided: {e0.elapsed_time(e1) / 40:.3f} ms/step "
              f"({sum(r.resampled for r in recs[3:])} resampling)", flush=True)
