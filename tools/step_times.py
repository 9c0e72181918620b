"""Per-step GPU time over a full C3 lambda path (device-decided steps), with
the resampling flag of each step.  python tools/step_times.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

data, _ = simulate_dataset(named_spec("c3"))
cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=1, init_burn=200, init_thin=5)
sched = S.make_schedule(2.0, 0.98, 100)
s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(sched.T + 1)]
recs = []
ev[1].record()
for t in range(2, sched.T + 1):
    recs.append(S.smc_step(s, data, sched, t, cfg, _defer=True))
    ev[t].record()
torch.cuda.synchronize()
S.resolve_records(s, recs)
ms = np.array([ev[t - 1].elapsed_time(ev[t]) for t in range(2, sched.T + 1)])
res = np.array([r.resampled for r in recs])
print(f"steps {len(ms)}: mean {ms.mean():.3f} ms, non-resampling {ms[~res].mean():.3f} ms "
      f"(median {np.median(ms[~res]):.3f}), resampling {ms[res].mean() if res.any() else float('nan'):.3f} ms "
      f"x{int(res.sum())}, first step {ms[0]:.3f} ms, total {ms.sum():.1f} ms")
