"""One C3 lambda step (RW-cov, 5 moves) inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off`.  Usage: python tools/profile_step.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
data, _ = simulate_dataset(named_spec("c3"))
cfg = S.SmcConfig(N=N, move_kernel="rw", moves=5, seed=0, init_burn=20, init_thin=1, init_chains=1024)
sched = S.make_schedule(2.0, 0.98, 100)
system, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
S.smc_step(system, data, sched, 2, cfg)
S.smc_step(system, data, sched, 3, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
S.smc_step(system, data, sched, 4, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled one step")
