import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1106_0322_b200.smc as S
from paper_1106_0322_b200.data import named_spec, simulate_dataset
data, _ = simulate_dataset(named_spec("c3"))
for thin in (1000, 10, 1000, 10):
    cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=1, init_burn=200, init_thin=5, init_chains=int(os.environ.get("INIT_CHAINS", "0")), snapshot_thin=thin)
    t0 = time.perf_counter()
    out = S.run_sampler(data, 1.0, S.make_schedule(2.0, 0.98, 100), cfg)
    print(thin, "wall", time.perf_counter() - t0, out.timings)
