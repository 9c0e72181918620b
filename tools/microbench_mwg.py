"""MwG (reference kernel) throughput: likelihood terms/s of one smc_step.
    python tools/microbench_mwg.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

for name, N, a in (("c1", 1024, 1.0), ("c2", 8192, 4.0), ("c3", 8192, 1.0), ("c3", 65536, 1.0)):
    data, _ = simulate_dataset(named_spec(name))
    cfg = S.SmcConfig(N=N, cycles=5, seed=0, init_burn=20, init_thin=1, init_chains=1024)
    sched = S.make_schedule(2.0, 0.98, 100)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s, _ = S.init_particles(data, S.GtPrior(a, 2.0 / a), cfg)
    torch.cuda.synchronize()
    ti = time.perf_counter() - t0
    S.smc_step(s, data, sched, 2, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(3, 6):
        S.smc_step(s, data, sched, t, cfg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    terms = N * cfg.cycles * data.p * data.n
    print(f"{name} N={N:6d} n={data.n} p={data.p}: {ms:9.2f} ms/step  {terms / ms / 1e9:7.3f} Tterms/s"
          f"  ({N * cfg.cycles * data.p / ms / 1e6:8.2f} G coord-updates/s)  init(20 burn) {ti:.2f}s")
