"""Initialisation time (parallel MwG chains, init_burn 2000, init_thin 5) at C3
for the subject-per-thread layout given by SPA_MWG_S (8 / 16 / 32)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.design import DeviceDesign  # noqa: E402

data, _ = simulate_dataset(named_spec(sys.argv[1] if len(sys.argv) > 1 else "c3"))
d = DeviceDesign.build(data.X, data.y)
for burn in (200, 2000):
    cfg = S.SmcConfig(N=65536, move_kernel="rw", init_burn=burn, init_thin=5)
    S.init_particles(data, S.GtPrior(1.0, 2.0), cfg, design=d)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sysm, acc = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg, design=d)
    torch.cuda.synchronize()
    print(f"S={os.environ.get('SPA_MWG_S', 'auto')} chains={S.resident_chains(d)} burn={burn}: "
          f"{time.perf_counter() - t0:.3f} s  acc={acc:.4f}", flush=True)
