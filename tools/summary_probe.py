"""Time / profile marginal_summaries on C3-sized particles (65536 x 500)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

data, _ = simulate_dataset(named_spec("c3"))
cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=0, init_burn=20, init_thin=1)
s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
S.marginal_summaries(s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if os.environ.get("PROFILE"):
    torch.cuda.profiler.start()
e0.record()
for _ in range(5):
    S.marginal_summaries(s)
e1.record()
torch.cuda.synchronize()
if os.environ.get("PROFILE"):
    torch.cuda.profiler.stop()
print(f"marginal_summaries {e0.elapsed_time(e1) / 5 * 1e3:.1f} us")
