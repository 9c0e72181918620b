"""One MwG kernel call (C3 shapes, 1024 particles, 5 sweeps) inside cudaProfilerStart/Stop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.design import DeviceDesign  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
data, _ = simulate_dataset(named_spec(name))
d = DeviceDesign.build(data.X, data.y)
s = S.ParticleSystem(d, int(sys.argv[2]) if len(sys.argv) > 2 else S.resident_chains(d), 1.0)
S._mwg(s, S.GtPrior(1.0, 2.0), 0.5, 2, 0, 0, 0, 0)
torch.cuda.synchronize()
torch.cuda.profiler.start()
S._mwg(s, S.GtPrior(1.0, 2.0), 0.5, 5, 0, 0, 0, 2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
