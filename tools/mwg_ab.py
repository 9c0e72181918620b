"""Init (MwG chains) wall time at C3, N=65536, burn 200, thin 5: auto chains
and a fixed 444 chains.  SPA_B200_LIB selects the library build (A/B)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.design import DeviceDesign  # noqa: E402

data, _ = simulate_dataset(named_spec(os.environ.get("MWG_CONFIG", "c3")))
print(os.environ.get("SPA_B200_LIB", "default"), "resident chains", S.resident_chains(DeviceDesign.build(data.X, data.y)))
for K in (0, 444, 0, 444):
    cfg = S.SmcConfig(N=int(os.environ.get("MWG_N", "65536")), move_kernel="rw", moves=5, seed=1, init_burn=200, init_thin=5, init_chains=K)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s, acc = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
    torch.cuda.synchronize()
    import hashlib
    h = hashlib.sha1(s.beta.cpu().numpy().tobytes() + s.ll.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"  K={K or 'auto'}: init {time.perf_counter() - t0:.3f} s  acc {acc:.4f}  mean ll {s.ll.mean().item():.3f}"
          f"  state {h}")
