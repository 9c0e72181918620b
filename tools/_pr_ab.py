import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1106_0322_b200.smc as S
from paper_1106_0322_b200 import _lib
from paper_1106_0322_b200.data import named_spec, simulate_dataset
from paper_1106_0322_b200.smc import _p, _stream
data, _ = simulate_dataset(named_spec("c3"))
cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=0, init_burn=20, init_thin=1, init_chains=1024)
sched = S.make_schedule(2.0, 0.98, 100)
s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
d = s.design
flush = torch.empty(256 * 2**20 // 4, device="cuda")
lw_t, lp_t = torch.empty_like(s.ll), torch.empty_like(s.ll)
ts = []
for rep in range(30):
    flush.add_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("spa_prior_reweight", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, 1.0, 1.9, 1.95, _p(lw_t), _p(lp_t), _stream())
    e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print(os.environ.get("SPA_B200_LIB"), f"prior_reweight median {ts[len(ts)//2]:.1f} us min {ts[0]:.1f}")
