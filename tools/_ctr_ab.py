"""rw_center (moments phase 2) A/B at C3: median time (L2 flushed) and a hash
of its outputs (transposed operand Dt, fixed-point delta).  SPA_B200_LIB
selects the library build."""
import hashlib, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1106_0322_b200.smc as S
from paper_1106_0322_b200 import _lib
from paper_1106_0322_b200.data import named_spec, simulate_dataset
from paper_1106_0322_b200.smc import _p, _stream
data, _ = simulate_dataset(named_spec("c3"))
cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=0, init_burn=20, init_thin=1, init_chains=1024)
s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
S._rw_factor(s, 2.38)
rw = s.rw_workspace()
wts = s.device_weights()
flush = torch.empty(256 * 2**20 // 4, device="cuda")
call = lambda: _lib.call("spa_rw_moments", _p(s.beta), s.N, s.ldb, s.q, _p(wts), _p(rw["ctr"]), 2, _p(rw["acc"]),
                         _p(rw["mws"]), rw["mws"].numel(), _stream())
ts = []
for rep in range(30):
    flush.add_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); call(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
rw["acc"].zero_(); call(); torch.cuda.synchronize()
ldk = (s.N + 63) // 64 * 64
h = hashlib.sha1(rw["mws"].view(torch.uint8)[: 2 * s.q * ldk].cpu().numpy().tobytes() + rw["acc"][: s.q].cpu().numpy().tobytes()).hexdigest()[:12]
print(os.path.basename(os.environ.get("SPA_B200_LIB", "default")), f"centre median {ts[len(ts)//2]:.1f} us min {ts[0]:.1f}  out {h}")
