"""prior_reweight A/B at C3 (N=65536): median time with L2 flushed between
launches, and a hash of (lw, lp) for the bit-identity check across builds.
SPA_B200_LIB selects the library build."""
import ctypes, hashlib, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1106_0322_b200.smc as S
from paper_1106_0322_b200 import _lib
from paper_1106_0322_b200.data import named_spec, simulate_dataset
from paper_1106_0322_b200.smc import _p, _stream
data, _ = simulate_dataset(named_spec(os.environ.get("PR_CONFIG", "c3")))
cfg = S.SmcConfig(N=int(os.environ.get("PR_N", "65536")), move_kernel="rw", moves=5, seed=0, init_burn=20, init_thin=1, init_chains=1024)
s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
d = s.design
flush = torch.empty(256 * 2**20 // 4, device="cuda")
lw_t, lp_t = torch.empty_like(s.ll), torch.empty_like(s.ll)
for a, c, cp in ((1.0, 1.9, 1.95), (4.0, 0.3, 0.31)):
    ts = []
    for rep in range(30):
        flush.add_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("spa_prior_reweight", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, a, c, cp, _p(lw_t), _p(lp_t), _stream())
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    h = hashlib.sha1(lw_t.cpu().numpy().tobytes() + lp_t.cpu().numpy().tobytes()).hexdigest()[:12]
    print(os.path.basename(os.environ.get("SPA_B200_LIB", "default")), f"a={a} c={c}: prior_reweight median {ts[len(ts)//2]:.1f} us min {ts[0]:.1f}  lw/lp {h}")
