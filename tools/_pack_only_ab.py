"""spa_rw_pack alone at C3 (N=65536): median time (L2 flushed) and a hash of
its outputs (A, ylin, lp) for the bit-identity check across builds.
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
S._rw_factor(s, 2.38)
rw, ws = s.rw_workspace(), s.ll_workspace()
zb = s.z_buffers(1)[0]
_lib.call("spa_rw_normals", s.N, s.q, 1, 4, 0, 0, _p(zb), _stream())
_lib.call("spa_rw_increments", s.N, s.q, s.ldb, s.factor_operand(), _p(zb), _p(rw["prop"]), _stream())
flush = torch.empty(256 * 2**20 // 4, device="cuda")
for a, c in ((1.0, 0.9), (float("inf"), 0.9)):
    ts = []
    for rep in range(40):
        flush.add_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("spa_rw_pack", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, _p(rw["prop"]), _p(ws["A"]),
                  _p(ws["ylin"]), a, c, _p(rw["lp_p"]), _stream())
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    h = hashlib.sha1(b"".join(t.contiguous().view(torch.uint8).cpu().numpy().tobytes() for t in (ws["A"], ws["ylin"], rw["lp_p"]))).hexdigest()[:12]
    print(os.path.basename(os.environ.get("SPA_B200_LIB", "default")), f"a={a}: pack median {ts[len(ts)//2]:.1f} us min {ts[0]:.1f}  out {h}", flush=True)
