"""CUDA-event timings of the lambda-step components at C3 (not under ncu).
    python tools/microbench.py [N]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200 import _lib  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.smc import _p, _stream  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
data, _ = simulate_dataset(named_spec("c3"))
cfg = S.SmcConfig(N=N, move_kernel="rw", moves=5, seed=0, init_burn=20, init_thin=1, init_chains=1024)
sched = S.make_schedule(2.0, 0.98, 100)
s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
for t in (2, 3):
    S.smc_step(s, data, sched, t, cfg)
torch.cuda.synchronize()
d = s.design
rw, ws = s.rw_workspace(), s.ll_workspace()
prior = S.GtPrior(1.0, sched.bs[3])


def timeit(name, fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1) / reps * 1e3:9.1f} us")


t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for t in range(4, 14):
    S.smc_step(s, data, sched, t, cfg)
t1.record()
torch.cuda.synchronize()
print(f"{'smc_step (mean of 10)':28s} {t0.elapsed_time(t1) / 10 * 1e3:9.1f} us")

timeit("reweight (prior mode 1+lse)", lambda: S._reweight_device(s, prior, S.GtPrior(1.0, sched.bs[2])), 5)
timeit("rw_factor (moments+chol)", lambda: S._rw_factor(s, 2.38))
timeit("chol only", lambda: _lib.call("spa_rw_factor", _p(rw["acc"]), s.q, 2.38, 1e-6, _p(rw["L"]), _p(rw["fws"]),
                                      _p(rw["info"]), None, _stream()))
timeit("prior mode 2", lambda: _lib.call("spa_prior_rows", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, 1.0,
                                         float(prior.c), float(prior.c), 2, _p(s.lp), _stream()))
zb = s.z_buffers(1)[0]
timeit("normals", lambda: _lib.call("spa_rw_normals", s.N, s.q, 1, 4, 0, 0, _p(zb), _stream()))
timeit("propose (gemm+pack)", lambda: _lib.call(
    "spa_rw_propose", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb, s.factor_operand(), 1, 4, 0, 0, _p(zb),
    _p(rw["prop"]), _p(ws["A"]), _p(ws["ylin"]), 1.0, float(prior.c), _p(rw["lp_p"]), _stream()))
lw_t, lp_t = torch.empty_like(s.ll), torch.empty_like(s.ll)
timeit("prior_reweight (fused)", lambda: _lib.call("spa_prior_reweight", ctypes.byref(d.struct), _p(s.beta), s.N, s.ldb,
                                                    1.0, float(prior.c), float(sched.bs[2]), _p(lw_t), _p(lp_t),
                                                    _stream()))
timeit("marginal summaries (3 q, 2 d)", lambda: S.marginal_summaries(s, (0.05, 0.5, 0.95), (0.05, 0.1)))
timeit("K1 loglik", lambda: _lib.call("spa_loglik_softplus", ctypes.byref(d.struct), _p(ws["A"]), s.N, _p(ws["sp"]),
                                      _p(ws["ws"]), ws["ws"].numel(), _stream()))
wts = s.device_weights()
timeit("centre pass (moments phase 2)", lambda: _lib.call(
    "spa_rw_moments", _p(s.beta), s.N, s.ldb, s.q, _p(wts), _p(rw["ctr"]), 2, _p(rw["acc"]), _p(rw["mws"]),
    rw["mws"].numel(), _stream()))
timeit("SYRK + reduce (phase 3)", lambda: _lib.call(
    "spa_rw_moments", _p(s.beta), s.N, s.ldb, s.q, _p(wts), None, 3, _p(rw["acc"]), _p(rw["mws"]),
    rw["mws"].numel(), _stream()))
# last: the accept writes the particle state
timeit("accept", lambda: _lib.call("spa_rw_accept", _p(s.beta), s.ldb, _p(rw["prop"]), s.q, s.N, _p(ws["ylin"]),
                                   _p(ws["sp"]), _p(rw["lp_p"]), _p(s.ll), _p(s.lp), 1, 4, 0, 0, _p(s.counter),
                                   _stream()))
