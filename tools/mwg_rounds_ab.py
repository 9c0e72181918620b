"""A/B of blocked MwG rounds (spa_mwg_set_rounds): per-coordinate latency of
the initialisation chains (K chains x sweeps, chain layout) and the whole
C3 init_particles (2000 burn sweeps), for the rounds in ROUNDS (default 1,2,4).
    python tools/mwg_rounds_ab.py [name=c3]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200 import _lib  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.design import DeviceDesign  # noqa: E402
from paper_1106_0322_b200.smc import _p, _stream  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
R = [int(v) for v in os.environ.get("ROUNDS", "1,2,4").split(",")]  # rounds to compare
data, _ = simulate_dataset(named_spec(name))
d = DeviceDesign.build(data.X, data.y)


def chain_time(K, sweeps, rounds):
    _lib.call("spa_mwg_set_rounds", rounds, 1)
    s = S.ParticleSystem(d, K, 1.0)
    bb = torch.empty((K, s.ldb), dtype=torch.float32, device="cuda")
    bl = torch.empty(K, dtype=torch.float64, device="cuda")
    bp = torch.empty(K, dtype=torch.float64, device="cuda")
    cnt = torch.zeros(K, dtype=torch.int64, device="cuda")

    def run(n, sweep0):
        _lib.call("spa_mwg_chain_slots", ctypes.byref(d.struct), _p(s.beta), K, s.ldb, 1.0, 2.0, 0.5, n, 1, 7, 0, 0,
                  0, sweep0, _p(s.ll), _p(s.lp), _p(bb), _p(bl), _p(bp), _p(cnt), 1, 0, _stream())

    run(20, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(sweeps, 20)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    acc = cnt.sum().item() / (K * (sweeps + 20) * d.q)
    return ms, acc, s.beta.clone()


for K in (148, 296):
    ref = None
    for rounds in R:
        ms, acc, b = chain_time(K, 40, rounds)
        same = "" if ref is None else (" identical" if torch.equal(ref, b) else " DIFFERENT")
        ref = b if ref is None else ref
        print(f"K={K} rounds={rounds}: {ms / 40 * 1e3:.1f} us/sweep, {ms / 40 / d.q * 1e6:.0f} ns/coord, "
              f"acc {acc:.3f}{same}", flush=True)

cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=1, init_burn=2000, init_thin=5)
prior1 = S.GtPrior(1.0, 2.0)
for rounds in R + R[:1]:
    _lib.call("spa_mwg_set_rounds", rounds, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sysm, acc = S.init_particles(data, prior1, cfg, False, design=d)
    torch.cuda.synchronize()
    print(f"init C3 burn 2000 rounds={rounds}: {time.perf_counter() - t0:.3f} s, acceptance {acc:.3f}, "
          f"ll sum {sysm.ll.sum().item():.6f}", flush=True)
    del sysm
# the lambda-step move (throughput layout): one call of 5 sweeps over M particles
M = 16384
for mr in R + R:
    _lib.call("spa_mwg_set_rounds", 4, mr)
    s = S.ParticleSystem(d, M, 1.0)
    s.beta.normal_(0.0, 0.05)
    cnt = torch.zeros(M, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("spa_mwg_move", ctypes.byref(d.struct), _p(s.beta), M, s.ldb, 1.0, 0.5, 0.5, 5, 3, 1, 2, 0, 0,
              _p(s.ll), _p(s.lp), _p(cnt), 1, 0, _stream())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"move M={M} 5 sweeps rounds={mr}: {ms:.2f} ms, {M * 5 * d.q * d.n / ms / 1e9:.3f} e12 terms/s, "
          f"acc {cnt.sum().item() / (M * 5 * d.q):.3f}", flush=True)
_lib.call("spa_mwg_set_rounds", 4, 4)
