"""CUDA-event time of one K1 launch (spa_loglik_softplus) at N=65536 on a named
workload (default c3), after 300 warm-up launches; an optional column count
truncates the design (stage-depth experiments):  python tools/k1_time.py [c3] [cols]"""
import ctypes
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200 import _lib  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.design import DeviceDesign  # noqa: E402
from paper_1106_0322_b200.smc import _p, _stream  # noqa: E402

data, _ = simulate_dataset(named_spec(sys.argv[1] if len(sys.argv) > 1 else "c3"))
X = data.X if len(sys.argv) < 3 else data.X[:, : int(sys.argv[2])]
d = DeviceDesign.build(X, data.y, False)
N = 65536
s = S.ParticleSystem(d, N, 1.0, False)
s.load_betas(np.random.default_rng(0).normal(0, 0.1, size=(N, d.q)))
ws = s.ll_workspace()
_lib.call("spa_pack_particles", ctypes.byref(d.struct), _p(s.beta), N, s.ldb, _p(ws["A"]), _p(ws["ylin"]), 1.0, 1.0,
          None, _stream())


def run():
    _lib.call("spa_loglik_softplus", ctypes.byref(d.struct), _p(ws["A"]), N, _p(ws["sp"]), _p(ws["ws"]),
              ws["ws"].numel(), _stream())


for _ in range(300):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"K1 n={d.n} q={d.q} kp={d.kp}: {us:.1f} us, {2.0 * d.n * d.q * N / us / 1e6:.0f} TFLOP/s algorithmic")
