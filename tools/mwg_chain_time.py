"""Per-sweep latency of the initialisation chains at C3: one chain-slot launch
of K chains x `sweeps` burn sweeps (the burn-in layout), CUDA events.
    python tools/mwg_chain_time.py [K=148] [sweeps=40] [name=c3]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200 import _lib  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402
from paper_1106_0322_b200.design import DeviceDesign  # noqa: E402
from paper_1106_0322_b200.smc import _p, _stream  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 148
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
data, _ = simulate_dataset(named_spec(sys.argv[3] if len(sys.argv) > 3 else "c3"))
d = DeviceDesign.build(data.X, data.y)
s = S.ParticleSystem(d, K, 1.0)
bb = torch.empty((K, s.ldb), dtype=torch.float32, device="cuda")
bl = torch.empty(K, dtype=torch.float64, device="cuda")
bp = torch.empty(K, dtype=torch.float64, device="cuda")
cnt = torch.zeros(K, dtype=torch.int64, device="cuda")


def run(n, sweep0):
    _lib.call("spa_mwg_chain_slots", ctypes.byref(d.struct), _p(s.beta), K, s.ldb, 1.0, 2.0, 0.5, n, 1, 7, 0, 0, 0,
              sweep0, _p(s.ll), _p(s.lp), _p(bb), _p(bl), _p(bp), _p(cnt), 1, 0, _stream())


run(20, 0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run(sweeps, 20)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"K={K} sweeps={sweeps} S={os.environ.get('SPA_MWG_S', 'auto')}: {ms:.2f} ms, {ms / sweeps * 1e3:.1f} us/sweep, "
      f"{ms / sweeps / d.q * 1e6:.0f} ns/coordinate, acceptance {cnt.sum().item() / (K * (sweeps + 20) * d.q):.3f}")
