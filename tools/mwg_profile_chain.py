"""One chain-slot launch (K chains x sweeps, the initialisation layout) for
ncu: python tools/mwg_profile_chain.py K sweeps rounds [name]"""
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

K, sweeps, rounds = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
data, _ = simulate_dataset(named_spec(sys.argv[4] if len(sys.argv) > 4 else "c3"))
d = DeviceDesign.build(data.X, data.y)
_lib.call("spa_mwg_set_rounds", rounds, 1)
s = S.ParticleSystem(d, K, 1.0)
bb = torch.empty((K, s.ldb), dtype=torch.float32, device="cuda")
bl = torch.empty(K, dtype=torch.float64, device="cuda")
bp = torch.empty(K, dtype=torch.float64, device="cuda")
cnt = torch.zeros(K, dtype=torch.int64, device="cuda")
for sw0 in (0, sweeps):
    _lib.call("spa_mwg_chain_slots", ctypes.byref(d.struct), _p(s.beta), K, s.ldb, 1.0, 2.0, 0.5, sweeps, 1, 7, 0, 0,
              0, sw0, _p(s.ll), _p(s.lp), _p(bb), _p(bl), _p(bp), _p(cnt), 1, 0, _stream())
torch.cuda.synchronize()
print("ok")
