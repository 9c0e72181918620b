"""Time spa_rw_factor alone on a random SPD matrix (q from argv)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
from paper_1106_0322_b200 import _lib  # noqa: E402
from paper_1106_0322_b200.smc import _p, _round_up, _stream  # noqa: E402
q = int(sys.argv[1]) if len(sys.argv) > 1 else 500
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rng = np.random.default_rng(0)
G = rng.normal(size=(q, q + 8)) / np.sqrt(q)
S = G @ G.T + 0.05 * np.eye(q)
acc = torch.zeros(q + q * q, dtype=torch.int64)
acc[q:] = torch.from_numpy(np.rint(np.tril(S) * 2.0**48).astype(np.int64).reshape(-1))
acc = acc.cuda()
kq = _round_up(q, 64)
L = torch.zeros((q, q), dtype=torch.float32, device="cuda")
fws = torch.zeros((_round_up(8 * q * q, 256) + _round_up(2 * q * kq, 256) + 8192) // 8 + 1, dtype=torch.float64,
                  device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
f = lambda: _lib.call("spa_rw_factor", _p(acc), q, 2.38, 1e-6, _p(L), _p(fws), _p(info), None, _stream())
f(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    f()
e1.record(); torch.cuda.synchronize()
print(f"q={q} spa_rw_factor {e0.elapsed_time(e1) / reps * 1e3:.1f} us")
