"""GPU time of the resampling pieces (CUPTI kernel durations via
torch.profiler, so host launch overhead is excluded): the exact scan
kernels, the ancestor search, gather and commit, with the gate on and off,
at C3 (N=65536, q=500) and C4 (N=2^20), log-normal weights (a reweighted
SMC population)."""
import collections
import re
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1106_0322_b200 import _lib  # noqa: E402
from paper_1106_0322_b200.smc import _p, _stream  # noqa: E402


def kernel_us(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    if os.environ.get("SPA_NO_PROFILER"):  # under ncu: plain launches only
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        return {}
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    tot = collections.defaultdict(float)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            m = re.search(r"(\w+_kernel)", e.name)
            name = m.group(1) if m else e.name.strip()
            tot[name] += e.device_time / reps
    return dict(tot)


for N in (65536, 1 << 20):
    q, ldb = 500, 512
    rng = np.random.default_rng(1)
    w = np.exp(rng.normal(0, 1.0, N))
    w /= w.sum()
    wd = torch.from_numpy(w).cuda()
    nb = _lib.load().spa_resample_workspace_bytes(N)
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    cum = torch.empty(N, dtype=torch.float64, device="cuda")
    mode = torch.zeros(1, dtype=torch.int32, device="cuda")
    k = kernel_us(lambda: _lib.call("spa_exact_cumsum", _p(wd), N, _p(cum), _p(mode), _p(ws), nb, _stream()))
    assert np.array_equal(cum.cpu().numpy(), np.cumsum(w))
    print(f"N={N} exact cumsum (fast path: {int(mode.item()) == 0}):",
          {n: round(v, 1) for n, v in k.items()}, flush=True)
    beta = torch.randn((N, ldb), device="cuda")
    alt = torch.empty_like(beta)
    ll, lp, lla, lpa, logw = (torch.zeros(N, dtype=torch.float64, device="cuda") for _ in range(5))
    anc = torch.empty(N, dtype=torch.int64, device="cuda")
    for g in (1.0, 0.0):
        gate = torch.full((1,), g, dtype=torch.float64, device="cuda")
        k = kernel_us(lambda: _lib.call("spa_resample_gated", _p(gate), _p(wd), N, 0.3 / N, _p(beta), _p(alt), ldb, q,
                                        _p(ll), _p(lla), _p(lp), _p(lpa), _p(logw), _p(anc), _p(ws), nb, _stream()))
        print(f"  gated resampling, gate={g:g}: total {sum(k.values()):.1f} us",
              {n: round(v, 1) for n, v in k.items()}, flush=True)
