"""Upper bounds on what the side work costs the lambda step (C3, 40 steps):
full step; no covariance rebuild after the first step; normals drawn once
(reused); both.  Timing-only experiment: the skipped variants are not valid
samplers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

data, _ = simulate_dataset(named_spec("c3"))
sched = S.make_schedule(2.0, 0.98, 100)
orig_factor, orig_normals = S._rw_factor, S._rw_normals_async


def run(skip_factor, skip_normals):
    calls = {"f": 0, "n": 0}
    ev = {}

    def factor(*a, **k):
        calls["f"] += 1
        if skip_factor and calls["f"] > 1:
            if k.get("centred") is not None:
                k["centred"].record()
            return None
        return orig_factor(*a, **k)

    def normals(system, config, t):
        calls["n"] += 1
        if skip_normals and calls["n"] > 1:
            e = torch.cuda.Event()
            e.record()
            return e
        return orig_normals(system, config, t)

    S._rw_factor, S._rw_normals_async = factor, normals
    cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=1, init_burn=20, init_thin=1, init_chains=1024)
    s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
    recs = [S.smc_step(s, data, sched, t, cfg, _defer=True) for t in (2, 3, 4)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for t in range(5, 45):
        recs.append(S.smc_step(s, data, sched, t, cfg, _defer=True))
    e1.record()
    torch.cuda.synchronize()
    S._rw_factor, S._rw_normals_async = orig_factor, orig_normals
    return e0.elapsed_time(e1) / 40


for rep in range(2):
    for sf, sn in ((False, False), (True, False), (False, True), (True, True)):
        print(f"skip factor {sf!s:5} skip normals {sn!s:5}: {run(sf, sn):.3f} ms/step", flush=True)
