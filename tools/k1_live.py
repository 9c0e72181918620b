"""K1's live per-launch time inside the C3 lambda step (CUDA events around
each launch on the main stream, as bench.py measures it) with the covariance
factor rebuilt every step (lag 1 / 2) or never (upper bound on the side
stream's interference)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

data, _ = simulate_dataset(named_spec("c3"))
sched = S.make_schedule(2.0, 0.98, 100)
orig = S._rw_factor
orig_launch = S._launch_normals
for mode in ("lag1", "lag2", "nofactor", "nofactor_nonormals"):
    calls = {"n": 0}

    def factor(*a, **k):
        calls["n"] += 1
        if mode.startswith("nofactor") and calls["n"] > 1:
            if k.get("centred") is not None:
                k["centred"].record()
            return None
        return orig(*a, **k)

    S._rw_factor = factor
    drawn = set()

    def launch(system, config, t, mv):  # nonormals: every move reuses its first draw
        if mode == "nofactor_nonormals" and mv in drawn:
            e = torch.cuda.Event()
            e.record()
            return e
        drawn.add(mv)
        return orig_launch(system, config, t, mv)

    S._launch_normals = launch
    cfg = S.SmcConfig(N=65536, move_kernel="rw", moves=5, seed=1, init_burn=20, init_thin=1, init_chains=1024,
                      rw_factor_lag=2 if mode == "lag2" else 1)
    s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
    recs = [S.smc_step(s, data, sched, t, cfg, _defer=True) for t in (2, 3, 4)]
    timer = bench.EventTimer(torch)
    S.KERNEL_TIMER = timer
    timer.enabled = True
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for t in range(5, 25):
        recs.append(S.smc_step(s, data, sched, t, cfg, _defer=True))
    e1.record()
    torch.cuda.synchronize()
    S.KERNEL_TIMER = None
    k1, n = timer.mean_ms("loglik")
    print(f"{mode:9s}: step {e0.elapsed_time(e1) / 20:.3f} ms, K1 {k1 * 1e3:.1f} us/launch live ({n} launches), "
          f"frac {327.68e9 / (k1 * 1e-3) / 1385e12:.3f}", flush=True)
S._rw_factor = orig
S._launch_normals = orig_launch
