"""GPU timeline of C3 lambda steps via torch.profiler (CUPTI kernel records):
per-kernel totals, GPU busy time and the idle gaps between kernels.
    python tools/timeline.py [steps]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1106_0322_b200.smc as S  # noqa: E402
from paper_1106_0322_b200.data import named_spec, simulate_dataset  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
torch.cuda.set_stream(S.sampler_stream())  # as run_sampler / bench.py
cfg_name = os.environ.get("TIMELINE_CONFIG", "c3")
Nn = int(os.environ.get("TIMELINE_N", "65536"))
data, _ = simulate_dataset(named_spec(cfg_name))
cfg = S.SmcConfig(N=Nn, move_kernel="rw", moves=5, seed=0, init_burn=20, init_thin=1, init_chains=min(1024, Nn))
sched = S.make_schedule(2.0, 0.98, 100)
s, _ = S.init_particles(data, S.GtPrior(1.0, 2.0), cfg)
for t in (2, 3, 4):
    S.smc_step(s, data, sched, t, cfg, _defer=True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for t in range(5, 5 + steps):
        S.smc_step(s, data, sched, t, cfg, _defer=True)
    torch.cuda.synchronize()

ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda x: x[0])
tot = defaultdict(float)
cnt = defaultdict(int)
for a, b, n in kern:
    tot[n[:70]] += b - a
    cnt[n[:70]] += 1
span = kern[-1][1] - kern[0][0]
# union of busy intervals (streams may overlap)
busy, cur_a, cur_b = 0.0, kern[0][0], kern[0][1]
gaps = []
for a, b, n in kern[1:]:
    if a > cur_b:
        busy += cur_b - cur_a
        gaps.append((a - cur_b, n[:50]))
        cur_a, cur_b = a, b
    else:
        cur_b = max(cur_b, b)
busy += cur_b - cur_a
print(f"steps={steps} span={span / steps:.1f} us/step busy={busy / steps:.1f} us/step "
      f"idle={(span - busy) / steps:.1f} us/step kernels={len(kern) / steps:.1f}/step")
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {v / steps:9.1f} us/step  x{cnt[n] / steps:5.1f}  {n}")
gaps.sort(reverse=True)
print("largest gaps (us, next kernel):")
for g, n in gaps[:15]:
    print(f"  {g:8.1f}  {n}")
if os.environ.get("TIMELINE_DUMP"):
    # the last step's kernels in start order (us from the step's first kernel)
    per = len(kern) // steps
    last = kern[-per:]
    t0 = last[0][0]
    print("last step, start/end us:")
    for a, b, n in last:
        print(f"  {a - t0:8.1f} {b - t0:8.1f} {b - a:7.1f}  {n[:70]}")
