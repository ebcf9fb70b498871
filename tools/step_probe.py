"""Where does the step time go?  Times estimate() graph replays (cfg2 fp32):
back to back (no flush), with the 256 MiB L2 flush between steps (as bench.py),
and with a tiny kernel between steps.  Exploration tool."""
import statistics
import sys

sys.path.insert(0, ".")
import torch

import __graft_entry__

__graft_entry__.ensure_built()
import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

c = P.baseline_config("cfg2")
plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, 32, c.taper, 1, 0)
x = torch.from_numpy(P.baseline_series(c)).cuda()
out = plan.empty_out()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tiny = torch.empty(1024, device="cuda")
for _ in range(5):
    plan.estimate(x, out)
torch.cuda.synchronize()
N = 200
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(N):
    plan.estimate(x, out)
b.record()
torch.cuda.synchronize()
print(f"back-to-back: {a.elapsed_time(b) / N * 1e3:.1f} us/step")
for name, between in (("flush", lambda i: flush.fill_(i & 0xFF)), ("tiny", lambda i: tiny.fill_(i))):
    ts = []
    for i in range(N):
        between(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.estimate(x, out)
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = [p.elapsed_time(q) * 1e3 for p, q in ts]
    print(f"{name} between steps: median {statistics.median(v):.1f} us, min {min(v):.1f}")
print(plan.time_stages(x, reps=50, out=out))
