"""Does a concurrent host->device copy slow the estimate kernels?  Times
plan.estimate (device-resident, graph replay) alone and while a 64 MiB
pinned H2D copy runs on another stream.  Exploration tool."""
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
host = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
dev = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()
for _ in range(5):
    plan.estimate(x, out)
torch.cuda.synchronize()


def timed(n=20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        plan.estimate(x, out)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


print(f"alone: {timed():.1f} us/step")
with torch.cuda.stream(side):
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(side)
    dev.copy_(host, non_blocking=True)
    c1.record(side)
t = timed()
torch.cuda.synchronize()
print(f"with concurrent 64 MiB H2D: {t:.1f} us/step; copy took {c0.elapsed_time(c1) * 1e3:.0f} us "
      f"({64 * 1.048576 / (c0.elapsed_time(c1) * 1e-3) / 1e3:.1f} GB/s)")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
dev.copy_(host, non_blocking=True)
b.record()
torch.cuda.synchronize()
print(f"copy alone: {a.elapsed_time(b) * 1e3:.0f} us ({64 * 1.048576 / (a.elapsed_time(b) * 1e-3) / 1e3:.1f} GB/s)")
