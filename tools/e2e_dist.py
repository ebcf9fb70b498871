"""Distribution of per-call host-path latency (hos_estimate_host, pinned
buffers, cfg2) over many calls.  Exploration tool.
  [HOS_STREAM=1] python tools/e2e_dist.py"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

c = P.baseline_config("cfg2")
plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, 32, c.taper, 1, 0)
xp = torch.from_numpy(P.baseline_series(c)).pin_memory()
op = torch.empty(plan.npoints, dtype=torch.complex64).pin_memory()
xn, on = xp.numpy(), op.numpy()
for _ in range(10):
    plan.estimate_host(xn, on)
ts = []
for _ in range(300):
    t0 = time.perf_counter()
    plan.estimate_host(xn, on)
    ts.append((time.perf_counter() - t0) * 1e6)
ts = np.array(ts)
print("p5/p25/p50/p75/p95 us:", np.percentile(ts, [5, 25, 50, 75, 95]).round(1), "frac<160:", round(float((ts < 160).mean()), 2))
