"""Host-path (e2e) anatomy: wall time of hos_estimate_host (zero-copy graph)
for cfg2 and for a tiny plan (fixed host + launch overhead), and the
_stream() lookup.  Exploration tool."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import __graft_entry__

__graft_entry__.ensure_built()
import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native


def wall(f, n=50):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        ts.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(ts), min(ts)


for name in ("cfg2", "cfg1"):
    c = P.baseline_config(name)
    plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, 32, c.taper, 1, 0)
    x = torch.from_numpy(P.baseline_series(c).astype(np.float32)).pin_memory()
    out = torch.empty(plan.npoints, dtype=torch.complex64).pin_memory()
    xn, on = x.numpy(), out.numpy()
    for _ in range(5):
        plan.estimate_host(xn, on)
    print(name, "estimate_host median/min us: %.1f / %.1f" % wall(lambda: plan.estimate_host(xn, on)))
print("_stream() us: %.2f / %.2f" % wall(lambda: plan._stream(), 200))
