"""Timeline of the streaming host path (HOS_STREAM=1): per-CTA K2 start,
first-data and end times (globaltimer) for a few traced calls.  Exploration
tool.   HOS_STREAM=1 python tools/stream_trace.py"""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

c = P.baseline_config("cfg2")
plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, 32, c.taper, 1, 0)
lib = _native.lib()
x = P.baseline_series(c)
xp = torch.from_numpy(x).pin_memory()
op = torch.empty(plan.npoints, dtype=torch.complex64).pin_memory()
for _ in range(5):
    plan.estimate_host(xp.numpy(), op.numpy())
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    plan.estimate_host(xp.numpy(), op.numpy())
    ts.append((time.perf_counter() - t0) * 1e6)
print("e2e us (graph):", np.round(sorted(ts)[:5], 1), "median", round(float(np.median(ts)), 1))
nw = 148 * 8
tr = torch.zeros(4 * nw + 1024, dtype=torch.int64, device="cuda")
lib.hos_plan_set_trace(plan.handle, ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    t0 = time.perf_counter()
    plan.estimate_host(xp.numpy(), op.numpy())
    print("traced call us:", round((time.perf_counter() - t0) * 1e6, 1))
torch.cuda.synchronize()
lib.hos_plan_set_trace(plan.handle, None)
t = tr.cpu().numpy()[:4 * nw].reshape(nw, 4).astype(np.float64)
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
start, first, end, sm = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 3]
print(f"K2 warps {used.sum()}: start {start.min():.1f}..{start.max():.1f} us; first data "
      f"{np.percentile(first, [0, 50, 100]).round(1)}; end {np.percentile(end, [0, 10, 50, 90, 100]).round(1)}")
print("distinct SMs used by K2:", len(set(sm.astype(int))))
