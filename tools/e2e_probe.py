"""e2e diagnostics: pinned H2D/D2H bandwidth and hos_estimate_host latency per chunk count."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

c = P.baseline_config("cfg2")
x = P.baseline_series(c)
xp = torch.from_numpy(x).pin_memory()
xd = torch.empty_like(xp, device="cuda")
for _ in range(5):
    xd.copy_(xp, non_blocking=True)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    xd.copy_(xp, non_blocking=True)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"H2D 4 MiB pinned: {statistics.median(ts) * 1e6:.1f} us = {x.nbytes / statistics.median(ts) / 1e9:.1f} GB/s")
for chunks in (1, 2, 4, 8):
    os.environ["HOS_E2E_CHUNKS"] = str(chunks)
    _native._plans.clear()
    plan = _native.get_plan(3, c.m, c.k, c.m3, True, 32, "hann", 1, 0)
    op = torch.empty(plan.npoints, dtype=torch.complex64).pin_memory()
    for _ in range(5):
        plan.estimate_host(xp.numpy(), op.numpy())
    ws = []
    for _ in range(50):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan.estimate_host(xp.numpy(), op.numpy())
        ws.append(time.perf_counter() - t0)
    print(f"chunks={chunks}: e2e median {statistics.median(ws) * 1e6:.1f} us  min {min(ws) * 1e6:.1f} us")
# device-side duration of the host-path graph (events on the launch stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for chunks in (1, 2, 4, 8):
    os.environ["HOS_E2E_CHUNKS"] = str(chunks)
    _native._plans.clear()
    plan = _native.get_plan(3, c.m, c.k, c.m3, True, 32, "hann", 1, 0)
    op = torch.empty(plan.npoints, dtype=torch.complex64).pin_memory()
    for _ in range(5):
        plan.estimate_host(xp.numpy(), op.numpy())
    ds = []
    for _ in range(30):
        torch.cuda.synchronize()
        e0.record()
        plan.estimate_host(xp.numpy(), op.numpy())
        e1.record()
        e1.synchronize()
        ds.append(e0.elapsed_time(e1) * 1e3)
    print(f"chunks={chunks}: device span median {statistics.median(ds):.1f} us")
