"""PCIe copy bandwidth (device events) and copy/compute overlap on this box."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

for mb in (0.5, 1, 4, 16, 64):
    n = int(mb * (1 << 20))
    hp = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts, td = [], []
    for i in range(12):
        e0.record(); d.copy_(hp, non_blocking=True); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        e0.record(); hp.copy_(d, non_blocking=True); e1.record(); e1.synchronize(); td.append(e0.elapsed_time(e1))
    h2d, d2h = statistics.median(ts[2:]), statistics.median(td[2:])
    print(f"{mb:5.1f} MiB  H2D {h2d * 1e3:7.1f} us ({n / h2d / 1e6:5.1f} GB/s)  D2H {d2h * 1e3:7.1f} us ({n / d2h / 1e6:5.1f} GB/s)")

c = P.baseline_config("cfg2")
x = P.baseline_series(c)
plan = _native.get_plan(3, c.m, c.k, c.m3, True, 32, "hann", 1, 0)
xd = torch.from_numpy(x).cuda()
for _ in range(5):
    plan.estimate(xd)
torch.cuda.synchronize()
s2 = torch.cuda.Stream()
hp = torch.empty(4 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ("compute", "copy", "both"):
    ts = []
    for _ in range(12):
        torch.cuda.synchronize()
        e0.record()
        if mode in ("copy", "both"):
            s2.wait_event(e0)
            with torch.cuda.stream(s2):
                d.copy_(hp, non_blocking=True)
        if mode in ("compute", "both"):
            plan.estimate(xd)
        e1.wait_stream(s2) if False else None
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{mode:8s} {statistics.median(ts[2:]) * 1e3:.1f} us")
