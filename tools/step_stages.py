"""Per-stage device times INSIDE one estimate (events between the kernels,
no graph replay), with the 256 MiB L2 flush before each step as bench.py
does, vs warm back-to-back.  Events between kernels break the PDL overlap,
so the sum exceeds the graph step; the per-stage cold/warm delta is the
point.  Exploration tool.   python tools/step_stages.py [cfg2]"""
import statistics
import sys

sys.path.insert(0, ".")
import torch

import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
c = P.baseline_config(name)
plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, 32, c.taper, c.batch, 0)
x = torch.from_numpy(P.baseline_series(c)).cuda()
out = plan.empty_out()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    plan.estimate(x, out)
plan.set_timing(True)
for mode in ("warm", "flushed"):
    acc = {}
    for i in range(40):
        if mode == "flushed":
            flush.fill_(i & 0xFF)
        plan.estimate(x, out)
        torch.cuda.synchronize()
        for k, v in plan.stage_ms().items():
            acc.setdefault(k, []).append(v * 1e3)
    med = {k: round(statistics.median(v), 2) for k, v in acc.items()}
    print(mode, med, "sum", round(sum(med.values()), 2))
plan.set_timing(False)
