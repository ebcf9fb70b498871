"""Warm-L2 per-stage breakdown of one estimate (cfg by argv[1]); diagnostics."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 32
c = P.baseline_config(name)
plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, prec, c.taper, c.batch, 0)
x = torch.from_numpy(P.baseline_series(c)).cuda()
for _ in range(5):
    plan.estimate(x)
plan.set_timing(True)
acc = {}
for _ in range(20):
    plan.estimate(x)
    for k, v in plan.stage_ms().items():
        acc.setdefault(k, []).append(v * 1e3)
plan.set_timing(False)
print(name, f"fp{prec}", " ".join(f"{k} {np.median(v):.1f}us" for k, v in acc.items()),
      f"total {sum(np.median(v) for v in acc.values()):.1f}us")
