"""Per-call wall time of hos_estimate_host on cfg2 over many back-to-back
calls (does the call time change after N calls / T ms?).  Exploration tool."""
import os
import subprocess
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import __graft_entry__

__graft_entry__.ensure_built()
import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

n_calls = int(sys.argv[1]) if len(sys.argv) > 1 else 120
gap_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
c = P.baseline_config("cfg2")
plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, 32, c.taper, 1, 0)
x = torch.from_numpy(P.baseline_series(c).astype(np.float32)).pin_memory()
out = torch.empty(plan.npoints, dtype=torch.complex64).pin_memory()
xn, on = x.numpy(), out.numpy()


def clocks():
    r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,pstate,pcie.link.gen.current,pcie.link.width.current",
                        "--format=csv,noheader"], capture_output=True, text=True)
    return r.stdout.strip()


print("before:", clocks())
ts = []
t_start = time.perf_counter()
stamps = []
for i in range(n_calls):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.estimate_host(xn, on)
    t1 = time.perf_counter()
    ts.append((t1 - t0) * 1e6)
    stamps.append((t0 - t_start) * 1e3)
    if gap_ms:
        time.sleep(gap_ms * 1e-3)
print("after:", clocks())
print("env", {k: v for k, v in os.environ.items() if k.startswith("HOS_")}, "gap_ms", gap_ms)
print("us:", " ".join("%.0f" % t for t in ts))
slow = [i for i, t in enumerate(ts) if t > 1.5 * min(ts)]
print("first slow call:", slow[0] if slow else None, "at ms", stamps[slow[0]] if slow else None)
