"""Per-warp timeline of k_triple_cta on a BASELINE config (hos_plan_set_trace):
per-CTA durations against their stage counts.  Exploration tool.
  python tools/k2cta_trace.py [cfg2]"""
import ctypes
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
c = P.baseline_config(name)
plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, 32, c.taper, c.batch, 0)
lib = _native.lib()
assert lib.hos_plan_k2_kind(plan.handle) == 1, "plan does not use k_triple_cta"
x = torch.from_numpy(P.baseline_series(c)).cuda()
out = plan.empty_out()
W = 16 if os.environ.get("HOS_K2_QUAD") == "1" else 8  # warps per k_triple_cta CTA
nctas = lib.hos_plan_nctas(plan.handle)
nw = 148 * W
tr = torch.zeros(4 * nw + 2 * 64 * W, dtype=torch.int64, device="cuda")
for _ in range(3):
    plan.estimate(x, out)
lib.hos_plan_set_trace(plan.handle, ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    plan.estimate(x, out)
torch.cuda.synchronize()
lib.hos_plan_set_trace(plan.handle, None)
tt = tr.cpu().numpy()
t = tt[:4 * nw].reshape(nw, 4).astype(np.float64)
st = tt[4 * nw:4 * nw + 64 * W].reshape(W, 64).astype(np.float64)
sd = tt[4 * nw + 64 * W:].reshape(W, 64).astype(np.float64)
t0 = t[:, 0].min()
start, first, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
cta = np.arange(nw) // W
print(f"start {start.min():.2f}..{start.max():.2f} us; first data {np.median(first - start):.2f} us after start "
      f"(max {np.max(first - start):.2f}); end {end.min():.2f}..{end.max():.2f} (median {np.median(end):.2f})")
ce = np.array([end[cta == i].max() for i in range(148)])
cs = np.array([start[cta == i].min() for i in range(148)])
order = np.argsort(-ce)
print("slowest CTAs (cta, start, end):", [(int(i), round(cs[i], 1), round(ce[i], 1)) for i in order[:8]])
print("fastest CTAs (cta, start, end):", [(int(i), round(cs[i], 1), round(ce[i], 1)) for i in order[-5:]])
print("CTA end percentiles 10/50/90:", np.percentile(ce, [10, 50, 90]).round(2))
w0 = st[0]
w0 = w0[w0 > 0]
print("traced CTA, warp 0: stage-ready gaps (us):", np.diff(w0 / 1e3).round(2).tolist())
base = st[st > 0].min()
for k in range(0, 24, 1):
    if not st[:, k].any():
        break
    print(f"stage {k:2d}: ready " + " ".join(f"{(st[w, k] - base) / 1e3:5.1f}" for w in range(W)) +
          " | done " + " ".join(f"{(sd[w, k] - base) / 1e3:5.1f}" for w in range(W)))
