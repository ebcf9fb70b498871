"""Per-warp K2 timeline on cfg2 (hos_plan_set_trace): launch ramp, first-data
latency, per-SM end spread.  Exploration tool."""
import ctypes
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import __graft_entry__

__graft_entry__.ensure_built()
import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

c = P.baseline_config("cfg2")
plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, 32, c.taper, 1, 0)
lib = _native.lib()
x = torch.from_numpy(P.baseline_series(c)).cuda()
out = plan.empty_out()
WPC = int(sys.argv[1]) if len(sys.argv) > 1 else 4  # warps per CTA of the build
nw = lib.hos_plan_nctas(plan.handle) * WPC
tr = torch.zeros(4 * nw, dtype=torch.int64, device="cuda")
for _ in range(3):
    plan.estimate(x, out)
lib.hos_plan_set_trace(plan.handle, ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    plan.estimate(x, out)
torch.cuda.synchronize()
lib.hos_plan_set_trace(plan.handle, None)
t = tr.cpu().numpy().reshape(nw, 4).astype(np.float64)
t0 = t[:, 0].min()
start, first, end, sm = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 3]
print(f"warps {nw}; start spread {start.min():.2f}..{start.max():.2f} us; first data {np.median(first - start):.2f} us "
      f"median after start; end {end.min():.2f}..{end.max():.2f} us (median {np.median(end):.2f})")
per_sm = {}
for s_, e_ in zip(sm, end):
    per_sm.setdefault(int(s_), []).append(e_)
ends = np.array([max(v) for v in per_sm.values()])
print(f"per-SM last end: min {ends.min():.2f} p10 {np.percentile(ends, 10):.2f} median {np.median(ends):.2f} "
      f"p90 {np.percentile(ends, 90):.2f} max {ends.max():.2f} us over {len(ends)} SMs")
dur = end - start
print(f"warp durations: min {dur.min():.2f} median {np.median(dur):.2f} max {dur.max():.2f} us")
# pattern of fast / slow warps inside an SM
wi = np.arange(nw) % WPC
cta = np.arange(nw) // WPC
for k in range(WPC):
    print(f"warp {k} of its CTA: median duration {np.median(dur[wi == k]):.2f} us")
rank_in_sm = np.zeros(nw, dtype=int)
for s_ in set(sm.astype(int)):
    idx = np.where(sm == s_)[0]
    ctas = sorted(set(cta[idx]))
    for i in idx:
        rank_in_sm[i] = ctas.index(cta[i])
for k in range(rank_in_sm.max() + 1):
    print(f"CTA #{k} on its SM (by index): median duration {np.median(dur[rank_in_sm == k]):.2f} us, "
          f"first data {np.median((first - start)[rank_in_sm == k]):.2f} us")
order = np.argsort(end)
print("5 earliest warps (gw, sm, warp, dur):", [(int(i), int(sm[i]), int(wi[i]), round(dur[i], 1)) for i in order[:5]])
pairs = {}
for s_ in set(sm.astype(int)):
    idx = np.where(sm == s_)[0]
    pairs[s_] = sorted(set(int(c_) for c_ in cta[idx]))
lo = [v[0] for v in pairs.values() if len(v) == 2]
hi = [v[1] for v in pairs.values() if len(v) == 2]
print(f"SMs with 2 CTAs: {len(lo)}; lower CTA index range {min(lo)}..{max(lo)}, upper {min(hi)}..{max(hi)}")
print("examples:", list(pairs.items())[:6])
