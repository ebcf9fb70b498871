"""Per-CTA timeline of the triple-product kernel on cfg2 (diagnostics)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

c = P.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, 32, c.taper, c.batch, 0)
x = torch.from_numpy(P.baseline_series(c)).cuda()
n = _native.lib().hos_plan_nctas(plan.handle)
tr = torch.zeros(8 * n * c.batch, dtype=torch.int64, device="cuda")
for _ in range(3):
    plan.estimate(x)
_native.lib().hos_plan_set_trace(plan.handle, ctypes.c_void_p(tr.data_ptr()))
plan.estimate(x)
torch.cuda.synchronize()
_native.lib().hos_plan_set_trace(plan.handle, None)
t = tr.cpu().numpy().reshape(-1, 8).astype(np.float64)
t0 = t[:, 0].min()
st, fd, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
print(f"CTAs {len(t)}  kernel span {en.max():.2f} us")
print(f"start   min/med/max {st.min():.2f} {np.median(st):.2f} {st.max():.2f}")
print(f"1st data-start med/max {np.median(fd - st):.2f} {np.max(fd - st):.2f}")
print(f"end     min/med/max {en.min():.2f} {np.median(en):.2f} {en.max():.2f}")
dur = en - st
print(f"dur     min/med/max {dur.min():.2f} {np.median(dur):.2f} {dur.max():.2f}")
order = np.argsort(-dur)[:8]
print("slowest CTAs (idx, dur, smid):", [(int(i), round(float(dur[i]), 2), int(t[i, 3])) for i in order])
sm = t[:, 3].astype(int)
per_sm = np.bincount(sm)
print("CTAs per SM histogram:", np.bincount(per_sm))
# structure of the spread
print("dur by CTA index (bins of 37):", [round(float(np.mean(dur[i:i + 37])), 1) for i in range(0, len(dur), 37)])
smd = np.zeros(per_sm.size)
for i in range(len(dur)):
    smd[sm[i]] = max(smd[sm[i]], en[i])
print("SM finish time min/med/max", smd.min().round(2), np.median(smd).round(2), smd.max().round(2))
print("SM finish by smid (bins of 16):", [round(float(np.mean(smd[i:i + 16])), 1) for i in range(0, len(smd), 16)])
# same SM: do its 3 CTAs have similar durations?
spread = [np.ptp(dur[sm == s]) for s in range(per_sm.size)]
print("within-SM duration spread med/max", np.median(spread).round(2), np.max(spread).round(2))
pl, dep, iss = (t[:, 7] - t0) / 1e3, (t[:, 6] - t0) / 1e3, (t[:, 4] - t0) / 1e3
print(f"piece list ready   med {np.median(pl - st):.2f} us after start")
print(f"dependency (K1) resolved med {np.median(dep):.2f} us (abs), max {dep.max():.2f}")
print(f"prologue issued    med {np.median(iss - dep):.2f} us after dependency")
print(f"first data         med {np.median(fd - iss):.2f} us after issue, max {np.max(fd - iss):.2f}")
print(f"warp0 total mbar wait med {np.median(t[:, 5]) / 1.965e3:.2f} us")
