"""What makes the step slower after the 256 MiB L2 flush?  Per-step device
time (events around one estimate) after: (a) a write flush (bench.py's),
(b) a read-only flush (L2 left clean), (c) a write flush then a read of x
(x back in L2), (d) a tiny kernel.  Exploration tool."""
import statistics
import sys

sys.path.insert(0, ".")
import torch

import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

c = P.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, 32, c.taper, c.batch, 0)
x = torch.from_numpy(P.baseline_series(c)).cuda()
out = plan.empty_out()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_r = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
tiny = torch.empty(1024, device="cuda")
sink = torch.empty(1, device="cuda")
for _ in range(5):
    plan.estimate(x, out)
modes = {
    "write flush": lambda i: flush.fill_(i & 0xFF),
    "read flush": lambda i: sink.copy_(flush_r.sum().view(1)),
    "write flush + read x": lambda i: (flush.fill_(i & 0xFF), sink.copy_(x.sum().view(1))),
    "write flush + read flush": lambda i: (flush.fill_(i & 0xFF), sink.copy_(flush_r.sum().view(1))),
    "tiny": lambda i: tiny.fill_(i),
}
for name, between in modes.items():
    ts = []
    for i in range(100):
        between(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.estimate(x, out)
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = [p.elapsed_time(q) * 1e3 for p, q in ts]
    print(f"{name:28s}: median {statistics.median(v):.1f} us, min {min(v):.1f}")
