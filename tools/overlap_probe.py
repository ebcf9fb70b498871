"""Does an async pinned H2D overlap with (a) a torch kernel, (b) our pipeline with/without graphs?"""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native

c = P.baseline_config("cfg2")
x = P.baseline_series(c)
xd = torch.from_numpy(x).cuda()
big = torch.randn(4096, 4096, device="cuda")
s2 = torch.cuda.Stream()
hp = torch.empty(4 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def measure(work, label):
    res = {}
    for mode in ("work", "copy", "both"):
        ts = []
        for _ in range(12):
            torch.cuda.synchronize()
            e0.record()
            if mode != "work":
                s2.wait_event(e0)
                with torch.cuda.stream(s2):
                    d.copy_(hp, non_blocking=True)
            if mode != "copy":
                work()
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[mode] = statistics.median(ts[2:])
    print(f"{label:28s} work {res['work']:7.1f}  copy {res['copy']:7.1f}  both {res['both']:7.1f} us")


measure(lambda: [big.mul_(1.0001) for _ in range(4)], "torch elementwise x4")
measure(lambda: big @ big, "torch matmul")
for ng in ("0", "1"):
    os.environ["HOS_NO_GRAPH"] = ng
    _native._plans.clear()
    plan = _native.get_plan(3, c.m, c.k, c.m3, True, 32, "hann", 1, 0)
    for _ in range(3):
        plan.estimate(xd)
    measure(lambda: plan.estimate(xd), f"hos estimate graph={ng == '0'}")
