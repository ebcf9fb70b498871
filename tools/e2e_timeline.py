import os, sys, torch
sys.path.insert(0, ".")
import paper_1805_11775_b200 as P
from paper_1805_11775_b200 import _native
c = P.baseline_config("cfg2"); x = P.baseline_series(c); xp = torch.from_numpy(x).pin_memory()
for ch in sys.argv[1:]:
    os.environ["HOS_E2E_CHUNKS"] = ch; os.environ.pop("HOS_E2E_TRACE", None); _native._plans.clear()
    plan = _native.get_plan(3, c.m, c.k, c.m3, True, 32, "hann", 1, 0)
    op = torch.empty(plan.npoints, dtype=torch.complex64).pin_memory()
    for _ in range(3): plan.estimate_host(xp.numpy(), op.numpy())
    os.environ["HOS_E2E_TRACE"] = "1"
    print("chunks", ch, flush=True)
    for _ in range(3): plan.estimate_host(xp.numpy(), op.numpy())
