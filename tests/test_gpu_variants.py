"""GPU parity of the launch variants a plan only takes under an environment
switch (read at plan creation, so each runs in a child process): the
per-warp staged K2 (k_triple_w) for every config, 8 x 16 tiles, the
streaming host path (front end and K2 concurrent, HOS_STREAM=1), the quad-row
16-warp K2 (HOS_K2_QUAD=1), both K2 refill hand-offs, the line-scan +
prefix-difference smoother for line grids (HOS_K4_TILES=0), the prefix-sum per-series
smoother (HOS_K4_SEP=0), and the host entry point with copy-engine chunks
(HOS_CHUNKS=2 / 8; the default reads the series over PCIe in the front end)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import numpy as np, torch
import paper_1805_11775_b200 as P
from paper_1805_11775_b200._native import get_plan
from conftest import north_star, golden, TOL_FP32, TOL_FP64
from oracle import hos_oracle as O
TOL = {{32: TOL_FP32, 64: TOL_FP64}}
for prec in (32, 64):
    # small grids against the oracle port (orders 3 and 4)
    for order, m, k, w in ((3, 128, 16, 5), (3, 256, 24, 7), (4, 64, 12, 5)):
        x = np.random.default_rng(order * 1000 + m + k).standard_normal(m * k)
        cfg = P.EstimationConfig(order, P.SegmentConfig(m=m, k=k), w, precision="fp%d" % prec, taper="hann")
        g = P.estimate_spectrum(P.TimeSeries(x), cfg)
        dom, ref = O.estimate(x, order, m, k, w, True, "hann")
        assert np.array_equal(g.indices, dom)
        e = O.north_star_error(g.values, ref)
        assert e <= TOL[prec], (order, m, k, w, prec, e)
    # cfg2 through the host entry point (pinned: zero-copy / streaming) vs the reference rows
    c = P.baseline_config("cfg2")
    x = P.baseline_series(c)
    plan = get_plan(3, c.m, c.k, c.m3, True, prec, "hann", 1, 0)
    dev = plan.estimate(torch.from_numpy(x).cuda()).cpu().numpy()
    xp = torch.from_numpy(x).pin_memory()
    op = torch.empty(plan.npoints, dtype=torch.complex64 if prec == 32 else torch.complex128).pin_memory()
    for _ in range(3):
        got = plan.estimate_host(xp.numpy(), op.numpy()).copy()
        assert north_star(got, dev) <= (1e-6 if prec == 32 else 1e-13)
    gl = golden("cfg2_rows.npz")
    assert north_star(got.astype(np.complex128)[gl["pos"]], gl["val"]) <= TOL[prec]
print("VARIANT-OK")
"""


@pytest.mark.parametrize("env", ["HOS_K2=warp", "HOS_K2_TILE=2", "HOS_STREAM=1", "HOS_CTA_DEPTH=4", "HOS_K2_QUAD=1",
                                 "HOS_K2_REFILL=empty", "HOS_K2_REFILL=last", "HOS_K2_SKEW=0", "HOS_K4_TILES=0", "HOS_K4_SEP=0", "HOS_K4_PIPE=0", "HOS_FRONT_R16=0",
                                 "HOS_CHUNKS=2", "HOS_CHUNKS=8"])
def test_variant_parity(cuda, env):
    k, v = env.split("=")
    code = CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env={**os.environ, k: v}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "VARIANT-OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


NATIVE_CHILD = r"""
import os, sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import numpy as np, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_1805_11775_b200 as P
from paper_1805_11775_b200.parallel import native_distributed_plan
from conftest import north_star
c = P.baseline_config("cfg2")
x = torch.from_numpy(P.baseline_series(c)).cuda()
for prec in ("fp32", "fp64"):
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=c.m, k=c.k), c.m3, precision=prec, taper="hann")
    plan = native_distributed_plan(cfg)
    ref = P.estimate_spectrum(x, cfg).values
    for _ in range(3):  # capture, then replays
        got = plan.estimate_distributed(x).cpu().numpy()
        assert north_star(got, ref) <= (1e-6 if prec == "fp32" else 1e-13), prec
dist.destroy_process_group()
print("NATIVE-OK")
"""


def test_native_distributed_plan_one_rank(cuda):
    """parallel.native_distributed_plan (dedicated NCCL communicator, the
    library's in-C-ABI collectives, graph replay) on a one-rank process group
    agrees with the single-GPU estimate."""
    code = NATIVE_CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "NATIVE-OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
