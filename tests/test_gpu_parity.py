"""GPU parity: libhos_b200 (through the drop-in API / C-ABI) vs the CPU
oracle and the reference's own golden outputs.

Bars (BASELINE.json north_star): max|dB|/max|B| <= 1e-5 in fp32 mode and
<= 1e-11 in fp64 mode, identical principal-domain indexing.
"""

import hashlib

import numpy as np
import pytest

from conftest import TOL_FP32, TOL_FP64, golden, max_rel_dev, north_star
from oracle import hos_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"fp32": TOL_FP32, "fp64": TOL_FP64}


def api():
    import paper_1805_11775_b200 as P

    return P


def small_cases():
    g = golden("small_cases.npz")
    for name in g["names"]:
        order, m, k, w, conj, seed, extra = (int(v) for v in g[f"{name}__meta"])
        yield str(name), order, m, k, w, bool(conj), g[f"{name}__x"], g[f"{name}__idx"], g[f"{name}__val"]


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("case", list(small_cases()), ids=lambda c: c[0])
def test_small_cases_vs_reference(cuda, case, prec):
    P = api()
    name, order, m, k, w, conj, x, idx, val = case
    cfg = P.EstimationConfig(order, P.SegmentConfig(m=m, k=k), w, conjugate_last=conj, precision=prec)
    g = P.estimate_spectrum(P.TimeSeries(x), cfg)
    assert np.array_equal(g.indices, idx)
    assert g.values.dtype == np.complex128
    err = north_star(g.values, val)
    assert err <= TOL[prec], f"{name} {prec}: {err:.3e}"
    if prec == "fp64":
        # the reference's own plan-equivalence bar, per point (tests/test_spectra.py:243-255)
        scale = max(float(np.abs(val).max()), 1e-300)
        assert np.all(np.abs(g.values - val) <= np.maximum(1e-9 * np.abs(val), 1e-12 * scale)), name


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_cfg1_full_tapered(cuda, prec):
    P = api()
    gl = golden("cfg1.npz")
    c = P.baseline_config("cfg1")
    x = P.baseline_series(c)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(gl["x_sha"])
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=c.m, k=c.k), c.m3, precision=prec, taper="hann")
    g = P.estimate_spectrum(P.TimeSeries(x), cfg)
    assert np.array_equal(g.indices, gl["idx"])
    assert north_star(g.values, gl["val_hann"]) <= TOL[prec]
    cfg0 = P.EstimationConfig(3, P.SegmentConfig(m=c.m, k=c.k), c.m3, precision=prec)
    g0 = P.estimate_spectrum(P.TimeSeries(x), cfg0)
    assert north_star(g0.values, gl["val_notaper"]) <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_cfg2_full_grid_vs_oracle(cuda, prec):
    """Headline config, whole grid: GPU (device-resident fp32 input) vs the
    oracle port (bit-exact with the reference, test_oracle.py) and the
    reference's golden rows."""
    import torch

    P = api()
    c = P.baseline_config("cfg2")
    x = P.baseline_series(c)
    gl = golden("cfg2_rows.npz")
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(gl["x_sha"])
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=c.m, k=c.k), c.m3, precision=prec, taper="hann")
    g = P.estimate_spectrum(torch.from_numpy(x).to(cuda), cfg)
    assert north_star(g.values[gl["pos"]], gl["val"]) <= TOL[prec]
    spec = O.segment_spectra(x, c.m, c.k, "hann")
    ref = O.parallel_efficient(spec, 3, c.m3, True, workers=8)
    err = north_star(g.values, ref)
    assert err <= TOL[prec], f"cfg2 {prec}: {err:.3e}"
    # ... and the reference's own whole grid (hospectra._compute_values on all 65,792 points)
    full = golden("cfg2_full.npz")
    assert len(g.values) == int(full["npoints"])
    err = north_star(g.values, full["val"])
    assert err <= TOL[prec], f"cfg2 {prec} vs reference full grid: {err:.3e}"
    if prec == "fp64":  # the reference's per-point bar (1e-9 relative, 1e-12 x max floor)
        d = np.abs(g.values - full["val"])
        assert np.all(d <= 1e-9 * np.abs(full["val"]) + 1e-12 * np.abs(full["val"]).max())


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_cfg4_full_grid_vs_reference(cuda, prec):
    """Trispectrum config, every point of the grid against the reference's own
    values (cfg4_full.npz from hospectra._compute_values)."""
    import torch

    P = api()
    c = P.baseline_config("cfg4")
    x = P.baseline_series(c)
    full = golden("cfg4_full.npz")
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(full["x_sha"])
    cfg = P.EstimationConfig(4, P.SegmentConfig(m=c.m, k=c.k), c.m3, precision=prec, taper="hann")
    g = P.estimate_spectrum(torch.from_numpy(x).to(cuda), cfg)
    assert len(g.values) == int(full["npoints"])
    err = north_star(g.values, full["val"])
    assert err <= TOL[prec], f"cfg4 {prec} vs reference full grid: {err:.3e}"
    if prec == "fp64":
        d = np.abs(g.values - full["val"])
        assert np.all(d <= 1e-9 * np.abs(full["val"]) + 1e-12 * np.abs(full["val"]).max())


@pytest.mark.parametrize("name,prec", [("cfg3", "fp32"), ("cfg3", "fp64"), ("cfg4", "fp32"), ("cfg4", "fp64")])
def test_baseline_rows_vs_reference(cuda, name, prec):
    import torch

    P = api()
    c = P.baseline_config(name)
    x = P.baseline_series(c)
    gl = golden(f"{name}_rows.npz")
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(gl["x_sha"])
    cfg = P.EstimationConfig(c.order, P.SegmentConfig(m=c.m, k=c.k), c.m3, precision=prec, taper="hann")
    g = P.estimate_spectrum(torch.from_numpy(x).to(cuda), cfg)
    assert np.array_equal(g.indices[gl["pos"]], gl["idx"])
    err = north_star(g.values[gl["pos"]], gl["val"])
    assert err <= TOL[prec], f"{name} {prec}: {err:.3e}"


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_cfg5_batch(cuda, prec):
    import torch

    P = api()
    c = P.baseline_config("cfg5")
    gl = golden("cfg5_series.npz")
    x = P.baseline_series(c)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(gl["x_sha"])
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=c.m, k=c.k), c.m3, precision=prec, taper="hann")
    vals = P.estimate_batch(torch.from_numpy(x).to(cuda), cfg)
    assert vals.shape == (c.batch, P.principal_domain(3, c.m).shape[0])
    for s in (0, 1, 4095):
        assert north_star(vals[s], gl[f"val_{s}"]) <= TOL[prec], s
    if prec == "fp64":
        return
    # batch rows == single-series estimates (the single-series plan splits the
    # segment sum into fp32 chunk partials, so they agree to fp32 rounding)
    for s in (7, 2048):
        one = P.estimate_spectrum(torch.from_numpy(x[s]).to(cuda), cfg)
        assert north_star(vals[s], one.values) <= 1e-6


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("order,m,k,w,conj", [(3, 64, 3, 5, True), (3, 50, 2, 4, False), (4, 32, 2, 3, True),
                                              (4, 30, 3, 4, False)])
def test_from_spectra_arbitrary_complex(cuda, order, m, k, w, conj, prec):
    """estimate_from_spectra accepts any complex spectra (no conjugate
    symmetry assumed), like the reference."""
    P = api()
    rng = np.random.default_rng(order * 100 + m)
    spec = rng.standard_normal((k, m)) + 1j * rng.standard_normal((k, m))
    cfg = P.EstimationConfig(order, P.SegmentConfig(m=m, k=k), w, conjugate_last=conj, precision=prec)
    g = P.estimate_from_spectra(P.SegmentSpectrumSet(spectra=spec), cfg)
    ref = O.efficient_values(spec, order, w, conj)
    assert north_star(g.values, ref) <= TOL[prec]


def test_dft_segments_matches_numpy(cuda):
    P = api()
    rng = np.random.default_rng(64)
    for m in (1, 2, 3, 7, 16, 33, 64, 1000):
        x = rng.standard_normal(3 * m)
        segs = P.segment_and_demean(P.TimeSeries(x), P.SegmentConfig(m=m, k=3))
        got = P.dft_segments(segs).spectra
        ref = np.fft.fft(segs.segments, axis=1)
        scale = max(float(np.abs(ref).max()), 1.0)
        assert np.max(np.abs(got - ref)) <= 1e-12 * scale, m


def test_reference_semantics(cuda):
    """Ports of hospectra tests/test_spectra.py:158-255 on the GPU path."""
    P = api()
    # constant series -> exactly zero grid
    for order in (3, 4):
        for prec in ("fp64", "fp32"):
            g = P.estimate_spectrum(P.TimeSeries(np.full(64, 2.5)),
                                    P.EstimationConfig(order, P.SegmentConfig(m=64), 5, precision=prec))
            assert np.all(g.values == 0)
    # window too large
    with pytest.raises(P.ParameterError, match="m3 < m/2"):
        P.EstimationConfig(3, P.SegmentConfig(m=64), 32)
    with pytest.raises(P.ParameterError, match="exceeds series length"):
        P.estimate_spectrum(P.TimeSeries(np.ones(100)), P.EstimationConfig(3, P.SegmentConfig(m=64, k=2), 5))
    # homogeneity alpha^3 / alpha^4
    rng = np.random.default_rng(6)
    x = rng.standard_normal(128)
    a = 1.7
    g1 = P.estimate_spectrum(P.TimeSeries(x), P.EstimationConfig(3, P.SegmentConfig(m=128), 5))
    g2 = P.estimate_spectrum(P.TimeSeries(a * x), P.EstimationConfig(3, P.SegmentConfig(m=128), 5))
    assert max_rel_dev(g2.values, a ** 3 * g1.values) < 1e-9
    h1 = P.estimate_spectrum(P.TimeSeries(x[:64]), P.EstimationConfig(4, P.SegmentConfig(m=64), 5))
    h2 = P.estimate_spectrum(P.TimeSeries(a * x[:64]), P.EstimationConfig(4, P.SegmentConfig(m=64), 5))
    assert max_rel_dev(h2.values, a ** 4 * h1.values) < 1e-9
    # conjugate variant differs, and every plan name gives identical values
    s = P.generate_qpc(0.1, 0.15, 64, 0.4, seed=10)
    wc = P.estimate_spectrum(s, P.EstimationConfig(3, P.SegmentConfig(m=64), 3, conjugate_last=True))
    nc = P.estimate_spectrum(s, P.EstimationConfig(3, P.SegmentConfig(m=64), 3, conjugate_last=False))
    assert not np.allclose(wc.values, nc.values)
    for plan in P.SmoothingPlan:
        got = P.estimate_spectrum(s, P.EstimationConfig(3, P.SegmentConfig(m=64), 3, plan, conjugate_last=False))
        assert np.array_equal(got.values, nc.values) and got.plan is plan
    # QPC peak at the coupled pair (tests/test_acceptance.py:239-249)
    q = P.generate_qpc(0.1, 0.15, 1024, 0.0, seed=7)
    for prec in ("fp64", "fp32"):
        g = P.estimate_spectrum(q, P.EstimationConfig(3, P.SegmentConfig(m=1024), 5, precision=prec))
        assert g.peak_point().k == (154, 102)
    gl = golden("qpc1024.npz")
    g = P.estimate_spectrum(q, P.EstimationConfig(3, P.SegmentConfig(m=1024), 5))
    assert north_star(g.values[gl["pos"]], gl["val"]) <= TOL_FP64 * 10


def test_parallel_estimate_invariant(cuda):
    P = api()
    s = P.generate_qpc(0.1, 0.15, 256, 0.4, seed=4)
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=256), 9)
    ref = P.estimate_spectrum(s, cfg)
    for p in (1, 2, 4, 8):
        for part in ("row_blocks", "point_blocks"):
            got = P.parallel_estimate(s, cfg, P.WorkerConfig(p=p, partition=part))
            assert np.array_equal(got.values, ref.values)
            assert np.array_equal(got.indices, ref.indices)


def test_deterministic_repeat(cuda):
    import torch

    P = api()
    c = P.baseline_config("cfg2")
    x = torch.from_numpy(P.baseline_series(c)).to(cuda)
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=c.m, k=c.k), c.m3, precision="fp32", taper="hann")
    a = P.estimate_spectrum(x, cfg).values
    b = P.estimate_spectrum(x, cfg).values
    assert np.array_equal(a, b)


@pytest.mark.parametrize("prec", [32, 64])
def test_host_entry_point_matches_device(cuda, prec):
    """hos_estimate_host: pageable buffers (copies) are bit-identical to the
    device path; page-locked ones (zero-copy graph) match it."""
    import torch

    from paper_1805_11775_b200._native import get_plan

    P = api()
    c = P.baseline_config("cfg2")
    x = P.baseline_series(c)
    plan = get_plan(3, c.m, c.k, c.m3, True, prec, "hann", 1, 0)
    dev = plan.estimate(torch.from_numpy(x).to(cuda)).cpu().numpy()
    host = plan.estimate_host(x)  # pageable: same launch sequence as the device path
    assert np.array_equal(dev, host)
    # pinned buffers: zero-copy graph (compare with a tolerance: the host path
    # may take a different launch configuration)
    xp = torch.from_numpy(x).pin_memory()
    op = torch.empty(plan.npoints, dtype=torch.complex64 if prec == 32 else torch.complex128).pin_memory()
    for _ in range(2):  # capture + replay
        pinned = plan.estimate_host(xp.numpy(), op.numpy()).copy()
        assert north_star(pinned, dev) <= (1e-6 if prec == 32 else 1e-13)
    gl = golden("cfg2_rows.npz")
    assert north_star(pinned.astype(np.complex128)[gl["pos"]], gl["val"]) <= TOL[f"fp{prec}"]


@pytest.mark.parametrize("order,m,k,w", [(3, 256, 12, 9), (4, 64, 6, 5)])
def test_shard_pipeline_single_gpu(cuda, order, m, k, w):
    """The multi-GPU building blocks on one GPU: partial raw sums of segment
    shards (hos_partial_raw), summed, then smoothing by output-row blocks
    (hos_smooth_raw) reproduces hos_estimate."""
    import torch

    from paper_1805_11775_b200._native import get_plan
    from paper_1805_11775_b200.parallel import shard_layout

    P = api()
    x = torch.from_numpy(np.random.default_rng(5).standard_normal(m * k)).to(cuda)
    plan = get_plan(order, m, k, w, True, 64, None, 1, 0)
    ref = plan.estimate(x).cpu().numpy()
    rows = (m - 1) // 2 + 1
    row_off = np.array([plan.row_point_offset(r) for r in range(rows + 1)])
    lay = shard_layout(k, row_off, plan.line_starts(), plan.rows_line_range, 3)
    raw = torch.zeros(plan.cells, dtype=torch.complex128, device=cuda)
    for r in range(3):
        part = torch.empty_like(raw)
        plan.partial_raw(x, lay.seg_bounds[r], lay.seg_bounds[r + 1], part)
        raw += part
    out = np.empty(plan.npoints, np.complex128)
    for r in range(3):
        r0, r1 = lay.row_bounds[r], lay.row_bounds[r + 1]
        l0 = lay.own_lines[r][0]
        c0 = int(plan.line_starts()[l0])
        n = plan.row_point_offset(r1) - plan.row_point_offset(r0)
        if n == 0:
            continue
        o = torch.empty(n, dtype=torch.complex128, device=cuda)
        plan.smooth_raw(raw[c0:], l0, r0, r1, o)
        out[lay.point_bounds[r]: lay.point_bounds[r + 1]] = o.cpu().numpy()
    assert north_star(out, ref) <= 1e-13


def _gloo_gpu_worker(rank, world, port, cfgs, q):
    """One rank of distributed_estimate with the real GPU engine (cuda:0 for
    every rank; gloo moves the collectives through the host, so the ranks'
    kernels never wait on each other)."""
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import __graft_entry__

        __graft_entry__.ensure_built()
        from paper_1805_11775_b200 import EstimationConfig, SegmentConfig, distributed_estimate

        res = []
        for order, m, k, w, prec, seed in cfgs:
            x = np.random.default_rng(seed).standard_normal(m * k)
            cfg = EstimationConfig(order, SegmentConfig(m=m, k=k), w, precision=prec, taper="hann")
            xd = torch.from_numpy(x).cuda()
            vals = distributed_estimate(xd, cfg).cpu().numpy()
            res.append(vals)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_gpu_engine_gloo(cuda, world):
    """Segment-sharded estimate through the GPU engine across `world` ranks
    (partial raw sums per shard, reduce-scatter / halo exchange, per-rank
    smoothing, all-gather) matches the oracle."""
    import socket

    import torch.multiprocessing as mp

    cfgs = [(3, 256, 13, 9, "fp64", 11), (3, 128, 9, 5, "fp32", 12), (4, 64, 7, 5, "fp64", 13)]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_gpu_worker, args=(r, world, port, cfgs, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for i, (order, m, k, w, prec, seed) in enumerate(cfgs):
        x = np.random.default_rng(seed).standard_normal(m * k)
        _, ref = O.estimate(x, order, m, k, w, True, "hann")
        tol = TOL_FP64 if prec == "fp64" else TOL_FP32
        for r in range(world):
            assert max_rel_dev(out[r][i], ref) <= tol, (world, r, i)


def _nccl_single_rank_comm():
    """A 1-rank NCCL communicator on the current device (ctypes on the
    libnccl.so.2 the process uses)."""
    import ctypes

    nccl = ctypes.CDLL("libnccl.so.2")

    class UniqueId(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_byte * 128)]

    uid = UniqueId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    assert nccl.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    return nccl, comm


@pytest.mark.parametrize("order,m,k,w,prec", [(3, 256, 13, 9, "fp64"), (4, 64, 7, 5, "fp64"), (3, 1024, 64, 9, "fp32")])
@pytest.mark.parametrize("p2p", ["1", "0"])
def test_capi_distributed_nccl_single_rank(cuda, monkeypatch, order, m, k, w, prec, p2p):
    """hos_comm_attach + hos_estimate_distributed on a 1-rank communicator
    match the oracle and the single-GPU path, with the reduce-scatter fused
    into the slot reduction as landing-slot stores (p2p=1: the rank's own
    landing buffer stands in for the owner's) and with NCCL's reduce-scatter
    (p2p=0); the multi-rank layout is the one pinned against
    parallel.shard_layout in test_api.py."""
    import torch

    from paper_1805_11775_b200 import _native

    monkeypatch.setenv("HOS_DIST_P2P", p2p)
    nccl, comm = _nccl_single_rank_comm()
    try:
        x = np.random.default_rng(order * 1000 + m).standard_normal(m * k)
        plan = _native.Plan(order, m, k, w, True, 64 if prec == "fp64" else 32, "hann", 1, 0)
        plan.comm_attach(comm.value, 0, 1)
        xd = torch.from_numpy(x).cuda()
        got = plan.estimate_distributed(xd).cpu().numpy()
        direct = plan.estimate(xd).cpu().numpy()
        _, ref = O.estimate(x, order, m, k, w, True, "hann")
        tol = TOL_FP64 if prec == "fp64" else TOL_FP32
        assert north_star(got, ref) <= tol
        assert north_star(got, direct) <= tol
    finally:
        nccl.ncclCommDestroy(comm)


def _sweep_cases():
    rng = np.random.default_rng(20260601)
    cases = []
    for order, ms in ((3, (4, 8, 12, 16, 31, 32, 64, 96, 128, 200, 256, 512)), (4, (8, 16, 24, 32, 50, 64, 128))):
        for m in ms:
            wmax = max(1, (m - 1) // 2 - 0)  # 2 m3 < m
            for _ in range(2):
                w = int(rng.integers(1, max(2, min(wmax, 12) + 1)))
                if 2 * w >= m:
                    w = max(1, (m - 1) // 2)
                k = int(rng.integers(1, 9))
                cases.append((order, m, k, w, bool(rng.integers(0, 2)), ["fp64", "fp32"][int(rng.integers(0, 2))],
                              [None, "hann"][int(rng.integers(0, 2))], int(rng.integers(0, 1 << 30))))
    return cases


@pytest.mark.parametrize("case", _sweep_cases(), ids=lambda c: "o%d_m%d_k%d_w%d_%s_%s_%s" % (
    c[0], c[1], c[2], c[3], "conj" if c[4] else "noconj", c[5], c[6] or "flat"))
def test_sweep_small_shapes(cuda, case):
    """Seeded sweep over small shapes (power-of-two and general M, odd tile
    counts, k not a multiple of the warp split, w = 1, both orders and
    precisions, taper on/off) against the oracle."""
    order, m, k, w, conj, prec, taper, seed = case
    P = api()
    x = np.random.default_rng(seed).standard_normal(m * k + 3)
    cfg = P.EstimationConfig(order, P.SegmentConfig(m=m, k=k), w, conjugate_last=conj, precision=prec, taper=taper)
    g = P.estimate_spectrum(P.TimeSeries(x), cfg)
    dom, ref = O.estimate(x, order, m, k, w, conj, taper)
    assert np.array_equal(g.indices, dom)
    if np.abs(ref).max() < 1e-12:
        # identically-zero estimate (e.g. m = 4: every point involves the demeaned
        # DC bin): the reference's values are rounding noise and max|B| is no
        # scale -- bound the absolute error by the compute precision instead
        assert np.abs(g.values).max() <= (1e-12 if prec == "fp64" else 1e-6)
    else:
        assert north_star(g.values, ref) <= (TOL_FP64 if prec == "fp64" else TOL_FP32)


@pytest.mark.parametrize("order,m,k,w,conj,prec", [(3, 64, 5, 5, True, 64), (3, 256, 9, 9, False, 32),
                                                   (4, 32, 4, 3, True, 32), (4, 64, 3, 5, False, 64)])
def test_k2_tile_step2(cuda, monkeypatch, order, m, k, w, conj, prec):
    """The 8 x 16 K2 tile shape (lane step 2, HOS_K2_TILE=2; auto-selected only
    for very short lines) matches the oracle and issues fewer cells."""
    import torch

    from paper_1805_11775_b200 import _native

    x = np.random.default_rng(m + k).standard_normal(m * k)
    _, ref = O.estimate(x, order, m, k, w, conj, "hann")
    issued = {}
    for step in ("2", "4"):
        monkeypatch.setenv("HOS_K2_TILE", step)
        plan = _native.Plan(order, m, k, w, conj, prec, "hann")
        out = plan.estimate(torch.from_numpy(x).cuda())
        issued[step] = plan.issued
        assert north_star(out.cpu().numpy(), ref) <= (TOL_FP64 if prec == 64 else TOL_FP32), step
    assert issued["2"] <= issued["4"]


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("m,k,w", [(384, 10, 3), (384, 9, 11), (256, 12, 5)])
def test_shifted_band_tilings_vs_oracle(cuda, prec, m, k, w):
    """Shapes whose best tiling starts with a short band (fewer regions than
    full 16-line bands): the shifted band lattice against the oracle port."""
    P = api()
    x = np.random.default_rng(m * 31 + k * 7 + w).standard_normal(m * k)
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=m, k=k), w, precision=prec, taper="hann")
    g = P.estimate_spectrum(P.TimeSeries(x), cfg)
    dom, ref = O.estimate(x, 3, m, k, w, True, "hann")
    assert np.array_equal(g.indices, dom)
    assert O.north_star_error(g.values, ref) <= TOL[prec]


def test_gpu_report_checksum_vs_oracle(cuda):
    """gpu_report: one timed GPU estimate as a BenchReport record whose
    checksum (sum |B|) equals the oracle grid's."""
    P = api()
    for n, w in ((128, 21), (256, 33)):
        x = P.generate_qpc(0.1, 0.15, n, 0.5, 1234)
        cfg = P.EstimationConfig(3, P.SegmentConfig(m=n, k=1), w)
        grid, r = P.gpu_report(x, cfg)
        dom, ref = O.estimate(x.samples, 3, n, 1, w, True, None)
        assert r.status == "ok" and r.n == n and r.M3 == w and r.P == 1
        assert abs(r.checksum - float(np.abs(ref).sum())) <= 1e-9 * float(np.abs(ref).sum())
        assert r.wall_seconds > 0 and r.peak_extra_bytes > 0
        assert P.reports_from_json(P.reports_to_json([r])) == [r]


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("batch,m,k,w", [(3, 128, 20, 5), (37, 256, 9, 7), (160, 128, 6, 3)])
def test_small_batches_vs_oracle(cuda, prec, batch, m, k, w):
    """Batches that do not fill the GPU with whole series: the K2 schedule
    cuts CTA ranges across series, so partial-slot counts differ per series."""
    import torch

    P = api()
    rng = np.random.default_rng(batch * 1000 + m + k)
    x = rng.standard_normal((batch, m * k))
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=m, k=k), w, precision=prec, taper="hann")
    vals = P.estimate_batch(torch.from_numpy(x).to(cuda), cfg)
    rows = range(batch) if batch <= 37 else (0, 1, batch // 2, batch - 1)
    for s in rows:
        dom, ref = O.estimate(x[s], 3, m, k, w, True, "hann")
        assert O.north_star_error(np.asarray(vals[s]), ref) <= TOL[prec], s


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("k,w,taper", [(5, 5, "hann"), (4, 9, None)])
def test_register_fft_front_end_vs_oracle(cuda, dtype, k, w, taper):
    """Large batches of m = 256 series in fp32 mode take the register-FFT front
    end (k_front_r16: >= 16 segment pairs per SM) and the pipelined smoother;
    odd k leaves the last pair with one segment; both input dtypes."""
    import torch

    P = api()
    batch, m = 1300, 256
    rng = np.random.default_rng(k * 100 + w)
    x = rng.standard_normal((batch, m * k)).astype(dtype)
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=m, k=k), w, precision="fp32", taper=taper)
    vals = P.estimate_batch(torch.from_numpy(x).to(cuda), cfg)
    assert vals.shape == (batch, P.principal_domain(3, m).shape[0])
    for s in (0, 1, 147, 148, batch // 2, batch - 1):
        dom, ref = O.estimate(x[s].astype(np.float64), 3, m, k, w, True, taper)
        assert O.north_star_error(np.asarray(vals[s]), ref) <= TOL["fp32"], s


def test_acceptance_criterion1_compare_grids(cuda):
    """The reference's acceptance criterion 1 (tests/test_acceptance.py:76-103)
    on the GPU path: for QPC series, every plan's fp64 grid is within
    compare_grids < 1e-9 of the NAIVE (materialized) oracle, orders 3 and 4."""
    P = api()
    worst = 0.0
    for order, sizes in ((3, (128, 256, 512)), (4, (64, 128))):
        for n in sizes:
            x = P.generate_qpc(0.1, 0.15, n, 0.5, 1234)
            spec = O.segment_spectra(x.samples, n, 1)
            for m3 in (5, 9, 17):
                ref = P.SpectrumGrid(order, n, m3, P.SmoothingPlan.NAIVE, O.principal_domain(order, n),
                                     O.materialized_values(spec, order, m3))
                for plan in P.SmoothingPlan:
                    cfg = P.EstimationConfig(order, P.SegmentConfig(m=n, k=1), m3, plan)
                    worst = max(worst, P.compare_grids(ref, P.estimate_spectrum(x, cfg)))
    assert worst < 1e-9, worst


def test_estimate_batch_of_one_keeps_batch_axis(cuda):
    P = api()
    x = np.random.default_rng(5).standard_normal((1, 64 * 4))
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=64, k=4), 3)
    vals = P.estimate_batch(x, cfg)
    assert vals.shape == (1, P.principal_domain(3, 64).shape[0])
    dom, ref = O.estimate(x[0], 3, 64, 4, 3)
    assert north_star(vals[0], ref) <= TOL_FP64


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_parallel_estimate_segment_split(cuda, prec):
    """WorkerConfig.p > 1 maps to a segment split over GPUs; here the shards
    are placed on one device (devices=[0]*p) so the split-and-sum path runs
    on a one-GPU box; values match the oracle within the precision's bar."""
    P = api()
    x = np.random.default_rng(31).standard_normal(128 * 12)
    cfg = P.EstimationConfig(3, P.SegmentConfig(m=128, k=12), 5, precision=prec, taper="hann")
    dom, ref = O.estimate(x, 3, 128, 12, 5, True, "hann")
    for p in (2, 3, 5):
        g = P.parallel_estimate(P.TimeSeries(x), cfg, P.WorkerConfig(p=p), devices=[0] * p)
        assert np.array_equal(g.indices, dom)
        assert north_star(g.values, ref) <= TOL[prec], p
