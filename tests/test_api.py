"""Host-side API of the drop-in (no GPU): configuration validation, plan
vocabulary, partitioning, interchange format and the multi-GPU shard layout.
Ports of hospectra tests/test_spectra.py, test_parallel.py, test_series.py."""

import csv
import json

import numpy as np
import pytest

from oracle import hos_oracle as O
from paper_1805_11775_b200 import (
    DataError,
    EstimationConfig,
    ParameterError,
    SegmentConfig,
    SmoothingPlan,
    SpectrumGrid,
    TimeSeries,
    WindowSpec,
    WorkerConfig,
    baseline_config,
    baseline_series,
    generate_gaussian_ar,
    generate_qpc,
    partition_domain,
    raw_bispectrum_value,
    raw_trispectrum_value,
    segment_and_demean,
    write_grid_csv,
)
from paper_1805_11775_b200.parallel import row_blocks, shard_layout


def test_timeseries_validation():
    assert TimeSeries([1, 2, 3]).samples.dtype == np.float64
    with pytest.raises(ParameterError):
        TimeSeries([])
    with pytest.raises(DataError, match="index 2"):
        TimeSeries([1.0, 2.0, np.nan])


def test_segment_config_validation():
    with pytest.raises(ParameterError):
        SegmentConfig(m=0)
    with pytest.raises(ParameterError, match=r"k\*m = 4\*32 = 128 exceeds series length n = 100"):
        SegmentConfig(m=32, k=4).validate_for(TimeSeries(np.zeros(100)))


def test_segment_and_demean_matches_reference_semantics():
    x = np.arange(10.0)
    s = segment_and_demean(TimeSeries(x), SegmentConfig(m=4, k=2))
    assert s.means_removed and s.segments.shape == (2, 4)
    assert np.allclose(s.segments, [[-1.5, -0.5, 0.5, 1.5], [-1.5, -0.5, 0.5, 1.5]])


def test_estimation_config_validation():
    seg = SegmentConfig(m=64)
    with pytest.raises(ParameterError, match="order must be 3 or 4"):
        EstimationConfig(2, seg, 5)
    with pytest.raises(ParameterError, match=">= 1"):
        EstimationConfig(3, seg, 0)
    with pytest.raises(ParameterError, match="m3 < m/2"):
        EstimationConfig(3, seg, 32)
    with pytest.raises(ParameterError, match="precision"):
        EstimationConfig(3, seg, 5, precision="fp16")
    with pytest.raises(ParameterError, match="taper"):
        EstimationConfig(3, seg, 5, taper="kaiser")
    cfg = EstimationConfig(3, seg, 5)
    assert cfg.plan is SmoothingPlan.EFFICIENT and cfg.conjugate_last and cfg.precision == "fp64"
    assert cfg.taper is None


def test_smoothing_plans_exactly_six():
    # hospectra tests/test_window_sums.py:313-325
    assert [p.name for p in SmoothingPlan] == ["NAIVE", "WS", "PREFIX", "FAST", "EFFICIENT", "STREAMING"]
    assert SmoothingPlan.parse("efficient") is SmoothingPlan.EFFICIENT
    with pytest.raises(ParameterError, match="valid plans"):
        SmoothingPlan.parse("turbo")
    assert SmoothingPlan.STREAMING.declared_extra_memory == "O(w)"


def test_window_spec():
    assert WindowSpec(3, "periodic").out_shape(5, 7) == (5, 7)
    assert WindowSpec(3).out_shape(5, 7) == (3, 5)
    with pytest.raises(ParameterError):
        WindowSpec(0)
    with pytest.raises(ParameterError):
        WindowSpec(3, "mirror")


def test_raw_values():
    # hospectra tests/test_spectra.py:67-102
    f = np.ones(4, complex)
    assert abs(raw_bispectrum_value(f, 1, 2) - 0.25) < 1e-15
    assert abs(raw_trispectrum_value(f, 1, 2, 3) - 0.25) < 1e-15
    rng = np.random.default_rng(3)
    f = rng.standard_normal(8) + 1j * rng.standard_normal(8)
    assert abs(raw_bispectrum_value(f, 5, 6) - f[5] * f[6] * np.conj(f[3]) / 8) < 1e-12
    assert abs(raw_bispectrum_value(f, 2, 3, False) - f[2] * f[3] * f[5] / 8) < 1e-12


def test_generators_match_reference_draws():
    s = generate_qpc(0.1, 0.15, 64, 0.4, seed=5)
    rng = np.random.default_rng(5)
    p1, p2 = rng.uniform(0.0, 2.0 * np.pi, size=2)
    t = np.arange(64.0)
    x = (np.cos(2 * np.pi * 0.1 * t + p1) + np.cos(2 * np.pi * 0.15 * t + p2)
         + np.cos(2 * np.pi * 0.25 * t + p1 + p2)) + rng.normal(0.0, 0.4, size=64)
    assert np.array_equal(s.samples, x)
    with pytest.raises(ParameterError):
        generate_qpc(0.3, 0.3, 64)
    with pytest.raises(ParameterError, match="unstable"):
        generate_gaussian_ar([1.5], 10)
    assert generate_gaussian_ar([0.5], 100, seed=1).n == 100


def test_baseline_configs():
    assert [c.name.split("_")[0] for c in (baseline_config(n) for n in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"))] == [
        "cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
    c = baseline_config("cfg2")
    assert (c.order, c.n, c.m, c.k, c.m3) == (3, 1 << 20, 1024, 1024, 9)
    x = baseline_series("cfg1")
    assert x.dtype == np.float64 and x.shape == (2048,)
    assert np.array_equal(x, baseline_series("cfg1"))  # seeded
    c5 = baseline_config("cfg5")
    assert baseline_series(c5, batch=2).shape == (2, c5.n)


# ---- partitioning (hospectra tests/test_parallel.py:19-56)


def test_partition_domain_ports():
    from paper_1805_11775_b200 import principal_domain

    dom = principal_domain(3, 16)
    assert np.array_equal(partition_domain(dom, WorkerConfig(p=1))[0], dom)
    parts = partition_domain(principal_domain(3, 8), WorkerConfig(p=4, partition="point_blocks"))
    assert sorted(len(p) for p in parts) == [1, 1, 2, 2]
    dom = principal_domain(3, 64)
    for mode in ("row_blocks", "point_blocks"):
        parts = partition_domain(dom, WorkerConfig(p=8, partition=mode))
        assert np.array_equal(np.concatenate([p for p in parts if len(p)]), dom)
    parts = partition_domain(dom, WorkerConfig(p=5))
    rows = [set(int(r) for r in p[:, 0]) for p in parts if len(p)]
    assert all(not (a & b) for a, b in zip(rows, rows[1:]))
    with pytest.raises(ParameterError):
        WorkerConfig(p=0)
    with pytest.raises(ParameterError):
        WorkerConfig(p=2, partition="diagonal")


# ---- interchange format (hospectra tests/test_spectra.py:299-323)


def test_write_grid_csv(tmp_path):
    dom = O.principal_domain(3, 16)
    rng = np.random.default_rng(1)
    vals = rng.standard_normal(len(dom)) + 1j * rng.standard_normal(len(dom))
    g = SpectrumGrid(order=3, m=16, m3=3, plan=SmoothingPlan.EFFICIENT, indices=dom, values=vals)
    path = tmp_path / "g.csv"
    write_grid_csv(g, path)
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["k1", "k2", "re", "im"]
    for row, idx, v in zip(rows[1:], dom, vals):
        assert [int(row[0]), int(row[1])] == list(idx)
        assert float(row[2]) == v.real and float(row[3]) == v.imag
    assert g.peak_point().k == tuple(int(v) for v in dom[np.argmax(np.abs(vals))])
    g4 = SpectrumGrid(4, 16, 3, SmoothingPlan.FAST, O.principal_domain(4, 16), np.zeros(len(O.principal_domain(4, 16))))
    write_grid_csv(g4, tmp_path / "g4.csv")
    assert open(tmp_path / "g4.csv").readline().strip() == "k1,k2,k3,re,im"


# ---- multi-GPU shard layout


def _geom3(m, w):
    """Order-3 dilated-domain lines, restated independently (SURVEY §8 D_h)."""
    h = w // 2
    lo, hi = -h, w - 1 - h
    rows = (m - 1) // 2 + 1
    stop = [min(k1, (m - 2 * k1 - 1) // 2) + 1 for k1 in range(rows)]
    cmax = [max(stop[k] - 1 for k in range(max(0, a - hi), min(rows - 1, a - lo) + 1)) + hi
            for a in range(lo, rows + hi)]
    line_start = np.concatenate([[0], np.cumsum([c - lo + 1 for c in cmax])]).astype(np.int64)
    row_off = np.concatenate([[0], np.cumsum(stop)]).astype(np.int64)
    return rows, lo, hi, cmax, line_start, row_off


@pytest.mark.parametrize("m,w,k,n", [(64, 5, 12, 2), (128, 9, 7, 3), (256, 4, 16, 8), (32, 3, 5, 4)])
def test_shard_layout_invariants(m, w, k, n):
    rows, lo, hi, cmax, line_start, row_off = _geom3(m, w)
    rlr = lambda r0, r1: (r0, r1 - 1 + (w - 1) + 1) if r1 > r0 else (r0, r0)
    lay = shard_layout(k, row_off, line_start, rlr, n)
    # segments and rows tile their ranges
    assert lay.seg_bounds[0] == 0 and lay.seg_bounds[-1] == k
    assert lay.row_bounds[0] == 0 and lay.row_bounds[-1] == rows
    assert lay.point_bounds[-1] == row_off[-1]
    # owned line blocks tile all lines; each rank's needed lines start in its own block
    assert lay.own_lines[0][0] == 0 and lay.own_lines[-1][1] == len(line_start) - 1
    for r in range(n):
        if r + 1 < n:
            assert lay.own_lines[r][1] == lay.own_lines[r + 1][0]
        if lay.row_bounds[r] < lay.row_bounds[r + 1]:
            assert lay.own_lines[r][0] <= lay.need_lines[r][0]
            assert lay.need_cells[r][1] - lay.own_cells[r][1] <= lay.halo or lay.halo_in_next is False
    assert lay.block >= max(c1 - c0 for c0, c1 in lay.own_cells)
    assert row_blocks(row_off, 1) == [0, rows]


@pytest.mark.parametrize("m,w,k,n", [(64, 5, 12, 2), (128, 9, 7, 3), (256, 4, 16, 8), (32, 3, 5, 4),
                                     (1024, 9, 1024, 8), (1024, 9, 1024, 3), (4096, 17, 2250, 8)])
def test_native_shard_layout_matches_python(m, w, k, n):
    """hos_shard_layout (the C-ABI multi-GPU path's layout) == parallel.shard_layout."""
    import __graft_entry__

    __graft_entry__.ensure_built()
    from paper_1805_11775_b200 import _native

    rows, lo, hi, cmax, line_start, row_off = _geom3(m, w)
    rlr = lambda r0, r1: (r0, r1 - 1 + (w - 1) + 1) if r1 > r0 else (r0, r0)
    lay = shard_layout(k, row_off, line_start, rlr, n)
    rec, (block, halo, in_next) = _native.shard_layout_native(3, m, k, w, n)
    assert list(rec[:, 0]) + [rec[-1, 1]] == lay.seg_bounds
    assert list(rec[:, 2]) + [rec[-1, 3]] == lay.row_bounds
    assert [tuple(v) for v in rec[:, 4:6]] == [tuple(v) for v in lay.own_lines]
    assert [tuple(v) for v in rec[:, 6:8]] == [tuple(v) for v in lay.need_lines]
    assert [tuple(v) for v in rec[:, 8:10]] == [tuple(v) for v in lay.own_cells]
    assert [tuple(v) for v in rec[:, 10:12]] == [tuple(v) for v in lay.need_cells]
    assert list(rec[:, 12]) + [rec[-1, 13]] == lay.point_bounds
    assert (block, halo, bool(in_next)) == (lay.block, lay.halo, lay.halo_in_next)


def test_report_json_schema():
    """BenchReport keeps the reference's JSON schema (hospectra/bench.py:58-80):
    the twelve keys, their types, round trip, rejection of foreign records."""
    import paper_1805_11775_b200 as P

    r = P.BenchReport(plan="EFFICIENT", order=3, n=256, M=256, K=1, M3=33, P=1, wall_seconds=0.5,
                      peak_extra_bytes=123, peak_rss_bytes=456, checksum=7.25)
    text = P.reports_to_json([r, r])
    assert P.reports_from_json(text) == [r, r]
    assert list(json.loads(text)[0]) == ["plan", "order", "n", "M", "K", "M3", "P", "wall_seconds",
                                         "peak_extra_bytes", "peak_rss_bytes", "checksum", "status"]
    assert r.status == "ok" and isinstance(r.wall_seconds, float)
    with pytest.raises(P.ParameterError):
        P.reports_from_json(json.dumps([{"plan": "EFFICIENT"}]))
    with pytest.raises(P.ParameterError):
        P.reports_from_json(json.dumps({"plan": "EFFICIENT"}))


def test_save_series_round_trip(tmp_path):
    import paper_1805_11775_b200 as P

    x = np.random.default_rng(3).standard_normal(257) * 1e3
    for fmt in ("csv", "raw64"):
        path = tmp_path / f"s.{fmt}"
        P.save_series(P.TimeSeries(x), path, fmt=fmt)
        assert np.array_equal(P.load_series(path, fmt=fmt).samples, x)
    with pytest.raises(P.ParameterError):
        P.save_series(P.TimeSeries(x), tmp_path / "s.bin", fmt="bin")


def test_compare_grids_semantics():
    """compare_grids is the reference's per-point relative deviation
    (hospectra/spectra.py:442-453): max|a-b| / max(|a|, |b|, 1e-12),
    0.0 on empty grids, ParameterError on mismatched grids."""
    import paper_1805_11775_b200 as P

    dom = O.principal_domain(3, 16)
    rng = np.random.default_rng(9)
    va = rng.standard_normal(len(dom)) + 1j * rng.standard_normal(len(dom))
    vb = va * (1 + 1e-7) + 1e-13
    vb[3] = 0.0
    a = P.SpectrumGrid(3, 16, 3, P.SmoothingPlan.EFFICIENT, dom, va)
    b = P.SpectrumGrid(3, 16, 3, P.SmoothingPlan.NAIVE, dom, vb)
    want = np.max(np.abs(va - vb) / np.maximum(np.maximum(np.abs(va), np.abs(vb)), 1e-12))
    assert P.compare_grids(a, b) == want == 1.0   # a zeroed point counts fully
    vb[3] = va[3]
    assert P.compare_grids(a, P.SpectrumGrid(3, 16, 3, P.SmoothingPlan.NAIVE, dom, vb)) < 2e-7
    tiny = P.SpectrumGrid(3, 16, 3, P.SmoothingPlan.NAIVE, dom, np.zeros(len(dom)) + 1e-14)
    zero = P.SpectrumGrid(3, 16, 3, P.SmoothingPlan.NAIVE, dom, np.zeros(len(dom), complex))
    assert P.compare_grids(tiny, zero) == pytest.approx(1e-2)   # the 1e-12 floor
    e = P.SpectrumGrid(3, 2, 1, P.SmoothingPlan.NAIVE, dom[:0], np.zeros(0, complex))
    assert P.compare_grids(e, e) == 0.0
    with pytest.raises(P.ParameterError):
        P.compare_grids(a, P.SpectrumGrid(3, 16, 5, P.SmoothingPlan.NAIVE, dom, va))
    with pytest.raises(P.ParameterError):
        P.compare_grids(a, P.SpectrumGrid(3, 16, 3, P.SmoothingPlan.NAIVE, dom[:-1], va[:-1]))
