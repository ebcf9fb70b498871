"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference (hospectra 0.1.0, pure Python) is imported read-only from
/root/reference/pkg/src; it cannot travel to the GPU box, so its outputs are
committed here as small fixtures.  Inputs are regenerated from seeds by
``paper_1805_11775_b200.signals`` / ``numpy.random.default_rng``; each
fixture stores a SHA-256 of its input so a generator drift is detected.

Fixtures:
  small_cases.npz   full grids of estimate_spectrum for many small configs
                    (orders 3/4, odd/even windows, conj on/off, k>1, w=1, tiny m)
  cfg1.npz          BASELINE cfg1 (n=2048 f64, M=128 K=16 w=5, Hann) full grid:
                    estimate_from_spectra on fft(hann * demeaned segments)
                    (the tapered oracle of SURVEY §0.1 #1) + untapered grid
  cfgN_rows.npz     BASELINE cfg2..cfg5: reference values on selected whole
                    output rows (k1) through the reference's own
                    _compute_values (hospectra/spectra.py:391) on the tapered
                    spectra; cfg5: full grids of selected series
  cfg2_full.npz,    BASELINE cfg2 / cfg4: the WHOLE grid (65,792 / 61,721 points) from the same seam
  cfg4_full.npz
  qpc1024.npz       the acceptance QPC case (generate_qpc(.1,.15,1024,0,seed 7),
                    m3=5): peak bin and values of selected rows
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import hospectra as H  # noqa: E402  (reference, read-only)
from hospectra.spectra import _compute_values  # noqa: E402

from paper_1805_11775_b200 import signals  # noqa: E402


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def hann(m):
    u = np.arange(m, dtype=np.float64)
    return 0.5 - 0.5 * np.cos(2.0 * np.pi * u / m)


def tapered_spectra(x64, m, k):
    seg = x64[: m * k].reshape(k, m).copy()
    seg -= seg.mean(axis=1, keepdims=True)
    return np.fft.fft(seg * hann(m)[None, :], axis=1)


# (name, order, m, k, m3, conj, seed, extra samples)
SMALL = [
    ("o3_m64_k4_w5", 3, 64, 4, 5, True, 11, 7),
    ("o3_m64_k4_w4_even", 3, 64, 4, 4, True, 12, 0),
    ("o3_m33_k2_w3_noconj", 3, 33, 2, 3, False, 13, 5),
    ("o3_m128_k3_w1", 3, 128, 3, 1, True, 14, 0),
    ("o3_m8_k1_w3", 3, 8, 1, 3, True, 15, 0),
    ("o3_m7_k2_w3_odd_m", 3, 7, 2, 3, True, 16, 1),
    ("o3_m256_k2_w17", 3, 256, 2, 17, True, 17, 0),
    ("o3_m100_k5_w9_noconj", 3, 100, 5, 9, False, 18, 3),
    ("o4_m32_k2_w3", 4, 32, 2, 3, True, 21, 0),
    ("o4_m64_k2_w5", 4, 64, 2, 5, True, 22, 0),
    ("o4_m33_k2_w4_noconj", 4, 33, 2, 4, False, 23, 2),
    ("o4_m8_k1_w3", 4, 8, 1, 3, True, 24, 0),
    ("o4_m48_k3_w6_even", 4, 48, 3, 6, True, 25, 0),
]


def make_small():
    out = {}
    for name, order, m, k, w, conj, seed, extra in SMALL:
        x = np.random.default_rng(seed).standard_normal(m * k + extra)
        cfg = H.EstimationConfig(order, H.SegmentConfig(m=m, k=k), w, H.SmoothingPlan.EFFICIENT,
                                 conjugate_last=conj)
        g = H.estimate_spectrum(H.TimeSeries(x), cfg)
        out[f"{name}__x"] = x
        out[f"{name}__idx"] = g.indices
        out[f"{name}__val"] = g.values
        out[f"{name}__meta"] = np.array([order, m, k, w, int(conj), seed, extra])
    # constant series -> exactly zero (tests/test_spectra.py:159-164)
    for order in (3, 4):
        x = np.full(64, 2.5)
        cfg = H.EstimationConfig(order, H.SegmentConfig(m=64, k=1), 5)
        g = H.estimate_spectrum(H.TimeSeries(x), cfg)
        assert np.all(g.values == 0)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), names=np.array([s[0] for s in SMALL]), **out)


def make_cfg1():
    c = signals.baseline_config("cfg1")
    x = signals.baseline_series(c).astype(np.float64)
    cfg = H.EstimationConfig(3, H.SegmentConfig(m=c.m, k=c.k), c.m3)
    spec = tapered_spectra(x, c.m, c.k)
    g = H.estimate_from_spectra(H.SegmentSpectrumSet(spectra=spec), cfg)
    g0 = H.estimate_spectrum(H.TimeSeries(x), cfg)
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), x_sha=sha(x), idx=g.indices, val_hann=g.values,
                        val_notaper=g0.values)


ROWS = {
    "cfg2": [0, 1, 100, 255, 256, 300, 511],
    "cfg3": [0, 40, 80, 1023, 2047],
    "cfg4": [0, 13, 28, 64, 127],
}


def rows_dom(order, m, rows):
    dom = H.principal_domain(order, m)
    sel = np.isin(dom[:, 0], rows)
    return dom, np.flatnonzero(sel)


def make_rows(name):
    c = signals.baseline_config(name)
    t0 = time.time()
    x = signals.baseline_series(c).astype(np.float64)
    xs = sha(signals.baseline_series(c))
    spec = tapered_spectra(x, c.m, c.k)
    cfg = H.EstimationConfig(c.order, H.SegmentConfig(m=c.m, k=c.k), c.m3)
    dom, pos = rows_dom(c.order, c.m, ROWS[name])
    vals = np.empty(len(pos), np.complex128)
    # whole rows are contiguous slices of the lexicographic domain
    cuts = np.flatnonzero(np.diff(pos) != 1) + 1
    for grp in np.split(np.arange(len(pos)), cuts):
        a, b = pos[grp[0]], pos[grp[-1]] + 1
        vals[grp] = _compute_values(H.SegmentSpectrumSet(spectra=spec), cfg, dom[a:b])
    np.savez_compressed(os.path.join(HERE, f"{name}_rows.npz"), x_sha=xs, rows=np.array(ROWS[name]),
                        pos=pos, idx=dom[pos], val=vals)
    print(name, "rows", len(pos), f"{time.time() - t0:.1f}s")


def make_full(name="cfg2"):
    """The WHOLE principal-domain grid of a BASELINE config from the reference's
    operator seam (single process, a few seconds for cfg2): cfg2_full.npz."""
    c = signals.baseline_config(name)
    t0 = time.time()
    x = signals.baseline_series(c).astype(np.float64)
    xs = sha(signals.baseline_series(c))
    spec = tapered_spectra(x, c.m, c.k)
    cfg = H.EstimationConfig(c.order, H.SegmentConfig(m=c.m, k=c.k), c.m3)
    dom = H.principal_domain(c.order, c.m)
    vals = _compute_values(H.SegmentSpectrumSet(spectra=spec), cfg, dom)
    np.savez_compressed(os.path.join(HERE, f"{name}_full.npz"), x_sha=xs, npoints=np.array(len(dom)), val=vals)
    print(name, "full grid", len(dom), f"{time.time() - t0:.1f}s")


def make_cfg5(series=(0, 1, 4095)):
    c = signals.baseline_config("cfg5")
    t0 = time.time()
    xall = signals.baseline_series(c)  # (4096, n) float32
    cfg = H.EstimationConfig(3, H.SegmentConfig(m=c.m, k=c.k), c.m3)
    out = {"x_sha": sha(xall), "series": np.array(series)}
    for s in series:
        spec = tapered_spectra(xall[s].astype(np.float64), c.m, c.k)
        g = H.estimate_from_spectra(H.SegmentSpectrumSet(spectra=spec), cfg)
        out[f"val_{s}"] = g.values
    out["idx"] = g.indices
    np.savez_compressed(os.path.join(HERE, "cfg5_series.npz"), **out)
    print("cfg5", f"{time.time() - t0:.1f}s")


def make_qpc():
    series = H.generate_qpc(0.1, 0.15, 1024, 0.0, seed=7)
    cfg = H.EstimationConfig(3, H.SegmentConfig(m=1024), 5)
    g = H.estimate_spectrum(series, cfg)
    (k1, k2), _ = g.peak_point()
    rows = [0, 100, 154, 255, 511]
    sel = np.flatnonzero(np.isin(g.indices[:, 0], rows))
    np.savez_compressed(os.path.join(HERE, "qpc1024.npz"), x_sha=sha(series.samples), peak=np.array([k1, k2]),
                        pos=sel, val=g.values[sel], absmax=np.abs(g.values).max())


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "cfg1", "qpc", "cfg2", "cfg2full", "cfg4", "cfg4full", "cfg5", "cfg3"]
    for w in which:
        if w == "small":
            make_small()
        elif w == "cfg1":
            make_cfg1()
        elif w == "cfg2full":
            make_full("cfg2")
        elif w == "cfg4full":
            make_full("cfg4")
        elif w == "qpc":
            make_qpc()
        elif w == "cfg5":
            make_cfg5()
        else:
            make_rows(w)
        print("done", w)
