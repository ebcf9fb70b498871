"""CPU oracle for the direct-method HOS hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The shipped estimator in
``paper_1805_11775_b200`` runs on the GPU and fails loudly without its CUDA
library; nothing there imports this file.

It restates, in NumPy, the reference ``hospectra`` 0.1.0 algorithm
(``/root/reference/pkg/src/hospectra``; abbreviated ``hospectra/X.py`` below):

* ``segment_spectra``      — segment + demean (``series.py:159-165``), optional
                             taper (extension), full-length
                             DFT (``dft.py:36-41``).
* ``principal_domain``     — closed-form row lengths (``spectra.py:133-168``).
* ``efficient_values``     — the default EFFICIENT plan end to end, restated
                             so that every floating-point operation happens in
                             the reference's order: the segment-averaged value
                             function (``spectra.py:227-263``), w-aligned
                             (2w-1)^2 patches with local prefix sums
                             (``tiled.py:36-47,96-118``), the 3-D plane ring
                             (``tiled.py:171-244``) and the final
                             ``/ w**(order-1)`` (``spectra.py:415``).  Pinned
                             bit-for-bit against the reference by
                             ``tests/golden`` (see ``tests/test_oracle.py``).
* ``materialized_values``  — the smooth-each-segment-then-average path of the
                             NAIVE plan (``spectra.py:207-224,351-388``), an
                             independent second oracle.
* ``spot_values``          — explicit window sums at chosen points, the
                             definition pinned by ``tests/test_spectra.py:190-210``;
                             used at full BASELINE sizes where a whole-grid
                             oracle run is too slow.
* ``parallel_efficient``   — the output-domain process fan-out of
                             ``parallel.py:62-162`` (row_blocks), used as the
                             multi-core CPU baseline.
"""

from __future__ import annotations

import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

__all__ = [
    "hann",
    "segment_spectra",
    "principal_domain",
    "domain_row_lengths",
    "efficient_values",
    "materialized_values",
    "spot_values",
    "estimate",
    "parallel_efficient",
    "north_star_error",
]


# ---------------------------------------------------------------------------
# front end


def hann(m: int) -> np.ndarray:
    """Periodic Hann taper 0.5 - 0.5 cos(2 pi u / m) (SURVEY §0.1 #1 pin)."""
    u = np.arange(m, dtype=np.float64)
    return 0.5 - 0.5 * np.cos(2.0 * np.pi * u / m)


def segment_spectra(x, m: int, k: int, taper=None) -> np.ndarray:
    """(k, m) complex128 spectra of the first k*m samples.

    Demean per segment in float64 (hospectra/series.py:163-164), multiply
    by the taper when one is given, then ``np.fft.fft`` along the segment
    axis (hospectra/dft.py:41).  Input is upcast to float64 exactly like
    ``TimeSeries`` does (hospectra/series.py:45)."""
    x = np.asarray(x, dtype=np.float64)
    if k * m > x.size:
        raise ValueError(f"k*m = {k}*{m} = {k * m} exceeds series length n = {x.size}")
    seg = x[: k * m].reshape(k, m).copy()
    seg -= seg.mean(axis=1, keepdims=True)
    if taper is not None:
        if isinstance(taper, str):
            if taper != "hann":
                raise ValueError(f"unknown taper {taper!r}")
            taper = hann(m)
        seg = seg * np.asarray(taper, dtype=np.float64)[None, :]
    return np.fft.fft(seg, axis=1)


def domain_row_lengths(m: int) -> np.ndarray:
    """Order-3 principal-domain row lengths, k1 = 0..(m-1)//2
    (hospectra/spectra.py:146-147)."""
    k1 = np.arange((m - 1) // 2 + 1)
    return np.minimum(k1, (m - 2 * k1 - 1) // 2) + 1


def principal_domain(order: int, m: int) -> np.ndarray:
    """Lexicographic principal-domain tuples (hospectra/spectra.py:133-168):
    order 3 ``0<=k2<=k1, k1+k2<m/2``; order 4 ``0<=k3<=k2<=k1, sum<m/2``."""
    out = []
    top = (m - 1) // 2 + 1
    for k1 in range(top):
        n2 = min(k1, (m - 2 * k1 - 1) // 2) + 1
        if order == 3:
            if n2 > 0:
                out.extend((k1, k2) for k2 in range(n2))
            continue
        for k2 in range(max(n2, 0)):
            n3 = min(k2, (m - 2 * k1 - 2 * k2 - 1) // 2) + 1
            if n3 > 0:
                out.extend((k1, k2, k3) for k3 in range(n3))
    if not out:
        return np.empty((0, order - 1), dtype=np.int32)
    return np.asarray(out, dtype=np.int32)


# ---------------------------------------------------------------------------
# EFFICIENT plan restatement (bit-exact with the reference)


class _SegmentProducts:
    """Segment-averaged raw products at shifted, wrapped indices.

    Restates the value functions of hospectra/spectra.py:227-263: indices
    arrive in output coordinates, are shifted by the window offset h and
    wrapped mod m; the last factor is read from a 2- (order 3) or 3-fold
    (order 4) concatenation so the index sum needs no wrap.  The segment
    sum runs sequentially in complex128 and is scaled by 1/(m k) once."""

    def __init__(self, spectra: np.ndarray, h: int, conj: bool, order: int):
        self.spectra = np.asarray(spectra, dtype=np.complex128)
        self.k, self.m = self.spectra.shape
        self.h = h
        reps = 2 if order == 3 else 3
        tiled = np.tile(self.spectra, (1, reps))
        self.last = np.conj(tiled) if conj else tiled
        self.scale = 1.0 / (self.m * self.k)

    def pair(self, rows, cols):
        m, h = self.m, self.h
        r = (np.asarray(rows) - h) % m
        c = (np.asarray(cols) - h) % m
        s = r + c
        total = None
        for f, g in zip(self.spectra, self.last):
            term = f[r] * f[c] * g[s]
            total = term if total is None else total + term
        return total * self.scale

    def triple(self, rows, cols, plane: int):
        m, h = self.m, self.h
        r = (np.asarray(rows) - h) % m
        c = (np.asarray(cols) - h) % m
        d = (int(plane) - h) % m
        s = r + c + d
        total = None
        for f, g in zip(self.spectra, self.last):
            term = (f[r] * f[c]) * (f[d] * g[s])
            total = term if total is None else total + term
        return total * self.scale


def _box_from_patch(patch: np.ndarray, w: int, nr: int, nc: int) -> np.ndarray:
    """w x w window sums of an (nr+w-1, nc+w-1) patch by local prefix sums
    and differences, rows first then columns (hospectra/tiled.py:36-47)."""
    if w == 1:
        return patch.copy()
    down = np.cumsum(patch, axis=0)
    band = down[w - 1:, :].copy()
    band[1:, :] -= down[: nr - 1, :]
    across = np.cumsum(band, axis=1)
    box = across[:, w - 1:].copy()
    box[:, 1:] -= across[:, : nc - 1]
    return box


def _row_runs(dom: np.ndarray):
    """(row, first, stop, flat offset) for each k1 run of a lex 2-column
    domain slice (hospectra/spectra.py:269-285)."""
    if len(dom) == 0:
        return []
    cut = np.flatnonzero(np.diff(dom[:, 0])) + 1
    starts = np.concatenate([[0], cut])
    ends = np.concatenate([cut, [len(dom)]])
    return [
        (int(dom[a, 0]), int(dom[a, 1]), int(dom[b - 1, 1]) + 1, int(a))
        for a, b in zip(starts, ends)
    ]


def _efficient_order3(prod: _SegmentProducts, w: int, dom: np.ndarray) -> np.ndarray:
    m = prod.m
    out = np.empty(len(dom), dtype=np.complex128)
    runs = _row_runs(dom)
    bands: dict[int, list] = {}
    for run in runs:
        bands.setdefault(run[0] - run[0] % w, []).append(run)
    for top in sorted(bands):
        members = bands[top]
        nr = min(w, m - top)
        lo = min(r[1] for r in members)
        hi = max(r[2] for r in members)
        left = lo - lo % w
        rows = np.arange(top, top + nr + w - 1)[:, None]
        while left < hi:
            nc = min(w, m - left)
            cols = np.arange(left, left + nc + w - 1)[None, :]
            box = _box_from_patch(prod.pair(rows, cols), w, nr, nc)
            for row, first, stop, off in members:
                a = max(first, left)
                b = min(stop, left + nc)
                if a < b:
                    dst = off + (a - first)
                    out[dst: dst + (b - a)] = box[row - top, a - left: b - left]
            left += w
    return out


def _efficient_order4(prod: _SegmentProducts, w: int, dom: np.ndarray) -> np.ndarray:
    m = prod.m
    out = np.empty(len(dom), dtype=np.complex128)
    if len(dom) == 0:
        return out
    brk = np.flatnonzero((np.diff(dom[:, 0]) != 0) | (np.diff(dom[:, 1]) != 0)) + 1
    first = np.concatenate([[0], brk])
    last = np.concatenate([brk, [len(dom)]])
    k1 = dom[first, 0].astype(np.int64)
    k2 = dom[first, 1].astype(np.int64)
    lo3 = dom[first, 2].astype(np.int64)
    hi3 = dom[last - 1, 2].astype(np.int64) + 1
    base = first.astype(np.int64)
    groups: dict[tuple, list] = {}
    for t in range(len(k1)):
        groups.setdefault((int(k1[t]) // w, int(k2[t]) // w), []).append(t)
    for key in sorted(groups):
        sel = np.asarray(groups[key])
        top, left = key[0] * w, key[1] * w
        nr, nc = min(w, m - top), min(w, m - left)
        rows = np.arange(top, top + nr + w - 1)[:, None]
        cols = np.arange(left, left + nc + w - 1)[None, :]
        ii, jj = k1[sel] - top, k2[sel] - left
        st, sp, bb = lo3[sel], hi3[sel], base[sel]

        def plane(p):
            return _box_from_patch(prod.triple(rows, cols, p), w, nr, nc)

        z0 = w * (int(st.min()) // w)
        ring = np.stack([plane(z0 + t) for t in range(w)])
        acc = ring.sum(axis=0)
        for z in range(z0, int(sp.max())):
            if z > z0:
                fresh = plane(z + w - 1)
                slot = (z - 1) % w
                if z % w == 0:
                    ring[slot] = fresh
                    acc = ring.sum(axis=0)
                else:
                    acc -= ring[slot]
                    acc += fresh
                    ring[slot] = fresh
            live = (st <= z) & (z < sp)
            if live.any():
                out[bb[live] + (z - st[live])] = acc[ii[live], jj[live]]
    return out


def efficient_values(spectra, order: int, m3: int, conj: bool = True, dom=None) -> np.ndarray:
    """EFFICIENT-plan values at ``dom`` (default: the whole principal
    domain), c128, lexicographic — the reference's ``_compute_values`` for
    plan EFFICIENT (hospectra/spectra.py:391-416)."""
    spectra = np.asarray(spectra, dtype=np.complex128)
    m = spectra.shape[1]
    if dom is None:
        dom = principal_domain(order, m)
    if len(dom) == 0:
        return np.empty(0, dtype=np.complex128)
    prod = _SegmentProducts(spectra, m3 // 2, conj, order)
    if order == 3:
        out = _efficient_order3(prod, m3, dom)
    else:
        out = _efficient_order4(prod, m3, dom)
    out /= float(m3) ** (order - 1)
    return out


# ---------------------------------------------------------------------------
# independent oracles


def materialized_values(spectra, order: int, m3: int, conj: bool = True) -> np.ndarray:
    """Smooth every segment's full periodic raw grid, then average
    (hospectra/spectra.py:207-224,351-388 with the NAIVE window sum).
    O(k m^2 w^2) / O(k m^3 w^3): small sizes only."""
    spectra = np.asarray(spectra, dtype=np.complex128)
    k, m = spectra.shape
    w, h = m3, m3 // 2
    dom = principal_domain(order, m)
    shape = (m,) * (order - 1)
    acc = np.zeros(shape, dtype=np.complex128)
    idx = np.arange(m)
    for f in spectra:
        g = np.conj(f) if conj else f
        if order == 3:
            raw = f[:, None] * f[None, :] * g[(idx[:, None] + idx[None, :]) % m] / m
        else:
            raw = (f[:, None, None] * f[None, :, None] * f[None, None, :]
                   * g[(idx[:, None, None] + idx[None, :, None] + idx[None, None, :]) % m] / m)
        sm = np.zeros_like(raw)
        offs = range(-h, w - h)
        if order == 3:
            for u in offs:
                for v in offs:
                    sm += np.roll(raw, (-u, -v), axis=(0, 1))
        else:
            for u in offs:
                for v in offs:
                    for t in offs:
                        sm += np.roll(raw, (-u, -v, -t), axis=(0, 1, 2))
        acc += sm
    acc /= k * float(w) ** (order - 1)
    return acc[tuple(dom.T)]


def spot_values(spectra, order: int, m3: int, points, conj: bool = True) -> np.ndarray:
    """Explicit periodic window sums of the segment-averaged raw product at
    the given points (the definition of tests/test_spectra.py:190-210):
    B(k) = w^-(order-1) sum_{offsets in [-h, w-1-h]^(order-1)} R(k+offsets),
    R = (1/(m K)) sum_i F_i(a) F_i(b) [F_i(c)] G_i(a+b[+c])."""
    spectra = np.asarray(spectra, dtype=np.complex128)
    k, m = spectra.shape
    w, h = m3, m3 // 2
    last = np.conj(spectra) if conj else spectra
    pts = np.asarray(points, dtype=np.int64).reshape(-1, order - 1)
    offs = np.arange(-h, w - h)
    out = np.empty(len(pts), dtype=np.complex128)
    for t, p in enumerate(pts):
        if order == 3:
            a = (p[0] + offs)[:, None] % m
            b = (p[1] + offs)[None, :] % m
            s = (a + b) % m
            raw = spectra[:, a] * spectra[:, b] * last[:, s]
        else:
            a = (p[0] + offs)[:, None, None] % m
            b = (p[1] + offs)[None, :, None] % m
            c = (p[2] + offs)[None, None, :] % m
            s = (a + b + c) % m
            raw = spectra[:, a] * spectra[:, b] * spectra[:, c] * last[:, s]
        out[t] = raw.sum() / (m * k) / float(w) ** (order - 1)
    return out


def estimate(x, order: int, m: int, k: int, m3: int, conj: bool = True, taper=None):
    """(indices, values) of the full estimator on series ``x``."""
    spec = segment_spectra(x, m, k, taper)
    dom = principal_domain(order, m)
    return dom, efficient_values(spec, order, m3, conj, dom)


# ---------------------------------------------------------------------------
# multi-core CPU baseline (output-domain fan-out, hospectra/parallel.py)


def _row_block_bounds(dom: np.ndarray, p: int) -> list[int]:
    """row_blocks cut offsets (hospectra/parallel.py:62-80)."""
    total = len(dom)
    if p == 1 or total == 0:
        return [0, total] + [total] * (p - 1)
    _, first_idx, counts = np.unique(dom[:, 0], return_index=True, return_counts=True)
    cum = np.cumsum(counts)
    targets = np.arange(1, p) * (total / p)
    gb = np.searchsorted(cum, targets, side="left") + 1
    cuts = [int(first_idx[b]) if b < len(first_idx) else total for b in gb]
    return [0] + cuts + [total]


def _worker(args):
    spectra, order, m3, conj, part = args
    return efficient_values(spectra, order, m3, conj, part)


def parallel_efficient(spectra, order: int, m3: int, conj: bool = True, workers: int | None = None,
                       dom=None) -> np.ndarray:
    """EFFICIENT values over ``dom`` computed by a process pool over
    row-block partitions; bit-identical to the serial sweep."""
    spectra = np.asarray(spectra, dtype=np.complex128)
    if dom is None:
        dom = principal_domain(order, spectra.shape[1])
    p = workers or os.cpu_count() or 1
    if p == 1 or len(dom) == 0:
        return efficient_values(spectra, order, m3, conj, dom)
    bounds = _row_block_bounds(dom, p)
    parts = [dom[bounds[i]: bounds[i + 1]] for i in range(p)]
    jobs = [(spectra, order, m3, conj, part) for part in parts if len(part)]
    import multiprocessing as mp

    with ProcessPoolExecutor(max_workers=p, mp_context=mp.get_context("spawn")) as pool:
        vals = list(pool.map(_worker, jobs))
    return np.concatenate(vals) if vals else np.empty(0, np.complex128)


# ---------------------------------------------------------------------------
# parity metric


def north_star_error(got, ref) -> float:
    """max|got - ref| / max|ref| (BASELINE.json north_star parity metric)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    if ref.size == 0:
        return 0.0
    scale = float(np.max(np.abs(ref)))
    if scale == 0.0:
        return float(np.max(np.abs(got - ref)))
    return float(np.max(np.abs(got - ref)) / scale)
