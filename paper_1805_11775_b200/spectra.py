"""Bispectrum / trispectrum estimation on the B200 (drop-in for
hospectra/spectra.py).

Same names, signatures, validation messages and output container as the
reference; the values come from the GPU pipeline of ``libhos_b200.so``:
segment + demean (+ taper) -> cuFFT -> FFMA2 triple/quad products over
the dilated principal domain -> fp64 per-line prefix scans -> box
differences -> lexicographic principal-domain values.

Extensions (keyword-only): ``EstimationConfig.precision``
("fp64" default for parity, "fp32" for throughput), ``EstimationConfig.taper``
(None | "hann"), ``device=`` on the estimators, ``estimate_batch`` for many
independent series, and CUDA-tensor series for device-resident inputs.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from ._native import _torch, domain_indices, domain_size, get_plan
from .dft import SegmentSpectrumSet
from .errors import ParameterError
from .series import SegmentConfig, TimeSeries
from .window_sums import SmoothingPlan

__all__ = [
    "EstimationConfig",
    "SpectrumPoint",
    "SpectrumGrid",
    "raw_bispectrum_value",
    "raw_trispectrum_value",
    "principal_domain",
    "domain_slice",
    "estimate_spectrum",
    "estimate_from_spectra",
    "estimate_batch",
    "compare_grids",
    "write_grid_csv",
]

_PRECISIONS = {"fp32": 32, "fp64": 64, 32: 32, 64: 64}


class SpectrumPoint(NamedTuple):
    """One principal-domain point: frequency-bin index tuple and value."""

    k: tuple
    value: complex


@dataclass(frozen=True)
class EstimationConfig:
    """Everything needed to turn a series into a smoothed spectrum
    (hospectra/spectra.py:60-79) plus the GPU extensions."""

    order: int
    segment: SegmentConfig
    m3: int
    plan: SmoothingPlan = SmoothingPlan.EFFICIENT
    conjugate_last: bool = True
    precision: str = field(default="fp64", kw_only=True)
    taper: str | None = field(default=None, kw_only=True)

    def __post_init__(self):
        if self.order not in (3, 4):
            raise ParameterError(f"order must be 3 or 4, got {self.order}")
        if self.m3 < 1:
            raise ParameterError(f"smoothing window must be >= 1, got {self.m3}")
        if 2 * self.m3 >= self.segment.m:
            raise ParameterError(
                f"smoothing window {self.m3} must satisfy m3 < m/2 "
                f"(segment length m = {self.segment.m})")
        if self.precision not in _PRECISIONS:
            raise ParameterError(f"precision must be 'fp32' or 'fp64', got {self.precision!r}")
        if self.taper not in (None, "hann"):
            raise ParameterError(f"taper must be None or 'hann', got {self.taper!r}")
        if not isinstance(self.plan, SmoothingPlan):
            raise ParameterError(f"plan must be a SmoothingPlan, got {self.plan!r}")

    @property
    def bits(self) -> int:
        return _PRECISIONS[self.precision]


@dataclass
class SpectrumGrid:
    """Smoothed estimate over the principal domain, parallel arrays in
    lexicographic order (hospectra/spectra.py:82-108)."""

    order: int
    m: int
    m3: int
    plan: SmoothingPlan
    indices: np.ndarray  # (npoints, order-1) int32
    values: np.ndarray   # (npoints,) complex128

    def point_dict(self) -> dict:
        return {tuple(int(v) for v in idx): val for idx, val in zip(self.indices, self.values)}

    def points(self):
        for idx, val in zip(self.indices, self.values):
            yield SpectrumPoint(tuple(int(v) for v in idx), complex(val))

    def peak_point(self) -> SpectrumPoint:
        t = int(np.argmax(np.abs(self.values)))
        return SpectrumPoint(tuple(int(v) for v in self.indices[t]), complex(self.values[t]))


def raw_bispectrum_value(f, k1: int, k2: int, conjugate_last: bool = True) -> complex:
    """``f[k1] f[k2] conj(f[(k1+k2) % m]) / m`` for one spectrum
    (hospectra/spectra.py:111-120)."""
    f = np.asarray(f)
    m = f.size
    last = f[(int(k1) + int(k2)) % m]
    if conjugate_last:
        last = np.conj(last)
    return complex(f[int(k1)] * f[int(k2)] * last / m)


def raw_trispectrum_value(f, k1: int, k2: int, k3: int, conjugate_last: bool = True) -> complex:
    """Fourth-order analogue (hospectra/spectra.py:123-130)."""
    f = np.asarray(f)
    m = f.size
    last = f[(int(k1) + int(k2) + int(k3)) % m]
    if conjugate_last:
        last = np.conj(last)
    return complex(f[int(k1)] * f[int(k2)] * f[int(k3)] * last / m)


def principal_domain(order: int, m: int) -> np.ndarray:
    """Lexicographic principal-domain tuples, int32 (npoints, order-1)
    (hospectra/spectra.py:133-168); enumerated by the library's closed-form
    row lengths."""
    if order not in (3, 4):
        raise ParameterError(f"order must be 3 or 4, got {order}")
    if m < 2:
        raise ParameterError(f"segment length must be >= 2, got {m}")
    return domain_indices(order, m, 0, domain_size(order, m))


def domain_slice(order: int, m: int, start: int, stop: int) -> np.ndarray:
    """``principal_domain(order, m)[start:stop]`` without building the whole
    domain (hospectra/spectra.py:171-196)."""
    if stop <= start:
        return np.empty((0, order - 1), dtype=np.int32)
    total = domain_size(order, m)
    if not (0 <= start < stop <= total):
        raise ParameterError(f"slice [{start}, {stop}) outside domain of size {total}")
    return domain_indices(order, m, start, stop)


def _plan_for(cfg: EstimationConfig, batch: int = 1, device=None):
    return get_plan(cfg.order, cfg.segment.m, cfg.segment.k, cfg.m3, cfg.conjugate_last, cfg.bits,
                    cfg.taper, batch, device)


def _grid(cfg: EstimationConfig, m: int, values: np.ndarray) -> SpectrumGrid:
    return SpectrumGrid(order=cfg.order, m=m, m3=cfg.m3, plan=cfg.plan,
                        indices=principal_domain(cfg.order, m), values=values)


def _to_host_c128(t) -> np.ndarray:
    return t.cpu().numpy().astype(np.complex128, copy=False)


def estimate_from_spectra(spec_set: SegmentSpectrumSet, cfg: EstimationConfig, *, device=None) -> SpectrumGrid:
    """Smoothing and averaging on precomputed segment DFTs
    (hospectra/spectra.py:419-431)."""
    if cfg.segment.m != spec_set.m or cfg.segment.k != spec_set.k:
        raise ParameterError(
            f"config ({cfg.segment.k}x{cfg.segment.m}) does not match "
            f"spectra ({spec_set.k}x{spec_set.m})")
    torch = _torch()
    plan = _plan_for(cfg, 1, device)
    cd = torch.complex64 if cfg.bits == 32 else torch.complex128
    spec = torch.as_tensor(np.ascontiguousarray(spec_set.spectra), device=f"cuda:{plan.device}").to(cd)
    out = plan.estimate_from_spectra(spec)
    return _grid(cfg, spec_set.m, _to_host_c128(out))


def estimate_spectrum(series, cfg: EstimationConfig, *, device=None) -> SpectrumGrid:
    """The direct method end to end (hospectra/spectra.py:434-439).

    ``series`` is a ``TimeSeries`` (host float64, the reference contract) or a
    1-D CUDA tensor (float32/float64) already resident on the device."""
    torch = _torch()
    if isinstance(series, TimeSeries):
        cfg.segment.validate_for(series)
        plan = _plan_for(cfg, 1, device)
        km = cfg.segment.k * cfg.segment.m
        x = torch.from_numpy(series.samples[:km]).to(f"cuda:{plan.device}")
    elif isinstance(series, torch.Tensor):
        if series.dim() != 1:
            raise ParameterError("a device series must be a 1-D tensor")
        cfg.segment.validate_for(np.empty(series.shape[0]))
        plan = _plan_for(cfg, 1, series.device.index if device is None else device)
        x = series
    else:
        raise ParameterError("series must be a TimeSeries or a CUDA tensor")
    out = plan.estimate(x)
    return _grid(cfg, cfg.segment.m, _to_host_c128(out))


def estimate_batch(x, cfg: EstimationConfig, *, device=None, to_host: bool = True):
    """Independent estimates of ``batch`` series (rows of ``x``: numpy
    (batch, n) or a CUDA tensor).  Returns (batch, npoints) values (host
    complex128 by default, or the device tensor with ``to_host=False``)."""
    torch = _torch()
    if isinstance(x, np.ndarray):
        if x.ndim != 2:
            raise ParameterError("batched series must be 2-D (batch, n)")
        cfg.segment.validate_for(np.empty(x.shape[1]))
        plan = _plan_for(cfg, x.shape[0], device)
        xt = torch.from_numpy(np.ascontiguousarray(x)).to(f"cuda:{plan.device}")
    else:
        if x.dim() != 2:
            raise ParameterError("batched series must be 2-D (batch, n)")
        cfg.segment.validate_for(np.empty(x.shape[1]))
        plan = _plan_for(cfg, x.shape[0], x.device.index if device is None else device)
        xt = x
    out = plan.estimate(xt).reshape(xt.shape[0], plan.npoints)  # (batch, npoints) for batch 1 too
    return _to_host_c128(out) if to_host else out


def compare_grids(a: SpectrumGrid, b: SpectrumGrid) -> float:
    """``max |a-b| / max(|a|, |b|, 1e-12)`` over the same domain
    (hospectra/spectra.py:442-453)."""
    if (a.order, a.m, a.m3) != (b.order, b.m, b.m3) or a.values.shape != b.values.shape:
        raise ParameterError(
            f"grid mismatch: ({a.order},{a.m},{a.m3},{a.values.shape}) vs "
            f"({b.order},{b.m},{b.m3},{b.values.shape})")
    if a.values.size == 0:
        return 0.0
    denom = np.maximum(np.maximum(np.abs(a.values), np.abs(b.values)), 1e-12)
    return float(np.max(np.abs(a.values - b.values) / denom))


def write_grid_csv(grid: SpectrumGrid, path) -> None:
    """Interchange format: header ``k1,k2[,k3],re,im``, one point per row in
    lexicographic order, 17 significant digits (hospectra/spectra.py:456-464)."""
    names = ["k1", "k2"] if grid.order == 3 else ["k1", "k2", "k3"]
    with open(str(path), "w", encoding="utf-8") as fh:
        fh.write(",".join(names + ["re", "im"]) + "\n")
        for idx, val in zip(grid.indices, grid.values):
            bins = ",".join(str(int(v)) for v in idx)
            fh.write(f"{bins},{val.real:.17g},{val.imag:.17g}\n")
