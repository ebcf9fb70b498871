"""Series container and segmentation (hospectra/series.py:29-92,159-165).

``TimeSeries`` / ``SegmentConfig`` / ``SegmentSet`` keep the reference's
fields, validation and messages so user code and tests port unchanged.
``segment_and_demean`` is the host-side utility of the reference API; the
estimator itself segments and demeans on the GPU (kernel K0) and never
calls it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DataError, ParameterError

__all__ = ["TimeSeries", "SegmentConfig", "SegmentSet", "segment_and_demean", "load_series"]


@dataclass(frozen=True)
class TimeSeries:
    """A finite real-valued sample sequence with provenance (float64)."""

    samples: np.ndarray
    source: str = ""

    def __post_init__(self):
        samples = np.asarray(self.samples, dtype=np.float64)
        object.__setattr__(self, "samples", samples)
        if samples.ndim != 1 or samples.size < 1:
            raise ParameterError("a time series needs at least one sample")
        finite = np.isfinite(samples)
        if not finite.all():
            raise DataError(f"non-finite sample at index {int(np.argmin(finite))}")

    @property
    def n(self) -> int:
        return int(self.samples.size)


@dataclass(frozen=True)
class SegmentConfig:
    """``k`` segments of ``m`` samples each."""

    m: int
    k: int = 1

    def __post_init__(self):
        if self.m < 1 or self.k < 1:
            raise ParameterError(
                f"segment length and count must be positive, got m={self.m}, k={self.k}")

    def validate_for(self, series) -> None:
        n = series.n if hasattr(series, "n") else int(np.asarray(series).shape[-1])
        if self.k * self.m > n:
            raise ParameterError(
                f"k*m = {self.k}*{self.m} = {self.k * self.m} exceeds series length n = {n}")


@dataclass(frozen=True)
class SegmentSet:
    """``k`` contiguous segments of ``m`` samples, optionally demeaned."""

    segments: np.ndarray  # (k, m)
    means_removed: bool = False

    @property
    def k(self) -> int:
        return int(self.segments.shape[0])

    @property
    def m(self) -> int:
        return int(self.segments.shape[1])


def segment_and_demean(series: TimeSeries, cfg: SegmentConfig) -> SegmentSet:
    """First k*m samples as (k, m) rows, each minus its own mean."""
    cfg.validate_for(series)
    rows = series.samples[: cfg.k * cfg.m].reshape(cfg.k, cfg.m).copy()
    rows -= rows.mean(axis=1, keepdims=True)
    return SegmentSet(segments=rows, means_removed=True)


def save_series(series: TimeSeries, path, fmt: str = "csv") -> None:
    """Write a series in a format ``load_series`` reads back exactly
    (hospectra/series.py:146-156): csv = one ``%.17g`` value per line, raw64
    = little-endian float64."""
    path = str(path)
    samples = np.asarray(series.samples, dtype=np.float64)
    if fmt == "csv":
        with open(path, "w", encoding="utf-8") as fh:
            for value in samples:
                fh.write(f"{value:.17g}\n")
    elif fmt == "raw64":
        samples.astype("<f8").tofile(path)
    else:
        raise ParameterError(f"unknown format {fmt!r}; expected csv or raw64")


def load_series(path, fmt: str = "csv") -> TimeSeries:
    """Read a series file in the reference's interchange formats
    (hospectra/series.py:95-140): ``csv`` = one decimal value per line, blank
    lines skipped, an optional single non-numeric header line; ``raw64`` =
    consecutive little-endian IEEE-754 float64 values.  Unreadable, empty,
    malformed or non-finite input raises DataError (with file:line for csv)."""
    path = str(path)
    if fmt not in ("csv", "raw64"):
        raise ParameterError(f"unknown series format {fmt!r} (csv or raw64)")
    try:
        data = open(path, "rb").read()
    except OSError as exc:
        raise DataError(f"cannot read {path}: {exc}") from exc
    if fmt == "raw64":
        if len(data) % 8:
            raise DataError(f"{path}: raw64 size {len(data)} is not a multiple of 8 bytes")
        vals = np.frombuffer(data, dtype="<f8").astype(np.float64)
        if vals.size == 0:
            raise DataError(f"{path}: empty input")
        bad = ~np.isfinite(vals)
        if bad.any():
            raise DataError(f"{path}: non-finite value at index {int(np.argmax(bad))}")
        return TimeSeries(vals, source=path)
    out = []
    for no, raw in enumerate(data.decode("utf-8").splitlines(), start=1):
        tok = raw.strip()
        if not tok:
            continue
        try:
            v = float(tok)
        except ValueError:
            if no == 1:
                continue  # header
            raise DataError(f"{path}:{no}: non-numeric value {tok!r}") from None
        if not np.isfinite(v):
            raise DataError(f"{path}:{no}: non-finite value {tok!r}")
        out.append(v)
    if not out:
        raise DataError(f"{path}: empty input")
    return TimeSeries(np.asarray(out, dtype=np.float64), source=path)
