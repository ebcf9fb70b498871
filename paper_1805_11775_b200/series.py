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

__all__ = ["TimeSeries", "SegmentConfig", "SegmentSet", "segment_and_demean"]


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
