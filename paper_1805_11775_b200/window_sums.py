"""Smoothing-plan vocabulary of the reference (hospectra/window_sums.py:47-118).

The reference offers six window-sum engines that all produce the same
values; the GPU estimator has one smoothing path (per-line fp64 prefix
scans + box differences) and accepts every plan name, returning identical
values whichever is chosen.  ``WindowSpec`` keeps the
reference's validation.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from .errors import ParameterError

__all__ = ["SmoothingPlan", "WindowSpec", "MATERIALIZED_PLANS", "STREAMING_PLANS"]


class SmoothingPlan(Enum):
    """The six window-sum engines of the reference."""

    NAIVE = "NAIVE"
    WS = "WS"
    PREFIX = "PREFIX"
    FAST = "FAST"
    EFFICIENT = "EFFICIENT"
    STREAMING = "STREAMING"

    @property
    def declared_work(self) -> str:
        return _DECLARED[self][0]

    @property
    def declared_extra_memory(self) -> str:
        return _DECLARED[self][1]

    @classmethod
    def parse(cls, name: str) -> "SmoothingPlan":
        try:
            return cls[name.upper()]
        except KeyError:
            valid = ", ".join(p.name for p in cls)
            raise ParameterError(f"unknown plan {name!r}; valid plans: {valid}") from None


_DECLARED = {
    SmoothingPlan.NAIVE: ("n^2 w^2", "O(1)"),
    SmoothingPlan.WS: ("n^2", "O(n^2)"),
    SmoothingPlan.PREFIX: ("n^2", "O(n^2)"),
    SmoothingPlan.FAST: ("n^2", "O(n w)"),
    SmoothingPlan.EFFICIENT: ("n^2", "O(w^2)"),
    SmoothingPlan.STREAMING: ("n^2 w", "O(w)"),
}

MATERIALIZED_PLANS = (SmoothingPlan.NAIVE, SmoothingPlan.WS, SmoothingPlan.PREFIX)
STREAMING_PLANS = (SmoothingPlan.FAST, SmoothingPlan.EFFICIENT, SmoothingPlan.STREAMING)


@dataclass(frozen=True)
class WindowSpec:
    """Square window of side ``w`` with a boundary rule."""

    w: int
    boundary: str = "valid"

    def __post_init__(self):
        if self.w < 1:
            raise ParameterError(f"window side must be >= 1, got {self.w}")
        if self.boundary not in ("valid", "periodic"):
            raise ParameterError(f"boundary must be 'valid' or 'periodic', got {self.boundary!r}")

    def out_shape(self, rows: int, cols: int) -> tuple[int, int]:
        if self.boundary == "valid":
            if self.w > min(rows, cols):
                raise ParameterError(f"window {self.w} exceeds matrix dimensions {rows}x{cols}")
            return rows - self.w + 1, cols - self.w + 1
        return rows, cols
