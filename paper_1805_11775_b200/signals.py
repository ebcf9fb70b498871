"""Seeded synthetic series for the BASELINE.json configurations.

BASELINE.json gives the signal formulas but no seeds; the seeds and the
draw order are pinned here: one
``numpy.random.default_rng(seed)`` per configuration (PCG64, platform
independent), phases drawn first, then the noise, in time order.

Also restates the two generators the reference itself ships,
``generate_qpc`` (hospectra/series.py:168-201) and ``generate_gaussian_ar``
(hospectra/series.py:204-237), with the same draw order so a given seed
yields the same samples.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ParameterError
from .series import TimeSeries

__all__ = [
    "BaselineConfig",
    "BASELINE_CONFIGS",
    "baseline_config",
    "baseline_series",
    "generate_qpc",
    "generate_gaussian_ar",
]


@dataclass(frozen=True)
class BaselineConfig:
    name: str
    order: int
    n: int          # samples per series
    m: int          # segment length M
    k: int          # segments K
    m3: int         # smoothing window side w = 2L+1
    dtype: str      # sample dtype handed to the estimator
    batch: int = 1  # independent series
    seed: int = 0
    taper: str | None = "hann"


#: The five BASELINE.json configurations, in file order.
BASELINE_CONFIGS = (
    BaselineConfig("cfg1_qpc", 3, 2048, 128, 16, 5, "float64", 1, 180511775),
    BaselineConfig("cfg2_bilinear", 3, 1 << 20, 1024, 1024, 9, "float32", 1, 180511776),
    BaselineConfig("cfg3_machinery", 3, 9_216_000, 4096, 2250, 17, "float32", 1, 180511777),
    BaselineConfig("cfg4_cubic_qpc", 4, 1 << 18, 256, 1024, 5, "float32", 1, 180511778),
    BaselineConfig("cfg5_returns", 3, 19_968, 256, 78, 7, "float32", 4096, 180511779),
)


def baseline_config(name: str) -> BaselineConfig:
    for c in BASELINE_CONFIGS:
        if c.name == name or c.name.split("_")[0] == name:
            return c
    raise ParameterError(f"unknown baseline config {name!r}")


def _qpc_small(rng, n):
    # x(i)=cos(2pi.1i+p1)+cos(2pi.15i+p2)+0.5cos(2pi.25i+p1+p2)+N(0,.5^2)
    p1, p2 = rng.uniform(0.0, 2.0 * np.pi, size=2)
    i = np.arange(n, dtype=np.float64)
    x = (np.cos(2 * np.pi * 0.10 * i + p1) + np.cos(2 * np.pi * 0.15 * i + p2)
         + 0.5 * np.cos(2 * np.pi * 0.25 * i + p1 + p2))
    return x + rng.normal(0.0, 0.5, size=n)


def _bilinear(rng, n):
    # x_t = e_t + 0.4 e_{t-1} e_{t-2}, e ~ N(0,1) iid, mean removed
    e = rng.standard_normal(n + 2)
    x = e[2:] + 0.4 * e[1:-1] * e[:-2]
    return x - x.mean()


def _machinery(rng, n):
    # fs = 2560 Hz; 25/50/75 Hz harmonics, amplitudes 1/.6/.3, phi3 = phi1+phi2, N(0,1)
    p1, p2 = rng.uniform(0.0, 2.0 * np.pi, size=2)
    t = np.arange(n, dtype=np.float64) / 2560.0
    x = (np.cos(2 * np.pi * 25 * t + p1) + 0.6 * np.cos(2 * np.pi * 50 * t + p2)
         + 0.3 * np.cos(2 * np.pi * 75 * t + p1 + p2))
    return x + rng.standard_normal(n)


def _cubic_qpc(rng, n):
    # cos at .05/.08/.11 with random phases + .5 cos(2pi .24 i + sum phases) + N(0,.5^2)
    ph = rng.uniform(0.0, 2.0 * np.pi, size=3)
    i = np.arange(n, dtype=np.float64)
    x = sum(np.cos(2 * np.pi * f * i + p) for f, p in zip((0.05, 0.08, 0.11), ph))
    x = x + 0.5 * np.cos(2 * np.pi * 0.24 * i + ph.sum())
    return x + rng.normal(0.0, 0.5, size=n)


def _returns(rng, n, batch):
    # x_t = e_t + 0.3 (e_{t-1}^2 - 1), e Student-t nu=4 scaled to unit variance;
    # series drawn one after another from the same generator
    out = np.empty((batch, n), dtype=np.float64)
    scale = 1.0 / math.sqrt(2.0)  # var(t_4) = 2
    for b in range(batch):
        e = rng.standard_t(4.0, size=n + 1) * scale
        out[b] = e[1:] + 0.3 * (e[:-1] ** 2 - 1.0)
    return out


def baseline_series(cfg: BaselineConfig | str, batch: int | None = None) -> np.ndarray:
    """Samples for a BASELINE config: shape (n,) or (batch, n), in the
    config's dtype.  ``batch`` truncates cfg5 to its first series (same
    samples as the full draw, since series are drawn in order)."""
    if isinstance(cfg, str):
        cfg = baseline_config(cfg)
    rng = np.random.default_rng(cfg.seed)
    kind = cfg.name.split("_", 1)[1]
    if kind == "qpc":
        x = _qpc_small(rng, cfg.n)
    elif kind == "bilinear":
        x = _bilinear(rng, cfg.n)
    elif kind == "machinery":
        x = _machinery(rng, cfg.n)
    elif kind == "cubic_qpc":
        x = _cubic_qpc(rng, cfg.n)
    else:
        x = _returns(rng, cfg.n, cfg.batch if batch is None else batch)
    return np.ascontiguousarray(x.astype(cfg.dtype))


# ---------------------------------------------------------------------------
# the reference's own generators (same draw order, same samples)


def generate_qpc(f1: float, f2: float, n: int, noise_sigma: float = 0.0, seed: int = 0) -> TimeSeries:
    """Three cosines at f1, f2, f1+f2 with the third phase locked to the
    sum of the first two, plus white Gaussian noise
    (hospectra/series.py:168-201)."""
    if not (0.0 < f1 and 0.0 < f2 and f1 + f2 < 0.5):
        raise ParameterError(f"need 0 < f1, f2 and f1+f2 < 0.5, got f1={f1}, f2={f2}")
    if noise_sigma < 0.0:
        raise ParameterError(f"noise_sigma must be >= 0, got {noise_sigma}")
    if n < 1:
        raise ParameterError(f"n must be >= 1, got {n}")
    rng = np.random.default_rng(seed)
    p1, p2 = rng.uniform(0.0, 2.0 * np.pi, size=2)
    t = np.arange(n, dtype=np.float64)
    x = (np.cos(2.0 * np.pi * f1 * t + p1) + np.cos(2.0 * np.pi * f2 * t + p2)
         + np.cos(2.0 * np.pi * (f1 + f2) * t + p1 + p2))
    if noise_sigma > 0:
        x = x + rng.normal(0.0, noise_sigma, size=n)
    return TimeSeries(x, source=f"qpc(f1={f1},f2={f2},n={n},sigma={noise_sigma},seed={seed})")


def generate_gaussian_ar(coeffs, n: int, seed: int = 0) -> TimeSeries:
    """Stable AR(p) driven by standard Gaussian noise, burn-in 10p
    (hospectra/series.py:204-237)."""
    a = np.asarray(list(coeffs), dtype=np.float64)
    if n < 1:
        raise ParameterError(f"n must be >= 1, got {n}")
    p = a.size
    if p:
        roots = np.roots(np.concatenate([[1.0], -a]))
        worst = float(np.max(np.abs(roots)))
        if worst >= 1.0:
            raise ParameterError(
                f"unstable AR coefficients: characteristic root magnitude {worst:.6g} >= 1")
    rng = np.random.default_rng(seed)
    burn = 10 * p
    eps = rng.standard_normal(n + burn)
    x = eps.copy() if p == 0 else np.empty(n + burn)
    if p:
        for t in range(n + burn):
            acc = eps[t]
            for j in range(min(p, t)):
                acc += a[j] * x[t - j - 1]
            x[t] = acc
    return TimeSeries(x[burn:].copy(), source=f"ar(coeffs={a.tolist()},n={n},seed={seed})")
