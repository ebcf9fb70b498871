"""Command line: ``estimate`` on the GPU.

Mirrors the reference's ``hospectra estimate`` (hospectra/cli.py:39-50,83-111):
same flags, validation messages and exit codes (0 success, 2 configuration
error, 1 I/O error), writing the same CSV grid (``write_grid_csv``).  Extra
flags: ``--device cuda[:N]`` (the GPU the estimate runs on), ``--precision
fp64|fp32`` and ``--taper none|hann``.  ``--threads`` / ``HOSPECTRA_THREADS``
are accepted for drop-in compatibility; on one GPU the result does not
depend on them (parallel_estimate is worker-count invariant).

    python -m paper_1805_11775_b200.cli estimate --input x.csv --seg-len 1024 \\
        --segments 1024 --window 9 --out grid.csv --device cuda:0 --precision fp32
"""

from __future__ import annotations

import argparse
import os
import sys

from .errors import DataError, ParameterError
from .parallel import WorkerConfig, parallel_estimate
from .series import SegmentConfig, load_series
from .spectra import EstimationConfig, write_grid_csv
from .window_sums import SmoothingPlan

PLAN_NAMES = [p.name for p in SmoothingPlan]


def _threads_default() -> int:
    try:
        return max(1, int(os.environ.get("HOSPECTRA_THREADS", "1")))
    except ValueError:
        return 1


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1805_11775_b200",
                                 description="GPU higher-order spectrum estimation (bispectrum/trispectrum).")
    sub = ap.add_subparsers(dest="command", required=True)
    est = sub.add_parser("estimate", help="estimate a spectrum from a series file")
    est.add_argument("--order", type=int, choices=(3, 4), default=3)
    est.add_argument("--input", required=True)
    est.add_argument("--format", choices=("csv", "raw64"), default="csv")
    est.add_argument("--seg-len", type=int, required=True, help="samples per segment (M)")
    est.add_argument("--segments", type=int, default=1, help="segment count (K)")
    est.add_argument("--window", type=int, required=True, help="smoothing window side (M3)")
    est.add_argument("--plan", choices=PLAN_NAMES, default="EFFICIENT")
    est.add_argument("--threads", type=int, default=None)
    est.add_argument("--conjugate", choices=("on", "off"), default="on")
    est.add_argument("--out", required=True)
    est.add_argument("--device", default="cuda", help="cuda or cuda:N")
    est.add_argument("--precision", choices=("fp64", "fp32"), default="fp64")
    est.add_argument("--taper", choices=("none", "hann"), default="none")
    est.set_defaults(func=cmd_estimate)
    return ap


def _device_index(text: str) -> int:
    if text == "cuda":
        return 0
    if text.startswith("cuda:") and text[5:].isdigit():
        return int(text[5:])
    raise ParameterError(f"--device must be cuda or cuda:N, got {text!r}")


def cmd_estimate(args) -> int:
    if args.seg_len < 2:
        raise ParameterError(f"--seg-len must be >= 2, got {args.seg_len}")
    if args.segments < 1:
        raise ParameterError(f"--segments must be >= 1, got {args.segments}")
    if args.window < 1 or 2 * args.window >= args.seg_len:
        raise ParameterError(f"--window {args.window} must satisfy 1 <= window < seg-len/2 "
                             f"(seg-len = {args.seg_len})")
    dev = _device_index(args.device)
    threads = args.threads if args.threads is not None else _threads_default()
    if threads < 1:
        raise ParameterError(f"--threads must be >= 1, got {threads}")
    series = load_series(args.input, args.format)
    if args.segments * args.seg_len > series.n:
        raise ParameterError(f"--segments * --seg-len = {args.segments * args.seg_len} exceeds "
                             f"series length {series.n}")
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the estimator needs a CUDA device")
    torch.cuda.set_device(dev)
    cfg = EstimationConfig(args.order, SegmentConfig(m=args.seg_len, k=args.segments), args.window,
                           plan=SmoothingPlan.parse(args.plan), conjugate_last=args.conjugate == "on",
                           precision=args.precision, taper=None if args.taper == "none" else args.taper)
    grid = parallel_estimate(series, cfg, WorkerConfig(p=threads))
    write_grid_csv(grid, args.out)
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except ParameterError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except (DataError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
