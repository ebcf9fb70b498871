"""ctypes binding of libhos_b200.so (include/hos.h) and the plan cache.

The shared library is built in-tree by ``__graft_entry__.build()``.  There
is no fallback: if the library or a CUDA device is missing, every estimator
entry point raises ``RuntimeError`` naming what is missing.  PyTorch is used
only for device memory and the current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
import threading
from collections import OrderedDict

import numpy as np

from .errors import DataError, ParameterError

__all__ = ["lib", "Plan", "get_plan", "HOS_F32", "HOS_F64", "HOS_C64", "HOS_C128", "LIB_PATH",
           "EXPORTED_SYMBOLS", "raise_for", "domain_size", "domain_indices"]

HOS_OK, HOS_EPARAM, HOS_EDATA, HOS_ECUDA, HOS_ENOMEM = 0, 1, 2, 3, 4
HOS_F32, HOS_F64, HOS_C64, HOS_C128 = 0, 1, 2, 3
TAPERS = {None: 0, "none": 0, "hann": 1}

LIB_PATH = os.environ.get("HOS_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhos_b200.so")

_i, _i64, _p, _d = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
_pp = ctypes.POINTER(ctypes.c_void_p)

#: every function declared in include/hos.h with (restype, argtypes)
EXPORTED_SYMBOLS = {
    "hos_version": (ctypes.c_char_p, []),
    "hos_last_error": (ctypes.c_char_p, []),
    "hos_domain_size": (_i64, [_i, _i]),
    "hos_domain_indices": (_i, [_i, _i, _i64, _i64, _p]),
    "hos_plan_create": (_i, [_pp, _i, _i, _i, _i, _i, _i, _i, _i, _i]),
    "hos_plan_destroy": (None, [_p]),
    "hos_plan_npoints": (_i64, [_p]),
    "hos_plan_cells": (_i64, [_p]),
    "hos_plan_units": (_i64, [_p]),
    "hos_plan_issued": (_i64, [_p]),
    "hos_plan_row_len": (_i64, [_p]),
    "hos_plan_device_bytes": (ctypes.c_size_t, [_p]),
    "hos_plan_launches": (_i, [_p]),
    "hos_estimate": (_i, [_p, _p, _i, _i64, _p, _p]),
    "hos_estimate_from_spectra": (_i, [_p, _p, _i, _p, _p]),
    "hos_segment_spectra": (_i, [_p, _p, _i, _i64, _p, _p]),
    "hos_dft_rows": (_i, [_p, _i, _i, _i, _i, _p, _p]),
    "hos_estimate_host": (_i, [_p, _p, _i, _i64, _p, _p]),
    "hos_plan_lines": (_i64, [_p]),
    "hos_plan_line_starts": (_i, [_p, _p]),
    "hos_partial_raw": (_i, [_p, _p, _i, _i, _i, _p, _p]),
    "hos_smooth_raw": (_i, [_p, _p, _i64, _i, _i, _p, _p]),
    "hos_row_point_offset": (_i64, [_p, _i]),
    "hos_rows_line_range": (_i, [_p, _i, _i, _p, _p]),
    "hos_peak_fp32": (_i, [_p, _p, _p]),
    "hos_peak_fp64": (_i, [_p, _p, _p]),
    "hos_plan_set_timing": (_i, [_p, _i]),
    "hos_plan_set_stamps": (_i, [_p, _p]),
    "hos_plan_nctas": (_i, [_p]),
    "hos_plan_k2_kind": (_i, [_p]),
    "hos_plan_kernel_ms": (_i, [_p, _p, _p]),
    "hos_plan_stage_ms": (_i, [_p, _p]),
    "hos_plan_set_trace": (_i, [_p, _p]),
    "hos_comm_attach": (_i, [_p, _p, _i, _i]),
    "hos_estimate_distributed": (_i, [_p, _p, _i, _p, _p]),
    "hos_shard_layout": (_i, [_i, _i, _i, _i, _i, _p]),
    "hos_cta_schedule_check": (_i, [_i, _i, _i, _i, _i, _i, _i, _i, _p]),
    "hos_plan_time_stages": (_i, [_p, _p, _i, _i64, _p, _i, _p, _p]),
}

_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load (once) and return the CDLL; raises RuntimeError when absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"libhos_b200.so not found at {LIB_PATH}; run __graft_entry__.build() "
                    "(the estimator has no CPU fallback)")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in EXPORTED_SYMBOLS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def raise_for(rc: int) -> None:
    if rc == HOS_OK:
        return
    msg = lib().hos_last_error().decode("utf-8", "replace")
    if rc == HOS_EPARAM:
        raise ParameterError(msg)
    if rc == HOS_EDATA:
        raise DataError(msg)
    raise RuntimeError(f"libhos_b200: {msg}")


def domain_size(order: int, m: int) -> int:
    n = lib().hos_domain_size(order, m)
    if n < 0:
        if order not in (3, 4):
            raise ParameterError(f"order must be 3 or 4, got {order}")
        raise ParameterError(f"segment length must be >= 2, got {m}")
    return int(n)


def domain_indices(order: int, m: int, start: int, stop: int) -> np.ndarray:
    n = max(0, stop - start)
    out = np.empty((n, order - 1), dtype=np.int32)
    if n:
        raise_for(lib().hos_domain_indices(order, m, start, stop, out.ctypes.data))
    return out


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the HOS estimator runs on the GPU only")
    return torch


class Plan:
    """Owns one hos_plan (cuFFT plan, scratch, geometry tables)."""

    def __init__(self, order, m, k, m3, conj=True, precision=64, taper=None, batch=1, device=None):
        torch = _torch()
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self.order, self.m, self.k, self.m3 = int(order), int(m), int(k), int(m3)
        self.conj, self.precision, self.batch = bool(conj), int(precision), int(batch)
        if taper not in TAPERS:
            raise ParameterError(f"unknown taper {taper!r}; expected None or 'hann'")
        self.taper = taper
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            raise_for(lib().hos_plan_create(ctypes.byref(handle), self.order, self.m, self.k, self.m3,
                                            int(self.conj), self.precision, TAPERS[taper], self.batch,
                                            self.device))
        self.handle = handle
        L = lib()
        self.npoints = int(L.hos_plan_npoints(handle))
        self.cells = int(L.hos_plan_cells(handle))
        self.units = int(L.hos_plan_units(handle))
        self.issued = int(L.hos_plan_issued(handle))
        self.row_len = int(L.hos_plan_row_len(handle))
        self.lines = int(L.hos_plan_lines(handle))
        self.complex_dtype = torch.complex64 if self.precision == 32 else torch.complex128

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.hos_plan_destroy(h)
            self.handle = None

    # -- helpers -------------------------------------------------------------

    def _stream(self):
        torch = _torch()
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def empty_out(self):
        torch = _torch()
        shape = (self.batch, self.npoints) if self.batch > 1 else (self.npoints,)
        return torch.empty(shape, dtype=self.complex_dtype, device=f"cuda:{self.device}")

    # -- entry points ----------------------------------------------------------

    def estimate(self, x, out=None):
        """x: CUDA tensor (n,) or (batch, n) float32/float64 -> complex values."""
        torch = _torch()
        if x.device.type != "cuda":
            raise ParameterError("series tensor must live on a CUDA device")
        if x.dtype not in (torch.float32, torch.float64):
            raise ParameterError(f"series dtype must be float32 or float64, got {x.dtype}")
        if x.stride(-1) != 1:
            x = x.contiguous()
        n = x.shape[-1]
        if self.k * self.m > n:
            raise ParameterError(
                f"k*m = {self.k}*{self.m} = {self.k * self.m} exceeds series length n = {n}")
        stride = x.stride(0) if x.dim() == 2 else n
        if x.dim() == 2 and x.shape[0] != self.batch:
            raise ParameterError(f"plan batch {self.batch} != series batch {x.shape[0]}")
        if out is None:
            out = self.empty_out()
        dt = HOS_F32 if x.dtype == torch.float32 else HOS_F64
        raise_for(lib().hos_estimate(self.handle, ctypes.c_void_p(x.data_ptr()), dt, stride,
                                     ctypes.c_void_p(out.data_ptr()), self._stream()))
        return out

    def estimate_from_spectra(self, spec, out=None):
        torch = _torch()
        if spec.dtype not in (torch.complex64, torch.complex128):
            raise ParameterError(f"spectra dtype must be complex64 or complex128, got {spec.dtype}")
        spec = spec.contiguous()
        if out is None:
            out = self.empty_out()
        dt = HOS_C64 if spec.dtype == torch.complex64 else HOS_C128
        raise_for(lib().hos_estimate_from_spectra(self.handle, ctypes.c_void_p(spec.data_ptr()), dt,
                                                  ctypes.c_void_p(out.data_ptr()), self._stream()))
        return out

    def segment_spectra(self, x):
        torch = _torch()
        x = x.contiguous()
        n = x.shape[-1]
        spec = torch.empty((self.batch * self.k, self.m), dtype=self.complex_dtype, device=x.device)
        dt = HOS_F32 if x.dtype == torch.float32 else HOS_F64
        raise_for(lib().hos_segment_spectra(self.handle, ctypes.c_void_p(x.data_ptr()), dt, n,
                                            ctypes.c_void_p(spec.data_ptr()), self._stream()))
        return spec

    def estimate_host(self, x_host: np.ndarray, out_host: np.ndarray | None = None):
        """Host buffers in/out through hos_estimate_host (copies inside)."""
        if x_host.dtype not in (np.float32, np.float64):
            raise ParameterError(f"series dtype must be float32 or float64, got {x_host.dtype}")
        x_host = np.ascontiguousarray(x_host)
        if out_host is None:
            cd = np.complex64 if self.precision == 32 else np.complex128
            out_host = np.empty((self.batch, self.npoints) if self.batch > 1 else (self.npoints,), cd)
        dt = HOS_F32 if x_host.dtype == np.float32 else HOS_F64
        stride = x_host.shape[-1]
        # synchronous: the plan's private stream (no torch stream lookup on this path)
        raise_for(lib().hos_estimate_host(self.handle, x_host.ctypes.data, dt, stride,
                                          out_host.ctypes.data, None))
        return out_host

    def partial_raw(self, x, seg_begin, seg_end, raw):
        torch = _torch()
        dt = HOS_F32 if x.dtype == torch.float32 else HOS_F64
        raise_for(lib().hos_partial_raw(self.handle, ctypes.c_void_p(x.data_ptr()), dt, seg_begin, seg_end,
                                        ctypes.c_void_p(raw.data_ptr()), self._stream()))
        return raw

    def smooth_raw(self, raw, line_begin, row_begin, row_end, out):
        raise_for(lib().hos_smooth_raw(self.handle, ctypes.c_void_p(raw.data_ptr()), int(line_begin),
                                       int(row_begin), int(row_end), ctypes.c_void_p(out.data_ptr()),
                                       self._stream()))
        return out

    def line_starts(self) -> np.ndarray:
        ls = np.empty(self.lines + 1, dtype=np.int64)
        raise_for(lib().hos_plan_line_starts(self.handle, ls.ctypes.data))
        return ls

    def rows_line_range(self, r0, r1):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        raise_for(lib().hos_rows_line_range(self.handle, r0, r1, ctypes.byref(a), ctypes.byref(b)))
        return int(a.value), int(b.value)

    def row_point_offset(self, row):
        return int(lib().hos_row_point_offset(self.handle, row))

    def set_timing(self, on: bool):
        raise_for(lib().hos_plan_set_timing(self.handle, int(on)))

    def set_stamps(self, buf):
        """In-step kernel stamps into a (16, 192) int64 CUDA tensor (None: off)."""
        raise_for(lib().hos_plan_set_stamps(self.handle, ctypes.c_void_p(buf.data_ptr() if buf is not None else 0)))

    def stage_ms(self):
        out = (ctypes.c_double * 6)()
        raise_for(lib().hos_plan_stage_ms(self.handle, out))
        return dict(zip(("prep", "fft", "extend", "triple", "scan", "box"), list(out)))

    def time_stages(self, x, reps=20, out=None):
        """Mean per-launch device ms of each stage over `reps` back-to-back
        launches (after one full estimate of x; x as in estimate())."""
        torch = _torch()
        if out is None:
            out = self.empty_out()
        n = x.shape[-1]
        stride = x.stride(0) if x.dim() == 2 else n
        dt = HOS_F32 if x.dtype == torch.float32 else HOS_F64
        res = (ctypes.c_double * 6)()
        raise_for(lib().hos_plan_time_stages(self.handle, ctypes.c_void_p(x.data_ptr()), dt, stride,
                                             ctypes.c_void_p(out.data_ptr()), reps, res, self._stream()))
        return dict(zip(("prep", "fft", "extend", "triple", "scan", "box"), list(res)))

    def comm_attach(self, nccl_comm: int, rank: int, nranks: int):
        """Attach an NCCL communicator (ncclComm_t as an int) of `nranks` ranks."""
        raise_for(lib().hos_comm_attach(self.handle, ctypes.c_void_p(nccl_comm), rank, nranks))

    def estimate_distributed(self, x, out=None):
        """Segment-sharded estimate of one series over the attached
        communicator; x: the full series (CUDA tensor) on every rank."""
        torch = _torch()
        if out is None:
            out = self.empty_out()
        dt = HOS_F32 if x.dtype == torch.float32 else HOS_F64
        raise_for(lib().hos_estimate_distributed(self.handle, ctypes.c_void_p(x.data_ptr()), dt,
                                                 ctypes.c_void_p(out.data_ptr()), self._stream()))
        return out

    def kernel_ms(self):
        t, tot = ctypes.c_double(), ctypes.c_double()
        raise_for(lib().hos_plan_kernel_ms(self.handle, ctypes.byref(t), ctypes.byref(tot)))
        return float(t.value), float(tot.value)


def shard_layout_native(order: int, m: int, k: int, m3: int, nranks: int):
    """hos_shard_layout as (per-rank rows of 14, (block, halo, in_next))."""
    import numpy as np

    out = np.zeros(14 * nranks + 3, dtype=np.int64)
    raise_for(lib().hos_shard_layout(order, m, k, m3, nranks, out.ctypes.data_as(ctypes.c_void_p)))
    return out[:14 * nranks].reshape(nranks, 14), tuple(int(v) for v in out[14 * nranks:])


def dft_rows(x, m: int, precision: int = 64):
    """Full complex spectra of the rows of a CUDA tensor x (rows*m reals)."""
    torch = _torch()
    x = x.contiguous()
    rows = x.numel() // m
    cd = torch.complex64 if precision == 32 else torch.complex128
    spec = torch.empty((rows, m), dtype=cd, device=x.device)
    dt = HOS_F32 if x.dtype == torch.float32 else HOS_F64
    with torch.cuda.device(x.device):
        stream = ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
        raise_for(lib().hos_dft_rows(ctypes.c_void_p(x.data_ptr()), dt, rows, m, precision,
                                     ctypes.c_void_p(spec.data_ptr()), stream))
    return spec


_plans: "OrderedDict[tuple, Plan]" = OrderedDict()
_plans_lock = threading.Lock()
_MAX_PLANS = 16


def get_plan(order, m, k, m3, conj=True, precision=64, taper=None, batch=1, device=None) -> Plan:
    """Cached plan for a configuration (LRU of 16)."""
    torch = _torch()
    if device is None:
        device = torch.cuda.current_device()
    key = (int(order), int(m), int(k), int(m3), bool(conj), int(precision), taper, int(batch), int(device))
    with _plans_lock:
        plan = _plans.get(key)
        if plan is not None:
            _plans.move_to_end(key)
            return plan
    plan = Plan(*key)
    with _plans_lock:
        _plans[key] = plan
        while len(_plans) > _MAX_PLANS:
            _plans.popitem(last=False)
    return plan
