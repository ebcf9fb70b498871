"""The C-ABI library loads, exports every symbol include/hos.h declares, and its
host-only entry points (principal domain, parameter validation) behave like the
reference -- no GPU needed.  Compute calls are covered by the -m gpu suite."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import hos_oracle as O

HEADER = os.path.join(ROOT, "include", "hos.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hos_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__

    __graft_entry__.ensure_built()
    from paper_1805_11775_b200 import _native

    return _native.lib()


def test_header_parses():
    syms = declared_symbols()
    assert "hos_estimate" in syms and "hos_plan_create" in syms and len(syms) >= 25


def test_every_declared_symbol_is_exported(lib):
    from paper_1805_11775_b200 import _native

    for name in declared_symbols():
        assert hasattr(lib, name), f"{name} declared in include/hos.h but not exported"
        assert name in _native.EXPORTED_SYMBOLS, f"{name} has no ctypes prototype"


def test_library_is_sm100a(lib):
    assert lib.hos_version().decode().endswith("sm_100a")
    so = os.path.join(ROOT, "paper_1805_11775_b200", "libhos_b200.so")
    blob = open(so, "rb").read()
    assert b"sm_100a" in blob


@pytest.mark.parametrize("order", [3, 4])
@pytest.mark.parametrize("m", [2, 3, 4, 7, 8, 16, 33, 64, 127, 256])
def test_domain_matches_oracle(lib, order, m):
    from paper_1805_11775_b200 import _native

    ref = O.principal_domain(order, m)
    assert _native.domain_size(order, m) == len(ref)
    assert np.array_equal(_native.domain_indices(order, m, 0, len(ref)), ref)


def test_domain_slice_and_errors(lib):
    from paper_1805_11775_b200 import ParameterError, domain_slice, principal_domain

    for order, m in ((3, 64), (3, 127), (4, 16)):
        dom = principal_domain(order, m)
        for a, b in ((0, len(dom)), (3, 11), (len(dom) // 2, len(dom))):
            assert np.array_equal(domain_slice(order, m, a, b), dom[a:b])
    with pytest.raises(ParameterError):
        domain_slice(3, 16, 0, 10_000)
    with pytest.raises(ParameterError, match="order must be 3 or 4"):
        principal_domain(5, 16)
    with pytest.raises(ParameterError, match="segment length must be >= 2"):
        principal_domain(3, 1)


def test_known_domains(lib):
    # hospectra tests/test_spectra.py:105-128
    from paper_1805_11775_b200 import principal_domain

    assert [tuple(p) for p in principal_domain(3, 2)] == [(0, 0)]
    assert [tuple(p) for p in principal_domain(3, 8)] == [(0, 0), (1, 0), (1, 1), (2, 0), (2, 1), (3, 0)]
    assert [tuple(p) for p in principal_domain(4, 4)] == [(0, 0, 0), (1, 0, 0)]


def _create(lib, *args):
    h = ctypes.c_void_p()
    rc = lib.hos_plan_create(ctypes.byref(h), *args)
    return rc, lib.hos_last_error().decode()


def test_plan_parameter_errors_without_gpu(lib):
    # validation happens before any device is touched; messages keep the
    # reference's fragments (hospectra/spectra.py:70-79)
    rc, msg = _create(lib, 3, 64, 2, 32, 1, 32, 0, 1, 0)
    assert rc == 1 and "m3 < m/2" in msg
    rc, msg = _create(lib, 5, 64, 2, 5, 1, 32, 0, 1, 0)
    assert rc == 1 and "order must be 3 or 4" in msg
    rc, msg = _create(lib, 3, 64, 0, 5, 1, 32, 0, 1, 0)
    assert rc == 1 and "positive" in msg
    rc, msg = _create(lib, 3, 64, 2, 5, 1, 16, 0, 1, 0)
    assert rc == 1 and "precision" in msg
    rc, msg = _create(lib, 3, 64, 2, 5, 1, 32, 7, 1, 0)
    assert rc == 1 and "taper" in msg
    rc, msg = _create(lib, 3, 64, 2, 0, 1, 32, 0, 1, 0)
    assert rc == 1 and "window" in msg


def test_estimators_fail_loudly_without_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1805_11775_b200 import EstimationConfig, SegmentConfig, TimeSeries, estimate_spectrum

    with pytest.raises(RuntimeError, match="CUDA device"):
        estimate_spectrum(TimeSeries(np.random.default_rng(0).standard_normal(128)),
                          EstimationConfig(3, SegmentConfig(m=64, k=2), 5))


SCHED_SHAPES = [
    # order, m, k, m3, precision, batch
    (3, 1024, 1024, 9, 32, 1),   # cfg2
    (3, 1024, 1024, 9, 64, 1),
    (3, 128, 16, 5, 32, 1),      # cfg1
    (3, 256, 78, 7, 32, 4096),   # cfg5
    (3, 256, 78, 7, 32, 37),     # a batch that does not divide the CTAs
    (4, 256, 1024, 5, 32, 1),    # cfg4
    (4, 64, 12, 5, 64, 3),
    (3, 512, 7, 3, 32, 1),       # fewer segments than a stage per CTA
    (3, 2048, 300, 11, 32, 1),
    (3, 4096, 2250, 17, 32, 1),  # cfg3: k_triple_w (not eligible)
    (3, 100, 50, 5, 32, 2),      # non-power-of-two M
]


@pytest.mark.parametrize("shape", SCHED_SHAPES, ids=lambda s: "o%d_m%d_k%d_w%d_p%d_b%d" % s)
@pytest.mark.parametrize("sms", [148, 132, 7])
@pytest.mark.parametrize("interleave", [0, 1])
def test_cta_schedule_covers_every_segment_once(lib, shape, sms, interleave):
    """hos_cta_schedule_check builds the k_triple_cta schedule on the host
    (no GPU) and verifies coverage, stage bounds, warp roles and partial-slot
    bookkeeping; here also the balance of the per-CTA stage counts."""
    import ctypes

    order, m, k, m3, prec, batch = shape
    if interleave and batch != 1:
        pytest.skip("the streaming schedule is for single series")
    stats = (ctypes.c_int64 * 12)()
    rc = lib.hos_cta_schedule_check(order, m, k, m3, prec, batch, sms, interleave, stats)
    assert rc == 0, lib.hos_last_error().decode()
    ctas, stages, smax, smin = stats[0], stats[1], stats[2], stats[3]
    if m == 4096:
        assert ctas == 0  # four whole rows per ring slot do not fit: per-warp staged kernel
        return
    if interleave and sms - 20 < 1:
        return
    assert 0 < ctas <= sms
    assert stats[4] >= 1 and stats[5] in (2, 4) and stats[6] >= 2
    groups = stats[7]
    assert stages >= batch * groups * -(-k // stats[10])  # each (series, group) needs ceil(k/4) stages at least
    assert smin >= 1 and smax >= smin
