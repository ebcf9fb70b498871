"""Series file formats and the ``estimate`` command line (ports of
hospectra tests/test_series.py load_series cases and tests/test_cli.py
argument checks; the GPU run itself is in the -m gpu part)."""

import csv
import os
import struct

import numpy as np
import pytest

from oracle import hos_oracle as O
from paper_1805_11775_b200 import DataError, ParameterError, load_series
from paper_1805_11775_b200 import cli


def test_load_series_csv(tmp_path):
    p = tmp_path / "x.csv"
    p.write_text("value\n1.5\n\n-2\n3e-1\n")
    s = load_series(p)
    assert np.array_equal(s.samples, [1.5, -2.0, 0.3]) and s.source == str(p)
    p.write_text("1\nabc\n")
    with pytest.raises(DataError, match=r"x.csv:2: non-numeric"):
        load_series(p)
    p.write_text("1\nnan\n")
    with pytest.raises(DataError, match="non-finite"):
        load_series(p)
    p.write_text("\n\n")
    with pytest.raises(DataError, match="empty"):
        load_series(p)
    with pytest.raises(DataError, match="cannot read"):
        load_series(tmp_path / "missing.csv")


def test_load_series_raw64(tmp_path):
    p = tmp_path / "x.bin"
    vals = [0.25, -1.0, 3.5]
    p.write_bytes(struct.pack("<3d", *vals))
    assert np.array_equal(load_series(p, "raw64").samples, vals)
    p.write_bytes(b"\x00" * 7)
    with pytest.raises(DataError, match="multiple of 8"):
        load_series(p, "raw64")
    p.write_bytes(struct.pack("<2d", 1.0, float("inf")))
    with pytest.raises(DataError, match="non-finite"):
        load_series(p, "raw64")
    with pytest.raises(ParameterError):
        load_series(p, "json")


def test_cli_validation_exit_codes(tmp_path, capsys):
    x = tmp_path / "x.csv"
    x.write_text("\n".join(str(v) for v in np.arange(64.0)))
    out = tmp_path / "g.csv"
    base = ["estimate", "--input", str(x), "--out", str(out)]
    assert cli.main(base + ["--seg-len", "32", "--window", "16"]) == 2
    assert "window < seg-len/2" in capsys.readouterr().err
    assert cli.main(base + ["--seg-len", "32", "--segments", "3", "--window", "5"]) == 2
    assert "exceeds series length 64" in capsys.readouterr().err
    assert cli.main(base + ["--seg-len", "32", "--window", "5", "--device", "tpu"]) == 2
    assert cli.main(["estimate", "--input", str(tmp_path / "nope.csv"), "--out", str(out), "--seg-len", "32",
                     "--window", "5"]) == 1
    assert not out.exists()


@pytest.mark.gpu
def test_cli_estimate_gpu(cuda, tmp_path):
    rng = np.random.default_rng(7)
    x = rng.standard_normal(128 * 6)
    src = tmp_path / "x.csv"
    src.write_text("\n".join(repr(float(v)) for v in x))
    out = tmp_path / "g.csv"
    assert cli.main(["estimate", "--input", str(src), "--seg-len", "128", "--segments", "6", "--window", "5",
                     "--out", str(out), "--device", "cuda:0", "--threads", "3"]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["k1", "k2", "re", "im"]
    dom, ref = O.estimate(x, 3, 128, 6, 5, True, None)
    got = np.array([complex(float(r[2]), float(r[3])) for r in rows[1:]])
    assert np.array_equal(np.array([[int(r[0]), int(r[1])] for r in rows[1:]]), dom)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.abs(ref).max()
