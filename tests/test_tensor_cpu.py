"""The .mosst format and seeded generation (paper_2511_05811_b200.tensor) vs
the reference (tensor.py:1-144): golden bytes, tensor_randn streams generated
by the reference itself (tests/golden/make_cli_golden.py), error classes."""

import os

import numpy as np
import pytest

from paper_2511_05811_b200 import errors
from paper_2511_05811_b200.tensor import DType, tensor_randn, tensor_read, tensor_write

HERE = os.path.dirname(os.path.abspath(__file__))

# test_tensor.py:13-18: tensor_write of E8M0 codes [[0,118,127],[128,254,1]], frozen bytes
GOLDEN_E8M0 = (b"MOSSTNSR\x01\x03\x02\x00\x00\x00\x02\x00\x00\x00\x00\x00\x00\x00"
               b"\x03\x00\x00\x00\x00\x00\x00\x00\x00v\x7f\x80\xfe\x01")


def test_golden_bytes(tmp_path):
    p = tmp_path / "c.mosst"
    tensor_write(np.array([[0, 118, 127], [128, 254, 1]], np.uint8), p, DType.E8M0)
    assert p.read_bytes() == GOLDEN_E8M0
    arr, tag = tensor_read(p)
    assert tag == DType.E8M0 and arr.tolist() == [[0, 118, 127], [128, 254, 1]]


def test_randn_matches_reference_streams():
    gold = np.load(os.path.join(HERE, "golden", "tensor_golden.npz"))
    cases = {"g_4": ([4], 7, "gaussian"), "g_3x5": ([3, 5], 11, "gaussian"), "l_64": ([64], 3, "laplace"),
             "o_32x64": ([32, 64], 5, "outlier_injected")}
    for name, (shape, seed, dist) in cases.items():
        got = tensor_randn(shape, seed=seed, dist=dist)
        assert got.dtype == np.float32 and np.array_equal(got, gold[name]), name


def test_reference_input_file_roundtrip(tmp_path):
    x, tag = tensor_read(os.path.join(HERE, "golden", "cli", "x.mosst"))
    assert tag == DType.F32 and x.shape == (64, 256)
    assert np.array_equal(x, tensor_randn([64, 256], seed=5, dist="outlier_injected"))
    p = tmp_path / "x.mosst"
    tensor_write(x, p)
    assert p.read_bytes() == open(os.path.join(HERE, "golden", "cli", "x.mosst"), "rb").read()


def test_format_errors(tmp_path):
    p = tmp_path / "bad.mosst"
    p.write_bytes(b"NOTMOSST" + b"\x00" * 16)
    with pytest.raises(errors.BadMagicError):
        tensor_read(p)
    p.write_bytes(GOLDEN_E8M0[:9])
    with pytest.raises(errors.TruncatedPayloadError):
        tensor_read(p)
    p.write_bytes(GOLDEN_E8M0[:8] + b"\x02" + GOLDEN_E8M0[9:])
    with pytest.raises(errors.VersionMismatchError):
        tensor_read(p)
    p.write_bytes(GOLDEN_E8M0[:-1])
    with pytest.raises(errors.TruncatedPayloadError):
        tensor_read(p)
    with pytest.raises(errors.InvalidShapeError):
        tensor_randn([4, 0], seed=1)
    with pytest.raises(errors.InvalidValueError):
        tensor_write(np.array([1.0, np.nan], np.float32), tmp_path / "n.mosst")
    with pytest.raises(errors.InvalidArgumentError):
        tensor_randn([4], seed=1, dist="cauchy")


def test_cli_host_paths():
    """CLI surface without a GPU: codec table, unsupported schemes -> JSON error + exit 1."""
    import subprocess
    import sys
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_2511_05811_b200.cli", *a], capture_output=True,
                                    text=True, cwd=os.path.dirname(HERE))
    r = run("codec-table", "--format", "e4m3")
    lines = r.stdout.strip().splitlines()
    assert r.returncode == 0 and lines[0] == "code,value" and len(lines) == 257
    assert lines[1 + 0x7E] == "126,448.0" and lines[1 + 0x38] == "56,1.0"      # test_fp8.py:59-68 anchors
    r = run("gemm", "--m", "4", "--n", "4", "--k", "33", "--scheme", "mx2", "--out", "/tmp/_g.json")
    assert r.returncode == 1 and '"error"' in r.stderr
