"""Fixtures for the .mosst / CLI parity tests, produced by the REFERENCE itself.

Run here, where /root/reference exists:
    python tests/golden/make_cli_golden.py
Imports ``mossq`` from /root/reference/pkg/src (read-only, never copied) and
writes:
  tests/golden/tensor_golden.npz   tensor_randn outputs (tensor.py:57-85) for
                                   several seeds / distributions / shapes
  tests/golden/cli/x.mosst         a seeded outlier_injected f32 input
  tests/golden/cli/ref_mx2*        `mossq quantize --scheme mx2` outputs
                                   (codes .mosst, micro .mosst, meta JSON)
  tests/golden/cli/ref_tensor*     `mossq quantize --scheme tensor` outputs
  tests/golden/cli/ref_group*      `mossq quantize --scheme group` outputs
  tests/golden/cli/ref_gemm.json   `mossq gemm --scheme mx2 --verify` report
  tests/golden/cli/ref_gemm_pergroup.json  `mossq gemm --scheme pergroup --verify` report
The GPU box never reads /root/reference; these files travel with the repo.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from click.testing import CliRunner  # noqa: E402
from mossq.cli import cli  # noqa: E402
from mossq.tensor import tensor_randn, tensor_write  # noqa: E402


def main():
    out = {}
    for name, shape, seed, dist in [("g_4", [4], 7, "gaussian"), ("g_3x5", [3, 5], 11, "gaussian"),
                                    ("l_64", [64], 3, "laplace"), ("o_32x64", [32, 64], 5, "outlier_injected")]:
        out[name] = tensor_randn(shape, seed=seed, dist=dist)
    np.savez(os.path.join(HERE, "tensor_golden.npz"), **out)

    d = os.path.join(HERE, "cli")
    x = tensor_randn([64, 256], seed=5, dist="outlier_injected")
    tensor_write(x, os.path.join(d, "x.mosst"))
    r = CliRunner()
    for scheme in ("mx2", "tensor", "group"):
        res = r.invoke(cli, ["quantize", "--scheme", scheme, "--in", os.path.join(d, "x.mosst"),
                             "--out", os.path.join(d, f"ref_{scheme}.mosst"),
                             "--meta", os.path.join(d, f"ref_{scheme}.json")])
        assert res.exit_code == 0, res.output
    res = r.invoke(cli, ["gemm", "--m", "128", "--n", "256", "--k", "512", "--scheme", "mx2", "--verify",
                         "--out", os.path.join(d, "ref_gemm.json")])
    assert res.exit_code == 0, res.output
    res = r.invoke(cli, ["gemm", "--m", "128", "--n", "256", "--k", "512", "--scheme", "pergroup", "--verify",
                         "--out", os.path.join(d, "ref_gemm_pergroup.json")])
    assert res.exit_code == 0, res.output
    for f in os.listdir(d):
        if f.endswith(".manifest.json"):
            os.remove(os.path.join(d, f))


if __name__ == "__main__":
    main()
