"""The GPU CLI (paper_2511_05811_b200.cli) against outputs of the reference's
own CLI on the same input (tests/golden/cli, made by make_cli_golden.py):
`quantize --scheme mx2|tensor` payloads byte-identical (.mosst codes and E8M0
micro codes) with equal metadata; `gemm --verify` within the FP32-accumulation
tolerance and with the reference's counters."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "cli")


def _cli(*args):
    r = subprocess.run([sys.executable, "-m", "paper_2511_05811_b200.cli", *args], capture_output=True, text=True,
                       cwd=os.path.dirname(HERE), timeout=300)
    assert r.returncode == 0, r.stderr
    return r


@pytest.mark.parametrize("scheme", ["mx2", "tensor", "group"])
def test_quantize_matches_reference_cli(tmp_path, scheme):
    out, meta = tmp_path / "q.mosst", tmp_path / "q.json"
    _cli("quantize", "--scheme", scheme, "--in", os.path.join(GOLD, "x.mosst"), "--out", str(out), "--meta", str(meta))
    assert out.read_bytes() == open(os.path.join(GOLD, f"ref_{scheme}.mosst"), "rb").read()
    got, ref = json.loads(meta.read_text()), json.load(open(os.path.join(GOLD, f"ref_{scheme}.json")))
    ref.pop("micro_scales_path", None)
    micro = got.pop("micro_scales_path", None)
    assert got == ref
    if scheme == "mx2":
        assert open(micro, "rb").read() == open(os.path.join(GOLD, "ref_mx2.mosst.micro.mosst"), "rb").read()
    assert (tmp_path / "q.mosst.manifest.json").exists()


@pytest.mark.parametrize("scheme", ["mx2", "pergroup"])
def test_gemm_verify_matches_reference_report(tmp_path, scheme):
    out = tmp_path / "g.json"
    r = _cli("gemm", "--m", "128", "--n", "256", "--k", "512", "--scheme", scheme, "--verify", "--out", str(out))
    ref_name = "ref_gemm.json" if scheme == "mx2" else "ref_gemm_pergroup.json"
    got, ref = json.loads(out.read_text()), json.load(open(os.path.join(GOLD, ref_name)))
    assert got["counters"] == ref["counters"]
    assert got["frobenius_rel_error"] <= 1e-5          # FP32 accumulation vs the float64 oracle
    assert "frobenius_rel_error=" in r.stdout
