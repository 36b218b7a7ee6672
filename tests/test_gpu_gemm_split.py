"""K2's tail split (csrc/gemm2.cu g2_unit): when the last wave of 256 x 256
pair tiles is at most half full, each tail tile runs as two half-K units on two
pairs and the second adds the first's FP32 partial before the epilogue.  This
happens on the Llama-7B shapes at seq 4096 (M = 4096: 256 tiles = 3.46 waves
on 74 pairs).  The result differs from the unsplit GEMM only by FP32
summation order, so the gates are the GEMM tolerance of SURVEY.md 8(c)
(test_gpu_parity_full.py), the amax epilogue stays exact, and accumulation
into FP32 (wgrad reduce-add) still adds exactly once."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_05811_b200 as P  # noqa: E402
from paper_2511_05811_b200.gemm import mx_gemm, mx_gemm_bkn  # noqa: E402
from paper_2511_05811_b200.quantize import quantize_mx2  # noqa: E402

from oracle import numpy_ref as R  # noqa: E402

from .helpers import rel_frob  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
F32_TOL = 1e-5
BF16_U = 2.0 ** -8


def host(t):
    return t.detach().cpu().numpy()


def _tiles(m, n):
    return (m // 256) * (n // 256)


def _splits(m, n, k=8192):
    if k < 8192:
        return False
    t = _tiles(m, n)
    pairs = min(t, torch.cuda.get_device_properties(0).multi_processor_count // 2)
    rem = t % pairs
    return rem > 0 and 2 * rem <= pairs


# (M, N, K) of the 7B step at seq 4096 that take the split path on 148 SMs
# (K >= 8192: the split's partial exchange costs more than half a shorter tile saves)
SPLIT_SHAPES = [(4096, 4096, 11008), (4096, 4096, 12288), (4096, 4096, 22016), (4096, 11008, 8192),
                (12288, 4096, 8192)]
NO_SPLIT_SHAPES = [(4096, 4096, 4096)]


@pytest.mark.parametrize("m,n,k", SPLIT_SHAPES + NO_SPLIT_SHAPES)
def test_split_shapes_vs_f64_oracle(m, n, k):
    assert _splits(m, n, k) == ((m, n, k) in SPLIT_SHAPES), "shape no longer (or now) exercises the tail split"
    torch.manual_seed(m + n + k)
    a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    a.view(-1)[::7919] *= 50
    w = torch.randn(n, k, device="cuda") * 0.02
    qa = quantize_mx2(a, row=True, micro=True)
    qw = P.quant_per_tensor(w)
    am = torch.zeros(1, device="cuda")
    d = mx_gemm(qa.codes, qa.sf, qa.g, qw.codes, None, qw.scale.reshape(1), out_dtype=torch.float32, amax_out=am)
    assert float(am) == float(d.abs().max())
    # every tail tile (the last rows of the raster) and a spread of others: sample rows of all m-pairs
    rng = np.random.default_rng(k)
    rows = np.unique(np.concatenate([rng.choice(m, 48, replace=False), np.arange(m - 256, m, 16)]))
    a_deq = R.dequantize_two_level(R.TwoLevel(host(qa.codes)[rows], float(qa.g), host(qa.micro)[rows]))
    b_deq = R.dequantize_per_tensor(host(qw.codes), float(qw.scale)).T
    ref = a_deq @ b_deq
    mag = np.abs(a_deq) @ np.abs(b_deq)
    got = host(d)[rows]
    assert float(np.max(np.abs(got - ref) / (mag + 1e-30))) <= F32_TOL
    assert rel_frob(got, ref) <= F32_TOL


def test_split_dgrad_bf16_and_amax():
    """MN-major dgrad (W as stored) at M = 4096, K = 11008 -> N = 4096, bf16 out."""
    m, k, n = 4096, 11008, 4096
    assert _splits(m, n, k)
    torch.manual_seed(3)
    a = quantize_mx2(torch.randn(m, k, device="cuda", dtype=torch.bfloat16), row=True, micro=True)
    w = P.quant_per_tensor(torch.randn(k, n, device="cuda") * 0.02)
    am = torch.zeros(1, device="cuda")
    d = mx_gemm_bkn(a.codes, a.sf, a.g, w.codes, w.scale.reshape(1), amax_out=am)
    assert float(am) == float(d.float().abs().max())
    rows = np.arange(0, m, 97)
    a_deq = R.dequantize_two_level(R.TwoLevel(host(a.codes)[rows], float(a.g), host(a.micro)[rows]))
    ref = a_deq @ R.dequantize_per_tensor(host(w.codes), float(w.scale))
    mag = np.abs(a_deq) @ np.abs(R.dequantize_per_tensor(host(w.codes), float(w.scale)))
    got = host(d.float())[rows]
    assert np.all(np.abs(got - ref) <= BF16_U * np.abs(ref) + 1.01 * F32_TOL * mag)


def test_split_accumulate_adds_once():
    """wgrad-style f32 accumulation (TMA reduce-add into main_grad): D0 + A.B."""
    m, n, k = 4096, 4096, 8192                     # dW[N_out, K_in], contraction over 8192 tokens
    assert _splits(m, n, k)
    torch.manual_seed(5)
    qa = quantize_mx2(torch.randn(m, k, device="cuda", dtype=torch.bfloat16), row=True)
    qb = quantize_mx2(torch.randn(n, k, device="cuda", dtype=torch.bfloat16), row=True)
    fresh = mx_gemm(qa.codes, qa.sf, qa.g, qb.codes, qb.sf, qb.g, out_dtype=torch.float32)
    d0 = torch.randn(m, n, device="cuda")
    acc = d0.clone()
    mx_gemm(qa.codes, qa.sf, qa.g, qb.codes, qb.sf, qb.g, out=acc, accumulate=True)
    want = d0 + fresh
    assert rel_frob(host(acc), host(want)) <= 1e-6
    # repeated launches reuse the flag words (re-zeroed by their consumers)
    for _ in range(5):
        again = mx_gemm(qa.codes, qa.sf, qa.g, qb.codes, qb.sf, qb.g, out_dtype=torch.float32)
        assert torch.equal(again, fresh)


_CHILD = r"""
import sys, torch
from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.quantize import quantize_mx2
torch.manual_seed(9)
qa = quantize_mx2(torch.randn(4096, 11008, device="cuda", dtype=torch.bfloat16), row=True)
qb = quantize_mx2(torch.randn(4096, 11008, device="cuda", dtype=torch.bfloat16), row=True)
d = mx_gemm(qa.codes, qa.sf, qa.g, qb.codes, qb.sf, qb.g, out_dtype=torch.float32)
torch.save(d.cpu(), sys.argv[1])
"""


def test_split_equals_unsplit_within_summation_order(tmp_path):
    """Same GEMM with MOSS_GEMM2_SPLIT=0 (whole tiles) and =1: the non-tail
    tiles are bit-identical, the tail tiles differ by FP32 reordering only."""
    outs = {}
    for flag in ("0", "1"):
        path = str(tmp_path / f"d{flag}.pt")
        r = subprocess.run([sys.executable, "-c", _CHILD, path], env=dict(os.environ, MOSS_GEMM2_SPLIT=flag),
                           capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[flag] = torch.load(path)
    d0, d1 = outs["0"], outs["1"]
    assert rel_frob(d1.numpy(), d0.numpy()) <= 1e-6
    m, n = d0.shape
    tile_diff = (d0 != d1).reshape(m // 256, 256, n // 256, 256).any(dim=3).any(dim=1)
    tiles = tile_diff.numel()
    pairs = min(tiles, torch.cuda.get_device_properties(0).multi_processor_count // 2)
    changed = int(tile_diff.sum())
    assert changed > 0, "no tile took the split path"
    assert changed <= tiles % pairs                # only the tail tiles may change
