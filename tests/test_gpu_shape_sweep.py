"""Randomized shape sweep of the quantizer and the GEMM through every kernel
path (single-launch TMA quantizer for 128-multiples, the generic fallback for
ragged shapes, f32 and bf16 inputs, 2-CTA and 1-CTA GEMMs, padded GEMMs):
quantizer outputs bit-exact vs the C oracle (oracle/moss_oracle.c), GEMM
within the FP32-accumulation tolerance of the float64 product of the GPU's
own codes.  Seeds are fixed, so a failure names its shape."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2511_05811_b200.fp8 import fp8_decode  # noqa: E402
from paper_2511_05811_b200.gemm import mx_gemm  # noqa: E402
from paper_2511_05811_b200.quantize import quantize_mx2  # noqa: E402

from .helpers import unswizzle_sf  # noqa: E402

RNG = np.random.default_rng(2026)
QSHAPES = [(int(r), int(c)) for r, c in zip(RNG.integers(1, 40, 24) * 32, RNG.integers(1, 48, 24) * 32)]
QSHAPES += [(128, 128), (256, 4096), (32, 32), (4096, 96)]


@pytest.mark.parametrize("rows,cols", QSHAPES)
def test_quantizer_shape_sweep(c_oracle, rows, cols):
    rng = np.random.default_rng(rows * 7919 + cols)
    x = (rng.standard_normal((rows, cols)) * np.exp(rng.uniform(-8, 8))).astype(np.float32)
    x[rng.random((rows, cols)) < 1e-3] *= 60.0
    for dtype in (torch.bfloat16, torch.float32):
        xt = torch.as_tensor(x, device="cuda").to(dtype)
        xe = xt.float().cpu().numpy()
        op = quantize_mx2(xt, row=True, col=True, micro=True)
        codes, micro, g, st = c_oracle.quant_two_level(xe)
        assert st == 0 and float(op.g) == g
        assert np.array_equal(op.codes.cpu().numpy(), codes), (rows, cols, dtype)
        assert np.array_equal(op.micro.cpu().numpy(), micro), (rows, cols, dtype)
        assert np.array_equal(unswizzle_sf(op.sf.cpu().numpy(), rows, cols // 32), micro)
        codes_t, micro_t, _, _ = c_oracle.quant_two_level(np.ascontiguousarray(xe.T))
        assert np.array_equal(op.codes_t.cpu().numpy(), codes_t), (rows, cols, dtype, "col")
        assert np.array_equal(op.micro_t.cpu().numpy(), micro_t), (rows, cols, dtype, "col")


GSHAPES = [(int(m), int(n), int(k)) for m, n, k in zip(RNG.integers(1, 24, 16) * 64, RNG.integers(1, 24, 16) * 64,
                                                       RNG.integers(1, 24, 16) * 128)]
GSHAPES += [(256, 256, 128), (512, 768, 1024), (128, 128, 128)]


@pytest.mark.parametrize("m,n,k", GSHAPES)
def test_gemm_shape_sweep(m, n, k):
    torch.manual_seed(m + 3 * n + 7 * k)
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    qa, qb = quantize_mx2(a, micro=True), quantize_mx2(b, micro=True)
    for out_dtype in (torch.float32, torch.bfloat16):
        d = mx_gemm(qa.codes, qa.sf, qa.g, qb.codes, qb.sf, qb.g, out_dtype=out_dtype)
        deq = lambda q, r: (fp8_decode(q.codes).double().view(r, k // 32, 32)
                            * torch.ldexp(torch.ones_like(q.micro, dtype=torch.float64),
                                          q.micro.to(torch.int64) - 127)[..., None]).view(r, k) * float(q.g)
        ref = deq(qa, m) @ deq(qb, n).t()
        rel = float((d.double() - ref).norm() / ref.norm())
        assert rel <= (1e-5 if out_dtype == torch.float32 else 4e-3), (m, n, k, out_dtype, rel)
