"""dgrad without a transposed weight copy: moss_gemm_mxf8_bkn reads the E4M3
weight codes W [K, N] as stored (MN-major tcgen05 B operand).  Must equal the
K-major GEMM on the materialised W^T bit for bit (same products, same K order),
at every Llama-7B dgrad shape."""

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2511_05811_b200.gemm import mx_gemm, mx_gemm_bkn  # noqa: E402
from paper_2511_05811_b200.quantize import quantize_mx2  # noqa: E402


@pytest.mark.parametrize("m,k,n", [(256, 128, 256), (512, 384, 768), (8192, 4096, 4096), (8192, 4096, 11008),
                                   (8192, 22016, 4096), (8192, 12288, 4096), (4096, 11008, 4096)])
def test_bkn_equals_transposed_copy(m, k, n):
    torch.manual_seed(m + k + n)
    dy = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    dy.view(-1)[::3001] *= 60.0
    q = quantize_mx2(dy)
    w = torch.randint(0, 256, (k, n), device="cuda", dtype=torch.uint8)
    w[(w & 0x7F) == 0x7F] = 0                    # no NaN codes
    s_a = q.g.reshape(1).float()
    s_w = torch.tensor([0.0123], device="cuda")
    ref = mx_gemm(q.codes, q.sf, s_a, w.t().contiguous(), None, s_w, out_dtype=torch.bfloat16)
    got = mx_gemm_bkn(q.codes, q.sf, s_a, w, s_w)
    assert got.shape == ref.shape
    assert torch.equal(got, ref), float((got.float() - ref.float()).abs().max())
