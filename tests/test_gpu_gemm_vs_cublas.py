"""Full-size cross-check of K2 against NVIDIA's library: on identical E4M3
codes and identical E8M0 scale buffers (the tcgen05 block-scale layout is
cuBLASLt's SWIZZLE_32_4_4), our GEMM and cuBLASLt MXFP8 (torch F.scaled_mm,
BlockWise1x32) must produce the same bf16 output for every fwd / dgrad /
wgrad shape of the Llama-7B linears — a size-independent
parity property at BASELINE's full sizes, complementing the float64-oracle
tolerance tests at oracle-friendly sizes."""

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.nn.functional as F  # noqa: E402

from paper_2511_05811_b200.gemm import mx_gemm  # noqa: E402
from paper_2511_05811_b200.quantize import quantize_mx2  # noqa: E402

T = 8192
SHAPES = []
for k, n in [(4096, 12288), (4096, 4096), (4096, 22016), (11008, 4096)]:
    SHAPES += [(T, n, k), (T, k, n), (n, k, T)]


@pytest.mark.skipif(not hasattr(F, "scaled_mm"), reason="torch without F.scaled_mm")
@pytest.mark.parametrize("m,n,k", SHAPES)
def test_gemm_equals_cublaslt_mxfp8(m, n, k):
    torch.manual_seed(m + n + k)
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    a.view(-1)[::4099] *= 40.0                  # outlier blocks: spread of E8M0 codes
    qa, qb = quantize_mx2(a), quantize_mx2(b)
    one = torch.ones(1, device="cuda")
    ours = mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out_dtype=torch.bfloat16)
    ref = F.scaled_mm(qa.codes.view(torch.float8_e4m3fn), qb.codes.view(torch.float8_e4m3fn).t(),
                      qa.sf.view(torch.float8_e8m0fnu), F.ScalingType.BlockWise1x32,
                      qb.sf.view(torch.float8_e8m0fnu), F.ScalingType.BlockWise1x32,
                      swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                      output_dtype=torch.bfloat16)
    exact = (ours == ref).float().mean().item()
    rel = ((ours.float() - ref.float()).norm() / ref.float().norm()).item()
    assert exact > 0.999 and rel < 1e-4, (exact, rel)


_RASTER_CHILD = r"""
import torch, torch.nn.functional as F
from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.quantize import quantize_mx2
one = torch.ones(1, device="cuda")
for m, n, k in [(8192, 22016, 4096), (22016, 8192, 4096), (4096, 11008, 11008)]:
    torch.manual_seed(m + 2 * n + k)
    qa = quantize_mx2(torch.randn(m, k, device="cuda", dtype=torch.bfloat16))
    qb = quantize_mx2(torch.randn(n, k, device="cuda", dtype=torch.bfloat16))
    ours = mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out_dtype=torch.bfloat16)
    ref = F.scaled_mm(qa.codes.view(torch.float8_e4m3fn), qb.codes.view(torch.float8_e4m3fn).t(),
                      qa.sf.view(torch.float8_e8m0fnu), F.ScalingType.BlockWise1x32,
                      qb.sf.view(torch.float8_e8m0fnu), F.ScalingType.BlockWise1x32,
                      swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                      output_dtype=torch.bfloat16)
    exact = (ours == ref).float().mean().item()
    assert exact > 0.999, (m, n, k, exact)
print("ok")
"""


@pytest.mark.skipif(not hasattr(F, "scaled_mm"), reason="torch without F.scaled_mm")
@pytest.mark.parametrize("budget_mb", ["8", "0"])
def test_raster_groups_equal_cublaslt(budget_mb):
    """The L2-budget raster (csrc/gemm2.cu g2_raster) only reorders tiles: with a
    tiny budget (many groups, both m-pair and n-tile orientations) and with the
    fixed 8-m-pair raster the outputs still equal cuBLASLt's."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, MOSS_GEMM2_L2MB=budget_mb)
    r = subprocess.run([sys.executable, "-c", _RASTER_CHILD], env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
