"""The per-group (COAT-style) comparator (csrc/pergroup.cu) against outputs
of the reference itself (tests/golden/make_pergroup_golden.py):
quant_per_group codes and scales bit-exact, gemm_pergroup_mainloop within the
FP32-accumulation tolerance of the reference's float64 result, same counters."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2511_05811_b200.gemm import gemm_pergroup_mainloop  # noqa: E402
from paper_2511_05811_b200.quantize import quant_per_group  # noqa: E402

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pergroup_golden.npz"))


def test_quant_per_group_bit_exact():
    for name in ("a", "b"):
        q = quant_per_group(torch.as_tensor(G[name], device="cuda"))
        assert np.array_equal(q.codes.cpu().numpy(), G[f"{name}_codes"])
        assert np.array_equal(q.scales.cpu().numpy(), G[f"{name}_scales"])
    q = quant_per_group(torch.as_tensor(G["a"], device="cuda").to(torch.bfloat16))
    assert q.codes.shape == (256, 512)


def test_gemm_pergroup_vs_reference():
    qa = quant_per_group(torch.as_tensor(G["a"], device="cuda"))
    qb = quant_per_group(torch.as_tensor(G["b"], device="cuda"))
    c, ctr = gemm_pergroup_mainloop(qa, qb)
    ref = G["c"]
    got = c.double().cpu().numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-5
    assert [ctr.mainloop_dequant_multiplies, ctr.epilogue_dequant_multiplies, ctr.block_scale_multiplies,
            ctr.mac_count] == G["counters"].tolist()


def test_gemm_pergroup_large_vs_float64():
    torch.manual_seed(5)
    a = torch.randn(1024, 4096, device="cuda")
    b = torch.randn(768, 4096, device="cuda")
    qa, qb = quant_per_group(a), quant_per_group(b)
    c, _ = gemm_pergroup_mainloop(qa, qb)
    from paper_2511_05811_b200.fp8 import fp8_decode
    da = (fp8_decode(qa.codes).double().view(1024, 32, 128) * qa.scales.double()[..., None]).view(1024, 4096)
    db = (fp8_decode(qb.codes).double().view(768, 32, 128) * qb.scales.double()[..., None]).view(768, 4096)
    ref = da @ db.t()
    assert float((c.double() - ref).norm() / ref.norm()) <= 1e-5
