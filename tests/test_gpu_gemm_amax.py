"""K2's amax epilogue: max|D| of the stored output, written by the GEMM for
the quantizer that consumes D (producer-fused amax, north_star (1);
the reduction it replaces is quantize.py:149-155).  Must equal max|D|
exactly — the quantizer's global scale, and so every code, depends on it."""

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_05811_b200 as P  # noqa: E402
from paper_2511_05811_b200 import nn as mnn  # noqa: E402
from paper_2511_05811_b200.gemm import mx_gemm, mx_gemm_bkn  # noqa: E402
from paper_2511_05811_b200.quantize import quantize_mx2  # noqa: E402


@pytest.mark.parametrize("m,n,k,dt", [(512, 512, 256, torch.bfloat16), (512, 384, 512, torch.bfloat16),
                                      (256, 256, 128, torch.float32), (200, 136, 96, torch.bfloat16),
                                      (8192, 4096, 4096, torch.bfloat16)])
def test_mx_gemm_amax_epilogue_exact(m, n, k, dt):
    torch.manual_seed(m + n + k)
    a = quantize_mx2(torch.randn(m, k, device="cuda", dtype=torch.bfloat16) * 3, row=True)
    b = quantize_mx2(torch.randn(n, k, device="cuda", dtype=torch.bfloat16), row=True)
    am = torch.full((1,), -1.0, device="cuda")
    d = mx_gemm(a.codes, a.sf, a.g, b.codes, b.sf, b.g, out_dtype=dt, amax_out=am)
    assert float(am) == float(d.float().abs().max())


@pytest.mark.parametrize("m,k,n", [(512, 256, 512), (8192, 11008, 4096), (8192, 4096, 4096)])
def test_mx_gemm_bkn_amax_epilogue_exact(m, k, n):
    torch.manual_seed(m + k + n)
    a = quantize_mx2(torch.randn(m, k, device="cuda", dtype=torch.bfloat16), row=True)
    w = P.quant_per_tensor(torch.randn(k, n, device="cuda") * 0.02)
    am = torch.zeros(1, device="cuda")
    d = mx_gemm_bkn(a.codes, a.sf, a.g, w.codes, w.scale.reshape(1), amax_out=am)
    assert float(am) == float(d.float().abs().max())


def test_amax_epilogue_reaches_the_next_quantizer(monkeypatch):
    """LayerStack: gate_up's dgrad hands O the amax of O's output-gradient, so
    every quantizer of the backward runs in producer-amax mode."""
    from paper_2511_05811_b200 import quantize as Q
    from paper_2511_05811_b200.workloads import LayerStack
    seen = []
    real = Q.quantize_mx2

    def spy(x2d, **kw):
        seen.append(kw.get("amax") is not None)
        return real(x2d, **kw)
    monkeypatch.setattr(mnn, "quantize_mx2", spy)
    torch.manual_seed(0)
    model = LayerStack(d_model=512, d_ffn=1024)
    x = torch.randn(1024, 512, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    loss = model(x)
    n_fwd = len(seen)
    loss.backward()
    bwd = seen[n_fwd:]
    assert len(bwd) == 4 and all(bwd), bwd                 # down, gate_up, o, qkv dY: all producer-amax
    assert seen[:n_fwd] == [False, True, True, True]       # x (step input) in-kernel; a, r, h from producers
