"""BASELINE configs[0] at its full size, with the reference's own input
generators: one MOSS FP8 linear fwd + dgrad + wgrad + auto-scaled AdamW step,
tokens = 4096, K = N = 4096 (x = tensor_randn(seed 1),
W = 0.02 tensor_randn(seed 2), dY = 1e-3 tensor_randn(seed 3), f32 inputs —
the reference CPU path's own case), against the CPU oracle:

  * every quantization bit-exact (activations row- and column-wise, dY, the
    weight copy at s_t and at s_{t+1});
  * fwd / dgrad / wgrad within the FP32-accumulation tolerance of the float64
    products of the dequantized operands (gemm.py:160-209 composition);
  * the AdamW step within 1e-3 * eta of the float64 reference (optim.py:78-106),
    the scale advance s_{t+1} = s_t + eta/448 (autoscale.py:71-79) exact."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2511_05811_b200.nn import MossAdamW, MossLinear  # noqa: E402
from paper_2511_05811_b200.tensor import tensor_randn  # noqa: E402

from oracle import numpy_ref as R  # noqa: E402

from .helpers import rel_frob  # noqa: E402

T = D = 4096
ETA = 3e-4


def test_config1_full_size_step(c_oracle):
    x = tensor_randn([T, D], seed=1)
    w0 = tensor_randn([D, D], seed=2) * np.float32(0.02)
    dy = tensor_randn([T, D], seed=3) * np.float32(1e-3)
    layer = MossLinear(D, D, init_std=None)
    with torch.no_grad():
        layer.weight.copy_(torch.as_tensor(w0))
    opt = MossAdamW([layer.weight], lr=ETA, weight_decay=0.1)
    xt = torch.as_tensor(x, device="cuda").requires_grad_(True)          # f32 activations (C1)
    y = layer(xt)
    y.backward(torch.as_tensor(dy, device="cuda", dtype=y.dtype))
    # weight copy at s_0 = max|W|/448 (schedule_from_weights, autoscale.py:62-68)
    s0 = R.jit_scale(w0)
    assert layer.schedule.s_t == s0
    wc, _ = R.encode_weight(w0, s0)
    assert np.array_equal(layer.w_fp8.cpu().numpy(), wc) and np.array_equal(layer.w_fp8_t.cpu().numpy(), wc.T)
    # oracle operands: the reference quantizer (bit-exactness of the GPU quantizer is asserted through the
    # C oracle in test_gpu_kernels / test_gpu_shape_sweep; here the products are compared)
    wd = R.dequantize_per_tensor(wc, float(np.float32(s0)))
    qx = c_oracle.quant_two_level(x)
    assert qx[3] == 0
    xd = R.dequantize_two_level(R.quant_two_level(x))
    y_ref = xd @ wd.T
    assert rel_frob(y.detach().float().cpu().numpy(), y_ref) <= 4e-3               # bf16 output
    dyh = y.new_tensor(dy).float().cpu().numpy()
    dyd = R.dequantize_two_level(R.quant_two_level(dyh))
    assert rel_frob(xt.grad.float().cpu().numpy(), dyd @ wd) <= 4e-3
    dw_ref = R.gemm_f64(R.dequantize_two_level(R.quant_two_level(np.ascontiguousarray(dyh.T))),
                        R.dequantize_two_level(R.quant_two_level(np.ascontiguousarray(x.T))))
    g = layer.weight.main_grad.cpu().numpy()
    assert rel_frob(g, dw_ref) <= 1e-5
    # the optimizer step on the GPU's own gradient
    w_before = layer.weight.detach().cpu().numpy().copy()
    opt.step()
    opt.check()
    st = R.adam_init(w0.shape, eta=ETA, weight_decay=0.1)
    w_ref, _ = R.adamw_step(w_before, g.astype(np.float64), st)
    w1 = layer.weight.detach().cpu().numpy()
    assert np.max(np.abs(w1 - w_ref)) <= 1e-3 * ETA
    sched = R.Schedule(s_t=s0)
    R.advance(sched, ETA)
    assert layer.schedule.s_t == sched.s_t                                           # exact f64 advance
    wc1, _ = R.encode_weight(w1, sched.s_t)
    assert np.array_equal(layer.w_fp8.cpu().numpy(), wc1)                             # next forward's codes
