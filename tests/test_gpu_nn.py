"""GPU parity of the training wrappers (MossLinear / MossAdamW) against the
composed CPU oracle:

  fwd   y  = deq(Q2(x))      . deq(E(W, s_t))^T            (train.py:168-174)
  dgrad dx = deq(Q2(dy))     . deq(E(W, s_t))              (composed; the reference bwd is fp)
  wgrad dW = deq(Q2(dy^T))   . deq(Q2(x^T))^T
  step  W' = adamw_step(W, dW); s_{t+1} = s_t + eta/448; W_fp8 = E(W', s_{t+1})
        every ``interval`` steps s = max|W'|/448           (optim.py:78-106, autoscale.py:71-96)

Q2 = quant_two_level (bit-exact on the GPU, test_gpu_kernels.py), E = the
per-tensor weight encode.  GEMM tolerance: FP32 accumulation (+ bf16 output
rounding where the output is bf16).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2511_05811_b200.nn import MossAdamW, MossLinear  # noqa: E402

from oracle import numpy_ref as R  # noqa: E402

from .helpers import rel_frob  # noqa: E402

BF16_TOL = 4e-3     # bf16 output rounding dominates (2^-9 relative)
F32_TOL = 1e-5


def host(t):
    return t.detach().float().cpu().numpy()


def deq2(x):
    return R.dequantize_two_level(R.quant_two_level(x))


@pytest.mark.parametrize("tokens,d_in,d_out", [(256, 512, 384), (1024, 4096, 4096), (512, 1024, 2816)])
def test_moss_linear_fwd_dgrad_wgrad(c_oracle, tokens, d_in, d_out):
    torch.manual_seed(tokens + d_in)
    layer = MossLinear(d_in, d_out)
    x = torch.randn(tokens, d_in, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    y = layer(x)
    dy = torch.randn(tokens, d_out, device="cuda", dtype=torch.bfloat16) * 1e-2
    y.backward(dy)
    w = host(layer.weight)
    s0 = layer.schedule.s_t
    assert s0 == float(np.abs(w).max()) / 448.0
    wc, _ = R.encode_weight(w, s0)
    assert np.array_equal(layer.w_fp8.cpu().numpy(), wc)                     # bit-exact weight copy
    assert np.array_equal(layer.w_fp8_t.cpu().numpy(), wc.T)
    w_deq = R.dequantize_per_tensor(wc, float(np.float32(s0)))
    xh, dyh = host(x), host(dy)
    y_ref = R.gemm_f64(deq2(xh), w_deq)
    assert rel_frob(host(y), y_ref) <= BF16_TOL
    dx_ref = deq2(dyh) @ w_deq
    assert rel_frob(host(x.grad), dx_ref) <= BF16_TOL
    dw_ref = R.gemm_f64(deq2(np.ascontiguousarray(dyh.T)), deq2(np.ascontiguousarray(xh.T)))
    assert rel_frob(host(layer.weight.main_grad), dw_ref) <= F32_TOL
    assert layer.weight.grad is None                      # wgrad went straight to main_grad


def test_adamw_autoscale_lifecycle(c_oracle):
    torch.manual_seed(7)
    layer = MossLinear(256, 512, interval=3)
    opt = MossAdamW(layer.parameters(), lr=1e-3, weight_decay=0.1)
    x = torch.randn(128, 256, device="cuda", dtype=torch.bfloat16)
    w_ref = host(layer.weight).astype(np.float64)
    layer(x)  # initialises the schedule (t = 0 max-reduction)
    sched = R.Schedule(s_t=R.jit_scale(w_ref), interval=3)
    st = R.adam_init(w_ref.shape, eta=1e-3, weight_decay=0.1)
    assert layer.schedule.s_t == sched.s_t
    for step in range(7):
        opt.zero_grad()
        y = layer(x)
        (y.float() ** 2).mean().backward()
        g = host(layer.weight.main_grad).astype(np.float64)
        w_before = host(layer.weight)
        opt.step()
        opt.check()
        # oracle step from the GPU's own W and gradient
        st_w, _ = R.adamw_step(w_before, g, st)
        R.advance(sched, 1e-3)
        if R.rescale_due(sched):
            R.rescale(host(layer.weight), sched)
        w_gpu = host(layer.weight)
        assert np.max(np.abs(w_gpu - st_w)) <= 2e-3 * 1e-3, step
        assert layer.schedule.t == sched.t and layer.schedule.last_rescale_step == sched.last_rescale_step
        assert layer.schedule.s_t == pytest.approx(sched.s_t, rel=1e-6), step
        wc, sat = R.encode_weight(w_gpu, layer.schedule.s_t)
        assert np.array_equal(layer.w_fp8.cpu().numpy(), wc), step          # codes for the next forward
        assert np.array_equal(layer.w_fp8_t.cpu().numpy(), wc.T), step
        assert float(layer.w_scale.item()) == float(np.float32(layer.schedule.s_t))
        # dominance: predicted scale never below the JIT scale (train.py:163-167)
        assert layer.schedule.s_t >= R.jit_scale(w_gpu) * (1 - 1e-7)
    assert [t for t, _ in opt.rescale_events] == [3, 6]
    assert int(opt.saturations.item()) == 0


def test_layer_stack_trains():
    from paper_2511_05811_b200.workloads import LayerStack
    torch.manual_seed(0)
    model = LayerStack(d_model=512, d_ffn=1024)
    opt = MossAdamW(model, lr=1e-3, weight_decay=0.0)
    x = torch.randn(1024, 512, device="cuda", dtype=torch.bfloat16)
    losses = []
    for _ in range(30):
        opt.zero_grad()
        loss = model(x)
        loss.backward()
        opt.step()
        losses.append(float(loss))
    opt.check()
    assert losses[-1] < 0.5 * losses[0]


def test_two_graph_steps_same_model_double_buffered():
    """Two CudaGraphSteps over one model/optimizer (double-buffered inputs, as the
    e2e pipeline uses them): both capture, and alternating replays give the same
    losses as a single graph fed by copies."""
    from paper_2511_05811_b200.nn import CudaGraphStep, MossAdamW
    from paper_2511_05811_b200.workloads import LayerStack

    def run(two):
        torch.manual_seed(0)
        model = LayerStack(d_model=512, d_ffn=1024, device="cuda")
        opt = MossAdamW(model, lr=1e-3)

        def fb(xin):
            loss = model(xin)
            loss.backward()
            return loss
        g = torch.Generator(device="cuda").manual_seed(5)
        data = [torch.randn(512, 512, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(8)]
        bufs = [torch.zeros(512, 512, device="cuda", dtype=torch.bfloat16).requires_grad_(True) for _ in range(2)]
        steps = [CudaGraphStep(fb, opt, (bufs[b],)) for b in range(2 if two else 1)]
        out = []
        for i, x in enumerate(data):
            b = i % len(steps)
            with torch.no_grad():
                bufs[b].copy_(x)
            out.append(float(steps[b](bufs[b])))
        return out

    assert run(True) == run(False)
