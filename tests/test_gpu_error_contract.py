"""Training-path error contract (optim.py:89-90 raises BEFORE mutating;
quantize.py:88 / fp8.py:219-222 raise in the forward): a step whose
activations, output-gradients or gradients hold NaN/Inf must leave the
optimizer exactly as it was after the last good step — FP32 masters,
moments, FP8 codes, per-tensor scales on the device, and the step counter and
scale schedules on the host — and check() must raise the reference's class.
The device half is gated (K3 skips when the flag word is set, which also
works under CUDA-graph replay); the host half is rolled back by check()."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from torch import nn  # noqa: E402

from paper_2511_05811_b200 import llama as L  # noqa: E402
from paper_2511_05811_b200.errors import InvalidValueError  # noqa: E402
from paper_2511_05811_b200.nn import CudaGraphStep, MossAdamW, MossLinear, raise_if_flagged  # noqa: E402
from paper_2511_05811_b200.trainer import make_optimizer  # noqa: E402

TINY = dict(vocab=512, d_model=128, n_layers=2, n_heads=4, d_ffn=256, max_seq=64, interval=50)


def _state(model, opt):
    dev = {}
    for n, p in model.named_parameters():
        dev[n] = p.detach().clone()
        st = opt.state.get(id(p))
        if st is not None:
            dev[n + ".m"], dev[n + ".v"] = st[0].clone(), st[1].clone()
        lay = getattr(p, "moss_layer", None)
        if lay is not None:
            dev[n + ".fp8"] = lay.w_fp8.clone()
            dev[n + ".scale"] = lay.w_scale.clone()
    host = (opt.t, [(l.schedule.s_t, l.schedule.t, l.schedule.last_rescale_step) for l in opt._moss_layers()])
    return dev, host


def _assert_same(a, b):
    assert a[1] == b[1], "host step counter / schedules"
    for k in a[0]:
        assert torch.equal(a[0][k], b[0][k]), k


def _setup(graph):
    torch.manual_seed(3)
    cfg = L.LlamaConfig(**TINY)
    model = L.LlamaModel(cfg)
    opt = make_optimizer(model, 2e-3, 100, 5)
    data = L.MarkovTokens(cfg.vocab, seed=2)
    sx = torch.zeros((4, 64), dtype=torch.long, device="cuda")
    sy = torch.zeros((4, 64), dtype=torch.long, device="cuda")

    def fb(xt, yt):
        loss = model(xt, yt)
        loss.backward()
        return loss
    graphed = CudaGraphStep(fb, opt, (sx, sy)) if graph else None

    def step():
        x, y = data.batch(4, 64)
        xt, yt = torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda")
        if graphed is not None:
            return graphed(xt, yt)
        opt.zero_grad()
        loss = fb(xt, yt)
        opt.step()
        return loss
    return model, opt, step


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("bad_steps", [1, 2])
def test_nonfinite_activation_skips_whole_step_and_rolls_back(graph, bad_steps):
    model, opt, step = _setup(graph)
    for _ in range(4):
        step()
        opt.check()
    emb = model.embed.detach()
    keep = emb.clone()
    emb.fill_(float("inf"))                    # every activation of the next forward is non-finite
    before = _state(model, opt)
    for _ in range(bad_steps):                 # check_every > 1: later steps are skipped too
        step()
    with pytest.raises(InvalidValueError):
        opt.check("poisoned step")
    _assert_same(_state(model, opt), before)   # nothing mutated, host rolled back
    emb.copy_(keep)                            # the run recovers from the last good step
    loss = step()
    opt.check("recovered step")
    assert torch.isfinite(loss).all() and opt.t == before[1][0] + 1


def test_nonfinite_replicated_gradient_gates_fp8_weight_updates():
    """A NaN in a gradient that no quantizer saw (a replicated parameter) is
    caught by the pre-update check: no K3 of the step runs, MOSS weights included."""
    torch.manual_seed(0)
    lin = MossLinear(64, 64)
    extra = nn.Parameter(torch.randn(64, device="cuda"))
    opt = MossAdamW(list(lin.parameters()) + [extra], lr=1e-3)
    x = torch.randn(32, 64, device="cuda", dtype=torch.bfloat16)
    for bad in (False, True):
        opt.zero_grad()
        lin(x).float().square().mean().backward()
        extra.grad = torch.zeros_like(extra)
        if bad:
            extra.grad[7] = float("nan")
            w0, c0, e0, t0 = lin.weight.detach().clone(), lin.w_fp8.clone(), extra.detach().clone(), opt.t
            s0 = lin.schedule.s_t
        opt.step()
        if not bad:
            opt.check()
    with pytest.raises(InvalidValueError, match="gradient"):
        opt.check()
    assert torch.equal(lin.weight.detach(), w0) and torch.equal(lin.w_fp8, c0) and torch.equal(extra.detach(), e0)
    assert opt.t == t0 and lin.schedule.s_t == s0
    raise_if_flagged("cuda")                   # flags were reset by the raise
