"""CPU reference of the MOSS training loop — TEST INFRASTRUCTURE ONLY.

Composes the reference's primitives (via oracle/numpy_ref) into the training
semantics the north_star asks for, in float64 on the CPU:
  forward  y  = deq(Q2(x)) . deq(E(W, s_t))^T            (train.py:168-174)
  dgrad    dx = deq(Q2(dy)) . deq(E(W, s_t))              (FP8 backward, composed:
  wgrad    dW = deq(Q2(dy^T)) . deq(Q2(x^T))^T             the reference bwd is fp)
  step     adamw_step (f64), s += eta/448, rescale every interval,
           E(W', s_{t+1}) for the next forward             (optim.py:78-106, autoscale.py:71-96)
where Q2 = quant_two_level and E = the per-tensor weight encode at the schedule
scale.  Used by tests/test_gpu_llama.py as the loss-curve reference of the
GPU run of the same Llama model.
"""

from __future__ import annotations

import numpy as np
import torch
from torch import nn

from . import numpy_ref as R


def _deq2(a32: np.ndarray) -> np.ndarray:
    """deq(quant_two_level(a)) in float64; the C restatement (pinned to the
    numpy one and to the reference's golden vectors) does the quantization."""
    from . import c_ref
    codes, micro, g, st = c_ref.load().quant_two_level_mt(a32)
    if st:
        raise ValueError("oracle quantization failed (non-finite or e8m0 range)")
    return R.dequantize_two_level(R.TwoLevel(codes, g, micro))


class _OracleLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, layer):
        shp = x.shape
        x32 = x.detach().reshape(-1, shp[-1]).numpy().astype(np.float32)
        wd = layer.w_deq()
        y = _deq2(x32) @ wd.T
        ctx.layer = layer
        ctx.x32 = x32
        ctx.wd = wd
        ctx.shp = shp
        return torch.from_numpy(y).view(*shp[:-1], wd.shape[0])

    @staticmethod
    def backward(ctx, dy):
        n = dy.shape[-1]
        dy32 = dy.detach().reshape(-1, n).numpy().astype(np.float32)
        dx = _deq2(dy32) @ ctx.wd
        dw = _deq2(np.ascontiguousarray(dy32.T)) @ _deq2(np.ascontiguousarray(ctx.x32.T)).T
        return torch.from_numpy(dx).view(ctx.shp), torch.from_numpy(dw), None


class OracleMossLinear(nn.Module):
    """float64 master weight + schedule + E4M3 codes at s_t (CPU)."""

    def __init__(self, d_in: int, d_out: int, interval: int):
        super().__init__()
        self.weight = nn.Parameter(torch.zeros(d_out, d_in, dtype=torch.float64))
        self.weight.oracle_layer = self
        self.interval = interval
        self.sched = None
        self.codes = None

    def init_from(self, w32: np.ndarray) -> None:
        with torch.no_grad():
            self.weight.copy_(torch.from_numpy(w32.astype(np.float64)))
        self.sched = R.Schedule(s_t=R.jit_scale(w32), interval=self.interval)   # autoscale.py:62-68
        self.encode()

    def encode(self) -> None:
        from . import c_ref        # == R.encode_weight bit for bit (tests/test_oracle.py)
        self.codes, _ = c_ref.load().encode_scaled(self.weight.detach().numpy().astype(np.float32),
                                                   np.float32(self.sched.s_t))   # train.py:113-118

    def w_deq(self) -> np.ndarray:
        return (R.fp8_decode(self.codes) * np.float32(self.sched.s_t)).astype(np.float64)

    def forward(self, x):
        return _OracleLinearFn.apply(x, self.weight, self)


class OracleAdamW:
    """adamw_step (f64) per parameter, then the autoscale lifecycle for MOSS weights."""

    def __init__(self, named_params, lr_schedule, weight_decay: float, no_decay):
        self.items = []
        for name, p in named_params:
            wd = 0.0 if no_decay(name, p) else weight_decay
            st = R.adam_init(tuple(p.shape), beta1=0.9, beta2=0.95, eta=0.0, weight_decay=wd, eps=1e-8)
            self.items.append((p, st))
        self.lr_schedule = lr_schedule
        self.t = 0

    def zero_grad(self):
        for p, _ in self.items:
            p.grad = None

    @torch.no_grad()
    def step(self):
        eta = self.lr_schedule(self.t)
        self.t += 1
        for p, st in self.items:
            if p.grad is None:
                continue
            st.eta = eta
            w_next, _ = R.adamw_step(p.detach().numpy(), p.grad.numpy(), st)
            p.copy_(torch.from_numpy(w_next))
            layer = getattr(p, "oracle_layer", None)
            if layer is not None:
                R.advance(layer.sched, eta)                              # autoscale.py:71-79
                if R.rescale_due(layer.sched):
                    R.rescale(p.detach().numpy(), layer.sched)           # autoscale.py:86-96
                layer.encode()                                           # next step's W codes


def seeded_init(model, seed: int, std: float = 0.02) -> None:
    """Device-independent initial parameters for a Llama model: parameter i
    (named_parameters order) is N(0, std^2) from a CPU torch generator seeded
    ``seed + i`` (1-D norm weights stay 1).  The GPU run and the CPU reference
    both start from these values, so a committed reference curve can be
    compared with a GPU run made later on another machine."""
    with torch.no_grad():
        for i, (_, p) in enumerate(model.named_parameters()):
            if p.dim() == 1:
                p.fill_(1.0)
                continue
            g = torch.Generator().manual_seed(seed + i)
            val = torch.randn(tuple(p.shape), generator=g, dtype=torch.float32) * std
            p.copy_(val.to(p.device, p.dtype))
            layer = getattr(p, "oracle_layer", None)
            if layer is not None:
                layer.init_from(val.numpy())


def reference_curve(cfg, *, steps: int, batch: int, seq: int, lr: float, warmup: int, data_seed: int,
                    init_seed: int, active: int | None = None, log=None) -> list:
    """The CPU float64 reference training run of ``cfg`` (a llama.LlamaConfig):
    every linear is an OracleMossLinear, the optimizer is OracleAdamW with the
    reference lr schedule (numpy_ref.lr_at = train.py:75-82), the data is
    MarkovTokens(cfg.vocab, data_seed, active=active)."""
    from paper_2511_05811_b200 import llama as L

    L._LINEAR_FACTORY = lambda c, i, o, d: OracleMossLinear(i, o, c.interval)
    try:
        ref = L.LlamaModel(L.LlamaConfig(**{**cfg.__dict__, "compute_dtype": torch.float64, "moss": True,
                                            "fused_ops": False}), device="cpu")
    finally:
        L._LINEAR_FACTORY = None
    ref = ref.double()
    seeded_init(ref, init_seed)
    sched = lambda t: R.lr_at(t, lr_peak=lr, warmup=warmup, steps=steps)
    opt = OracleAdamW(ref.named_parameters(), sched, 0.1, L.LlamaModel.no_decay)
    data = L.MarkovTokens(cfg.vocab, seed=data_seed, active=active)
    losses = []
    for step in range(steps):
        x, y = data.batch(batch, seq)
        opt.zero_grad()
        loss = ref(torch.as_tensor(x), torch.as_tensor(y))
        loss.backward()
        opt.step()
        losses.append(float(loss))
        if log is not None:
            log(step, losses[-1])
    return losses
