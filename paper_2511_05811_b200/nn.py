"""Torch training wrappers for the MOSS hot path: the FP8 linear autograd
function and the auto-scaling AdamW optimizer (BASELINE.json north_star).

The reference has no torch layer; its training semantics are the step loop
of train.py:151-203, which these wrappers reproduce:
  * forward: activations two-level quantized (quant_two_level, train.py:171),
    weights encoded per tensor at the schedule scale s_t current at the start
    of the step (train.py:168);
  * the FP8 GEMMs apply block scales in the tensor core and the global
    scales in the epilogue (gemm.py:115-129);
  * optimizer: AdamW (optim.py:78-106), then s <- s + eta/448
    (autoscale.py:71-79) and a JIT rescale every ``interval`` steps
    (autoscale.py:82-96).  K3 fuses the update with the FP8 weight copy at
    s_{t+1}, which is exactly what the next forward needs.
The backward runs in FP8 too (north_star (2)): dgrad = Q(dY) . W (W codes
transposed by K3), wgrad = Q(dY^T) . Q(X^T) (column-wise codes of X stashed
by the forward instead of the bf16 activation).  The reference backward is
full precision (train.py:187-192); see DESIGN.md for the composed oracle.

Errors: data-dependent conditions accumulate in a device flag word per
device; ``MossAdamW.check()`` (or ``raise_if_flagged``) raises the
reference's exception classes at the step boundary.
"""

from __future__ import annotations

import math
from typing import Callable, Iterable

import numpy as np
import torch
from torch import nn

from . import _lib
from .autoscale import ScaleSchedule, auto_scale_advance, rescale_due
from .errors import InvalidArgumentError, InvalidShapeError
from .fp8 import E4M3
from .gemm import mx_gemm
from .optim import adam_params
from .quantize import quantize_mx2

__all__ = ["MossLinearFunction", "MossLinear", "MossAdamW", "device_flags", "raise_if_flagged"]

_FLAGS: dict[str, _lib.FlagWord] = {}


def device_flags(device) -> _lib.FlagWord:
    key = str(torch.device(device))
    if key not in _FLAGS:
        _FLAGS[key] = _lib.FlagWord(device)
    return _FLAGS[key]


def raise_if_flagged(device="cuda", where: str = "") -> None:
    fw = device_flags(device)
    try:
        fw.raise_if_set(where)
    finally:
        fw.reset()


def _aligned_2d(x: torch.Tensor, k: int) -> torch.Tensor:
    x2 = x.reshape(-1, k)
    if x2.dtype != torch.bfloat16 and x2.dtype != torch.float32:
        x2 = x2.to(torch.bfloat16)
    if not x2.is_contiguous() or x2.data_ptr() % 16:
        x2 = x2.contiguous().clone() if x2.data_ptr() % 16 else x2.contiguous()
    return x2


class MossLinearFunction(torch.autograd.Function):
    """y = x W^T with MOSS FP8 forward, dgrad and wgrad (three tcgen05 GEMMs)."""

    @staticmethod
    def forward(ctx, x: torch.Tensor, weight: torch.Tensor, layer: "MossLinear") -> torch.Tensor:
        k = x.shape[-1]
        n = layer.out_features
        x2d = _aligned_2d(x, k)
        need_w = weight.requires_grad
        flags = device_flags(x.device)
        op = quantize_mx2(x2d, row=True, col=need_w, flags=flags)
        y = mx_gemm(op.codes, op.sf, op.g, layer.w_fp8, None, layer.w_scale, out_dtype=torch.bfloat16)
        ctx.layer = layer
        ctx.need_w = need_w
        ctx.x_shape = x.shape
        ctx.x_dtype = x.dtype
        # FP8 activation stash: column-wise codes of X for wgrad (1 B/elem instead of bf16)
        ctx.x_t = (op.codes_t, op.sf_t, op.g) if need_w else None
        return y.view(*x.shape[:-1], n)

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        layer = ctx.layer
        n = layer.out_features
        need_x = ctx.needs_input_grad[0]
        dy2d = _aligned_2d(dy, n)
        flags = device_flags(dy.device)
        opd = quantize_mx2(dy2d, row=need_x, col=ctx.need_w, flags=flags)
        dx = None
        if need_x:
            dx = mx_gemm(opd.codes, opd.sf, opd.g, layer.w_fp8_t, None, layer.w_scale, out_dtype=torch.bfloat16)
            dx = dx.view(ctx.x_shape)
            if dx.dtype != ctx.x_dtype:
                dx = dx.to(ctx.x_dtype)
        if ctx.need_w:
            xc_t, xsf_t, xg = ctx.x_t
            w = layer.weight
            if getattr(w, "main_grad", None) is None:
                w.main_grad = torch.empty_like(w, dtype=torch.float32)
                w.grad_fresh = True
            mx_gemm(opd.codes_t, opd.sf_t, opd.g, xc_t, xsf_t, xg, out=w.main_grad,
                    accumulate=not getattr(w, "grad_fresh", True))
            w.grad_fresh = False
            ctx.x_t = None
            hook = getattr(w, "grad_ready_hook", None)
            if hook is not None:
                hook(w)
        return dx, None, None


class MossLinear(nn.Module):
    """FP8 (MOSS) linear layer, y = x W^T, no bias (Llama-style).

    Keeps the FP32 master weight as the Parameter and, as buffers, its E4M3
    copy (and transpose for dgrad) encoded at the schedule scale s_t, plus
    f32(s_t) on the device.  Weight gradients land in ``weight.main_grad``
    (FP32), written directly by the wgrad GEMM.
    """

    def __init__(self, in_features: int, out_features: int, bias: bool = False, device="cuda",
                 interval: int = 500, init_std: float | None = 0.02):
        super().__init__()
        if bias:
            raise InvalidArgumentError("MossLinear has no bias (Llama-style linears)")
        if in_features % 32 or out_features % 32:
            raise InvalidShapeError("in/out features must be multiples of 32")
        self.in_features, self.out_features = in_features, out_features
        w = torch.empty(out_features, in_features, dtype=torch.float32, device=device)
        if init_std is not None:
            w.normal_(0.0, init_std)
        self.weight = nn.Parameter(w)
        self.weight.moss_layer = self
        self.register_buffer("w_fp8", torch.zeros(out_features, in_features, dtype=torch.uint8, device=device),
                             persistent=False)
        self.register_buffer("w_fp8_t", torch.zeros(in_features, out_features, dtype=torch.uint8, device=device),
                             persistent=False)
        self.register_buffer("w_scale", torch.ones(1, dtype=torch.float32, device=device), persistent=False)
        self.register_buffer("w_amax", torch.zeros(1, dtype=torch.float32, device=device), persistent=False)
        self.interval = interval
        self.schedule: ScaleSchedule | None = None

    @torch.no_grad()
    def init_fp8(self) -> None:
        """schedule_from_weights (autoscale.py:62-68) + the t=0 weight encode."""
        flags = device_flags(self.weight.device)
        amax = self.w_amax
        _lib.amax(self.weight.detach(), amax, flags)
        s0 = float(amax.item())
        s0 = s0 / E4M3.max_value if s0 > 0 else 1.0
        self.schedule = ScaleSchedule(s0=s0, s_t=s0, t=0, interval=self.interval, delta_max=E4M3.max_value)
        self.encode_weight()

    @torch.no_grad()
    def encode_weight(self) -> None:
        """W_fp8 = e4m3(f32(W)/f32(s_t)) (train.py:113-118) + transpose, one launch."""
        s = float(np.float32(self.schedule.s_t))
        self.w_scale.fill_(s)
        _lib.encode_scaled(self.weight.detach(), device_flags(self.weight.device), scale_host=s,
                           codes=self.w_fp8, codes_t=self.w_fp8_t if self.out_features % 32 == 0 else None)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if self.schedule is None:
            self.init_fp8()
        return MossLinearFunction.apply(x, self.weight, self)

    def extra_repr(self) -> str:
        return f"in_features={self.in_features}, out_features={self.out_features}, fp8=e4m3(mx2 act, per-tensor W)"


class MossAdamW:
    """AdamW with MOSS automatic weight scaling (optim.py + autoscale.py),
    one fused kernel launch per parameter per step.

    MossLinear weights: update + s_{t+1} = s_t + eta/448 + FP8 copy (and
    transpose) at s_{t+1}; every ``interval`` steps the scale snaps to
    max|W|/448 (one amax read-back) and the copy is re-encoded.
    Other parameters (embeddings, norms, head): the same kernel, no copy.
    Gradients: ``p.main_grad`` for MossLinear weights, ``p.grad`` otherwise
    (both FP32); ``grad_scale`` multiplies them (DP averaging).
    """

    def __init__(self, params: Iterable[nn.Parameter] | nn.Module, lr: float = 3e-4,
                 betas: tuple[float, float] = (0.9, 0.95), eps: float = 1e-8, weight_decay: float = 0.1,
                 lr_schedule: Callable[[int], float] | None = None, decoupled_decay: bool = True,
                 no_decay: Callable[[str, nn.Parameter], bool] | None = None):
        if isinstance(params, nn.Module):
            named = list(params.named_parameters())
        else:
            named = [(f"p{i}", p) for i, p in enumerate(params)]
        if not (0.0 <= betas[0] < 1.0 and 0.0 <= betas[1] < 1.0):
            raise InvalidArgumentError("betas must lie in [0, 1)")
        self.params = [p for _, p in named if p.requires_grad]
        for p in self.params:
            if p.dtype != torch.float32:
                raise InvalidArgumentError("MossAdamW keeps FP32 master parameters")
            if p.numel() % 8:
                raise InvalidShapeError("parameter numel must be a multiple of 8")
        self.wd_of = {id(p): (0.0 if (no_decay and no_decay(n, p)) else weight_decay) for n, p in named}
        self.lr, self.betas, self.eps = lr, betas, eps
        self.lr_schedule = lr_schedule
        self.decoupled = decoupled_decay
        self.t = 0
        self.grad_scale = 1.0
        self.state = {id(p): (torch.zeros_like(p), torch.zeros_like(p)) for p in self.params}
        self.saturations = torch.zeros(1, dtype=torch.int32, device=self.params[0].device) if self.params else None
        self.rescale_events: list[tuple[int, int]] = []

    def zero_grad(self) -> None:
        for p in self.params:
            if hasattr(p, "moss_layer"):
                p.grad_fresh = True
            elif p.grad is not None:
                p.grad = None

    def current_lr(self) -> float:
        return self.lr_schedule(self.t) if self.lr_schedule is not None else self.lr

    @torch.no_grad()
    def step(self, lr: float | None = None) -> None:
        eta = self.current_lr() if lr is None else lr
        self.t += 1
        b1, b2 = self.betas
        for p in self.params:
            layer = getattr(p, "moss_layer", None)
            g = p.main_grad if layer is not None else p.grad
            if g is None:
                continue
            m, v = self.state[id(p)]
            hp = adam_params(eta, b1, b2, self.eps, self.wd_of[id(p)], self.t, self.decoupled, self.grad_scale)
            flags = device_flags(p.device)
            if layer is None:
                rows, cols = (p.shape[0], p.shape[1]) if p.dim() == 2 and p.shape[1] % 8 == 0 else (1, p.numel())
                _lib.adamw_fp8(p.data, g, m, v, rows, cols, hp, 0.0, flags)
                continue
            sched = layer.schedule
            auto_scale_advance(sched, eta)                       # O(1), autoscale.py:71-79
            rows, cols = p.shape
            if rescale_due(sched):                               # autoscale.py:82-96
                _lib.adamw_fp8(p.data, g, m, v, rows, cols, hp, 0.0, flags, w_amax=layer.w_amax)
                amax = float(layer.w_amax.item())
                sched.s_t = amax / E4M3.max_value if amax > 0 else 1.0
                sched.last_rescale_step = sched.t
                self.rescale_events.append((self.t, id(p)))
                layer.encode_weight()
            else:
                s = float(np.float32(sched.s_t))
                _lib.adamw_fp8(p.data, g, m, v, rows, cols, hp, s, flags, w_fp8=layer.w_fp8,
                               w_fp8_t=layer.w_fp8_t, w_amax=layer.w_amax, n_saturated=self.saturations)
                layer.w_scale.fill_(s)

    def check(self, where: str = "MossAdamW") -> None:
        """Raise pending device-side errors (non-finite grads/activations, E8M0 range)."""
        devs = {str(p.device) for p in self.params}
        for d in devs:
            raise_if_flagged(d, where)

    def dominance_violations(self) -> int:
        """s_auto < s_jit count over MOSS weights right now (train.py:163-167); syncs."""
        bad = 0
        for p in self.params:
            layer = getattr(p, "moss_layer", None)
            if layer is not None:
                jit = float(layer.w_amax.item()) / E4M3.max_value
                bad += int(layer.schedule.s_t < jit)
        return bad


def cosine_lr(peak: float, warmup: int, total: int, floor_frac: float = 0.1) -> Callable[[int], float]:
    """lr_at of train.py:75-82 as a schedule for MossAdamW."""
    def f(step: int) -> float:
        if step < warmup:
            return peak * (step + 1) / warmup
        span = max(1, total - warmup)
        progress = min(1.0, (step - warmup) / span)
        floor = peak * floor_frac
        return floor + 0.5 * (peak - floor) * (1.0 + math.cos(math.pi * progress))
    return f
