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

import gc
import math
from typing import Callable, Iterable

import numpy as np
import torch
from torch import nn

from . import _lib
from .autoscale import ScaleSchedule, auto_scale_advance, rescale_due
from .errors import InvalidArgumentError, InvalidShapeError
from .fp8 import E4M3
from .gemm import mx_gemm, mx_gemm_bkn
from .optim import adam_params
from .quantize import quantize_mx2

__all__ = ["MossLinearFunction", "MossLinear", "MossAdamW", "CudaGraphStep", "device_flags", "raise_if_flagged", "cosine_lr"]

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


# How each activation / output-gradient quantization got its tensor amax
# (("fwd" | "bwd"), ("producer" | "in_kernel")) -> count: evidence that the
# producer-fused amax reaches the quantizers (CudaGraphStep records the counts
# of its captured step).
QUANT_MODES: dict = {}


def _count_mode(where: str, amax) -> None:
    key = (where, "producer" if amax is not None else "in_kernel")
    QUANT_MODES[key] = QUANT_MODES.get(key, 0) + 1


class MossLinearFunction(torch.autograd.Function):
    """y = x W^T with MOSS FP8 forward, dgrad and wgrad (three tcgen05 GEMMs)."""

    # The FP32 master weight is an autograd input only so that autograd tracks
    # the dependency; its gradient is returned as None and instead written by
    # the wgrad GEMM straight into ``weight.main_grad`` (FP32, possibly a DP
    # bucket view), with no extra pass over the gradient.
    # ``amax`` (optional, device f32 [1]) is max|x| computed by the kernel that
    # produced x (producer-fused amax): the quantizer then skips its reduction.
    # ``dx_consumer`` (optional MossLinear): the layer that quantizes this layer's
    # dX as ITS output-gradient (e.g. through a residual add) — the dgrad GEMM then
    # writes max|dX| for it (the amax epilogue) and that quantizer skips its reduction.
    @staticmethod
    def forward(ctx, x: torch.Tensor, weight: torch.Tensor, layer: "MossLinear",
                amax: torch.Tensor | None = None, dx_consumer: "MossLinear | None" = None) -> torch.Tensor:
        k = x.shape[-1]
        n = layer.out_features
        x2d = _aligned_2d(x, k)
        if x2d.data_ptr() != x.data_ptr() or x2d.dtype != x.dtype:
            amax = None                                 # the quantized tensor is not the producer's
        need_w = weight.requires_grad
        flags = device_flags(x.device)
        fp8_bwd = layer.fp8_backward
        _count_mode("fwd", amax)
        op = quantize_mx2(x2d, row=True, col=need_w and fp8_bwd, flags=flags, amax=amax)
        y = mx_gemm(op.codes, op.sf, op.g, layer.w_fp8, None, layer.w_scale, out_dtype=torch.bfloat16)
        ctx.layer = layer
        ctx.dx_consumer = dx_consumer
        ctx.fp8_bwd = fp8_bwd
        if not fp8_bwd:
            # reference semantics (train.py:187-192): backward in full precision at the
            # unquantized activation and the FP32 master weight
            ctx.save_for_backward(x2d)
        ctx.need_w = need_w
        ctx.x_shape = x.shape
        ctx.x_dtype = x.dtype
        # FP8 activation stash: column-wise codes of X for wgrad (1 B/elem instead of bf16)
        ctx.x_t = (op.codes_t, op.sf_t, op.g) if (need_w and fp8_bwd) else None
        return y.view(*x.shape[:-1], n)

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        layer = ctx.layer
        n = layer.out_features
        need_x = ctx.needs_input_grad[0]
        if not ctx.fp8_bwd:
            return MossLinearFunction._backward_fp(ctx, dy, layer, need_x)
        dy2d = _aligned_2d(dy, n)
        flags = device_flags(dy.device)
        dy_amax = layer.take_dy_amax(dy2d)
        _count_mode("bwd", dy_amax)
        opd = quantize_mx2(dy2d, row=need_x, col=ctx.need_w, flags=flags, amax=dy_amax)
        dx = None
        if need_x:
            dx = torch.empty((dy2d.shape[0], layer.in_features), dtype=torch.bfloat16, device=dy.device)
            am = ctx.dx_consumer.offer_dy_amax(dx) if ctx.dx_consumer is not None else None
            mx_gemm_bkn(opd.codes, opd.sf, opd.g, layer.w_fp8, layer.w_scale, out=dx, amax_out=am)   # dY W, W as stored
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
        return dx, None, None, None, None

    @staticmethod
    def _backward_fp(ctx, dy, layer, need_x):
        (x2d,) = ctx.saved_tensors
        dy2d = dy.reshape(-1, layer.out_features)
        w = layer.weight
        dx = None
        if need_x:
            dx = (dy2d @ w.detach().to(dy2d.dtype)).view(ctx.x_shape).to(ctx.x_dtype)
        if ctx.need_w:
            gw = dy2d.t().float() @ x2d.float()
            if getattr(w, "main_grad", None) is None or getattr(w, "grad_fresh", True):
                if getattr(w, "main_grad", None) is None:
                    w.main_grad = torch.empty_like(w, dtype=torch.float32)
                w.main_grad.copy_(gw)
            else:
                w.main_grad.add_(gw)
            w.grad_fresh = False
            hook = getattr(w, "grad_ready_hook", None)
            if hook is not None:
                hook(w)
        layer.take_dy_amax(dy2d)
        return dx, None, None, None, None


class MossLinear(nn.Module):
    """FP8 (MOSS) linear layer, y = x W^T, no bias (Llama-style).

    Keeps the FP32 master weight as the Parameter and, as buffers, its E4M3
    copy (and transpose for dgrad) encoded at the schedule scale s_t, plus
    f32(s_t) on the device.  Weight gradients land in ``weight.main_grad``
    (FP32), written directly by the wgrad GEMM.
    """

    def __init__(self, in_features: int, out_features: int, bias: bool = False, device="cuda",
                 interval: int = 500, init_std: float | None = 0.02, fp8_backward: bool = True):
        super().__init__()
        self.fp8_backward = fp8_backward   # False: the reference's full-precision backward (train.py:187-192)
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
        self.register_buffer("w_scale", torch.ones(1, dtype=torch.float32, device=device), persistent=False)
        self.register_buffer("w_amax", torch.zeros(1, dtype=torch.float32, device=device), persistent=False)
        self.interval = interval
        self.schedule: ScaleSchedule | None = None
        # producer-fused amax of this layer's output-gradient (set by the
        # backward of the op that consumes our output, read by our backward)
        self.register_buffer("dy_amax", torch.zeros(1, dtype=torch.float32, device=device), persistent=False)
        self._dy_amax_ptr = None
        # set by zero.Zero1 when this weight's FP8 codes arrive by an async
        # all-gather: a callable that makes the current stream wait for them
        self.fp8_pending = None

    @property
    def w_fp8_t(self) -> torch.Tensor:
        """W_fp8^T as a view: no transposed copy is kept — the dgrad GEMM reads
        W_fp8 [out, in] as stored through an MN-major operand (gemm.mx_gemm_bkn)."""
        return self.w_fp8.t()

    def offer_dy_amax(self, dy: torch.Tensor) -> torch.Tensor:
        """Called by the producer of dY before it launches: returns the amax
        buffer to fill and remembers which tensor it describes."""
        self._dy_amax_ptr = (dy.data_ptr(), tuple(dy.shape))
        return self.dy_amax

    def take_dy_amax(self, dy2d: torch.Tensor) -> torch.Tensor | None:
        """The producer's amax if it describes exactly ``dy2d`` (else None)."""
        want, self._dy_amax_ptr = self._dy_amax_ptr, None
        if want is None or want[0] != dy2d.data_ptr() or dy2d.dtype != torch.bfloat16:
            return None
        n = 1
        for s in want[1]:
            n *= s
        return self.dy_amax if n == dy2d.numel() else None

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
        """W_fp8 = e4m3(f32(W)/f32(s_t)) (train.py:113-118), one launch."""
        s = float(np.float32(self.schedule.s_t))
        self.w_scale.fill_(s)
        _lib.encode_scaled(self.weight.detach(), device_flags(self.weight.device), scale_host=s, codes=self.w_fp8)

    def forward(self, x: torch.Tensor, amax: torch.Tensor | None = None,
                dx_consumer: "MossLinear | None" = None) -> torch.Tensor:
        """``amax``: max|x| from x's producer; ``dx_consumer``: the MossLinear that
        quantizes dX as its output-gradient (gets max|dX| from the dgrad epilogue)."""
        if self.schedule is None:
            self.init_fp8()
        if self.fp8_pending is not None:
            pending, self.fp8_pending = self.fp8_pending, None
            pending()
        return MossLinearFunction.apply(x, self.weight, self, amax, dx_consumer)

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

    A step is ``prepare()`` (host, O(1) per parameter: the schedule advance
    of autoscale.py:71-79, bias corrections, the per-parameter kernel
    arguments staged in a pinned ring and sent with ONE stream-ordered H2D
    copy) followed by ``launch()`` (the kernels, which read those arguments
    from device memory — so ``launch`` can be captured in a CUDA graph and
    replayed).  ``step()`` does both.  Rescale steps need the amax of the
    updated weights on the host and run eagerly (``launch(rescale=True)``).
    """

    _WORDS = 12            # moss_adam_params (10 words, word 9 = step) + enc scale (word 10), padded to 48 B
    _ENC = 10
    _RING = 8

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
        if not self.params:
            raise InvalidArgumentError("no trainable parameters")
        for p in self.params:
            if p.dtype != torch.float32:
                raise InvalidArgumentError("MossAdamW keeps FP32 master parameters")
            if p.numel() % 8:
                raise InvalidShapeError("parameter numel must be a multiple of 8")
            layer = getattr(p, "moss_layer", None)
            if layer is not None and layer.schedule is None:
                layer.init_fp8()                       # schedule_from_weights at t = 0
        self.wd_of = {id(p): (0.0 if (no_decay and no_decay(n, p)) else weight_decay) for n, p in named}
        self.lr, self.betas, self.eps = lr, betas, eps
        self.lr_schedule = lr_schedule
        self.decoupled = decoupled_decay
        self.t = 0
        self.grad_scale = 1.0
        dev = self.params[0].device
        intervals = {p.moss_layer.interval for p in self.params if hasattr(p, "moss_layer")}
        if len(intervals) > 1:
            # one rescale cadence per optimizer: rescale steps run eagerly and
            # CudaGraphStep decides eager-vs-replay from it (autoscale.py:82-96)
            raise InvalidArgumentError(f"MossLinear layers of one optimizer must share the rescale interval, "
                                       f"got {sorted(intervals)}")
        # moments are allocated at the first update (lazily), so parameters handed to
        # a sharded driver (zero.Zero1.shard) never hold full-size m, v
        self.state: dict[int, tuple | None] = {id(p): None for p in self.params}
        self.index = {id(p): i for i, p in enumerate(self.params)}
        self.sharded: set[int] = set()      # parameters whose update is done elsewhere (zero.Zero1)
        self.saturations = torch.zeros(1, dtype=torch.int32, device=dev)
        self.rescale_events: list[tuple[int, int]] = []
        n = len(self.params)
        self.hp_dev = torch.zeros(n * self._WORDS, dtype=torch.float32, device=dev)
        self.hp_pinned = torch.zeros(self._RING, n * self._WORDS, dtype=torch.float32).pin_memory()
        self._ring_events: list = [None] * self._RING
        self._slot = 0
        self._rescale_pending = False
        # host state before each step prepared since the last clean check():
        # restored when a device error gate skipped that step's update
        self._snapshots: dict[int, tuple] = {}

    def shard(self, params) -> None:
        """Hand the update of ``params`` to a sharded driver (zero.Zero1): their
        moments are not kept here, ``launch`` skips them; ``prepare`` still
        advances their schedules and stages their kernel arguments."""
        for p in params:
            self.sharded.add(id(p))
            self.state[id(p)] = None

    def record_ptr(self, p) -> int:
        """Device address of p's staged kernel arguments (moss_adam_params + encode scale)."""
        return self.hp_dev.data_ptr() + self.index[id(p)] * self._WORDS * 4

    def enc_ptr(self, p) -> int:
        """Device address of p's staged encode scale f32(s_{t+1})."""
        return self.record_ptr(p) + self._ENC * 4

    def _moss_layers(self):
        return [p.moss_layer for p in self.params if hasattr(p, "moss_layer")]

    def _snapshot(self) -> tuple:
        return (self.t, [(l.schedule.s_t, l.schedule.t, l.schedule.last_rescale_step) for l in self._moss_layers()])

    def _restore(self, snap: tuple) -> None:
        self.t = snap[0]
        for layer, (s_t, t, last) in zip(self._moss_layers(), snap[1]):
            layer.schedule.s_t, layer.schedule.t, layer.schedule.last_rescale_step = s_t, t, last
        self._rescale_pending = False

    def zero_grad(self, set_to_none: bool = True) -> None:
        for p in self.params:
            if hasattr(p, "moss_layer"):
                p.grad_fresh = True
            elif p.grad is not None:
                if set_to_none:
                    p.grad = None
                else:
                    p.grad.zero_()

    def current_lr(self) -> float:
        return self.lr_schedule(self.t) if self.lr_schedule is not None else self.lr

    def rescale_due_next(self) -> bool:
        """Will the coming step end with a rescale (autoscale.py:82-83)?"""
        for p in self.params:
            layer = getattr(p, "moss_layer", None)
            if layer is not None:
                sc = layer.schedule
                return (sc.t + 1) - sc.last_rescale_step >= sc.interval
        return False

    def prepare(self, lr: float | None = None) -> bool:
        """Host half of a step; returns True when this step must rescale (eager launch)."""
        eta = self.current_lr() if lr is None else lr
        self._snapshots[self.t + 1] = self._snapshot()
        if len(self._snapshots) > 1024:                # never checked: keep the recent ones
            self._snapshots.pop(min(self._snapshots))
        self.t += 1
        b1, b2 = self.betas
        bc1, bc2 = 1.0 - b1 ** self.t, 1.0 - b2 ** self.t
        slot = self._slot
        self._slot = (slot + 1) % self._RING
        ev = self._ring_events[slot]
        if ev is not None:
            ev.synchronize()                                   # the copy that last read this slot is done
        buf = self.hp_pinned[slot].numpy().reshape(-1, self._WORDS)
        ibuf = buf.view(np.uint32)
        buf[:, 0] = eta
        buf[:, 1] = b1
        buf[:, 2] = b2
        buf[:, 3] = self.eps
        buf[:, 5] = bc1
        buf[:, 6] = bc2
        ibuf[:, 7] = int(self.decoupled)
        buf[:, 8] = self.grad_scale
        ibuf[:, 9] = self.t                                    # recorded by K3 if its error gate skips
        rescale = False
        for i, p in enumerate(self.params):
            buf[i, 4] = self.wd_of[id(p)]
            layer = getattr(p, "moss_layer", None)
            if layer is not None:
                sched = layer.schedule
                auto_scale_advance(sched, eta)                 # O(1), autoscale.py:71-79
                rescale |= rescale_due(sched)
                buf[i, self._ENC] = np.float32(sched.s_t)
        self.hp_dev.copy_(self.hp_pinned[slot], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._ring_events[slot] = ev
        self._rescale_pending = rescale
        return rescale

    @torch.no_grad()
    def launch(self, rescale: bool | None = None) -> None:
        """Device half of a step: one fused kernel per parameter (graph-capturable when not rescaling)."""
        rescale = self._rescale_pending if rescale is None else rescale
        base = self.hp_dev.data_ptr()
        stride = self._WORDS * 4
        # gradients the error gate cannot vouch for — not made by an FP8 GEMM from
        # flag-checked operands — are checked BEFORE any update of the step, so a
        # non-finite one skips every K3 launch (optim.py:89-90 raises before mutating)
        for p in self.params:
            layer = getattr(p, "moss_layer", None)
            if layer is None and p.grad is not None:
                _lib.check_finite(p.grad, device_flags(p.device))
            elif layer is not None and not layer.fp8_backward and getattr(p, "main_grad", None) is not None:
                _lib.check_finite(p.main_grad, device_flags(p.device))
        for i, p in enumerate(self.params):
            if id(p) in self.sharded:
                continue
            layer = getattr(p, "moss_layer", None)
            g = p.main_grad if layer is not None else p.grad
            if g is None:
                continue
            st = self.state[id(p)]
            if st is None:
                st = self.state[id(p)] = (torch.zeros_like(p), torch.zeros_like(p))
            m, v = st
            flags = device_flags(p.device)
            p_dev = base + i * stride
            if layer is None:
                rows, cols = (p.shape[0], p.shape[1]) if p.dim() == 2 and p.shape[1] % 8 == 0 else (1, p.numel())
                _lib.adamw_fp8_dev(p.data, g, m, v, rows, cols, p_dev, None, flags)
                continue
            rows, cols = p.shape
            if rescale:
                _lib.adamw_fp8_dev(p.data, g, m, v, rows, cols, p_dev, None, flags, w_amax=layer.w_amax)
            else:
                _lib.adamw_fp8_dev(p.data, g, m, v, rows, cols, p_dev, p_dev + self._ENC * 4, flags,
                                   scale_out=layer.w_scale,
                                   w_fp8=layer.w_fp8, w_amax=layer.w_amax,
                                   n_saturated=self.saturations)
        if rescale:
            self._finish_rescale()

    def _finish_rescale(self) -> None:
        """JIT snap of every MOSS scale to max|W'|/448 and re-encode (autoscale.py:86-96)."""
        self.check("rescale step")          # a gated (skipped) update leaves no amax to snap to
        mine = [p for p in self.params if hasattr(p, "moss_layer") and id(p) not in self.sharded]
        if not mine:
            self._rescale_pending = False
            return
        # every layer's max|W'| in ONE device->host read (not one sync per layer)
        amaxes = torch.cat([p.moss_layer.w_amax.view(1) for p in mine]).cpu().tolist()
        for p, amax in zip(mine, amaxes):
            layer = p.moss_layer
            sched = layer.schedule
            sched.s_t = amax / E4M3.max_value if amax > 0 else 1.0
            sched.last_rescale_step = sched.t
            self.rescale_events.append((self.t, id(p)))
            layer.encode_weight()
        self._rescale_pending = False

    def step(self, lr: float | None = None) -> None:
        self.launch(self.prepare(lr))

    def check(self, where: str = "MossAdamW") -> None:
        """Raise pending device-side errors (non-finite grads/activations, E8M0 range).

        The error gate in K3 skipped every update from the first flagged step
        on, so before raising, the host half (step counter, scale schedules)
        is rolled back to its state before that step: host and device agree
        and the optimizer is exactly as it was after the last good step."""
        first = None
        bad = []
        for d in sorted({str(p.device) for p in self.params}):
            bits, skipped = device_flags(d).read()
            if bits:
                bad.append(d)
                if skipped != _lib.NO_STEP:
                    first = skipped if first is None else min(first, skipped)
        if bad:
            if first is not None and first in self._snapshots:
                self._restore(self._snapshots[first])
            self._snapshots.clear()
            for d in bad:
                raise_if_flagged(d, where)
        self._snapshots.clear()

    def dominance_violations(self) -> int:
        """s_auto < s_jit count over MOSS weights right now (train.py:163-167); syncs."""
        bad = 0
        for p in self.params:
            layer = getattr(p, "moss_layer", None)
            if layer is not None:
                jit = float(layer.w_amax.item()) / E4M3.max_value
                bad += int(layer.schedule.s_t < jit)
        return bad


class CudaGraphStep:
    """A whole training step (forward, backward, gradient exchange, fused
    optimizer kernels) captured once in a CUDA graph and replayed.

    ``step_fn(*inputs) -> loss`` must run forward + backward; the gradient
    exchange (``buckets``: dist.GradBuckets or zero.Zero1 — their NCCL
    collectives are captured on the comm stream, which forks from and joins
    the capture stream) and the optimizer's device half are captured after
    it.  Per replay the host only runs ``prepare()`` (O(1) per parameter + one
    H2D copy) and ``graph.replay()``.  Steps that end with a rescale (every
    ``interval`` steps) run eagerly, exactly like the uncaptured path.
    """

    def __init__(self, step_fn, opt: MossAdamW, static_inputs: tuple, zero_grad=None, buckets=None):
        self.fn, self.opt, self.inputs = step_fn, opt, static_inputs
        self.buckets = buckets
        if buckets is not None:
            if getattr(buckets, "overlap_gather", False):
                # a gather issued at the end of one replay and waited in the next
                # forward would be a dependency between two graph launches
                buckets.overlap_gather = False
            base = zero_grad or buckets.reset
        else:
            base = zero_grad or (lambda: opt.zero_grad(set_to_none=True))

        def zero_all():
            base()
            for t in self.inputs:                 # inputs that require grad (dX of the first layer)
                if isinstance(t, torch.Tensor) and t.requires_grad:
                    t.grad = None
        self.zero_grad = zero_all
        self.graph = None
        self.loss = None

    def _fwd_bwd(self) -> torch.Tensor:
        loss = self.fn(*self.inputs).detach()
        if self.buckets is not None:
            self.buckets.finish()
        return loss

    def _prepare(self) -> bool:
        b = self.buckets
        return b.prepare() if hasattr(b, "prepare") else self.opt.prepare()

    def _launch(self, rescale: bool) -> None:
        b = self.buckets
        b.launch(rescale) if hasattr(b, "launch") else self.opt.launch(rescale)

    def _capture(self) -> None:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        # warm-up on the capture stream (autograd / allocator state), as torch requires
        with torch.cuda.stream(s):
            for _ in range(2):                 # forward/backward only: no optimizer state change
                self.zero_grad()
                self._fwd_bwd()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        # No Python GC during the capture: a collection there can run the destructors of
        # stale objects (e.g. c10d Work handles of earlier eager collectives) whose CUDA
        # calls on the legacy stream invalidate the capture.  thread_local: other threads'
        # CUDA calls (the NCCL watchdog) do not count against this capture.
        gc.collect()
        gc_was_on = gc.isenabled()
        gc.disable()
        try:
            before = dict(QUANT_MODES)
            with torch.cuda.graph(self.graph, stream=s, capture_error_mode="thread_local"):
                # zeroing is part of the step: replays re-zero the bucket accumulators.
                # detached loss: the captured autograd graph (and the AccumulateGrad nodes bound to
                # this capture stream) must not outlive the capture, or a later capture of
                # the same model on another stream picks up a cross-stream dependency
                self.zero_grad()
                self.loss = self._fwd_bwd()
                self._launch(False)
            self.capture_quant_modes = {f"{w}/{m}": QUANT_MODES.get((w, m), 0) - before.get((w, m), 0)
                                        for (w, m) in QUANT_MODES}
        finally:
            if gc_was_on:
                gc.enable()
        torch.cuda.current_stream().wait_stream(s)

    def __call__(self, *inputs) -> torch.Tensor:
        with torch.no_grad():                       # static inputs may be leaves that require grad
            for dst, src in zip(self.inputs, inputs):
                if src is not dst:
                    dst.copy_(src, non_blocking=True)
        if self.opt.rescale_due_next() or self.graph is None:
            # eager step (rescale, or the step before the first capture)
            self.zero_grad()
            loss = self._fwd_bwd()                    # detached: drop the eager autograd graph
            self._launch(self._prepare())
            if self.graph is None:
                self._capture()
            return loss
        if self._prepare():
            raise RuntimeError("rescale due inside a replayed step")     # rescale_due_next() said no
        self.graph.replay()
        return self.loss


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
