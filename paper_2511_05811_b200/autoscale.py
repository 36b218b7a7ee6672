"""Automatic per-tensor weight scaling — drop-in for mossq.autoscale's
training functions (reference autoscale.py:36-96).  ``interval_sweep``
(autoscale.py:99-148) is an offline ablation and out of scope.

The schedule stays a host-side O(1) object, exactly as in the reference:
``auto_scale_advance`` touches no weight data (autoscale.py:71-79).  The only
device work is the rescale max-reduction every ``interval`` steps
(autoscale.py:86-96), done by the K0 amax kernel (or fused into K3).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch

from . import _lib
from .errors import InvalidArgumentError, InvalidValueError
from .fp8 import Fp8Format
from .quantize import PerTensorQuant, quant_per_tensor

__all__ = ["ScaleSchedule", "schedule_from_weights", "jit_scale", "auto_scale_advance", "rescale_due",
           "rescale_interval"]


@dataclass
class ScaleSchedule:
    s0: float
    s_t: float
    t: int
    interval: int
    delta_max: float
    last_rescale_step: int = 0
    eta_schedule: Callable[[int], float] | None = None

    def __post_init__(self):
        if self.interval < 1:
            raise InvalidArgumentError("interval must be >= 1")
        if self.s0 <= 0.0 or self.s_t <= 0.0:
            raise InvalidValueError("scales must be positive")


def device_amax(w: torch.Tensor) -> torch.Tensor:
    """max|w| as a 1-element f32 device tensor (K0); raises on NaN/Inf."""
    x = w.detach()
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.float()
    x = x.contiguous().reshape(-1)
    if x.data_ptr() % 16:
        x = x.clone()
    out = torch.empty(1, dtype=torch.float32, device=x.device)
    flags = _lib.FlagWord(x.device)
    _lib.amax(x, out, flags)
    flags.raise_if_set("jit_scale")
    return out


def jit_scale(w, fmt: Fp8Format) -> float:
    """max|w| / max_value, 1.0 for all-zero w (autoscale.py:53-59)."""
    if not isinstance(w, torch.Tensor) or not w.is_cuda:
        w = torch.as_tensor(w, device="cuda")
    try:
        amax = float(device_amax(w).item())
    except Exception as e:
        raise InvalidValueError("jit_scale requires finite weights") from e
    return amax / fmt.max_value if amax > 0.0 else 1.0


def schedule_from_weights(w, fmt: Fp8Format, interval: int = 500,
                          eta_schedule: Callable[[int], float] | None = None) -> ScaleSchedule:
    """The one max-reduction at t = 0 (autoscale.py:62-68)."""
    s0 = jit_scale(w, fmt)
    return ScaleSchedule(s0=s0, s_t=s0, t=0, interval=interval, delta_max=fmt.max_value,
                         last_rescale_step=0, eta_schedule=eta_schedule)


def auto_scale_advance(sched: ScaleSchedule, current_eta: float | None = None) -> ScaleSchedule:
    """s += eta / max_value; t += 1.  O(1), no weight data (autoscale.py:71-79)."""
    if current_eta is None:
        if sched.eta_schedule is None:
            raise InvalidArgumentError("no eta given and schedule has no eta_schedule")
        current_eta = sched.eta_schedule(sched.t)
    sched.s_t += current_eta / sched.delta_max
    sched.t += 1
    return sched


def rescale_due(sched: ScaleSchedule) -> bool:
    return sched.t - sched.last_rescale_step >= sched.interval


def rescale_interval(w, sched: ScaleSchedule, fmt: Fp8Format) -> PerTensorQuant:
    """Snap s_t to the JIT value of w and re-encode (autoscale.py:86-96)."""
    if not rescale_due(sched):
        raise InvalidArgumentError(
            f"rescale not due: t={sched.t}, last={sched.last_rescale_step}, interval={sched.interval}")
    if fmt.max_value != sched.delta_max:
        raise InvalidArgumentError("format does not match the schedule's delta_max")
    sched.s_t = jit_scale(w, fmt)
    sched.last_rescale_step = sched.t
    return quant_per_tensor(w if isinstance(w, torch.Tensor) else torch.as_tensor(w, dtype=torch.float32), fmt)
