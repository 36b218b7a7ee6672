"""AdamW on the GPU — drop-in for mossq.optim's training functions
(reference optim.py:52-106).  The bound checkers (optim.py:109-212) are
offline analysis and are out of scope.

``adamw_step(w, g, state)`` keeps the reference's contract: returns
(w_next, state, delta), advances state in place, raises InvalidValueError
on a non-finite gradient before mutating anything.  The arithmetic is the
fused sm_100a kernel (K3) in FP32 with FP32 moments (the reference uses
float64; tests state the tolerance).  The training path uses the same kernel
through ``MossAdamW`` (nn.py), fused with the FP8 weight copy.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .errors import InvalidArgumentError, InvalidShapeError, InvalidValueError

__all__ = ["OptimizerState", "init_state", "adamw_step", "adam_params"]


@dataclass
class OptimizerState:
    m: torch.Tensor
    v: torch.Tensor
    t: int = 0
    beta1: float = 0.9
    beta2: float = 0.95
    eta: float = 1e-3
    weight_decay: float = 0.1
    eps: float = 1e-8
    decoupled_decay: bool = True


def init_state(shape, *, beta1: float = 0.9, beta2: float = 0.95, eta: float = 1e-3,
               weight_decay: float = 0.1, eps: float = 1e-8, decoupled_decay: bool = True,
               device="cuda") -> OptimizerState:
    """Zero moments at t = 0 (optim.py:65-75)."""
    if not (0.0 <= beta1 < 1.0 and 0.0 <= beta2 < 1.0):
        raise InvalidArgumentError("betas must lie in [0, 1)")
    shape = tuple(shape)
    return OptimizerState(m=torch.zeros(shape, dtype=torch.float32, device=device),
                          v=torch.zeros(shape, dtype=torch.float32, device=device), t=0, beta1=beta1,
                          beta2=beta2, eta=eta, weight_decay=weight_decay, eps=eps,
                          decoupled_decay=decoupled_decay)


def adam_params(lr: float, beta1: float, beta2: float, eps: float, weight_decay: float, t: int,
                decoupled: bool, grad_scale: float = 1.0) -> _lib.AdamParams:
    """Kernel hyper-parameters for step number t (>= 1); bias corrections in f64."""
    return _lib.AdamParams(lr=lr, beta1=beta1, beta2=beta2, eps=eps, weight_decay=weight_decay,
                           bc1=1.0 - beta1 ** t, bc2=1.0 - beta2 ** t, decoupled=int(decoupled),
                           grad_scale=grad_scale)


def _as_2d(t: torch.Tensor) -> tuple[int, int]:
    n = t.numel()
    if t.dim() == 2 and t.shape[1] % 8 == 0:
        return t.shape[0], t.shape[1]
    if n % 8 == 0:
        return 1, n
    raise InvalidShapeError("the fused AdamW kernel needs numel % 8 == 0")


def adamw_step(w, g, state: OptimizerState):
    """One AdamW step (optim.py:78-106) on the GPU; returns (w_next, state, delta)."""
    if not isinstance(w, torch.Tensor) or not w.is_cuda:
        w = torch.as_tensor(w, dtype=torch.float32, device="cuda")
    if not isinstance(g, torch.Tensor) or not g.is_cuda:
        g = torch.as_tensor(g, dtype=torch.float32, device="cuda")
    if tuple(w.shape) != tuple(g.shape) or tuple(w.shape) != tuple(state.m.shape):
        raise InvalidShapeError(f"shape mismatch: w{tuple(w.shape)} g{tuple(g.shape)} m{tuple(state.m.shape)}")
    if not bool(torch.isfinite(g).all()):
        raise InvalidValueError("gradient contains NaN/Inf")
    w_old = w.float()
    w_next = w_old.clone().contiguous()
    gf = g.contiguous() if g.dtype in (torch.float32, torch.bfloat16) else g.float().contiguous()
    rows, cols = _as_2d(w_next)
    state.t += 1
    p = adam_params(state.eta, state.beta1, state.beta2, state.eps, state.weight_decay, state.t,
                    state.decoupled_decay)
    flags = _lib.FlagWord(w.device)
    _lib.adamw_fp8(w_next, gf, state.m, state.v, rows, cols, p, 0.0, flags)
    delta = w_old - w_next
    if state.decoupled_decay and state.weight_decay != 0.0:
        delta = delta - state.eta * state.weight_decay * w_old
    return w_next, state, delta
