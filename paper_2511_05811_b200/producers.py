"""Autograd wrappers of the producer kernels (csrc/producers.cu): the Llama
ops that make each FP8 linear's input and output-gradient, with the tensor
amax computed in the same pass (producer-fused amax).

Forward: RMSNorm -> (y, amax) feeds MossLinear(y, amax=...) of qkv / gate_up;
SwiGLU -> (h, amax) feeds the down projection.  Backward: each op writes
amax(dX) into the buffer of the MossLinear whose output-gradient dX is
(``consumer.offer_dy_amax``), so that layer's two-level quantizer runs in
producer-amax mode: one read of dY, no reduction pass.

The residual add is folded into the next RMSNorm (``AddRMSNormFn``):
x' = x + delta and y = norm(x') in one kernel; its backward adds the
residual-stream gradient into dx in the same kernel.
"""

from __future__ import annotations

import torch

from . import _lib

__all__ = ["RMSNormFn", "AddRMSNormFn", "SwiGLUFn", "RopeQKVFn", "CrossEntropyFn", "Sum3Fn", "AddFn",
           "MeanSquareFn"]


def _c2(t: torch.Tensor, d: int) -> torch.Tensor:
    t2 = t.reshape(-1, d)
    return t2 if t2.is_contiguous() else t2.contiguous()


def _amax_buf(consumer, out: torch.Tensor) -> torch.Tensor | None:
    return consumer.offer_dy_amax(out) if consumer is not None else None


class RMSNormFn(torch.autograd.Function):
    """y = norm(x) * w; returns (y, amax(y)).  ``consumer``: the MossLinear whose
    dY is dx (None when x's producer does not quantize its gradient)."""

    @staticmethod
    def forward(ctx, x, weight, eps: float, consumer):
        d = x.shape[-1]
        x2 = _c2(x, d)
        T = x2.shape[0]
        y = torch.empty_like(x2)
        rstd = torch.empty(T, dtype=torch.float32, device=x.device)
        amax = torch.empty(1, dtype=torch.float32, device=x.device)
        _lib.rmsnorm_fwd(x2, None, None, weight, eps, y, rstd, amax)
        ctx.save_for_backward(x2, weight, rstd)
        ctx.consumer, ctx.shape = consumer, x.shape
        ctx.mark_non_differentiable(amax)
        ctx.set_materialize_grads(False)     # no zero-filled gradient for the amax output
        return y.view(x.shape), amax

    @staticmethod
    def backward(ctx, dy, _damax):
        if dy is None:
            return None, None, None, None
        x2, weight, rstd = ctx.saved_tensors
        d = x2.shape[1]
        dx = torch.empty_like(x2)
        dw = torch.zeros_like(weight)
        _lib.rmsnorm_bwd(_c2(dy, d), x2, weight, rstd, None, dx, dw, _amax_buf(ctx.consumer, dx))
        return dx.view(ctx.shape), dw, None, None


class AddRMSNormFn(torch.autograd.Function):
    """x' = x + delta; y = norm(x') * w; returns (x', y, amax(y)).
    Backward: dx' (residual stream) + norm'(dy) -> the gradient of both x and
    delta; ``consumer`` is the MossLinear that produced delta (its dY)."""

    @staticmethod
    def forward(ctx, x, delta, weight, eps: float, consumer):
        d = x.shape[-1]
        x2, d2 = _c2(x, d), _c2(delta, d)
        T = x2.shape[0]
        xn = torch.empty_like(x2)
        y = torch.empty_like(x2)
        rstd = torch.empty(T, dtype=torch.float32, device=x.device)
        amax = torch.empty(1, dtype=torch.float32, device=x.device)
        _lib.rmsnorm_fwd(x2, d2, xn, weight, eps, y, rstd, amax)
        ctx.save_for_backward(xn, weight, rstd)
        ctx.consumer, ctx.shape = consumer, x.shape
        ctx.mark_non_differentiable(amax)
        ctx.set_materialize_grads(False)     # no zero-filled gradient for the amax output
        return xn.view(x.shape), y.view(x.shape), amax

    @staticmethod
    def backward(ctx, dxn, dy, _damax):
        if dxn is None and dy is None:
            return None, None, None, None, None
        xn, weight, rstd = ctx.saved_tensors
        d = xn.shape[1]
        dx = torch.empty_like(xn)
        dw = torch.zeros_like(weight)
        if dy is None:
            dy = torch.zeros_like(xn)
        _lib.rmsnorm_bwd(_c2(dy, d), xn, weight, rstd, None if dxn is None else _c2(dxn, d), dx, dw,
                         _amax_buf(ctx.consumer, dx))
        g = dx.view(ctx.shape)
        return g, g, dw, None, None


class SwiGLUFn(torch.autograd.Function):
    """gu = [gate | up] -> (h = silu(gate) * up, amax(h)); ``consumer`` is the
    gate_up MossLinear (its dY is dgu)."""

    @staticmethod
    def forward(ctx, gu, consumer):
        f2 = gu.shape[-1]
        gu2 = _c2(gu, f2)
        h = torch.empty(gu2.shape[0], f2 // 2, dtype=gu.dtype, device=gu.device)
        amax = torch.empty(1, dtype=torch.float32, device=gu.device)
        _lib.swiglu_fwd(gu2, h, amax)
        ctx.save_for_backward(gu2)
        ctx.consumer, ctx.shape = consumer, gu.shape
        ctx.mark_non_differentiable(amax)
        ctx.set_materialize_grads(False)     # no zero-filled gradient for the amax output
        return h.view(*gu.shape[:-1], f2 // 2), amax

    @staticmethod
    def backward(ctx, dh, _damax):
        if dh is None:
            return None, None
        (gu2,) = ctx.saved_tensors
        dgu = torch.empty_like(gu2)
        _lib.swiglu_bwd(_c2(dh, gu2.shape[1] // 2), gu2, dgu, _amax_buf(ctx.consumer, dgu))
        return dgu.view(ctx.shape), None


class RopeQKVFn(torch.autograd.Function):
    """qkv [B, S, 3*H*hd] -> q, k, v [B, H, S, hd] (q, k rotated).  Backward
    assembles dqkv with the inverse rotation; ``consumer`` is the qkv layer."""

    @staticmethod
    def forward(ctx, qkv, cos, sin, n_heads: int, consumer):
        B, S, three_d = qkv.shape
        hd = three_d // (3 * n_heads)
        qkv = qkv if qkv.is_contiguous() else qkv.contiguous()
        # q, k, v in [B, S, H, hd] memory, returned as [B, H, S, hd] views: SDPA then
        # leaves its output in that memory order and the O projection's input
        # (out.transpose(1, 2).reshape(B, S, d)) is a view, not a transpose copy
        q = torch.empty(B, S, n_heads, hd, dtype=qkv.dtype, device=qkv.device)
        k, v = torch.empty_like(q), torch.empty_like(q)
        _lib.rope_fwd(qkv, cos, sin, q, k, v, B, S, n_heads, hd, bshd=True)
        ctx.save_for_backward(cos, sin)
        ctx.dims, ctx.consumer = (B, S, n_heads, hd), consumer
        return q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2)

    @staticmethod
    def backward(ctx, dq, dk, dv):
        cos, sin = ctx.saved_tensors
        B, S, H, hd = ctx.dims

        def bshd(t):
            # [B, H, S, hd]-shaped gradient -> [B, S, H, hd] memory (a view when SDPA
            # produced it in that order, as it does for [B, S, H, hd]-strided inputs)
            if t is None:
                return torch.zeros(B, S, H, hd, dtype=torch.bfloat16, device=cos.device)
            tt = t.transpose(1, 2)
            return tt if tt.is_contiguous() else tt.contiguous()
        dq, dk, dv = bshd(dq), bshd(dk), bshd(dv)
        dqkv = torch.empty(B, S, 3 * H * hd, dtype=dq.dtype, device=dq.device)
        _lib.rope_bwd(dq, dk, dv, cos, sin, dqkv, _amax_buf(ctx.consumer, dqkv.view(B * S, -1)), B, S, H, hd,
                      bshd=True)
        return dqkv, None, None, None, None


class CrossEntropyFn(torch.autograd.Function):
    """mean_t (logsumexp(x_t) - x_t[y_t]) on bf16 logits [T, V] in f32 math,
    one read of the logits forward, one read + one bf16 write backward (the
    torch path materialises an f32 copy of the logits and an f32 gradient)."""

    @staticmethod
    def forward(ctx, logits, targets):
        V = logits.shape[-1]
        lg = _c2(logits, V)
        tg = targets.reshape(-1).contiguous()
        T = lg.shape[0]
        lse = torch.empty(T, dtype=torch.float32, device=lg.device)
        loss = torch.empty(T, dtype=torch.float32, device=lg.device)
        _lib.cross_entropy_fwd(lg, tg, lse, loss)
        ctx.save_for_backward(lg, tg, lse)
        ctx.shape = logits.shape
        return loss.mean()

    @staticmethod
    def backward(ctx, g):
        lg, tg, lse = ctx.saved_tensors
        scale = (g.float() / lg.shape[0]).reshape(1).contiguous()
        d = torch.empty_like(lg)
        _lib.cross_entropy_bwd(lg, tg, lse, scale, d)
        return d.view(ctx.shape), None


# ---------------------------------------------------------------- glue of the LayerStack benchmark workload
class Sum3Fn(torch.autograd.Function):
    """qkv [T, 3d] -> (q + k + v, amax); backward broadcasts da to [da, da, da]
    with amax for ``consumer`` (the qkv layer)."""

    @staticmethod
    def forward(ctx, qkv, consumer):
        d3 = qkv.shape[-1]
        x = _c2(qkv, d3)
        out = torch.empty(x.shape[0], d3 // 3, dtype=x.dtype, device=x.device)
        amax = torch.empty(1, dtype=torch.float32, device=x.device)
        _lib.glue(0, x, out, amax, T=x.shape[0], d=d3 // 3)
        ctx.consumer, ctx.shape = consumer, qkv.shape
        ctx.mark_non_differentiable(amax)
        ctx.set_materialize_grads(False)     # no zero-filled gradient for the amax output
        return out.view(*qkv.shape[:-1], d3 // 3), amax

    @staticmethod
    def backward(ctx, da, _):
        if da is None:
            return None, None
        d = ctx.shape[-1] // 3
        da2 = _c2(da, d)
        out = torch.empty(da2.shape[0], 3 * d, dtype=da2.dtype, device=da2.device)
        _lib.glue(1, da2, out, _amax_buf(ctx.consumer, out), T=da2.shape[0], d=d)
        return out.view(ctx.shape), None


class AddFn(torch.autograd.Function):
    """(x + y, amax(x + y)) in one pass; the gradient passes to both inputs."""

    @staticmethod
    def forward(ctx, x, y):
        d = x.shape[-1]
        x2, y2 = _c2(x, d), _c2(y, d)
        out = torch.empty_like(x2)
        amax = torch.empty(1, dtype=torch.float32, device=x.device)
        _lib.glue(2, x2, out, amax, y=y2, T=x2.shape[0], d=d)
        ctx.mark_non_differentiable(amax)
        ctx.set_materialize_grads(False)     # no zero-filled gradient for the amax output
        return out.view(x.shape), amax

    @staticmethod
    def backward(ctx, g, _):
        return g, g


class MeanSquareFn(torch.autograd.Function):
    """mean((y + b)^2) in f32 over a bf16 tensor (b: optional fixed bf16 offset of y's
    shape); backward dy = 2 (y + b) g / n (bf16) with amax for ``consumer`` (the layer
    that produced y)."""

    @staticmethod
    def forward(ctx, y, consumer, offset=None):
        d = y.shape[-1]
        y2 = _c2(y, d)
        b2 = _c2(offset, d) if offset is not None else None
        acc = torch.empty(1 + _lib.SUMSQ_PARTIALS, dtype=torch.float32, device=y.device)
        _lib.sumsq(y2, acc, scale=1.0 / y2.numel(), offset=b2)   # the mean, in-kernel (no torch scalar op)
        ctx.save_for_backward(y2)
        ctx.b2, ctx.consumer, ctx.shape = b2, consumer, y.shape
        return acc[0]

    @staticmethod
    def backward(ctx, g):
        (y2,) = ctx.saved_tensors
        g = g if g.dtype == torch.float32 else g.float()
        dy = torch.empty_like(y2)
        # dy = (y + b) * f32(g * 2/n), the factor formed in-kernel from the incoming gradient
        _lib.glue(3, y2, dy, _amax_buf(ctx.consumer, dy), y=ctx.b2, scale=g.contiguous(), alpha=2.0 / y2.numel(),
                  T=y2.shape[0], d=y2.shape[1])
        return dy.view(ctx.shape), None, None
