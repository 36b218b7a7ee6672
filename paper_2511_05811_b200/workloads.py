"""Benchmark / parity workloads built only from the public training API.

``LayerStack`` is BASELINE config 2 as a training step: the five Llama-7B
linear shapes of one decoder layer (QKV 4096->12288, O 4096->4096,
gate/up 4096->2x11008 fused, down 11008->4096) at M tokens, chained with
cheap bf16 glue so that every linear sees a real forward input and a real
backward gradient:

    qkv = QKV(x); a = q + k + v              (stand-in for attention mixing)
    r = x + O(a); h = silu(gate(r)) * up(r); y = down(h); loss = mean((y + b)^2)

b is a fixed N(0, 1) bf16 offset (seeded, one per input shape): the optimum is
y = -b, not y = 0.  With plain mean(y^2) the stack learns to output zero, its
output-gradients shrink step after step and, after ~200 steps, span more binades
than E8M0 can (a block max below g 2^-127: the reference's E8m0RangeError); the
offset keeps the gradient statistics stationary over any number of steps.

The glue ops are producer kernels (producers.py) as in the Llama decoder:
each writes the amax of the tensor it makes, so the quantizers of a/r/h (fwd)
and of the qkv/gate_up/down output-gradients run in producer-amax mode (one
read, no reduction); o's output-gradient is the gate_up dgrad GEMM's output,
whose amax comes from the GEMM epilogue.  Only x (the step's input) is
quantized with the in-kernel amax.

The residual branch does not back-propagate into the step input x (x's
gradient is the QKV dgrad only): no autograd add of two gradient paths, so
every kernel of the step is one of ours (bench.py lists the rest).

One step = forward + backward (FP8 fwd/dgrad/wgrad for every linear, each
input and gradient two-level quantized row- and column-wise) + MossAdamW
(fused update + autoscale + FP8 weight copy).  GEMM FLOPs per step:
6 * M * sum(N*K) = 6 * M * 202.4M.
"""

from __future__ import annotations

import torch
from torch import nn

from .nn import MossLinear
from .producers import AddFn, MeanSquareFn, Sum3Fn, SwiGLUFn

LLAMA7B_SHAPES = {"qkv": (4096, 12288), "o": (4096, 4096), "gate_up": (4096, 22016), "down": (11008, 4096)}


class LayerStack(nn.Module):
    def __init__(self, d_model: int = 4096, d_ffn: int = 11008, device="cuda", interval: int = 500,
                 loss_offset: bool = True):
        super().__init__()
        self.d, self.f = d_model, d_ffn
        self.qkv = MossLinear(d_model, 3 * d_model, device=device, interval=interval)
        self.o = MossLinear(d_model, d_model, device=device, interval=interval)
        self.gate_up = MossLinear(d_model, 2 * d_ffn, device=device, interval=interval)
        self.down = MossLinear(d_ffn, d_model, device=device, interval=interval)
        self._offsets: dict = {}
        self.loss_offset = loss_offset      # False: plain mean(y^2) (short runs only, see above)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        a, am = Sum3Fn.apply(self.qkv(x), self.qkv)              # a = q + k + v
        # residual r = x + O(a); its gradient is not propagated back into the step
        # input (x's gradient is the qkv dgrad alone), so no autograd sum of the two
        # paths runs: every kernel of the step is one of ours
        r, am = AddFn.apply(x.detach(), self.o(a, am))
        # gate_up's dX is O's output-gradient (AddFn passes it through): the dgrad
        # epilogue hands O its amax
        h, am = SwiGLUFn.apply(self.gate_up(r, am, dx_consumer=self.o), self.gate_up)
        b = self.offset(x) if self.loss_offset else None
        return MeanSquareFn.apply(self.down(h, am), self.down, b)    # mean((y + b)^2)

    def offset(self, x: torch.Tensor) -> torch.Tensor:
        """The loss offset b for x's shape: N(0, 1) bf16 from a fixed seed, made once."""
        key = (tuple(x.shape), x.device)
        b = self._offsets.get(key)
        if b is None:
            if x.is_cuda and torch.cuda.is_current_stream_capturing():
                raise RuntimeError("LayerStack: run one eager step at this input shape before graph capture")
            g = torch.Generator(device=x.device).manual_seed(2718)
            b = torch.randn(*x.shape[:-1], self.d, device=x.device, generator=g).to(torch.bfloat16)
            self._offsets[key] = b
        return b

    def gemm_flops_per_token(self) -> int:
        return 6 * sum(m.in_features * m.out_features for m in (self.qkv, self.o, self.gate_up, self.down))
