"""Training loop for the Llama workloads: the step ordering of train.py:151-203
(forward with FP8 weights encoded at s_t, backward, AdamW, scale advance /
rescale) driven through MossLinear + MossAdamW, with an optional DP gradient
exchange (dist.GradBuckets)."""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import TrainDivergedError
from .llama import LlamaModel, MarkovTokens
from .nn import MossAdamW, cosine_lr


@dataclass
class TrainLog:
    loss: list = field(default_factory=list)
    lr: list = field(default_factory=list)
    step_ms: list = field(default_factory=list)

    def smoothed(self, window: int = 20) -> np.ndarray:
        """Trailing moving average (train.py:85-94)."""
        s = np.asarray(self.loss, dtype=np.float64)
        c = np.cumsum(s)
        out = np.empty_like(s)
        for i in range(len(s)):
            lo = max(0, i - window + 1)
            out[i] = (c[i] - (c[lo - 1] if lo else 0.0)) / (i - lo + 1)
        return out


def make_optimizer(model: LlamaModel, lr: float, steps: int, warmup: int, weight_decay: float = 0.1):
    return MossAdamW(model, lr=lr, betas=(0.9, 0.95), eps=1e-8, weight_decay=weight_decay,
                     lr_schedule=cosine_lr(lr, warmup, steps), no_decay=LlamaModel.no_decay)


def train(model: LlamaModel, data: MarkovTokens, *, steps: int, batch: int, seq: int, lr: float = 1e-3,
          warmup: int = 20, weight_decay: float = 0.1, buckets=None, divergence_threshold: float = 1e6,
          check_every: int = 1, cuda_graph: bool = False) -> TrainLog:
    """``cuda_graph=True`` captures forward + backward + the gradient exchange
    (``buckets``) + the optimizer kernels once and replays the graph each step
    (nn.CudaGraphStep); rescale steps run eagerly."""
    opt = make_optimizer(model, lr, steps, warmup, weight_decay)
    if callable(buckets):                            # a factory: e.g. lambda opt: Zero1(opt)
        buckets = buckets(opt)
    if buckets is not None:
        opt.grad_scale = buckets.grad_scale
    dev = next(model.parameters()).device
    log = TrainLog()
    graphed = None
    if cuda_graph:
        from .nn import CudaGraphStep
        sx = torch.zeros((batch, seq), dtype=torch.long, device=dev)
        sy = torch.zeros((batch, seq), dtype=torch.long, device=dev)

        def fb(xt, yt):
            loss = model(xt, yt)
            loss.backward()
            return loss
        # the gradient exchange (all-reduce buckets or ZeRO-1) is captured with the step
        graphed = CudaGraphStep(fb, opt, (sx, sy), buckets=buckets)
    for step in range(steps):
        x, y = data.batch(batch, seq)
        xt = torch.as_tensor(x, device=dev)
        yt = torch.as_tensor(y, device=dev)
        log.lr.append(opt.current_lr())
        if graphed is not None:
            loss = graphed(xt, yt)
        else:
            if buckets is not None:
                buckets.reset()
            else:
                opt.zero_grad()
            loss = model(xt, yt)
            loss.backward()
            if buckets is not None:
                buckets.finish()
            if hasattr(buckets, "step"):
                buckets.step()                       # zero.Zero1: sharded update + FP8 all-gather
            else:
                opt.step()
        lv = float(loss.detach())
        if step % check_every == 0:
            opt.check(f"step {step}")
        if not math.isfinite(lv) or lv > divergence_threshold:
            raise TrainDivergedError(f"loss {lv} at step {step}")
        log.loss.append(lv)
    if hasattr(buckets, "sync"):
        buckets.sync()                               # land the last step's overlapped FP8 all-gathers
    return log
