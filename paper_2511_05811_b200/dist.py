"""Data-parallel gradient exchange: bucketed all-reduce overlapped with backward
(BASELINE.json north_star (4)).

The reference is single-process (train.py); the paper trained
with FSDP/ZeRO-2 on 8xH200.  Here every rank holds the full
FP32 master weights, quantizes its own activations (per-rank global amax,
a documented semantic difference from the single-GPU global batch) and
exchanges FP32 gradients once per step:

  * gradients live in flat FP32 bucket buffers (~``bucket_mb`` each),
    filled in reverse layer order; MossLinear wgrad GEMMs write straight into
    them (``weight.main_grad`` is a bucket view), other parameters get
    ``param.grad`` as a bucket view (autograd accumulates in place);
  * when the last gradient of a bucket is produced, the bucket's all-reduce
    (SUM) is launched on a dedicated communication stream, ordered after the
    producing kernels with a CUDA event, so it overlaps the rest of backward;
  * ``finish()`` makes the compute stream wait for all buckets; the 1/world
    average is fused into the optimizer kernel (MossAdamW.grad_scale).

W, m, v, s_t and the FP8 weight copies stay bit-identical across ranks:
they are deterministic functions of the all-reduced gradients and of eta.
Works with NCCL (CUDA tensors, comm stream) and gloo (CPU tensors, tests).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch
import torch.distributed as dist
from torch import nn

__all__ = ["GradBuckets"]


@dataclass
class _Bucket:
    buf: torch.Tensor
    params: list = field(default_factory=list)
    pending: int = 0
    work: object = None
    launched: bool = False


class GradBuckets:
    def __init__(self, params, bucket_mb: float = 64.0, group=None, always_communicate: bool = False):
        if isinstance(params, nn.Module):
            params = list(params.parameters())
        self.params = [p for p in params if p.requires_grad]
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        # world 1 normally skips the collectives; tests force them (NCCL world 1 under graph capture)
        self.communicate = self.world > 1 or (always_communicate and dist.is_initialized())
        dev = self.params[0].device
        self.cuda = dev.type == "cuda"
        self.comm_stream = torch.cuda.Stream(device=dev) if self.cuda else None
        cap = int(bucket_mb * 1024 * 1024 // 4)
        self.buckets: list[_Bucket] = []
        self.bucket_of: dict[int, _Bucket] = {}
        # reverse registration order == the order backward produces gradients
        cur: list = []
        size = 0
        for p in reversed(self.params):
            cur.append(p)
            size += p.numel()
            if size >= cap:
                self._make_bucket(cur, size, dev)
                cur, size = [], 0
        if cur:
            self._make_bucket(cur, size, dev)
        self.timing = False                 # bench: CUDA events around each bucket's all-reduce
        self.comm_events: list = []
        self._hooks = []
        for p in self.params:
            if hasattr(p, "moss_layer"):
                p.grad_ready_hook = self._ready
            else:
                self._hooks.append(p.register_post_accumulate_grad_hook(self._ready))
        self.reset()

    def _make_bucket(self, plist, size, dev):
        buf = torch.zeros(size, dtype=torch.float32, device=dev)
        b = _Bucket(buf=buf, params=list(plist))
        off = 0
        for p in plist:
            view = buf[off: off + p.numel()].view_as(p)
            if hasattr(p, "moss_layer"):
                p.main_grad = view
                p.grad_fresh = True
            else:
                p.grad = view
            self.bucket_of[id(p)] = b
            off += p.numel()
        self.buckets.append(b)

    def reset(self) -> None:
        """Start of a step: re-arm buckets, zero the in-place accumulators."""
        for b in self.buckets:
            b.pending = len(b.params)
            b.work = None
            b.launched = False
            for p in b.params:
                if hasattr(p, "moss_layer"):
                    p.grad_fresh = True
                else:
                    if p.grad is None or p.grad.data_ptr() != self._view_ptr(b, p):
                        p.grad = self._view(b, p)
                    p.grad.zero_()

    def _view(self, b: _Bucket, p) -> torch.Tensor:
        off = 0
        for q in b.params:
            if q is p:
                return b.buf[off: off + p.numel()].view_as(p)
            off += q.numel()
        raise KeyError

    def _view_ptr(self, b: _Bucket, p) -> int:
        return self._view(b, p).data_ptr()

    def _ready(self, p) -> None:
        b = self.bucket_of[id(p)]
        b.pending -= 1
        if b.pending == 0:
            self._launch(b)

    def _launch(self, b: _Bucket) -> None:
        if b.launched:
            return
        b.launched = True
        if not self.communicate:
            return
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(b.buf.device))
            self.comm_stream.wait_event(ev)
            with torch.cuda.stream(self.comm_stream):
                if self.timing:
                    s = torch.cuda.Event(enable_timing=True)
                    s.record(self.comm_stream)
                b.work = dist.all_reduce(b.buf, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
                if self.timing:
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(self.comm_stream)
                    self.comm_events.append((b.buf.numel() * 4, s, e))
        else:
            b.work = dist.all_reduce(b.buf, op=dist.ReduceOp.SUM, group=self.group, async_op=True)

    def finish(self) -> None:
        """All gradients summed across ranks; compute stream ordered after the comms."""
        for b in self.buckets:
            if not b.launched:
                self._launch(b)
        for b in self.buckets:
            if b.work is not None:
                b.work.wait()
        if self.cuda and self.communicate:
            torch.cuda.current_stream(self.buckets[0].buf.device).wait_stream(self.comm_stream)

    @property
    def grad_scale(self) -> float:
        return 1.0 / self.world

    def comm_summary(self) -> dict | None:
        """All-reduce bytes and bus bandwidth 2(n-1)/n x bytes / time (NCCL's busbw) over the timed events."""
        if not self.comm_events:
            return None
        torch.cuda.synchronize()
        nbytes = sum(b for b, _, _ in self.comm_events)
        ms = sum(s.elapsed_time(e) for _, s, e in self.comm_events)
        return {"allreduce_bytes": nbytes, "allreduce_ms": ms, "launches": len(self.comm_events),
                "busbw_gbs": 2 * (self.world - 1) / self.world * nbytes / (ms / 1e3) / 1e9 if ms > 0 else None}

    def total_bytes(self) -> int:
        return sum(b.buf.numel() * 4 for b in self.buckets)
