"""ZeRO-1 for the MOSS weights: sharded optimizer state, FP8 weight all-gather
(the paper's FP8-communication claim, PAPER.md:15,
334-365).

Data parallel over ``world`` ranks, one process per GPU.  For every
MossLinear weight W (the FP8 linears, ~96 % of a Llama's parameters):

  * backward: the wgrad GEMM writes the FP32 gradient into a flat bucket;
    when the bucket's last gradient is produced, a reduce-scatter (SUM) on
    the communication stream leaves each rank the summed gradient of ITS
    1/world slice of the bucket — overlapped with the rest of backward;
  * step: each rank runs the fused AdamW + autoscale + FP8-copy kernel (K3)
    on its slice only: the FP32 master values, moments m, v and the E4M3
    codes of that slice (moments are allocated for the slice only: 8/world
    bytes per parameter instead of 8);
  * the E4M3 codes of every slice are all-gathered (1 byte per parameter on
    the wire, not 4: the FP8 all-gather) into the codes buffer the forward
    GEMMs read; the dgrad GEMM reads the same codes as an MN-major operand, so
    no transposed copy has to be rebuilt.  With
    ``overlap_gather`` (default) the all-gathers are issued asynchronously in
    forward layer order at the end of ``step`` and each MossLinear waits for
    its bucket's gather only when the next forward reaches
    it, so the exchange overlaps the preceding layers' forward compute;
  * scales: s_t advances on the host identically on every rank
    (autoscale.py:71-79, O(1), no data); a rescale step (autoscale.py:86-96)
    max-all-reduces the per-slice amax of W' (one small collective), snaps
    s_t = amax/448 everywhere and re-encodes the slices.

Non-MOSS parameters (embeddings, norms, head) stay replicated: all-reduce
(dist.GradBuckets) and the full update on every rank.

Layout: a bucket holds whole parameters, each padded to a multiple of 256
elements; the bucket length is a multiple of 256 * world, so every slice
boundary and every parameter/slice intersection is 256-aligned and the
slice update runs as [n/256, 256] tiles of the same K3 kernel.

Invariants (tests/test_zero_cpu.py, tests/test_gpu_zero.py): after each
step every rank holds identical FP8 codes, transposed codes and scales; at
world_size 1 the result is bit-identical to the replicated MossAdamW step.
On a rank, master values outside its slices are stale by design: the forward
and the FP8 backward consume only the FP8 codes (the full-precision backward,
which would read them, is rejected).  ``gather_master()`` all-gathers the
FP32 masters, e.g. before ``model.state_dict()`` for a checkpoint.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .dist import GradBuckets
from .errors import InvalidArgumentError
from .fp8 import E4M3
from .nn import MossAdamW, device_flags

__all__ = ["Zero1"]

ALIGN = 256


@dataclass
class _Part:
    param: torch.nn.Parameter
    lo: int          # range [lo, hi) in the parameter's flat index space
    hi: int
    soff: int        # offset of lo inside this rank's slice


@dataclass
class _Bucket:
    params: list
    offsets: dict                      # id(p) -> offset in the bucket
    length: int
    grad: torch.Tensor                 # f32 [length]
    codes: torch.Tensor                # u8 [length]
    gshard: torch.Tensor               # f32 [length/world]: summed gradient slice
    m: torch.Tensor                    # f32 [length/world]
    v: torch.Tensor
    parts: list = field(default_factory=list)
    pending: int = 0
    work: object = None
    launched: bool = False


def _flat2d(n: int) -> tuple[int, int]:
    return (n // ALIGN, ALIGN) if n % ALIGN == 0 else (1, n)


class Zero1:
    """Sharded MOSS optimizer + gradient exchange.  Same host interface as
    dist.GradBuckets (``reset``, ``finish``, ``grad_scale``) plus ``step``,
    which replaces ``opt.step()``."""

    def __init__(self, opt: MossAdamW, bucket_mb: float = 64.0, group=None, overlap_gather: bool = True):
        self.opt = opt
        self.overlap_gather = overlap_gather
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        moss = [p for p in opt.params if hasattr(p, "moss_layer")]
        rest = [p for p in opt.params if not hasattr(p, "moss_layer")]
        for p in moss:
            if not getattr(p.moss_layer, "fp8_backward", True):
                # the full-precision backward (train.py:187-192) reads the FP32 master
                # weight, which is only current on this rank's slices
                raise InvalidArgumentError("ZeRO-1 needs the FP8 backward (MossLinear(fp8_backward=True))")
        self.moss = moss
        self.dev = moss[0].device if moss else opt.params[0].device
        self.cuda = self.dev.type == "cuda"
        self.comm_stream = torch.cuda.Stream(device=self.dev) if self.cuda else None
        self.dp = GradBuckets(rest, bucket_mb=bucket_mb, group=group) if rest else None
        opt.shard(moss)
        cap = int(bucket_mb * 1024 * 1024 // 4)
        self.buckets: list[_Bucket] = []
        self.bucket_of: dict[int, _Bucket] = {}
        cur, size = [], 0
        for p in reversed(moss):                 # backward produces gradients in reverse order
            cur.append(p)
            size += -(-p.numel() // ALIGN) * ALIGN
            if size >= cap:
                self._make_bucket(cur)
                cur, size = [], 0
        if cur:
            self._make_bucket(cur)
        for p in moss:
            p.grad_ready_hook = self._ready
        self.reset()

    # ------------------------------------------------------------------ layout
    def _make_bucket(self, plist) -> None:
        offsets, off = {}, 0
        for p in plist:
            offsets[id(p)] = off
            off += -(-p.numel() // ALIGN) * ALIGN
        unit = ALIGN * self.world
        length = -(-off // unit) * unit
        S = length // self.world
        z = lambda n, dt: torch.zeros(n, dtype=dt, device=self.dev)
        grad = z(length, torch.float32)
        b = _Bucket(params=list(plist), offsets=offsets, length=length, grad=grad,
                    codes=z(length, torch.uint8), gshard=grad if self.world == 1 else z(S, torch.float32),
                    m=z(S, torch.float32), v=z(S, torch.float32))
        lo_r, hi_r = self.rank * S, (self.rank + 1) * S
        for p in plist:
            o, n = offsets[id(p)], p.numel()
            a, e = max(o, lo_r), min(o + n, hi_r)
            if a < e:
                b.parts.append(_Part(p, a - o, e - o, a - lo_r))
            layer = p.moss_layer
            p.main_grad = b.grad[o:o + n].view_as(p)
            p.grad_fresh = True
            view = b.codes[o:o + n].view(layer.w_fp8.shape)
            view.copy_(layer.w_fp8)             # the t=0 codes (identical on every rank)
            layer._buffers["w_fp8"] = view
            self.bucket_of[id(p)] = b
        self.buckets.append(b)

    # ------------------------------------------------------------------ gradient exchange
    @property
    def grad_scale(self) -> float:
        return 1.0 / self.world

    def reset(self) -> None:
        for b in self.buckets:
            b.pending, b.work, b.launched = len(b.params), None, False
            for p in b.params:
                p.grad_fresh = True
        if self.dp is not None:
            self.dp.reset()

    def _ready(self, p) -> None:
        b = self.bucket_of[id(p)]
        b.pending -= 1
        if b.pending == 0:
            self._launch_rs(b)

    def _launch_rs(self, b: _Bucket) -> None:
        if b.launched:
            return
        b.launched = True
        if self.world == 1:
            return                              # gshard aliases grad: the whole bucket is this rank's slice
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.dev))
            self.comm_stream.wait_event(ev)
            with torch.cuda.stream(self.comm_stream):
                b.work = dist.reduce_scatter_tensor(b.gshard, b.grad, op=dist.ReduceOp.SUM, group=self.group,
                                                    async_op=True)
        else:
            b.work = dist.reduce_scatter_tensor(b.gshard, b.grad, op=dist.ReduceOp.SUM, group=self.group,
                                                async_op=True)

    def finish(self) -> None:
        for b in self.buckets:
            if not b.launched:
                self._launch_rs(b)
        for b in self.buckets:
            if b.work is not None:
                b.work.wait()
        if self.cuda and self.world > 1:
            torch.cuda.current_stream(self.dev).wait_stream(self.comm_stream)
        if self.dp is not None:
            self.dp.finish()

    # ------------------------------------------------------------------ kernels (swappable in CPU tests)
    def _update_part(self, b: _Bucket, part: _Part, rescale: bool) -> None:
        """K3 on one slice part: AdamW + FP8 codes at s_{t+1} (or only amax on rescale steps)."""
        p, layer = part.param, part.param.moss_layer
        n = part.hi - part.lo
        rows, cols = _flat2d(n)
        o = b.offsets[id(p)]
        w = p.data.view(-1)[part.lo:part.hi].view(rows, cols)
        g = b.gshard[part.soff:part.soff + n].view(rows, cols)
        m = b.m[part.soff:part.soff + n].view(rows, cols)
        v = b.v[part.soff:part.soff + n].view(rows, cols)
        rec = self.opt.record_ptr(p)
        flags = device_flags(self.dev)
        if rescale:
            _lib.adamw_fp8_dev(w, g, m, v, rows, cols, rec, None, flags, w_amax=layer.w_amax)
        else:
            codes = b.codes[o + part.lo:o + part.hi].view(rows, cols)
            _lib.adamw_fp8_dev(w, g, m, v, rows, cols, rec, rec + MossAdamW._ENC * 4, flags, scale_out=layer.w_scale, w_fp8=codes,
                               w_amax=layer.w_amax, n_saturated=self.opt.saturations)

    def _encode_part(self, b: _Bucket, part: _Part, scale: float) -> None:
        """Rescale re-encode of one slice part: codes = e4m3(W / f32(s)) (train.py:113-118)."""
        p = part.param
        n = part.hi - part.lo
        rows, cols = _flat2d(n)
        o = b.offsets[id(p)]
        w = p.data.view(-1)[part.lo:part.hi].view(rows, cols)
        codes = b.codes[o + part.lo:o + part.hi].view(rows, cols)
        _lib.encode_scaled(w, device_flags(self.dev), scale_host=scale, codes=codes)

    def _set_scale(self, layer, idx: int) -> None:
        """w_scale of a layer with no slice on this rank: copy the staged f32(s_{t+1})."""
        w = MossAdamW._WORDS
        e = MossAdamW._ENC
        layer.w_scale.copy_(self.opt.hp_dev[idx * w + e: idx * w + e + 1])

    def _transpose(self, layer) -> None:
        """Nothing to rebuild: the dgrad GEMM reads W_fp8 as stored (MN-major
        operand, gemm.mx_gemm_bkn), so the gathered codes are the whole update.
        (tests/test_zero_cpu.py swaps in a host transpose for its stub layers.)"""

    # ------------------------------------------------------------------ step
    @torch.no_grad()
    def step(self, lr: float | None = None) -> None:
        self.launch(self.prepare(lr))

    def prepare(self, lr: float | None = None) -> bool:
        """Host half of the step (schedule advance, staged kernel arguments);
        True when this step rescales."""
        self.sync()                              # codes of the previous step must have landed
        return self.opt.prepare(lr)

    @torch.no_grad()
    def launch(self, rescale: bool) -> None:
        """Device half: replicated updates, K3 on this rank's slices, the FP8
        all-gather (graph-capturable when not rescaling and not overlapped)."""
        opt = self.opt
        opt.launch(rescale)                      # replicated parameters (sharded ones are skipped)
        local = set()
        for b in self.buckets:
            for part in b.parts:
                self._update_part(b, part, rescale)
                local.add(id(part.param))
        for p in self.moss:
            if id(p) not in local:
                if rescale:
                    p.moss_layer.w_amax.zero_()
                else:
                    self._set_scale(p.moss_layer, opt.index[id(p)])
        if rescale:
            self._rescale()
        self._gather()

    def _rescale(self) -> None:
        """JIT snap s_t = max|W'|/448 on every rank (autoscale.py:86-96): one MAX all-reduce."""
        self.opt.check("rescale step")          # a gated (skipped) update leaves no amax to snap to
        amax = torch.cat([p.moss_layer.w_amax.view(1) for p in self.moss])
        if self.world > 1:
            dist.all_reduce(amax, op=dist.ReduceOp.MAX, group=self.group)
        host = amax.cpu().numpy()
        opt = self.opt
        for p, a in zip(self.moss, host):
            layer = p.moss_layer
            sched = layer.schedule
            sched.s_t = float(a) / E4M3.max_value if a > 0 else 1.0
            sched.last_rescale_step = sched.t
            opt.rescale_events.append((opt.t, id(p)))
            layer.w_amax.fill_(float(a))
            layer.w_scale.fill_(float(np.float32(sched.s_t)))
        for b in self.buckets:
            for part in b.parts:
                self._encode_part(b, part, float(np.float32(part.param.moss_layer.schedule.s_t)))
        opt._rescale_pending = False

    def _gather(self) -> None:
        """FP8 all-gather of every bucket's codes, then the local W_fp8^T rebuild
        (deferred to each layer's next forward when ``overlap_gather``)."""
        if self.overlap_gather and dist.is_initialized():
            # (also at world 1, where the in-place gather is a copy onto itself:
            # keeps this path exercised by the single-GPU tests)
            for b in reversed(self.buckets):      # buckets were built in backward order
                S = b.length // self.world
                work = dist.all_gather_into_tensor(b.codes, b.codes[self.rank * S:(self.rank + 1) * S],
                                                   group=self.group, async_op=True)
                for p in b.params:
                    p.moss_layer.fp8_pending = self._arrival(work, p.moss_layer)
            return
        if self.world > 1:
            for b in self.buckets:
                S = b.length // self.world
                dist.all_gather_into_tensor(b.codes, b.codes[self.rank * S:(self.rank + 1) * S], group=self.group)
        for p in self.moss:
            self._transpose(p.moss_layer)

    def _arrival(self, work, layer):
        def arrived() -> None:
            work.wait()                           # NCCL: a stream dependency, no host block
            self._transpose(layer)
        return arrived

    def sync(self) -> None:
        """Complete every pending FP8 all-gather (codes current on this rank)."""
        for p in self.moss:
            layer = p.moss_layer
            if layer.fp8_pending is not None:
                pending, layer.fp8_pending = layer.fp8_pending, None
                pending()

    @torch.no_grad()
    def gather_master(self) -> None:
        """All-gather the FP32 master weights of every MOSS parameter so that each
        rank holds the full, current values (checkpointing: state_dict)."""
        for b in self.buckets:
            S = b.length // self.world
            flat = torch.zeros(b.length, dtype=torch.float32, device=self.dev)
            lo_r = self.rank * S
            for part in b.parts:
                o = b.offsets[id(part.param)]
                flat[o + part.lo:o + part.hi] = part.param.data.view(-1)[part.lo:part.hi]
            if self.world > 1:
                dist.all_gather_into_tensor(flat, flat[lo_r:lo_r + S].clone(), group=self.group)
            for p in b.params:
                o = b.offsets[id(p)]
                p.data.view(-1).copy_(flat[o:o + p.numel()])

    def state_bytes(self) -> int:
        """Optimizer-state bytes held by this rank for the MOSS weights (m, v slices)."""
        return sum(b.m.numel() * 8 for b in self.buckets)
