"""World-size-2 gloo test of the ZeRO-1 orchestration (paper_2511_05811_b200.zero).

CPU stand-ins replace the three device kernels (K3 slice update, slice
re-encode, byte transpose) with the oracle's reference arithmetic
(oracle/numpy_ref: adamw_step, encode_weight), so this checks what the host
code owns: the bucket/slice layout (256-aligned parts), the reduce-scatter
of the gradients, the slice updates at the shared scale schedule, the
max-all-reduce + re-encode of a rescale step, and the FP8 all-gather +
transposed copy — against a single-process replicated computation of the
same steps.  The GPU kernels themselves are covered by test_gpu_zero.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from torch import nn

SHAPES = [(64, 96), (40, 32), (256, 48), (8, 16)]     # mixed sizes: parts straddle slice boundaries
STEPS, INTERVAL, LR = 5, 3, 1e-2


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _Layer:
    def __init__(self, out, inn, seed):
        from oracle import numpy_ref as R
        g = torch.Generator().manual_seed(seed)
        self.weight = nn.Parameter(torch.randn(out, inn, generator=g) * 0.02)
        self.weight.moss_layer = self
        s0 = R.jit_scale(self.weight.detach().numpy())
        self.schedule = R.Schedule(s_t=s0, interval=INTERVAL)
        codes, _ = R.encode_weight(self.weight.detach().numpy(), s0)
        self.w_fp8 = torch.from_numpy(codes.copy())
        self.w_fp8_t = self.w_fp8.t().contiguous()
        self.w_scale = torch.tensor([np.float32(s0)])
        self.w_amax = torch.zeros(1)
        self.fp8_pending = None        # set by Zero1's overlapped all-gather
        self._buffers = {}

    def __setattr__(self, k, v):
        object.__setattr__(self, k, v)

    def __getattribute__(self, k):
        bufs = object.__getattribute__(self, "__dict__").get("_buffers", {})
        return bufs[k] if k in bufs else object.__getattribute__(self, k)


class _StubOpt:
    """The MossAdamW host half Zero1 relies on (prepare / launch / check / records)."""
    _WORDS = 12
    _ENC = 10

    def __init__(self, layers):
        self.params = [lay.weight for lay in layers]
        self.index = {id(p): i for i, p in enumerate(self.params)}
        self.hp_dev = torch.zeros(len(self.params) * self._WORDS)
        self.saturations = torch.zeros(1, dtype=torch.int32)
        self.rescale_events, self.t, self.grad_scale, self._rescale_pending = [], 0, 1.0, False
        self.state = {}

    def shard(self, params):
        self.sharded = {id(p) for p in params}

    def record_ptr(self, p):
        return self.index[id(p)]

    def prepare(self, lr=None):
        from oracle import numpy_ref as R
        self.t += 1
        due = False
        for i, p in enumerate(self.params):
            sched = p.moss_layer.schedule
            R.advance(sched, LR)
            due |= R.rescale_due(sched)
            self.hp_dev[i * self._WORDS + self._ENC] = float(np.float32(sched.s_t))
        self._rescale_pending = due
        return due

    def launch(self, rescale=None):
        pass

    def check(self, where=""):
        pass


def _adam_states(shapes):
    from oracle import numpy_ref as R
    return [R.adam_init(s, eta=LR, weight_decay=0.1) for s in shapes]


def _install_cpu_kernels(z, states_by_param):
    """Oracle stand-ins for the K3 slice update, slice encode and transpose."""
    from oracle import numpy_ref as R

    def update(b, part, rescale):
        p = part.param
        n = part.hi - part.lo
        st = states_by_param[id(p)][(part.lo, part.hi)]
        w = p.data.view(-1)[part.lo:part.hi].double().numpy()
        g = b.gshard[part.soff:part.soff + n].double().numpy() * z.grad_scale
        w2, _ = R.adamw_step(w, g, st)
        p.data.view(-1)[part.lo:part.hi] = torch.from_numpy(w2.astype(np.float32))
        layer = p.moss_layer
        if rescale:
            layer.w_amax.fill_(float(np.abs(w2.astype(np.float32)).max()))
        else:
            s = float(z.opt.hp_dev[z.opt.index[id(p)] * 12 + 10])
            codes, _ = R.encode_weight(w2.astype(np.float32), s)
            o = b.offsets[id(p)]
            b.codes[o + part.lo:o + part.hi] = torch.from_numpy(codes.reshape(-1))
            layer.w_amax.fill_(float(np.abs(w2.astype(np.float32)).max()))
            layer.w_scale.fill_(s)

    def encode(b, part, scale):
        p = part.param
        o = b.offsets[id(p)]
        codes, _ = R.encode_weight(p.data.view(-1)[part.lo:part.hi].numpy(), scale)
        b.codes[o + part.lo:o + part.hi] = torch.from_numpy(codes.reshape(-1))

    def transpose(layer):
        layer.w_fp8_t.copy_(layer.w_fp8.t())

    z._update_part, z._encode_part, z._transpose = update, encode, transpose


def _grads(rank, step):
    g = torch.Generator().manual_seed(1000 + 17 * step + rank)
    return [torch.randn(s, generator=g) * 1e-2 for s in SHAPES]


def _worker(rank, world, port, q, overlap=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_05811_b200.zero as Z
        layers = [_Layer(o, i, seed=k) for k, (o, i) in enumerate(SHAPES)]
        opt = _StubOpt(layers)
        z = Z.Zero1(opt, bucket_mb=0.02, overlap_gather=overlap)   # ~5k floats per bucket: several buckets
        assert len(z.buckets) >= 2
        # every part is 256-aligned inside its parameter, slices tile each bucket
        for b in z.buckets:
            assert b.length % (256 * world) == 0
            for part in b.parts:
                assert part.lo % 256 == 0 or part.lo == 0
        states = {}
        for b in z.buckets:
            for part in b.parts:
                states.setdefault(id(part.param), {})[(part.lo, part.hi)] = _adam_states([(part.hi - part.lo,)])[0]
        _install_cpu_kernels(z, states)
        for step in range(STEPS):
            z.reset()
            for lay, g in zip(layers, _grads(rank, step)):
                lay.weight.main_grad.copy_(g)            # the wgrad GEMM's output
                lay.weight.grad_ready_hook(lay.weight)
            z.finish()
            z.step()
            if overlap:
                # async all-gathers are in flight until a forward (or sync) consumes them
                assert all(lay.fp8_pending is not None for lay in layers)
        z.sync()
        assert all(lay.fp8_pending is None for lay in layers)
        z.gather_master()                                  # full FP32 masters on every rank (checkpoints)
        # numpy copies: torch tensors in a spawn queue die with the child's shared-memory handles
        q.put((rank, [(lay.w_fp8.numpy().copy(), lay.w_fp8_t.numpy().copy(), float(lay.w_scale),
                       lay.schedule.s_t, lay.schedule.last_rescale_step, lay.weight.data.numpy().copy())
                      for lay in layers], "", z.state_bytes()))
    except Exception as e:  # surface worker failures immediately
        q.put((rank, None, repr(e), 0))
        raise
    finally:
        dist.destroy_process_group()


def _replicated_reference(world):
    """Single-process: summed gradients, full-tensor AdamW, encode at the schedule scale."""
    from oracle import numpy_ref as R
    layers = [_Layer(o, i, seed=k) for k, (o, i) in enumerate(SHAPES)]
    states = _adam_states([(o * i,) for o, i in SHAPES])
    for step in range(STEPS):
        gsum = [sum(_grads(r, step)[k] for r in range(world)) for k in range(len(SHAPES))]
        due = False
        for lay in layers:
            R.advance(lay.schedule, LR)
            due |= R.rescale_due(lay.schedule)
        for k, lay in enumerate(layers):
            w = lay.weight.data.view(-1).double().numpy()
            g = gsum[k].view(-1).double().numpy() / world
            w2, _ = R.adamw_step(w, g, states[k])
            lay.weight.data.view(-1)[:] = torch.from_numpy(w2.astype(np.float32))
        for lay in layers:
            wf = lay.weight.data.numpy()
            if due:
                amax = float(np.abs(wf).max())
                lay.schedule.s_t = amax / 448.0 if amax > 0 else 1.0
                lay.schedule.last_rescale_step = lay.schedule.t
            codes, _ = R.encode_weight(wf, float(np.float32(lay.schedule.s_t)))
            lay.w_fp8 = torch.from_numpy(codes.copy())
            lay.w_scale = torch.tensor([np.float32(lay.schedule.s_t)])
    return layers


@pytest.mark.parametrize("world,overlap", [(2, True), (2, False)])
def test_zero1_matches_replicated_world2(world, overlap):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, overlap)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, lay_state, err, sbytes = q.get(timeout=180)
        assert lay_state is not None, f"rank {rank}: {err}"
        out[rank] = (lay_state, sbytes)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    ref = _replicated_reference(world)
    for rank in range(world):
        for (codes, codes_t, scale, s_t, last, master), lay in zip(out[rank][0], ref):
            assert np.array_equal(master, lay.weight.data.numpy()), f"rank {rank}: gathered FP32 masters"
            assert np.array_equal(codes, lay.w_fp8.numpy()), f"rank {rank}: gathered FP8 codes"
            assert np.array_equal(codes_t, lay.w_fp8.t().numpy()), f"rank {rank}: transposed codes"
            assert scale == float(lay.w_scale) and s_t == lay.schedule.s_t
            assert last == 3                          # the rescale at step 3 (interval 3) happened everywhere
    # sharded optimizer state: each rank keeps ~1/world of the moments
    total = sum(-(-o * i // 256) * 256 for o, i in SHAPES)
    assert out[0][1] <= (total * 8) // world + 8 * 256 * world * 4
