"""World-size-2 gloo tests of the DP gradient exchange (paper_2511_05811_b200.dist).

Covers the host logic of north_star (4) on CPU: bucket assignment in reverse
parameter order, in-place accumulation into bucket views, the MossLinear-style
ready hook (main_grad written by the kernel, then ``grad_ready_hook``), launch
on bucket completion, and the SUM + 1/world averaging contract.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from torch import nn


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _FakeMossLayer:
    pass


def _worker(rank: int, world: int, port: int, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_05811_b200.dist import GradBuckets
        torch.manual_seed(0)
        model = nn.Sequential(nn.Linear(64, 128), nn.ReLU(), nn.Linear(128, 32))
        # one "MOSS" parameter whose gradient is produced outside autograd
        moss_w = nn.Parameter(torch.zeros(16, 32))
        moss_w.moss_layer = _FakeMossLayer()
        params = list(model.parameters()) + [moss_w]
        buckets = GradBuckets(params, bucket_mb=0.01)   # ~2.6k floats: forces several buckets
        assert len(buckets.buckets) >= 2
        # bucket order follows reverse registration order
        first = buckets.buckets[0].params
        assert first[0] is moss_w
        results = []
        for it in range(2):
            buckets.reset()
            torch.manual_seed(100 + rank + 10 * it)
            x = torch.randn(8, 64)
            loss = model(x).pow(2).mean()
            loss.backward()
            # "kernel" writes main_grad then signals, like MossLinearFunction.backward
            moss_w.main_grad.copy_(torch.full((16, 32), float(rank + 1 + it)))
            moss_w.grad_ready_hook(moss_w)
            buckets.finish()
            # reference: local grads all-reduced by hand
            torch.manual_seed(100 + rank + 10 * it)
            ref_model = nn.Sequential(nn.Linear(64, 128), nn.ReLU(), nn.Linear(128, 32))
            ref_model.load_state_dict(model.state_dict())
            ref_model(x).pow(2).mean().backward()
            for p_ref, p in zip(ref_model.parameters(), model.parameters()):
                g = p_ref.grad.clone()
                dist.all_reduce(g)
                assert torch.allclose(p.grad, g, atol=1e-6), "bucketed grad != all-reduced grad"
            want = sum(float(r + 1 + it) for r in range(world))
            assert torch.all(moss_w.main_grad == want)
            assert buckets.grad_scale == 1.0 / world
            results.append(float(sum(p.grad.abs().sum() for p in model.parameters())))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


def test_grad_buckets_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    out = dict(q.get(timeout=10) for _ in range(2))
    assert out[0] == pytest.approx(out[1])      # identical summed grads on both ranks
