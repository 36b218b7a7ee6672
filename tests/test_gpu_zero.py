"""ZeRO-1 (zero.Zero1) on the GPU at world_size 1 over NCCL: the sharded
driver — flat 256-aligned slices through the K3 kernel, codes in the
bucket buffer the GEMMs read (dgrad reads them as stored, MN-major),
rescale through the max-all-reduce path — must train exactly like the
replicated MossAdamW (same init, same data).  The multi-rank collectives are
covered on CPU by test_zero_cpu.py (gloo, world 2)."""

import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2511_05811_b200 import _lib  # noqa: E402
from paper_2511_05811_b200 import llama as L  # noqa: E402
from paper_2511_05811_b200.trainer import train  # noqa: E402
from paper_2511_05811_b200.zero import Zero1  # noqa: E402

TINY = dict(vocab=512, d_model=128, n_layers=2, n_heads=4, d_ffn=256, max_seq=64, interval=4)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_zero1_world1_matches_replicated():
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    try:
        runs = {}
        for zero in (False, True):
            torch.manual_seed(7)
            model = L.LlamaModel(L.LlamaConfig(**TINY))
            log = train(model, L.MarkovTokens(512, seed=2), steps=10, batch=4, seq=64, lr=2e-3, warmup=2,
                        buckets=(lambda opt: Zero1(opt, bucket_mb=0.5)) if zero else None)
            lay = [m for m in model.modules() if hasattr(m, "w_fp8")]
            runs[zero] = (np.array(log.loss), [l.w_fp8.clone() for l in lay], [l.w_fp8_t.clone() for l in lay],
                          [float(l.w_scale) for l in lay], [l.schedule.last_rescale_step for l in lay],
                          [p.detach().clone() for p in model.parameters()])
        a, b = runs[False], runs[True]
        assert np.allclose(a[0], b[0], rtol=1e-3, atol=0), (a[0], b[0])
        for x, y in zip(a[1], b[1]):
            assert (x == y).float().mean().item() > 0.999
        for x, y in zip(b[1], b[2]):
            assert torch.equal(x.t(), y)                 # transposed copy rebuilt exactly
        assert a[3] == pytest.approx(b[3], rel=1e-6)
        assert a[4] == b[4] and max(a[4]) == 8           # rescales at steps 4 and 8 on both paths
        for x, y in zip(a[5], b[5]):
            assert torch.allclose(x, y, rtol=1e-4, atol=1e-6)
    finally:
        dist.destroy_process_group()
