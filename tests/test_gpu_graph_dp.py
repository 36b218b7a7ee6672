"""CUDA-graph training steps WITH the gradient exchange captured
(nn.CudaGraphStep(buckets=...)), as bench.py times every N: the bucketed
NCCL all-reduce (forced at world 1 so the collectives really run inside the
captured graph) and ZeRO-1 must train exactly like their eager steps."""

import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2511_05811_b200 import llama as L  # noqa: E402
from paper_2511_05811_b200.dist import GradBuckets  # noqa: E402
from paper_2511_05811_b200.trainer import train  # noqa: E402
from paper_2511_05811_b200.zero import Zero1  # noqa: E402

TINY = dict(vocab=512, d_model=128, n_layers=2, n_heads=4, d_ffn=256, max_seq=64, interval=7)


@pytest.fixture(scope="module", autouse=True)
def nccl_world1():
    if dist.is_initialized():
        yield
        return
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def _run(kind, graph, steps=30):
    torch.manual_seed(11)
    cfg = L.LlamaConfig(**TINY)
    model = L.LlamaModel(cfg)
    if kind == "allreduce":
        b = GradBuckets(model, bucket_mb=0.25, always_communicate=True)     # several buckets
        assert b.communicate and len(b.buckets) > 1
    else:
        b = lambda opt: Zero1(opt, bucket_mb=0.25)
    log = train(model, L.MarkovTokens(cfg.vocab, seed=5), steps=steps, batch=8, seq=64, lr=2e-3, warmup=5,
                buckets=b, cuda_graph=graph)
    blk = model.blocks[0]
    return np.array(log.loss), blk.qkv.schedule.s_t, blk.qkv.schedule.last_rescale_step, blk.qkv.w_fp8.clone()


@pytest.mark.parametrize("kind", ["allreduce", "zero1"])
def test_graphed_exchange_matches_eager(kind):
    eager = _run(kind, False)
    graph = _run(kind, True)
    assert np.isfinite(graph[0]).all()
    assert np.allclose(graph[0], eager[0], rtol=2e-2, atol=0), (graph[0][-5:], eager[0][-5:])
    assert graph[1] == eager[1] and graph[2] == eager[2] == 28          # s_t and rescale cadence (interval 7)
    assert (graph[3] == eager[3]).float().mean().item() > 0.99
    assert graph[0][-1] < graph[0][0]


@pytest.mark.slow
def test_bench_two_ranks_end_to_end():
    """bench.py --gpus 2 spawns two ranks and runs the whole N > 1 path (bucketed
    all-reduce DP on the layer step, the 7B-shape decoder truncated to 2 layers,
    max-over-ranks timing, the communicator record).  On this one-GPU box the two
    ranks share cuda:0 over gloo (MOSS_BENCH_SHARED_GPU); the driver's 8-GPU run
    uses NCCL with the step graph-captured."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["MOSS_BENCH_SHARED_GPU"] = "1"
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                        "--layers", "2", "--llama-steps", "2", "--no-fp8-roof", "--tokens", "4096"],
                       capture_output=True, text=True, timeout=1200, env=env, cwd=root)
    assert p.returncode == 0, p.stderr[-3000:]
    d = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["config"]["global_batch_tokens"] == 2 * 4096
    assert d["collectives"]["communicator"]["world_size"] == 2
    assert d["collectives"]["allreduce_bytes"] > 0
    assert d["llama7b"]["n_gpus"] == 2 and d["llama7b"]["tokens_per_s"] > 0
    assert d["llama7b_batch2"]["n_gpus"] == 2 and d["llama7b_batch2"]["tokens_per_gpu_per_step"] == 2 * 4096
    assert d["value"] > 0 and d["e2e"]["value"] > 0
