"""Two data-parallel ranks on ONE GPU (gloo carries CUDA tensors through host
staging; NCCL refuses two ranks per device): exercises the multi-rank
training path with the real kernels — DP all-reduce buckets (dist.GradBuckets)
and ZeRO-1 (zero.Zero1) — and checks the invariant both must keep: every
rank ends each step with bit-identical FP8 weight codes, transposed codes and
scales, and both modes train the same model identically."""

import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(step, rank, world, tokens=512):
    """Rank's shard of the global batch of ``step`` (the same global batch for any world size)."""
    g = torch.Generator(device="cuda").manual_seed(1000 + step)
    full = torch.randn(tokens, 512, device="cuda", dtype=torch.bfloat16, generator=g)
    n = tokens // world
    return full[rank * n:(rank + 1) * n].contiguous()


def _worker(rank, world, port, mode, q, steps=4):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_05811_b200.dist import GradBuckets
        from paper_2511_05811_b200.nn import MossAdamW
        from paper_2511_05811_b200.workloads import LayerStack
        from paper_2511_05811_b200.zero import Zero1
        torch.manual_seed(0)                                     # identical init on every rank
        model = LayerStack(d_model=512, d_ffn=1024, device="cuda", interval=3, loss_offset=False)
        opt = MossAdamW(model, lr=1e-3)
        ex = Zero1(opt, bucket_mb=1.0) if mode == "zero1" else GradBuckets(model, bucket_mb=1.0)
        opt.grad_scale = ex.grad_scale
        losses = []
        for step in range(steps):                                # includes a rescale at step 3
            x = _batch(step, rank, world)                        # this rank's shard of the global batch
            ex.reset()
            loss = model(x)
            loss.backward()
            ex.finish()
            if mode == "zero1":
                ex.step()
            else:
                opt.step()
            opt.check("dp")
            losses.append(float(loss))
        if mode == "zero1":
            ex.sync()                                            # land the overlapped FP8 all-gathers
        mods = [model.qkv, model.o, model.gate_up, model.down]
        q.put((rank, [m.w_fp8.cpu().numpy() for m in mods], [m.w_fp8_t.cpu().numpy() for m in mods],
               [float(m.w_scale) for m in mods], losses))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, None, repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def _run(mode, steps=4):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q, steps)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        rank, codes, codes_t, scales, losses = q.get(timeout=600)
        assert codes is not None, f"rank {rank}: {codes_t}"
        out[rank] = (codes, codes_t, scales, losses)
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    return out


def test_dp_ranks_stay_identical():
    import numpy as np
    res = {mode: _run(mode) for mode in ("allreduce", "zero1")}
    for mode, out in res.items():
        for a, b in zip(out[0][0], out[1][0]):
            assert np.array_equal(a, b), f"{mode}: FP8 codes differ across ranks"
        for a, b in zip(out[0][1], out[1][1]):
            assert np.array_equal(a, b), f"{mode}: transposed codes differ across ranks"
        assert out[0][2] == out[1][2]
    # ZeRO-1 trains the same model as the all-reduce DP (same summed gradients, same update)
    for a, b in zip(res["allreduce"][0][0], res["zero1"][0][0]):
        assert (a == b).mean() > 0.999
    assert np.allclose(res["allreduce"][0][3], res["zero1"][0][3], rtol=1e-3)


DP_STEPS = 40
DP_BAND = 0.02          # per step, relative, 2-rank mean loss vs the 1-GPU loss on the same global batch


def test_dp_matches_single_gpu_at_same_global_batch():
    """2 ranks x 256 tokens vs 1 process x 512 tokens, same global batches, 40
    steps (13 rescales at interval 3): the loss curves agree within DP_BAND at
    every step (n-GPU curve within a stated band of the 1-GPU
    curve); the loss falls by more than half over the run.  The only semantic difference is the
    per-rank activation amax; it perturbs FP8 gradients at the
    quantization-noise level, which Adam's sign-like early steps turn into
    different updates of near-zero-gradient weights, so weights are not
    compared element-wise here (the invariant is rank-to-rank identity, above)."""
    import numpy as np

    from paper_2511_05811_b200.nn import MossAdamW
    from paper_2511_05811_b200.workloads import LayerStack
    torch.manual_seed(0)
    model = LayerStack(d_model=512, d_ffn=1024, device="cuda", interval=3, loss_offset=False)
    opt = MossAdamW(model, lr=1e-3)
    single = []
    for step in range(DP_STEPS):
        opt.zero_grad()
        loss = model(_batch(step, 0, 1))
        loss.backward()
        opt.step()
        opt.check()
        single.append(float(loss))
    dp = _run("allreduce", steps=DP_STEPS)
    dp_loss = (np.array(dp[0][3]) + np.array(dp[1][3])) / 2          # mean of the ranks' shard losses
    gap = np.abs(dp_loss - np.array(single)) / np.array(single)
    print(f"DP vs 1-GPU over {DP_STEPS} steps: max gap {gap.max():.4f}, loss {single[0]:.4f} -> {single[-1]:.4f}")
    assert single[-1] < 0.5 * single[0]
    assert gap.max() <= DP_BAND, gap
