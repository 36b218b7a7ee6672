"""Training-loop parity (BASELINE config 3 semantics) on the Llama decoder.

1. tiny Llama, 120 steps: the GPU run (MossLinear + MossAdamW, bf16 glue)
   vs the CPU float64 reference of the same model whose linears and
   optimizer are the composed oracle (oracle/train_ref.py) — smoothed loss
   curves within a stated band;
2. ~125M Llama (d 768, 12 layers, SwiGLU 2048, vocab 32000), 600 steps:
   MOSS FP8 vs the same model with bf16 linears; the reference's own
   quant-vs-fp band is 5 % of the smoothed final loss (test_train.py:53-60),
   the band here is 2 % (measured on B200: 0.17 % at 1000 steps / lr 6e-4,
   0.40 % at 600 steps / lr 3e-4 / batch 32; profiles/r01_llama_parity.txt).
   Short runs (< ~300 steps) are dominated by when each run escapes the
   Markov-chain loss plateau and are not a meaningful band.
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2511_05811_b200 import llama as L  # noqa: E402
from paper_2511_05811_b200.nn import cosine_lr  # noqa: E402
from paper_2511_05811_b200.trainer import TrainLog, train  # noqa: E402

TINY = dict(vocab=512, d_model=128, n_layers=2, n_heads=4, d_ffn=256, max_seq=64)
TINY_BAND = 0.05        # max relative gap of the smoothed curves after warm-up
TINY_FINAL_BAND = 0.03


def _cpu_reference_curve(gpu_model, cfg, steps, batch, seq, lr, warmup, seed):
    from oracle.train_ref import OracleAdamW, OracleMossLinear
    L._LINEAR_FACTORY = lambda c, i, o, d: OracleMossLinear(i, o, c.interval)
    try:
        ref = L.LlamaModel(L.LlamaConfig(**{**cfg.__dict__, "compute_dtype": torch.float64}), device="cpu")
    finally:
        L._LINEAR_FACTORY = None
    ref = ref.double()
    with torch.no_grad():
        for (n, p_ref), (n2, p) in zip(ref.named_parameters(), gpu_model.named_parameters()):
            assert n == n2
            w = p.detach().float().cpu().numpy()
            layer = getattr(p_ref, "oracle_layer", None)
            if layer is not None:
                layer.init_from(w)
            else:
                p_ref.copy_(torch.from_numpy(w.astype(np.float64)))
    opt = OracleAdamW(ref.named_parameters(), cosine_lr(lr, warmup, steps), 0.1, L.LlamaModel.no_decay)
    data = L.MarkovTokens(cfg.vocab, seed=seed)
    losses = []
    for _ in range(steps):
        x, y = data.batch(batch, seq)
        opt.zero_grad()
        loss = ref(torch.as_tensor(x), torch.as_tensor(y))
        loss.backward()
        opt.step()
        losses.append(float(loss))
    return losses


@pytest.mark.slow
def test_tiny_llama_gpu_vs_cpu_reference_loss_curve():
    steps, batch, seq, lr, warmup, seed = 120, 8, 64, 2e-3, 12, 3
    torch.manual_seed(seed)
    cfg = L.LlamaConfig(**TINY)
    model = L.LlamaModel(cfg)
    init = {n: p.detach().clone() for n, p in model.named_parameters()}
    log = train(model, L.MarkovTokens(cfg.vocab, seed=seed), steps=steps, batch=batch, seq=seq, lr=lr,
                warmup=warmup)
    with torch.no_grad():
        for n, p in model.named_parameters():
            p.copy_(init[n])
    torch.set_num_threads(max(1, __import__("os").cpu_count()))
    ref = _cpu_reference_curve(model, cfg, steps, batch, seq, lr, warmup, seed)
    gpu_s = log.smoothed(20)
    ref_log = TrainLog(loss=ref)
    ref_s = ref_log.smoothed(20)
    gap = np.abs(gpu_s - ref_s) / ref_s
    print(f"tiny llama: gpu final {gpu_s[-1]:.4f} cpu-ref final {ref_s[-1]:.4f} "
          f"max smoothed gap after warm-up {gap[warmup:].max():.4f}")
    assert ref_s[-1] < 0.6 * math.log(cfg.vocab)           # the reference itself learns
    assert gap[warmup:].max() <= TINY_BAND
    assert gap[-1] <= TINY_FINAL_BAND


@pytest.mark.slow
def test_llama_125m_moss_vs_bf16_band():
    steps, batch, seq, lr, warmup = 600, 8, 256, 6e-4, 60
    finals = {}
    for moss in (True, False):
        torch.manual_seed(0)
        cfg = L.LlamaConfig(**{**L.LLAMA_125M.__dict__, "moss": moss, "max_seq": seq})
        model = L.LlamaModel(cfg)
        log = train(model, L.MarkovTokens(cfg.vocab, seed=1, active=2048), steps=steps, batch=batch, seq=seq,
                    lr=lr, warmup=warmup, cuda_graph=True)
        finals[moss] = float(log.smoothed(50)[-1])
        if moss:
            losses = log.loss
        del model
        torch.cuda.empty_cache()
    gap = abs(finals[True] - finals[False]) / finals[False]
    print(f"125M: moss {finals[True]:.4f} bf16 {finals[False]:.4f} gap {gap:.4f}")
    assert losses[-1] < losses[0] * 0.7
    assert gap <= 0.02


def _run_125m(name):
    """The GPU run of tests/golden/make_llama125m_curve.py's RUNS[name]: same
    seeded init (oracle.train_ref.seeded_init), same Markov data, same schedule."""
    import os
    import sys
    from oracle.train_ref import seeded_init
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(here, "golden"))
    import make_llama125m_curve as M
    run = M.RUNS[name]
    ref = np.load(M.path(name))
    cfg = L.LlamaConfig(**{**L.LLAMA_125M.__dict__, "max_seq": run["seq"]})
    model = L.LlamaModel(cfg)
    seeded_init(model, run["init_seed"])
    log = train(model, L.MarkovTokens(cfg.vocab, seed=run["data_seed"], active=run["active"]), steps=run["steps"],
                batch=run["batch"], seq=run["seq"], lr=run["lr"], warmup=run["warmup"], cuda_graph=True)
    gpu, ref = np.asarray(log.loss), np.asarray(ref["loss"])
    assert len(gpu) == len(ref) == run["steps"]
    gpu_s = TrainLog(loss=list(gpu)).smoothed(20)
    ref_s = TrainLog(loss=list(ref)).smoothed(20)
    return gpu, ref, gpu_s, ref_s, np.abs(gpu_s - ref_s) / ref_s, run


# BASELINE configs[2]: ~125M Llama decoder, 200 steps, GPU (MossLinear + MossAdamW,
# fused bf16 producers, CUDA-graph replays) vs the CPU float64 reference of the same
# model (composed MOSS oracle linears, adamw_step + autoscale, lr_at), committed by
# tests/golden/make_llama125m_curve.py.  Bands per regime (see that script):
C3_PLATEAU_BAND = 0.01      # 20-step smoothed curves, point by point, warm-up .. step 100
C3_CONVERGED_BAND = 0.02    # smoothed loss over the last 20 steps, after the chain is learned
# converge run, point by point: the first descent (warm-up .. step 44) within 1 % (measured 0.03 %); the
# second drop (steps ~45-100) runs a few steps ahead on the GPU (max 9 % at step 67 — a timing shift, the
# curves meet again: tools/c3_converge_gap.py), so it is not compared; from step 100 within 2 % (1.5 %)
C3_DESCENT_BAND = 0.01


@pytest.mark.slow
def test_llama_125m_gpu_vs_cpu_reference_descent_and_plateau():
    gpu, ref, gpu_s, ref_s, gap, run = _run_125m("plateau")
    w = run["warmup"]
    print(f"125M plateau run: max smoothed gap steps {w}..99 = {gap[w:100].max():.5f}; "
          f"step 199 gpu {gpu_s[-1]:.4f} ref {ref_s[-1]:.4f}")
    assert ref[99] < 0.75 * ref[0] and gpu[99] < 0.75 * gpu[0]          # both descend
    assert gap[w:100].max() <= C3_PLATEAU_BAND


@pytest.mark.slow
def test_llama_125m_gpu_vs_cpu_reference_converged_loss():
    gpu, ref, gpu_s, ref_s, gap, run = _run_125m("converge")
    w = run["warmup"]
    print(f"125M converge run: final smoothed gpu {gpu_s[-1]:.4f} ref {ref_s[-1]:.4f} gap {gap[-1]:.4f}; "
          f"max smoothed gap steps {w}..44 = {gap[w:45].max():.4f}, steps 100.. = {gap[100:].max():.4f}")
    assert ref_s[-1] < 0.3 * ref[0] and gpu_s[-1] < 0.3 * gpu[0]        # both learn the chain
    assert gap[-1] <= C3_CONVERGED_BAND
    assert gap[w:45].max() <= C3_DESCENT_BAND           # first descent, point by point
    assert gap[100:].max() <= C3_CONVERGED_BAND         # after the second drop, point by point


def test_cuda_graph_training_matches_eager():
    """CUDA-graph replays (nn.CudaGraphStep) give the same training as eager
    steps: identical data and init -> loss curves equal up to FP nondeterminism,
    FP8 weight copies and schedules identical, rescale steps handled eagerly."""
    curves = {}
    states = {}
    for graph in (False, True):
        torch.manual_seed(11)
        cfg = L.LlamaConfig(**{**TINY, "interval": 7})
        model = L.LlamaModel(cfg)
        log = train(model, L.MarkovTokens(cfg.vocab, seed=5), steps=30, batch=8, seq=64, lr=2e-3, warmup=5,
                    cuda_graph=graph)
        curves[graph] = np.array(log.loss)
        blk = model.blocks[0]
        states[graph] = (blk.qkv.schedule.s_t, blk.qkv.schedule.last_rescale_step, blk.qkv.w_fp8.clone())
    assert np.allclose(curves[True], curves[False], rtol=2e-2, atol=0)
    assert states[True][0] == states[False][0] and states[True][1] == states[False][1] == 28
    agree = (states[True][2] == states[False][2]).float().mean().item()
    assert agree > 0.99


@pytest.mark.slow
def test_llama7b_shape_band_deconfounded():
    """configs[3] semantics at the Llama-2-7B layer shape (d 4096, ffn 11008, 32 heads,
    vocab 32000, seq 4096; 8 of the 32 layers to keep the test short — the full-depth
    run is profiles/r02_llama7b_band_deconfounded.txt, tools/band_7b_v2.py): pairs that
    differ in ONE thing, same init, data and CUDA-graph stepping.  MOSS FP8 linears vs
    bf16 linears (torch glue both), and our fused producers vs torch glue (MOSS both).
    Bands: final smoothed loss within 1 %, second half of the run within 2 % (the steep
    descent right after warm-up shifts by a step or two and is not compared)."""
    import gc
    steps, warm = 150, 15
    runs = {"moss_fused": dict(moss=True, fused_ops=True), "moss_torchglue": dict(moss=True, fused_ops=False),
            "bf16_torchglue": dict(moss=False, fused_ops=False)}
    res = {}
    for name, kw in runs.items():
        torch.manual_seed(0)
        cfg = L.LlamaConfig(**{**L.LLAMA2_7B.__dict__, "n_layers": 8, "max_seq": 4096, **kw})
        model = L.LlamaModel(cfg)
        log = train(model, L.MarkovTokens(cfg.vocab, seed=1, active=128), steps=steps, batch=1, seq=4096, lr=3e-4,
                    warmup=warm, cuda_graph=True)
        res[name] = log.smoothed(25)
        assert res[name][-1] < 0.15 * log.loss[0]                      # every run learns the chain
        del model, log
        gc.collect()
        torch.cuda.empty_cache()
    for a, b in (("moss_torchglue", "bf16_torchglue"), ("moss_fused", "moss_torchglue")):
        gap = np.abs(res[a] - res[b]) / res[b]
        print(f"7B shape x8: {a} vs {b}: final {gap[-1]:.4f}, second half max {gap[steps // 2:].max():.4f}")
        assert gap[-1] <= 0.01
        assert gap[steps // 2:].max() <= 0.02
