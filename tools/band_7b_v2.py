"""configs[3] loss band at the full Llama-2-7B shape, deconfounded:
every run uses the SAME glue and the SAME stepping (CUDA-graph replays), so a
pair differs in one thing only:
    moss_torchglue  vs bf16_torchglue : MOSS FP8 linears vs bf16 linears (torch RMSNorm/RoPE/SwiGLU/CE)
    moss_fused      vs moss_torchglue : our producer kernels vs torch glue (MOSS linears both)
Same init (torch.manual_seed(0)), same synthetic Markov tokens.  Regime: a chain of
`active` states the model learns smoothly (the 4096-state chain of round 1 has a
chaotic plateau escape that moves by ~100 steps under any numerical change).
    python tools/band_7b_v2.py STEPS LR ACTIVE LAYERS
Prints smoothed(25) losses at quarters, the max smoothed gap after warm-up and the
final gap per pair, and step times."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_05811_b200 import llama as L  # noqa: E402
from paper_2511_05811_b200.trainer import train  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
lr = float(sys.argv[2]) if len(sys.argv) > 2 else 3e-4
active = int(sys.argv[3]) if len(sys.argv) > 3 else 128
layers = int(sys.argv[4]) if len(sys.argv) > 4 else 32
seq, warm = 4096, max(10, steps // 10)
runs = {"moss_fused": dict(moss=True, fused_ops=True), "moss_torchglue": dict(moss=True, fused_ops=False),
        "bf16_torchglue": dict(moss=False, fused_ops=False)}
res, ms = {}, {}
for name, kw in runs.items():
    torch.manual_seed(0)
    cfg = L.LlamaConfig(**{**L.LLAMA2_7B.__dict__, "n_layers": layers, "max_seq": seq, **kw})
    model = L.LlamaModel(cfg)
    t0 = time.time()
    log = train(model, L.MarkovTokens(cfg.vocab, seed=1, active=active), steps=steps, batch=1, seq=seq, lr=lr,
                warmup=warm, cuda_graph=True)
    ms[name] = (time.time() - t0) / steps * 1e3
    res[name] = log.smoothed(25)
    print(f"{name}: first {log.loss[0]:.4f} last {log.loss[-1]:.4f} smoothed last {res[name][-1]:.4f} "
          f"wall {ms[name]:.0f} ms/step", flush=True)
    del model, log
    gc.collect()
    torch.cuda.empty_cache()
print(f"# 7B shape x{layers} layers, seq {seq}, batch 1, {steps} steps, lr {lr}, warm-up {warm}, {active} Markov states")
for q in (0.25, 0.5, 0.75, 1.0):
    i = int(q * steps) - 1
    print("  at %.2f: " % q + "  ".join(f"{n} {res[n][i]:.4f}" for n in runs))
for a, b in (("moss_torchglue", "bf16_torchglue"), ("moss_fused", "moss_torchglue"), ("moss_fused", "bf16_torchglue")):
    gap = np.abs(res[a] - res[b]) / res[b]
    print(f"  {a} vs {b}: max smoothed gap after warm-up {gap[warm:].max():.4f} (at step {warm + int(gap[warm:].argmax())}), "
          f"final {gap[-1]:.4f}")
