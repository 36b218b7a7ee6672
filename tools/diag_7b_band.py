"""configs[3] loss behaviour at the full Llama-2-7B shape (32 layers, d 4096,
ffn 11008, seq 4096, batch 1): MOSS FP8 linears (fwd/dgrad/wgrad MXFP8,
auto-scaled AdamW) vs the same model with bf16 linears, same init, same
synthetic Markov-chain tokens, CUDA-graph steps.  Prints smoothed losses and
the relative gap at quarters of the run, plus step times."""
import os
import sys
import gc
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_05811_b200 import llama as L
from paper_2511_05811_b200.trainer import train

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
lr = float(sys.argv[2]) if len(sys.argv) > 2 else 3e-4
layers = int(sys.argv[3]) if len(sys.argv) > 3 else 32
seq = 4096
res, ms = {}, {}
for name, kw in (("moss", dict(moss=True)), ("bf16", dict(moss=False))):
    torch.manual_seed(0)
    cfg = L.LlamaConfig(**{**L.LLAMA2_7B.__dict__, "n_layers": layers, "max_seq": seq, **kw})
    model = L.LlamaModel(cfg)
    t0 = time.time()
    log = train(model, L.MarkovTokens(cfg.vocab, seed=1, active=4096), steps=steps, batch=1, seq=seq, lr=lr,
                warmup=max(10, steps // 10), cuda_graph=(name == "moss"))   # bf16 eager: no graph pool
    ms[name] = (time.time() - t0) / steps * 1e3
    res[name] = log.smoothed(25)
    print(f"{name}: first {log.loss[0]:.4f} last {log.loss[-1]:.4f} wall {ms[name]:.0f} ms/step", flush=True)
    del model, log
    gc.collect()
    torch.cuda.empty_cache()
    print(f"  memory after {name}: {torch.cuda.memory_allocated() / 2**30:.1f} GiB allocated", flush=True)
gap = np.abs(res["moss"] - res["bf16"]) / res["bf16"]
for q in (0.25, 0.5, 0.75, 1.0):
    i = int(q * steps) - 1
    print(f"7B-shape x{layers} layers, {steps} steps, lr {lr}, at {q:.2f}: bf16 {res['bf16'][i]:.4f} "
          f"moss {res['moss'][i]:.4f} gap {gap[i]:.4f}", flush=True)
