"""Activation memory of one Llama-2-7B-shape forward (seq 4096, batch 1):
MOSS FP8 linears (FP8 row/col codes stashed for backward, producer kernels)
vs the same model with bf16 linears and torch ops.  Memory held between the
end of forward and backward = what autograd saved.  Diagnostic (the paper's
activation-memory claim)."""
import gc
import sys

import torch

from paper_2511_05811_b200 import llama as L
from paper_2511_05811_b200.trainer import make_optimizer

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
seq = 4096
for name, moss in (("moss", True), ("bf16", False)):
    cfg = L.LlamaConfig(**{**L.LLAMA2_7B.__dict__, "n_layers": layers, "max_seq": seq, "moss": moss})
    model = L.LlamaModel(cfg)
    opt = make_optimizer(model, 3e-4, 100, 10)
    tok = torch.randint(0, cfg.vocab, (1, seq + 1), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    x, y = tok[:, :-1].contiguous(), tok[:, 1:].contiguous()
    for _ in range(2):
        opt.zero_grad()
        model(x, y).backward()
        opt.step()
    torch.cuda.synchronize()
    gc.collect()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    loss = model(x, y)
    torch.cuda.synchronize()
    held = torch.cuda.memory_allocated() - base
    loss.backward()
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    print(f"{name}: activations held after forward {held / 1e9:.3f} GB for {layers} layers "
          f"({held / 1e9 / layers:.3f} GB/layer incl. head), fwd+bwd transient peak {peak / 1e9:.3f} GB", flush=True)
    del model, opt, loss, x, y, tok
    gc.collect()
    torch.cuda.empty_cache()
