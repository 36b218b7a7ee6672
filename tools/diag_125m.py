"""configs[2] diagnostic: the ~125M Llama on Markov tokens, bf16 linears vs MOSS FP8
(fwd+bwd) vs MOSS FP8 forward with full-precision backward, two learning rates;
smoothed final / mid-run losses.  argv: steps."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_05811_b200 import llama as L
from paper_2511_05811_b200.trainer import train
steps, batch, seq = int(sys.argv[1]) if len(sys.argv) > 1 else 200, 8, 256
for lr, warm in ((1e-3, 20), (3e-4, 40)):
    for name, kw in (("bf16", dict(moss=False)), ("moss fp8 fwd+bwd", dict(moss=True)), ("moss fp8 fwd, fp bwd", dict(moss=True, fp8_backward=False))):
        torch.manual_seed(0)
        cfg = L.LlamaConfig(**{**L.LLAMA_125M.__dict__, "max_seq": seq, **kw})
        model = L.LlamaModel(cfg)
        log = train(model, L.MarkovTokens(cfg.vocab, seed=1, active=2048), steps=steps, batch=batch, seq=seq, lr=lr, warmup=warm, cuda_graph=True)
        print(f"lr {lr:g} {name:22s} final(20) {np.mean(log.loss[-20:]):.4f}  at 50% {np.mean(log.loss[steps//2-10:steps//2+10]):.4f}", flush=True)
        del model; torch.cuda.empty_cache()
