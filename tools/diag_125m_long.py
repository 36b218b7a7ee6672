"""configs[2] long-horizon band: ~125M Llama, bf16 vs MOSS FP8 linears, one lr.
argv: steps lr warmup [batch]."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_05811_b200 import llama as L
from paper_2511_05811_b200.trainer import train
steps = int(sys.argv[1]); lr = float(sys.argv[2]); warm = int(sys.argv[3]); batch = int(sys.argv[4]) if len(sys.argv) > 4 else 8
seq = 256
res = {}
for name, kw in (("bf16", dict(moss=False)), ("moss", dict(moss=True))):
    torch.manual_seed(0)
    cfg = L.LlamaConfig(**{**L.LLAMA_125M.__dict__, "max_seq": seq, **kw})
    model = L.LlamaModel(cfg)
    log = train(model, L.MarkovTokens(cfg.vocab, seed=1, active=2048), steps=steps, batch=batch, seq=seq, lr=lr, warmup=warm, cuda_graph=True)
    res[name] = log.smoothed(50)
    del model; torch.cuda.empty_cache()
gap = np.abs(res["moss"] - res["bf16"]) / res["bf16"]
for q in (0.25, 0.5, 0.75, 1.0):
    i = int(q * steps) - 1
    print(f"steps {steps} lr {lr} batch {batch} at {q:.2f}: bf16 {res['bf16'][i]:.4f} moss {res['moss'][i]:.4f} gap {gap[i]:.4f}", flush=True)
