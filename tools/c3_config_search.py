"""Pick a configs[2] run (lr, warmup, active vocab, batch) whose loss curve is
numerically STABLE: the GPU product path (MOSS linears, fused bf16 producers)
against the same model with f32 torch glue (a proxy for the f64 CPU reference)
from the same seeded init and data; prints the max smoothed gap per config."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.train_ref import seeded_init  # noqa: E402
from paper_2511_05811_b200 import llama as L  # noqa: E402
from paper_2511_05811_b200.trainer import TrainLog, train  # noqa: E402

configs = [dict(lr=6e-4, warmup=40, active=256), dict(lr=3e-4, warmup=40, active=256),
           dict(lr=3e-4, warmup=20, active=128), dict(lr=6e-4, warmup=40, active=128),
           dict(lr=4e-4, warmup=40, active=256)]
steps, batch, seq = 200, 8, 256
for c in configs:
    curves = {}
    for mode in ("fused_bf16", "glue_f32"):
        kw = {} if mode == "fused_bf16" else {"fused_ops": False, "compute_dtype": torch.float32}
        cfg = L.LlamaConfig(**{**L.LLAMA_125M.__dict__, "max_seq": seq, **kw})
        model = L.LlamaModel(cfg)
        seeded_init(model, 7)
        log = train(model, L.MarkovTokens(cfg.vocab, seed=1, active=c["active"]), steps=steps, batch=batch, seq=seq,
                    lr=c["lr"], warmup=c["warmup"], cuda_graph=mode == "fused_bf16")
        curves[mode] = np.asarray(log.loss)
        del model
        torch.cuda.empty_cache()
    a = TrainLog(loss=list(curves["fused_bf16"])).smoothed(20)
    b = TrainLog(loss=list(curves["glue_f32"])).smoothed(20)
    gap = np.abs(a - b) / b
    jumps = [float(np.max(np.diff(v))) for v in curves.values()]
    print(c, f"first {curves['fused_bf16'][0]:.3f} last bf16 {a[-1]:.4f} f32 {b[-1]:.4f} maxgap {gap[c['warmup']:].max():.4f} "
          f"final {gap[-1]:.4f} max step-up {jumps[0]:.3f}/{jumps[1]:.3f}", flush=True)
