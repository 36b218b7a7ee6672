"""Two CudaGraphSteps over the same model/optimizer (double-buffered inputs).  Diagnostic."""
import sys
import traceback

import torch

from paper_2511_05811_b200.nn import CudaGraphStep, MossAdamW
from paper_2511_05811_b200.workloads import LayerStack

dev = torch.device("cuda")
model = LayerStack(d_model=1024, d_ffn=2048, device=dev)
opt = MossAdamW(model, lr=3e-4)
rg = sys.argv[1] == "1"


def fwd_bwd(xin):
    loss = model(xin)
    loss.backward()
    return loss


xs = [torch.randn(1024, 1024, device=dev, dtype=torch.bfloat16).requires_grad_(rg) for _ in range(3)]
gs = []
for i in range(3):
    try:
        g = CudaGraphStep(fwd_bwd, opt, (xs[i],))
        g(xs[i]); g(xs[i]); torch.cuda.synchronize()
        gs.append(g)
        print("graph", i, "ok", flush=True)
    except Exception:
        traceback.print_exc(limit=3)
        break
