"""One eager LayerStack step (configs[1]) inside cudaProfilerStart/Stop, after
warm-up steps: run under `ncu --profile-from-start off` to capture exactly the
step's launches (e.g. per-kernel DRAM bytes with --cache-control none, so the
producer -> consumer L2 reuse inside the step is what gets measured)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_05811_b200.nn import MossAdamW
from paper_2511_05811_b200.workloads import LayerStack

dev = torch.device("cuda")
model = LayerStack(device=dev)
opt = MossAdamW(model, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
x = torch.randn(8192, model.d, device=dev, dtype=torch.bfloat16)


def step():
    opt.zero_grad()
    loss = model(x)
    loss.backward()
    opt.step()
    return loss


runner = step
if "--graph" in sys.argv:        # the timed mode: one replay of the captured step
    from paper_2511_05811_b200.nn import CudaGraphStep
    one = torch.ones((), device=dev)

    def fwd_bwd(xin):
        loss = model(xin)
        loss.backward(one)
        return loss
    xg = x.clone().requires_grad_(True)
    g = CudaGraphStep(fwd_bwd, opt, (xg,))
    runner = lambda: g(xg)
for _ in range(4):
    runner()
torch.cuda.synchronize()
torch.cuda.profiler.start()
runner()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
