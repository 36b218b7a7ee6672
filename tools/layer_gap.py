"""Where does the LayerStack step time go beyond the kernel sum?  A: CUDA-graph
replay; B: eager step with the host issued ahead (device sleep); per replay
distribution.  Diagnostic only."""
import statistics

import torch

from paper_2511_05811_b200.nn import CudaGraphStep, MossAdamW
from paper_2511_05811_b200.workloads import LayerStack

dev = torch.device("cuda")
model = LayerStack(device=dev)
opt = MossAdamW(model, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
x = torch.randn(8192, model.d, device=dev, dtype=torch.bfloat16)


def fwd_bwd(xin):
    loss = model(xin)
    loss.backward()
    return loss


def step(xin):
    opt.zero_grad()
    loss = fwd_bwd(xin)
    opt.step()
    return loss


for _ in range(3):
    step(x)
torch.cuda.synchronize()
ev = lambda: torch.cuda.Event(enable_timing=True)
# B: eager, host ahead
bt = []
for _ in range(10):
    torch.cuda._sleep(30_000_000)
    a, b = ev(), ev()
    a.record()
    step(x)
    b.record()
    torch.cuda.synchronize()
    bt.append(a.elapsed_time(b))
g = CudaGraphStep(fwd_bwd, opt, (x,))
for _ in range(3):
    g(x)
torch.cuda.synchronize()
at = []
for _ in range(20):
    a, b = ev(), ev()
    a.record()
    g(x)
    b.record()
    torch.cuda.synchronize()
    at.append(a.elapsed_time(b))
a, b = ev(), ev()
a.record()
for _ in range(50):
    g(x)
b.record()
torch.cuda.synchronize()
print(f"eager host-ahead: median {statistics.median(bt):.3f} ms  min {min(bt):.3f}")
print(f"graph single replay: median {statistics.median(at):.3f} ms  min {min(at):.3f}  max {max(at):.3f}")
print(f"graph 50 back-to-back: {a.elapsed_time(b) / 50:.3f} ms/step")
ct = []
for _ in range(20):
    torch.cuda._sleep(40_000_000)
    a, b = ev(), ev()
    a.record()
    g(x)
    b.record()
    torch.cuda.synchronize()
    ct.append(a.elapsed_time(b))
print(f"graph replay after idle: median {statistics.median(ct):.3f} ms  min {min(ct):.3f}  max {max(ct):.3f}")
print("single replays in order:", " ".join(f"{t:.2f}" for t in at))
