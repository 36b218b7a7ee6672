"""Per-kernel CUPTI durations of the configs[1] layer step: eager steps
(back to back, no sleep) vs CUDA-graph replays of the same step, in launch
order.  Diagnostic for the in-step kernel rates."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2511_05811_b200.nn import CudaGraphStep, MossAdamW
from paper_2511_05811_b200.workloads import LayerStack

dev = torch.device("cuda")
model = LayerStack(device=dev)
opt = MossAdamW(model, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
x = torch.randn(8192, model.d, device=dev, dtype=torch.bfloat16).requires_grad_(True)
one = torch.ones((), device=dev)


def fwd_bwd(xin):
    loss = model(xin)
    loss.backward(one)
    return loss


def step(xin):
    opt.zero_grad()
    loss = fwd_bwd(xin.detach().requires_grad_(True))
    opt.step()
    return loss


for _ in range(3):
    step(x)
g = CudaGraphStep(fwd_bwd, opt, (x.detach().clone().requires_grad_(True),))
for _ in range(3):
    g(x)
torch.cuda.synchronize()
print("captured quant amax modes:", getattr(g, "capture_quant_modes", None))


def prof(fn, reps=5):
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        for _ in range(reps):
            fn(x)
        torch.cuda.synchronize()
    evs = [e for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA and "moss::" in e.name]
    return evs, reps


for name, fn in (("eager", step), ("replay", g), ("eager", step), ("replay", g)):
    evs, reps = prof(fn)
    per = len(evs) // reps
    last = evs[-per:]
    tot = {}
    for e in evs:
        k = e.name.split("(")[0].split("<")[0].replace("moss::", "")
        tot[k] = tot.get(k, 0.0) + e.device_time / reps
    print(name, {k: round(v, 1) for k, v in tot.items()}, "sum", round(sum(tot.values()), 1))
    print("   last step:", [(e.name.split("(")[0].split("<")[0].replace("moss::", "")[:10], round(e.device_time, 1))
                          for e in last])
