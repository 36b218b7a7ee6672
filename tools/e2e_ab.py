"""A/B in one process: plain graph replays (HBM-resident input) vs the e2e
loop (pinned H2D prefetch on a copy stream + per-step loss D2H), alternated
to separate the pipeline cost from thermal drift.  Diagnostic only."""
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


static_x = x.clone()
g = CudaGraphStep(fwd_bwd, opt, (static_x,))
for _ in range(4):
    g(x)
torch.cuda.synchronize()
x_host = x.cpu().pin_memory()
stage = [torch.empty_like(x) for _ in range(2)]
cstream = torch.cuda.Stream()
ready = [torch.cuda.Event() for _ in range(2)]
consumed = [torch.cuda.Event() for _ in range(2)]
steps = 30


def plain():
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        g(static_x)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


def plain_copy():
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        g(x)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


def e2e():
    loss_host = torch.empty(steps, dtype=torch.float32).pin_memory()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()

    def prefetch(i):
        b = i % 2
        with torch.cuda.stream(cstream):
            cstream.wait_event(s)
            if i >= 2:
                cstream.wait_event(consumed[b])
            stage[b].copy_(x_host, non_blocking=True)
            ready[b].record(cstream)

    prefetch(0)
    for i in range(steps):
        b = i % 2
        if i + 1 < steps:
            prefetch(i + 1)
        torch.cuda.current_stream().wait_event(ready[b])
        loss = g(stage[b])
        consumed[b].record()
        loss_host[i].copy_(loss.detach().reshape(()), non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


for r in range(3):
    print(f"round {r}: plain {plain():.3f} ms  plain+D2D {plain_copy():.3f} ms  e2e {e2e():.3f} ms  plain {plain():.3f} ms")
