"""Kernel list of one eager LayerStack step (torch profiler): which launches
are ours (moss/csrc) and which are torch glue.  Diagnostic only."""
import torch
from torch.profiler import ProfilerActivity, profile

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


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=90))
