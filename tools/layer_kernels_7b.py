"""Kernel sequence (names, durations) of ONE Llama-2-7B-shape decoder layer
fwd+bwd+step (seq 4096) in launch order: which launches are not ours."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2511_05811_b200.llama import LLAMA2_7B, LlamaConfig, LlamaModel  # noqa: E402
from paper_2511_05811_b200.trainer import make_optimizer  # noqa: E402

cfg = LlamaConfig(**{**LLAMA2_7B.__dict__, "n_layers": 2})
model = LlamaModel(cfg)
opt = make_optimizer(model, 3e-4, 1000, 10)
tok = torch.randint(0, cfg.vocab, (1, 4097), device="cuda")
x, y = tok[:, :-1].contiguous(), tok[:, 1:].contiguous()


def step():
    opt.zero_grad()
    loss = model(x, y)
    loss.backward()
    opt.step()


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
tot = {}
for e in evs:
    ours = "moss::" in e.name
    print(f"{'  ' if ours else '**'} {e.time_range.elapsed_us():8.1f} us  {e.name[:110]}")
    k = "ours" if ours else "other"
    tot[k] = tot.get(k, 0) + e.time_range.elapsed_us()
print(tot)
