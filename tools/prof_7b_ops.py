"""Which torch ops launch the non-moss kernels of the 7B-shape step (profiler
with shapes, 2 layers).  Diagnostic only."""
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2511_05811_b200.llama import LLAMA2_7B, LlamaConfig, LlamaModel
from paper_2511_05811_b200.trainer import make_optimizer

cfg = LlamaConfig(**{**LLAMA2_7B.__dict__, "n_layers": 2})
model = LlamaModel(cfg)
opt = make_optimizer(model, 3e-4, 1000, 10)
tok = torch.randint(0, cfg.vocab, (1, 4097), device="cuda")
x, y = tok[:, :-1].contiguous(), tok[:, 1:].contiguous()


def step():
    opt.zero_grad()
    model(x, y).backward()
    opt.step()


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages(group_by_input_shape=True).table(sort_by="cuda_time_total", row_limit=45,
                                                          max_name_column_width=60, max_shapes_column_width=70))
