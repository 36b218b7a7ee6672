"""torch-profiler kernel table of the Llama-2-7B-shape step (argv: layers; seq 4096,
batch 1): shares of K2, K3, K1, producers, SDPA, head."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_05811_b200.llama import LLAMA2_7B, LlamaConfig, LlamaModel
from paper_2511_05811_b200.trainer import make_optimizer
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = LlamaConfig(**{**LLAMA2_7B.__dict__, "n_layers": layers})
model = LlamaModel(cfg)
opt = make_optimizer(model, 3e-4, 1000, 10)
tok = torch.randint(0, cfg.vocab, (1, 4097), device="cuda")
x, y = tok[:, :-1].contiguous(), tok[:, 1:].contiguous()
def step():
    opt.zero_grad(); loss = model(x, y); loss.backward(); opt.step()
for _ in range(3): step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2): step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=90))
