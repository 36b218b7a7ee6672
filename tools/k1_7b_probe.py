"""K1 launch durations inside the Llama-2-7B-shape step (2 layers, seq 4096, batch 1,
CUDA-graph replays; CUPTI): forward vs backward quantizations of the same shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2511_05811_b200 import llama as L  # noqa: E402
from paper_2511_05811_b200.nn import CudaGraphStep  # noqa: E402
from paper_2511_05811_b200.trainer import make_optimizer  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
torch.manual_seed(0)
cfg = L.LlamaConfig(**{**L.LLAMA2_7B.__dict__, "n_layers": 2, "max_seq": 4096})
model = L.LlamaModel(cfg)
opt = make_optimizer(model, 3e-4, 10_000, 100)
tok = torch.randint(0, cfg.vocab, (B, 4097), device="cuda")
x, y = tok[:, :-1].contiguous(), tok[:, 1:].contiguous()
one = torch.ones((), device="cuda")


def fb(xt, yt):
    loss = model(xt, yt)
    loss.backward(one)
    return loss


g = CudaGraphStep(fb, opt, (x.clone(), y.clone()))
for _ in range(20):
    g(x, y)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        g(x, y)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
q = [e.device_time for e in evs if "quant_mx2" in e.name]
n = len(q) // 5
print(f"MOSS_Q4_REV={os.environ.get('MOSS_Q4_REV', '1')} batch {B}: K1 us per launch (median of 5 replays):",
      np.round(np.median(np.array(q).reshape(5, n), 0), 1).tolist())
