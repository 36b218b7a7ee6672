"""A/B of a launch-time switch inside the layer step's CUDA graph, one process:
one graph captured per setting of an environment variable read at launch time
(default MOSS_Q4_DYN=1,0: K1's dynamic vs static tile schedule; e.g.
`python tools/k1_dyn_graph_ab.py 8 MOSS_PDL=0,1`); replays alternate in blocks,
CUPTI durations of the 8 K1 launches per step (medians over the blocks), the
step time and the idle time between kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2511_05811_b200.nn import CudaGraphStep, MossAdamW  # noqa: E402
from paper_2511_05811_b200.workloads import LayerStack  # noqa: E402

torch.manual_seed(0)
model = LayerStack(device="cuda")
opt = MossAdamW(model, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
x = torch.randn(8192, 4096, device="cuda", dtype=torch.bfloat16).requires_grad_(True)
one = torch.ones((), device="cuda")


def fwd_bwd(xin):
    loss = model(xin)
    loss.backward(one)
    return loss


VAR, VALS = (sys.argv[2].split("=") if len(sys.argv) > 2 else ("MOSS_Q4_DYN", "1,0"))
graphs = {}
for v in VALS.split(","):
    os.environ[VAR] = v
    g = CudaGraphStep(fwd_bwd, opt, (x.detach().clone().requires_grad_(True),))
    g(x)
    g(x)
    graphs[v] = g
k1 = {v: [] for v in graphs}
step = {v: [] for v in graphs}
busy = {v: [] for v in graphs}
for blk in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    for v, g in graphs.items():
        for _ in range(10):
            g(x)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            s.record()
            for _ in range(5):
                g(x)
            e.record()
            torch.cuda.synchronize()
        q = [ev.device_time for ev in prof.events() if "quant_mx2" in ev.name]
        kev = sorted((ev.time_range.start, ev.time_range.end) for ev in prof.events()
                     if ev.device_type == torch.autograd.DeviceType.CUDA)
        span = kev[-1][1] - kev[0][0]
        covered, cur_s, cur_e = 0.0, None, None        # union of kernel intervals
        for a, b in kev:
            if cur_e is None or a > cur_e:
                if cur_e is not None:
                    covered += cur_e - cur_s
                cur_s, cur_e = a, b
            else:
                cur_e = max(cur_e, b)
        covered += cur_e - cur_s
        busy[v].append((span - covered) / 5)
        k1[v].append(np.array(q).reshape(5, -1).mean(0))
        step[v].append(s.elapsed_time(e) / 5)
for v in graphs:
    a = np.median(np.stack(k1[v]), 0)
    print(f"{VAR}={v}: step {np.median(step[v]):.3f} ms; idle between kernels {np.median(busy[v]):.1f} us/step; "
          f"K1 us per launch {np.round(a, 1).tolist()} sum {a.sum():.1f}")
