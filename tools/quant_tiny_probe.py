"""K1 producer-mode rate on well-scaled data vs late-training-gradient data
(tensor amax ~2^-40, block maxima spread over 70 binades: most blocks outside
the fast path's eff range -> the general path).  CUPTI medians, us."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2511_05811_b200 import _lib  # noqa: E402
from paper_2511_05811_b200.quantize import sf_buffer  # noqa: E402

fl = _lib.FlagWord()
rows, cols = 8192, 12288
torch.manual_seed(0)
base = torch.randn(rows, cols, device="cuda")
rs = torch.pow(2.0, -torch.randint(0, 70, (rows, 1), device="cuda").float())
data = {"randn": base.to(torch.bfloat16), "tiny-gradient": (base * 2.0 ** -40 * rs).to(torch.bfloat16)}
codes = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
sf = sf_buffer(rows, cols, "cuda")
ct = torch.empty(cols, rows, dtype=torch.uint8, device="cuda")
sft = sf_buffer(cols, rows, "cuda")
g = torch.empty(1, device="cuda")
for name, x in data.items():
    am = x.float().abs().max().reshape(1)

    def q():
        _lib.quant_mx2_fused(x, am, fl, amax_given=True, codes=codes, sf=sf, codes_t=ct, sf_t=sft, g_out=g)
    for _ in range(3):
        q()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            q()
        torch.cuda.synchronize()
    t = sorted(e.device_time for e in prof.events() if "quant_mx2" in e.name)
    med = t[len(t) // 2]
    print(f"{name:14s} {rows}x{cols} producer-amax row+col: {med:7.1f} us  {rows * cols * 4.0625 / med / 1e3:6.0f} GB/s")
fl.raise_if_set("probe")
