"""Which 32-element blocks of the LayerStack's activations and output-gradients
take K1's general (IEEE-division) path instead of the branch-free fast path
(csrc/quant_v4.cu q4_block: g outside [2^-60, 2^60), 0 < block max < 2^-100,
or eff = g 2^e outside [2^-60, 2^60)), per quantized tensor, row- and
column-wise blocks; plus the fraction of warps (32 consecutive blocks of a
thread group) that contain at least one such block (a warp vote sends the
whole warp down the general path)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_05811_b200 import nn as mnn
from paper_2511_05811_b200.nn import MossAdamW
from paper_2511_05811_b200.workloads import LayerStack

seen = []
real = mnn.quantize_mx2


def spy(x2d, **kw):
    seen.append(x2d.detach().float().clone())
    return real(x2d, **kw)


mnn.quantize_mx2 = spy
torch.manual_seed(1234)
dev = torch.device("cuda")
model = LayerStack(device=dev)
opt = MossAdamW(model, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
torch.manual_seed(4321)
x = torch.randn(8192, model.d, device=dev, dtype=torch.bfloat16).requires_grad_(True)
for it in range(3):
    seen.clear()
    opt.zero_grad()
    loss = model(x.detach().requires_grad_(True))
    loss.backward()
    opt.step()
torch.cuda.synchronize()


def stats(t, name):
    amax = float(t.abs().max())
    g = amax / 448.0 if amax > 0 else 1.0
    eg = math.floor(math.log2(g)) + 127
    fast_g = 67 <= eg <= 186
    emin = max(67 - eg, -127)
    emax = min(186 - eg, 127)
    out = []
    for label, blocks in (("row", t.reshape(t.shape[0], -1, 32)), ("col", t.t().reshape(t.shape[1], -1, 32))):
        bm = blocks.abs().amax(-1)
        s = bm / 448.0
        e = torch.ceil(torch.log2(torch.clamp(s, min=1e-45) / g))
        e = torch.where(bm > 0, e, torch.zeros_like(e))
        tiny = (bm > 0) & (bm < 2.0 ** -100)
        slow = tiny | (e < emin) | (e > emax) | (not fast_g)
        frac = float(slow.float().mean())
        out.append(f"{label}: slow blocks {frac:.2e}")
    print(f"{name:22s} {tuple(t.shape)} amax {amax:.3e} g 2^{eg - 127:+d}  " + "  ".join(out), flush=True)


names = ["x (QKV in)", "a (O in)", "r (gate_up in)", "h (down in)", "dY down", "dY gate_up", "dY O", "dY QKV"]
for i, t in enumerate(seen):
    stats(t, names[i] if i < len(names) else f"#{i}")
