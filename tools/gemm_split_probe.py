"""Tail split A/B: the Llama-7B GEMM shapes at seq 4096 (M = 4096 fwd/dgrad,
M = N_out for wgrad), 30 back-to-back launches each, CUDA events per launch
(median).  Run twice: MOSS_GEMM2_SPLIT=0 and =1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.quantize import quant_per_tensor, quantize_mx2

T = 4096
shapes = []
for k, n in [(4096, 12288), (4096, 4096), (4096, 22016), (11008, 4096)]:
    shapes += [("fwd", T, n, k), ("dgrad", T, k, n), ("wgrad", n, k, T)]
tot = 0.0
for kind, m, n, k in shapes:
    a = quantize_mx2(torch.randn(m, k, device="cuda", dtype=torch.bfloat16), row=True)
    w = quant_per_tensor(torch.randn(n, k, device="cuda") * 0.02)
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    f = lambda: mx_gemm(a.codes, a.sf, a.g, w.codes, None, w.scale.reshape(1), out=out)
    for _ in range(5):
        f()
    ev = []
    for _ in range(30):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); f(); e.record(); ev.append((s, e))
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in ev)
    ms = ts[len(ts) // 2]
    tiles = (m // 256) * (n // 256)
    tot += ms
    print(f"split={os.environ.get('MOSS_GEMM2_SPLIT', '1')} {kind:5s} {m}x{n}x{k} tiles {tiles:5d} "
          f"waves {tiles / 74:5.2f}: {ms * 1e3:7.1f} us {2 * m * n * k / ms / 1e9:6.0f} TF/s", flush=True)
    del a, w, out
print(f"split={os.environ.get('MOSS_GEMM2_SPLIT', '1')} total {tot * 1e3:.1f} us")
