"""K3 in isolation: fused AdamW + FP8 copy (+ transposed copy) on Llama-7B
weight shapes; CUDA events without per-iteration host sync, median of 20.
GB/s = algorithmic bytes (16 read + 12 written + 1 per code
copy per parameter) / time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_05811_b200 import _lib
from paper_2511_05811_b200.optim import adam_params

def timeit(fn, iters=20, warm=3):
    for _ in range(warm): fn()
    ev = []
    for _ in range(iters):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); ev.append((s, e))
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in ev)
    return ts[len(ts) // 2]
fl = _lib.FlagWord()
p = adam_params(3e-4, 0.9, 0.95, 1e-8, 0.1, 1, True)
for rows, cols in [(4096, 4096), (12288, 4096), (22016, 4096), (4096, 11008), (32000, 4096)]:
    w = torch.randn(rows, cols, device="cuda") * 0.02
    g = torch.randn(rows, cols, device="cuda") * 1e-3
    m = torch.zeros_like(w); v = torch.zeros_like(w)
    w8 = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
    w8t = torch.empty(cols, rows, dtype=torch.uint8, device="cuda")
    n = rows * cols
    t2 = timeit(lambda: _lib.adamw_fp8(w, g, m, v, rows, cols, p, 0.001, fl, w_fp8=w8, w_fp8_t=w8t))
    t0 = timeit(lambda: _lib.adamw_fp8(w, g, m, v, rows, cols, p, 0.001, fl))
    print(f"adamw {rows}x{cols}: +fp8+fp8T {t2*1e3:7.1f} us {n*30/t2/1e6:5.0f} GB/s | plain {t0*1e3:7.1f} us "
          f"{n*28/t0/1e6:5.0f} GB/s", flush=True)
fl.raise_if_set("probe")
