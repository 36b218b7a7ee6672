"""Quick kernel timing probe (CUDA events, inputs > L2 or L2 flushed)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_05811_b200 import _lib
from paper_2511_05811_b200.quantize import quantize_mx2, quant_per_tensor
from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.optim import adam_params

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]

M = 8192
for (K, N) in [(4096, 12288), (4096, 4096), (4096, 11008), (11008, 4096)]:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda") * 0.02
    qa = quantize_mx2(a, row=True)
    qw = quant_per_tensor(w)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    f = lambda: mx_gemm(qa.codes, qa.sf, qa.g, qw.codes, None, qw.scale.reshape(1), out=out)
    ms = timeit(f)
    print(f"gemm M={M} K={K} N={N}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.0f} TFLOP/s", flush=True)
    fq = lambda: quantize_mx2(a, row=True, col=False)
    ms = timeit(fq)
    print(f"quant row  {M}x{K}: {ms:.3f} ms  {M*K*(2+1+1/32)/ms/1e6:.0f} GB/s (alg)", flush=True)
    fq2 = lambda: quantize_mx2(a, row=True, col=True)
    ms = timeit(fq2)
    print(f"quant row+col {M}x{K}: {ms:.3f} ms  {M*K*(2+2+2/32)/ms/1e6:.0f} GB/s (alg)", flush=True)

rows, cols = 11008, 4096
w = torch.randn(rows, cols, device="cuda") * 0.02
g = torch.randn(rows, cols, device="cuda") * 1e-3
m = torch.zeros_like(w); v = torch.zeros_like(w)
w8 = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
w8t = torch.empty(cols, rows, dtype=torch.uint8, device="cuda")
fl = _lib.FlagWord()
p = adam_params(3e-4, 0.9, 0.95, 1e-8, 0.1, 1, True)
fa = lambda: _lib.adamw_fp8(w, g, m, v, rows, cols, p, 0.001, fl, w_fp8=w8, w_fp8_t=w8t)
ms = timeit(fa)
print(f"adamw_fp8 {rows}x{cols}: {ms:.3f} ms  {rows*cols*30/ms/1e6:.0f} GB/s (alg 30 B/param)", flush=True)
