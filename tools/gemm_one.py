"""Run one config-2 GEMM a few times (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_05811_b200.quantize import quantize_mx2, quant_per_tensor
from paper_2511_05811_b200.gemm import mx_gemm
M, K, N = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 4096, 12288))]
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
w = torch.randn(N, K, device="cuda") * 0.02
qa = quantize_mx2(a, row=True)
qw = quant_per_tensor(w)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    mx_gemm(qa.codes, qa.sf, qa.g, qw.codes, None, qw.scale.reshape(1), out=out)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    mx_gemm(qa.codes, qa.sf, qa.g, qw.codes, None, qw.scale.reshape(1), out=out)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"variant={os.environ.get('MOSS_GEMM_VARIANT','2')} M={M} K={K} N={N}: {ms:.3f} ms {2*M*N*K/ms/1e9:.0f} TFLOP/s")
