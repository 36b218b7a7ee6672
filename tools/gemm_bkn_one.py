"""One MN-major dgrad GEMM (8192 x 4096 x 22016: gate/up dgrad) and one K-major forward GEMM, for ncu."""
import torch

from paper_2511_05811_b200.gemm import mx_gemm, mx_gemm_bkn
from paper_2511_05811_b200.quantize import quantize_mx2

q = quantize_mx2(torch.randn(8192, 22016, device="cuda", dtype=torch.bfloat16))
w = torch.randint(0, 0x70, (22016, 4096), device="cuda", dtype=torch.uint8)
s = torch.ones(1, device="cuda")
for _ in range(2):
    mx_gemm_bkn(q.codes, q.sf, s, w, s)
qx = quantize_mx2(torch.randn(8192, 4096, device="cuda", dtype=torch.bfloat16))
wf = torch.randint(0, 0x70, (22016, 4096), device="cuda", dtype=torch.uint8)
for _ in range(2):
    mx_gemm(qx.codes, qx.sf, s, wf, None, s)
torch.cuda.synchronize()
