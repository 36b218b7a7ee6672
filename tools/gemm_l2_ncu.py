"""One launch each of our K2 and cuBLASLt MXFP8 (torch F.scaled_mm) on the same
codes/scales (8192 x 12288 x 4096), for an ncu comparison of L2 -> SM traffic:
    ncu --metrics <list> -k regex:"gemm|nvjet|cutlass|sm100" python tools/gemm_l2_ncu.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2511_05811_b200.gemm import mx_gemm  # noqa: E402
from paper_2511_05811_b200.quantize import quantize_mx2  # noqa: E402

M, N, K = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 12288, 4096))]
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
qa, qb = quantize_mx2(a, row=True), quantize_mx2(b, row=True)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
one = torch.ones(1, device="cuda")
A8, B8 = qa.codes.view(torch.float8_e4m3fn), qb.codes.view(torch.float8_e4m3fn).t()
sa, sb = qa.sf.view(torch.float8_e8m0fnu), qb.sf.view(torch.float8_e8m0fnu)
for _ in range(2):
    mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out=out)
    F.scaled_mm(A8, B8, sa, F.ScalingType.BlockWise1x32, sb, F.ScalingType.BlockWise1x32,
                swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                output_dtype=torch.bfloat16)
torch.cuda.synchronize()
print("ok")
