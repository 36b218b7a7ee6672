"""One launch each of our GEMM and cuBLAS MXFP8 (F.scaled_mm) per shape, for
an ncu --set full comparison.  argv: list of M,N,K."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.quantize import quantize_mx2
shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(8192, 12288, 4096)]
one = torch.ones(1, device="cuda")
for (m, n, k) in shapes:
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    qa = quantize_mx2(a, row=True); qb = quantize_mx2(b, row=True)
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out=out)
    F.scaled_mm(qa.codes.view(torch.float8_e4m3fn), qb.codes.view(torch.float8_e4m3fn).t(), qa.sf.view(torch.float8_e8m0fnu),
                F.ScalingType.BlockWise1x32, qb.sf.view(torch.float8_e8m0fnu), F.ScalingType.BlockWise1x32,
                swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4, output_dtype=torch.bfloat16)
    torch.cuda.synchronize()
