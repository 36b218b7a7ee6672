"""One launch each of: quant v3 row+col (8192x11008), our GEMM and cuBLAS MXFP8 on qkv.fwd
(8192x12288x4096) -- the target list for an ncu --set full capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
from paper_2511_05811_b200 import _lib
from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.quantize import quantize_mx2, sf_buffer
fl = _lib.FlagWord()
x = torch.randn(8192, 11008, device="cuda", dtype=torch.bfloat16)
am = torch.zeros(1, device="cuda"); _lib.amax(x, am, fl)
codes = torch.empty(8192, 11008, dtype=torch.uint8, device="cuda"); sf = sf_buffer(8192, 11008, "cuda")
ct = torch.empty(11008, 8192, dtype=torch.uint8, device="cuda"); sft = sf_buffer(11008, 8192, "cuda")
g = torch.empty(1, device="cuda")
for _ in range(2):
    _lib.quant_mx2(x, am, fl, codes=codes, sf=sf, codes_t=ct, sf_t=sft, g_out=g)
for _ in range(2):
    _lib.quant_mx2_fused(x, am, fl, codes=codes, sf=sf, codes_t=ct, sf_t=sft, g_out=g)
for _ in range(2):
    _lib.quant_mx2_fused(x, am, fl, amax_given=True, codes=codes, sf=sf, codes_t=ct, sf_t=sft, g_out=g)
a = torch.randn(8192, 4096, device="cuda", dtype=torch.bfloat16)
b = torch.randn(12288, 4096, device="cuda", dtype=torch.bfloat16)
qa = quantize_mx2(a, row=True); qb = quantize_mx2(b, row=True)
one = torch.ones(1, device="cuda")
out = torch.empty(8192, 12288, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out=out)
A8 = qa.codes.view(torch.float8_e4m3fn); B8 = qb.codes.view(torch.float8_e4m3fn).t()
for _ in range(2):
    F.scaled_mm(A8, B8, qa.sf.view(torch.float8_e8m0fnu), F.ScalingType.BlockWise1x32, qb.sf.view(torch.float8_e8m0fnu),
                F.ScalingType.BlockWise1x32, swizzle_a=F.SwizzleType.SWIZZLE_32_4_4,
                swizzle_b=F.SwizzleType.SWIZZLE_32_4_4, output_dtype=torch.bfloat16)
torch.cuda.synchronize()
