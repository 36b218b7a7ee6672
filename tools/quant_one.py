"""One producer-amax row+col quantization of an 8192 x 4096 bf16 tensor (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_05811_b200 import _lib
from paper_2511_05811_b200.quantize import sf_buffer
rows, cols = 8192, 4096
x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
am = x.abs().max().float().reshape(1)
fl = _lib.FlagWord()
codes = torch.empty(rows, cols, dtype=torch.uint8, device="cuda"); sf = sf_buffer(rows, cols, "cuda")
ct = torch.empty(cols, rows, dtype=torch.uint8, device="cuda"); sft = sf_buffer(cols, rows, "cuda")
g = torch.empty(1, device="cuda")
for _ in range(3):
    _lib.quant_mx2_fused(x, am, fl, amax_given=True, codes=codes, sf=sf, codes_t=ct, sf_t=sft, g_out=g)
torch.cuda.synchronize()
