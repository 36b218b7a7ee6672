"""Strides of the SDPA output for [B,S,H,hd]-viewed vs contiguous [B,H,S,hd]
inputs: does O-projection input need a transpose copy?  Diagnostic only."""
import torch, torch.nn.functional as F
B,S,H,hd = 1, 4096, 32, 128
qkv = torch.randn(B, S, 3, H, hd, device="cuda", dtype=torch.bfloat16, requires_grad=True)
q = qkv[:, :, 0].transpose(1, 2); k = qkv[:, :, 1].transpose(1, 2); v = qkv[:, :, 2].transpose(1, 2)
print("q strides", q.stride())
o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
print("o shape", o.shape, "strides", o.stride(), "transpose contiguous:", o.transpose(1, 2).is_contiguous())
qc = torch.empty(B, S, H, hd, device="cuda", dtype=torch.bfloat16).normal_().requires_grad_(True)
kc = torch.empty(B, S, H, hd, device="cuda", dtype=torch.bfloat16).normal_().requires_grad_(True)
vc = torch.empty(B, S, H, hd, device="cuda", dtype=torch.bfloat16).normal_().requires_grad_(True)
o2 = F.scaled_dot_product_attention(qc.transpose(1,2), kc.transpose(1,2), vc.transpose(1,2), is_causal=True)
print("o2 strides", o2.stride(), o2.transpose(1,2).is_contiguous())
do = torch.randn_like(o2.transpose(1,2)).transpose(1,2)
o2.backward(do)
print("grad strides", qc.grad.stride(), kc.grad.stride(), vc.grad.stride())
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    o2 = F.scaled_dot_product_attention(qc.transpose(1,2), kc.transpose(1,2), vc.transpose(1,2), is_causal=True)
    o2.backward(do)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=8, max_name_column_width=70))
