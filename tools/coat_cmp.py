"""Ablation (the paper's Fig. 1 / Table 7 contrast):
MOSS MX epilogue-dequant GEMM (K2) vs the per-group main-loop-dequant GEMM
(csrc/pergroup.cu) on the Llama-7B layer shapes, same FLOPs, CUDA events,
back-to-back launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_05811_b200 import _lib
from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.quantize import quant_per_group, quantize_mx2

def timeit(fn, n=10):
    for _ in range(3): fn()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
one = torch.ones(1, device="cuda")
tot_f = tot_mx = tot_pg = 0.0
print(f"{'shape':14s} {'M':>6s} {'N':>6s} {'K':>6s} | MX (ours) TF/s | per-group TF/s | ratio")
for name, K, N in [("qkv", 4096, 12288), ("o", 4096, 4096), ("gate_up", 4096, 22016), ("down", 11008, 4096)]:
    for tag, (m, n, k) in [("fwd", (8192, N, K)), ("dgrad", (8192, K, N)), ("wgrad", (N, K, 8192))]:
        a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
        qa, qb = quantize_mx2(a), quantize_mx2(b)
        out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        t_mx = timeit(lambda: mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out=out))
        pa, pb = quant_per_group(a), quant_per_group(b)
        sa_t, sb_t = pa.scales.t().contiguous(), pb.scales.t().contiguous()
        t_pg = timeit(lambda: _lib.gemm_pergroup(pa.codes, sa_t, pb.codes, sb_t, out))
        f = 2.0 * m * n * k
        tot_f += f; tot_mx += t_mx; tot_pg += t_pg
        print(f"{name + '.' + tag:14s} {m:6d} {n:6d} {k:6d} | {f / t_mx / 1e9:14.0f} | {f / t_pg / 1e9:14.0f} | {t_pg / t_mx:5.2f}x")
print(f"layer total: MX {tot_f / tot_mx / 1e9:.0f} TF/s, per-group {tot_f / tot_pg / 1e9:.0f} TF/s, "
      f"per-group takes {tot_pg / tot_mx:.2f}x the time")
