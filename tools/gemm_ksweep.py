"""Per-tile fixed cost of the GEMM: time(K) over K at fixed M, N, ours vs
cuBLAS MXFP8; intercept / tiles-per-pair = the per-tile bubble."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.nn.functional as F
from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.quantize import quantize_mx2
def timeit(fn, iters=20, warm=5):
    for _ in range(warm): fn()
    ev = []
    for _ in range(iters):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); ev.append((s, e))
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in ev)
    return ts[len(ts) // 2]
one = torch.ones(1, device="cuda")
M, N = 8192, 9472     # 32 x 37 = 1184 pair tiles = 16 waves of 74 pairs exactly
res = {"ours": [], "cublas": []}
Ks = [1024, 2048, 4096, 8192]
for K in Ks:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16); b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    qa = quantize_mx2(a); qb = quantize_mx2(b)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t1 = timeit(lambda: mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out=out))
    A8 = qa.codes.view(torch.float8_e4m3fn); B8 = qb.codes.view(torch.float8_e4m3fn).t()
    t2 = timeit(lambda: F.scaled_mm(A8, B8, qa.sf.view(torch.float8_e8m0fnu), F.ScalingType.BlockWise1x32,
                                    qb.sf.view(torch.float8_e8m0fnu), F.ScalingType.BlockWise1x32,
                                    swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                                    output_dtype=torch.bfloat16))
    res["ours"].append(t1); res["cublas"].append(t2)
    fl = 2 * M * N * K
    print(f"K={K}: ours {t1*1e3:8.1f} us {fl/t1/1e9:6.0f} TF/s | cublas {t2*1e3:8.1f} us {fl/t2/1e9:6.0f} TF/s", flush=True)
for k, v in res.items():
    slope, icpt = np.polyfit(Ks, v, 1)
    print(f"{k}: per-wave fixed cost {icpt*1e3/16:.2f} us, per-K-block(128) time {slope*128*1e3/16:.3f} us")
