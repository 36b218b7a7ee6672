"""Per-tile timeline of K2 from a debug build (-DG2_TIMELINE): globaltimer
stamps of the MMA warp (E0 tile start after tmem_empty, E1 first k-block
issued, E2 tmem_full commit issued) and of epilogue warp 0 of the leader CTA
(E3 tmem_full seen, E4 TMEM drained, E5 tmem_empty arrived).
    nvcc ... -DG2_TIMELINE -o paper_2511_05811_b200/_build/libmoss_tl.so csrc/*.cu
    MOSS_B200_LIB=paper_2511_05811_b200/_build/libmoss_tl.so python tools/gemm_timeline.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_05811_b200 import _lib
from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.quantize import quantize_mx2

M, N, K = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 9472, 4096))]
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
qa, qb = quantize_mx2(a), quantize_mx2(b)
one = torch.ones(1, device="cuda")
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out=out)
torch.cuda.synchronize()
buf = np.zeros(74 * 64 * 8, dtype=np.uint64)
lib = _lib.lib()
lib.moss_g2_timeline.argtypes = [ctypes.c_void_p]
assert lib.moss_g2_timeline(buf.ctypes.data) == 0
t = buf.reshape(74, 64, 8).astype(np.int64)
tiles = (M // 256) * (N // 256)
n_it = -(-tiles // 74)
t0 = t[:, 0, 0].min()
per = []
for p in range(74):
    for i in range(n_it - 1):
        e = t[p, i]
        nx = t[p, i + 1]
        if (nx == 0).any() or (e == 0).any():
            continue
        per.append([e[4] - e[3], e[5] - e[4], nx[0] - e[5], nx[1] - nx[0], nx[3] - e[3], e[3] - e[2]])
per = np.array(per, dtype=np.float64)
names = ["drain (E4-E3)", "arrive (E5-E4)", "arrive->mma wake (E0'-E5)", "first kblock issue (E1'-E0')",
         "tile period (E3'-E3)", "commit issue->full seen (E3-E2)"]
print(f"GEMM {M}x{N}x{K}: {tiles} tiles, {n_it} per pair; medians over {len(per)} handoffs (us):")
for j, nm in enumerate(names):
    print(f"  {nm:34s} {np.median(per[:, j]) / 1e3:8.3f}   p10 {np.percentile(per[:, j], 10) / 1e3:7.3f}"
          f"   p90 {np.percentile(per[:, j], 90) / 1e3:7.3f}")
print("first tile start spread (us):", (t[:, 0, 0].max() - t0) / 1e3, " last full seen:", (t[:, :n_it, 3].max() - t0) / 1e3)
