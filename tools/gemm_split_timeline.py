"""Per-unit timeline of K2 with the tail split (debug build -DG2_TIMELINE):
for each pair and unit, E0 (MMA: unit start after tmem_empty), E2 (MMA:
last commit issued), E3 (epilogue: accumulator full seen), E5 (epilogue:
TMEM released).  Prints when each round of units starts/ends (us from the
first unit start) so a slow tail is visible.
    nvcc <build flags> -DG2_TIMELINE -shared -o paper_2511_05811_b200/_build/libmoss_tl.so csrc/*.cu
    MOSS_B200_LIB=paper_2511_05811_b200/_build/libmoss_tl.so python tools/gemm_split_timeline.py M N K"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_05811_b200 import _lib
from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.quantize import quantize_mx2

M, N, K = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 4096))]
qa = quantize_mx2(torch.randn(M, K, device="cuda", dtype=torch.bfloat16))
qb = quantize_mx2(torch.randn(N, K, device="cuda", dtype=torch.bfloat16))
one = torch.ones(1, device="cuda")
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out=out)
torch.cuda.synchronize()
buf = np.zeros(74 * 64 * 8, dtype=np.uint64)
lib = _lib.lib()
lib.moss_g2_timeline.argtypes = [ctypes.c_void_p]
assert lib.moss_g2_timeline(buf.ctypes.data) == 0
t = buf.reshape(74, 64, 8).astype(np.int64)
t0 = t[:, 0, 0][t[:, 0, 0] > 0].min()
print(f"split={os.environ.get('MOSS_GEMM2_SPLIT', '1')} GEMM {M}x{N}x{K}")
entry = (t[:, 1, 7] - t0) / 1e3
print(f" kernel entry per pair: {entry.min():7.2f}..{entry.max():7.2f}")
for i in range(8):
    e = t[:, i]
    ok = e[:, 0] > 0
    if not ok.any():
        break
    r = (e[ok] - t0) / 1e3
    f6 = r[:, 6][e[ok][:, 6] > 0]
    print(f" round {i}: pairs {ok.sum():3d}  start {r[:, 0].min():7.2f}..{r[:, 0].max():7.2f}  "
          f"commit {r[:, 2].min():7.2f}..{r[:, 2].max():7.2f}  full-seen {r[:, 3].min():7.2f}..{r[:, 3].max():7.2f}  "
          f"released {r[:, 5].min():7.2f}..{r[:, 5].max():7.2f}  "
          + (f"split-flag {f6.min():7.2f}..{f6.max():7.2f}" if f6.size else ""))
done = (t[:, 0, 7] - t0) / 1e3
print(f" epilogue done per pair: {done.min():7.2f}..{done.max():7.2f}")
