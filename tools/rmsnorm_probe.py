"""RMSNorm producer kernels at the 7B width (T = 4096 rows of d = 4096, with the
residual add / residual gradient): algorithmic GB/s of fwd and bwd, 20
back-to-back launches each, CUDA events.  MOSS_RMS_V2 selects the variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import torch  # noqa: E402

from paper_2511_05811_b200 import _lib  # noqa: E402

T, d = int(os.environ.get("T", 4096)), 4096
x = torch.randn(T, d, device="cuda", dtype=torch.bfloat16)
delta = torch.randn_like(x)
xo, y = torch.empty_like(x), torch.empty_like(x)
w = torch.randn(d, device="cuda")
rstd = torch.empty(T, device="cuda")
am = torch.empty(1, device="cuda")
dy, dres, dx = torch.randn_like(x), torch.randn_like(x), torch.empty_like(x)
dw = torch.zeros(d, device="cuda")


def timed(fn, nbytes, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return {"us": ms * 1e3, "gbs": nbytes / (ms / 1e3) / 1e9}


out = {"mode": os.environ.get("MOSS_RMS_V2", "1"), "T": T, "d": d}
out["fwd_residual"] = timed(lambda: _lib.rmsnorm_fwd(x, delta, xo, w, 1e-5, y, rstd, am), T * d * 8)
out["fwd_plain"] = timed(lambda: _lib.rmsnorm_fwd(x, None, None, w, 1e-5, y, rstd, am), T * d * 4)
out["bwd_residual"] = timed(lambda: _lib.rmsnorm_bwd(dy, xo, w, rstd, dres, dx, dw, am), T * d * 8)
out["bwd_plain"] = timed(lambda: _lib.rmsnorm_bwd(dy, xo, w, rstd, None, dx, dw, am), T * d * 6)
print(json.dumps(out))
