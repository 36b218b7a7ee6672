"""Per-CTA timeline of the last K1 launch of a layer step from a debug build
(-DQ4_TIMELINE): entry, first tile in smem, exit (globaltimer), cycles, SM id —
eager step vs CUDA-graph replay (the qkv output-gradient quantizer, 8192x12288,
is the step's last K1 launch).
    nvcc ... -DQ4_TIMELINE -o paper_2511_05811_b200/_build/libmoss_q4tl.so csrc/*.cu
    MOSS_B200_LIB=paper_2511_05811_b200/_build/libmoss_q4tl.so python tools/k1_timeline.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_05811_b200 import _lib  # noqa: E402
from paper_2511_05811_b200.nn import CudaGraphStep, MossAdamW  # noqa: E402
from paper_2511_05811_b200.workloads import LayerStack  # noqa: E402

lib = _lib.lib()
lib.moss_q4_timeline.argtypes = [ctypes.c_void_p]
buf = np.zeros(1024 * 8, dtype=np.uint64)


def read(title):
    torch.cuda.synchronize()
    assert lib.moss_q4_timeline(buf.ctypes.data) == 0
    t = buf.reshape(-1, 8).astype(np.int64)
    G = int(t[0, 7])
    t = t[:G]
    t0 = t[:, 0].min()
    entry, first, exit_ = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
    mhz = t[:, 3] / (t[:, 2] - t[:, 0]) * 1e3
    print(f"== {title}: {G} CTAs, {int(t[0, 6])} elems; kernel span {exit_.max():.1f} us")
    q = lambda a: " ".join(f"{v:7.1f}" for v in np.percentile(a, [0, 10, 50, 90, 100]))
    print(f"  entry  us   (min p10 p50 p90 max) {q(entry)}")
    print(f"  first tile  (min p10 p50 p90 max) {q(first)}")
    print(f"  exit   us   (min p10 p50 p90 max) {q(exit_)}")
    print(f"  MHz         (min p10 p50 p90 max) {q(mhz)}")
    print(f"  tiles/CTA   {np.bincount(t[:, 5])[np.bincount(t[:, 5]) > 0]} at {np.nonzero(np.bincount(t[:, 5]))[0]}")
    sms = np.bincount(t[:, 4], minlength=148)
    print(f"  CTAs per SM: {np.bincount(sms)} (index = CTAs on an SM)")
    late = entry > 5
    if late.any():
        print(f"  {late.sum()} CTAs entered > 5 us after the first; their SMs: {sorted(set(t[late, 4].tolist()))[:20]}")


torch.manual_seed(0)
model = LayerStack(device="cuda")
opt = MossAdamW(model, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
x = torch.randn(8192, 4096, device="cuda", dtype=torch.bfloat16).requires_grad_(True)
one = torch.ones((), device="cuda")


def fwd_bwd(xin):
    loss = model(xin)
    loss.backward(one)
    return loss


def eager_step():
    opt.zero_grad()
    fwd_bwd(x.detach().requires_grad_(True))
    opt.step()


N = int(sys.argv[1]) if len(sys.argv) > 1 else 50
for _ in range(N):
    eager_step()
read(f"eager step ({N} steps)")
g = CudaGraphStep(fwd_bwd, opt, (x.detach().clone().requires_grad_(True),))
for _ in range(N):
    g(x)
read(f"graph replay ({N} replays)")
for _ in range(N):
    eager_step()
read(f"eager step again ({N} steps)")
