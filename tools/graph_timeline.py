"""Kernel timeline of the bench's layer step INSIDE its CUDA graph: every
launch of ours is bracketed by external CUDA events captured into the graph,
so a replay yields each kernel's duration and the idle gap before it — what
the sum of per-kernel times misses against the step time.

    python tools/graph_timeline.py [--replays 20] [--tokens 8192]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2511_05811_b200 import _lib  # noqa: E402
from paper_2511_05811_b200.nn import CudaGraphStep, MossAdamW  # noqa: E402
from paper_2511_05811_b200.workloads import LayerStack  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--replays", type=int, default=20)
ap.add_argument("--tokens", type=int, default=8192)
args = ap.parse_args()
dev = torch.device("cuda")
torch.manual_seed(0)
model = LayerStack(device=dev)
opt = MossAdamW(model, lr=3e-4)
x = torch.randn(args.tokens, 4096, device=dev, dtype=torch.bfloat16).requires_grad_(True)
one = torch.ones((), device=dev)


def fb(xin):
    loss = model(xin)
    loss.backward(one)
    return loss


g = CudaGraphStep(fb, opt, (x,))
g(x)                                   # eager step
_lib.INSTR.start(timing=True, external=True)
g._capture()                           # re-capture with the events inside the graph
_lib.INSTR.stop()
recs = list(_lib.INSTR.records)
torch.cuda.synchronize()
for _ in range(3):
    g(x)
torch.cuda.synchronize()
acc = None
whole = []
for _ in range(args.replays):
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    g(x)
    e0.record()
    torch.cuda.synchronize()
    whole.append(s0.elapsed_time(e0))
    first = recs[0][2]
    row = []
    prev_end = None
    for kind, work, s, e in recs:
        t0 = first.elapsed_time(s)
        dur = s.elapsed_time(e)
        gap = 0.0 if prev_end is None else prev_end.elapsed_time(s)
        row.append((dur, gap))
        prev_end = e
    acc = row if acc is None else [(a[0] + b[0], a[1] + b[1]) for a, b in zip(acc, row)]
n = args.replays
out = []
for (kind, work, _, _), (d, gp) in zip(recs, acc):
    out.append({"kind": kind, "ms": d / n, "gap_before_ms": gp / n,
                "rate": (work / (d / n / 1e3) / (1e12 if kind == "gemm" else 1e9)) if d else None})
tot_k = sum(o["ms"] for o in out)
tot_g = sum(o["gap_before_ms"] for o in out)
span = recs[0][2].elapsed_time(recs[-1][3])
print(json.dumps({"launches": len(out), "sum_kernel_ms": tot_k, "sum_gap_ms": tot_g, "first_to_last_ms": span,
                  "replay_ms_median": sorted(whole)[len(whole) // 2], "kernels": out}, indent=1))
