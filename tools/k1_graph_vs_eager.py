"""Diagnostic: one K1 launch (producer-amax, row+col) on the same buffers, eager vs
captured in a CUDA graph, and inside a graph that also holds a big wgrad-style
GEMM + a streaming producer ahead of it.  CUPTI durations (us)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2511_05811_b200 import _lib  # noqa: E402
from paper_2511_05811_b200.quantize import sf_buffer  # noqa: E402


def k1_us(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    q = sorted(e.device_time for e in prof.events() if "quant_mx2" in e.name)
    return round(q[len(q) // 2], 1), len(q)


fl = _lib.FlagWord()
for rows, cols in [(8192, 22016), (8192, 4096)]:
    x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
    am = x.abs().max().float().reshape(1)
    codes = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
    sf = sf_buffer(rows, cols, "cuda")
    ct = torch.empty(cols, rows, dtype=torch.uint8, device="cuda")
    sft = sf_buffer(cols, rows, "cuda")
    g = torch.empty(1, device="cuda")

    def q():
        _lib.quant_mx2_fused(x, am, fl, amax_given=True, codes=codes, sf=sf, codes_t=ct, sf_t=sft, g_out=g)
    e = k1_us(q)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        q()
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        q()
    gg = k1_us(gr.replay)
    # graph allocating its own outputs (graph pool) like the training step
    gr2 = torch.cuda.CUDAGraph()
    holder = {}
    with torch.cuda.graph(gr2):
        c2 = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
        s2 = sf_buffer(rows, cols, "cuda")
        ct2 = torch.empty(cols, rows, dtype=torch.uint8, device="cuda")
        st2 = sf_buffer(cols, rows, "cuda")
        x2 = x * 1.0
        _lib.quant_mx2_fused(x2, am, fl, amax_given=True, codes=c2, sf=s2, codes_t=ct2, sf_t=st2, g_out=g)
        holder["o"] = (c2, s2, ct2, st2, x2)
    gp = k1_us(gr2.replay)
    print(f"{rows}x{cols}: eager {e}  graph(same buffers) {gg}  graph(pool buffers, input made in-graph) {gp}", flush=True)
fl.raise_if_set("probe")
