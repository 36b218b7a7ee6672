"""K0/K1 in isolation: two-launch (amax + quantize) vs the fused single launch,
row-only and row+col, on Llama-7B activation shapes (CUDA events, L2 flushed
between iterations, median of 20).  GB/s are algorithmic bytes (input read
once + codes + scales written once) / time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_05811_b200 import _lib
from paper_2511_05811_b200.quantize import sf_buffer

flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
def timeit(fn, iters=20, warm=5):
    """No host sync inside the loop: the 80 us flush kernel keeps the GPU queue
    ahead of the host, so the events bracket device time only (no launch gaps)."""
    for _ in range(warm): fn()
    ev = []
    for _ in range(iters):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); ev.append((s, e))
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in ev)
    return ts[len(ts) // 2]
fl = _lib.FlagWord()
for rows, cols in [(4096, 4096), (8192, 4096), (8192, 11008), (8192, 12288), (8192, 22016)]:
    x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
    n = rows * cols
    am = torch.zeros(1, device="cuda")
    codes = torch.empty(rows, cols, dtype=torch.uint8, device="cuda"); sf = sf_buffer(rows, cols, "cuda")
    ct = torch.empty(cols, rows, dtype=torch.uint8, device="cuda"); sft = sf_buffer(cols, rows, "cuda")
    g = torch.empty(1, device="cuda")
    t_am = timeit(lambda: _lib.amax(x, am, fl))
    t_r2 = timeit(lambda: (_lib.amax(x, am, fl), _lib.quant_mx2(x, am, fl, codes=codes, sf=sf, g_out=g)))
    t_rc2 = timeit(lambda: (_lib.amax(x, am, fl), _lib.quant_mx2(x, am, fl, codes=codes, sf=sf, codes_t=ct, sf_t=sft, g_out=g)))
    t_r1 = timeit(lambda: _lib.quant_mx2_fused(x, am, fl, codes=codes, sf=sf, g_out=g))
    t_rc1 = timeit(lambda: _lib.quant_mx2_fused(x, am, fl, codes=codes, sf=sf, codes_t=ct, sf_t=sft, g_out=g))
    t_rcp = timeit(lambda: _lib.quant_mx2_fused(x, am, fl, amax_given=True, codes=codes, sf=sf, codes_t=ct, sf_t=sft, g_out=g))
    br, brc = n * (2 + 1 + 1 / 32), n * (2 + 2 + 2 / 32)
    print(f"{rows}x{cols}: amax {2*n/t_am/1e6:5.0f} GB/s | row: 2-launch {t_r2*1e3:6.1f} us {br/t_r2/1e6:5.0f} GB/s, "
          f"fused {t_r1*1e3:6.1f} us {br/t_r1/1e6:5.0f} GB/s | row+col: 2-launch {t_rc2*1e3:6.1f} us {brc/t_rc2/1e6:5.0f}, "
          f"fused {t_rc1*1e3:6.1f} us {brc/t_rc1/1e6:5.0f}, producer-amax {t_rcp*1e3:6.1f} us {brc/t_rcp/1e6:5.0f} GB/s",
          flush=True)
fl.raise_if_set("probe")
