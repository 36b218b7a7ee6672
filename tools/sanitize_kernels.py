"""Small invocations of K1 (fused single launch: in-kernel amax + grid
barrier, and producer-amax mode), K2 (2-CTA tcgen05 GEMM, K-major and
MN-major B, f32 accumulate) and K3 (AdamW + FP8 copy), for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_kernels.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2511_05811_b200 import _lib  # noqa: E402
from paper_2511_05811_b200.gemm import mx_gemm, mx_gemm_bkn  # noqa: E402
from paper_2511_05811_b200.optim import adam_params  # noqa: E402
from paper_2511_05811_b200.quantize import quant_per_tensor, quantize_mx2  # noqa: E402

torch.manual_seed(0)
dev = "cuda"
fl = _lib.FlagWord(dev)
which = sys.argv[1:] or ["k1", "k2", "k3", "step"]
if "k1" in which:
    for rows, cols in [(256, 512), (384, 1024)]:
        x = torch.randn(rows, cols, device=dev, dtype=torch.bfloat16)
        q = quantize_mx2(x, row=True, col=True, flags=fl)                       # single launch, grid barrier
        am = x.float().abs().max().reshape(1)
        q2 = quantize_mx2(x, row=True, col=True, flags=fl, amax=am)             # producer-amax mode
        torch.cuda.synchronize()
        os.environ["MOSS_Q4_DYN"] = "2"                                          # dynamic tile tail
        q3 = quantize_mx2(x, row=True, col=True, flags=fl, amax=am)
        q3 = quantize_mx2(x, row=True, col=True, flags=fl, amax=am)             # counter reset
        os.environ.pop("MOSS_Q4_DYN")
        xt = (x.float() * torch.pow(2.0, -torch.randint(40, 110, (rows, 1), device=dev).float())).to(torch.bfloat16)
        q4 = quantize_mx2(xt, row=True, col=True, flags=fl)                      # general (scaled) path
        torch.cuda.synchronize()
        assert torch.equal(q.codes, q2.codes) and torch.equal(q.codes_t, q2.codes_t)
    print("k1 ok", flush=True)
if "k2" in which:
    m, n, k = 512, 512, 512
    a = quantize_mx2(torch.randn(m, k, device=dev, dtype=torch.bfloat16), row=True, col=False, flags=fl)
    b = quantize_mx2(torch.randn(n, k, device=dev, dtype=torch.bfloat16), row=True, col=False, flags=fl)
    y = mx_gemm(a.codes, a.sf, a.g, b.codes, b.sf, b.g, out_dtype=torch.bfloat16)
    acc = torch.zeros(m, n, device=dev, dtype=torch.float32)
    mx_gemm(a.codes, a.sf, a.g, b.codes, b.sf, b.g, out=acc, accumulate=True)               # TMA reduce-add epilogue
    w = quant_per_tensor(torch.randn(k, n, device=dev) * 0.02)
    z = mx_gemm_bkn(a.codes, a.sf, a.g, w.codes, w.scale.reshape(1))                         # MN-major B
    torch.cuda.synchronize()
    assert torch.isfinite(y.float()).all() and torch.isfinite(acc).all() and torch.isfinite(z.float()).all()
    print("k2 ok", flush=True)
if "k3" in which:
    rows, cols = 256, 512
    w = torch.randn(rows, cols, device=dev) * 0.02
    g = torch.randn_like(w) * 1e-3
    mm, vv = torch.zeros_like(w), torch.zeros_like(w)
    codes = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
    amax = torch.zeros(1, device=dev)
    _lib.adamw_fp8(w, g, mm, vv, rows, cols, adam_params(1e-3, 0.9, 0.95, 1e-8, 0.1, 1, True), 1e-4, fl,
                   w_fp8=codes, w_amax=amax)
    torch.cuda.synchronize()
    print("k3 ok", flush=True)
if "step" in which:
    # one LayerStack training step at small shapes: every producer / glue kernel (incl. the
    # offset loss), the quantizers in producer-amax mode, the GEMMs with the amax epilogue, K3
    from paper_2511_05811_b200.nn import MossAdamW
    from paper_2511_05811_b200.workloads import LayerStack
    model = LayerStack(d_model=256, d_ffn=512, device=dev)
    opt = MossAdamW(model, lr=1e-3)
    xs = torch.randn(256, 256, device=dev, dtype=torch.bfloat16)
    for _ in range(2):
        opt.zero_grad()
        loss = model(xs.detach().requires_grad_(True))
        loss.backward()
        opt.step()
    torch.cuda.synchronize()
    opt.check("sanitize step")
    print("step ok", flush=True)
fl.raise_if_set("sanitize")
