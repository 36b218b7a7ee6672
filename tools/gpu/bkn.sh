timeout 300 python -m pytest tests/test_gpu_gemm_bkn.py -q -x 2>&1 | tail -3
timeout 200 python - <<'PY'
import torch
from paper_2511_05811_b200.gemm import mx_gemm, mx_gemm_bkn
from paper_2511_05811_b200.quantize import quantize_mx2
for m, k, n in [(8192, 4096, 4096), (8192, 4096, 11008), (8192, 22016, 4096), (8192, 12288, 4096)]:
    q = quantize_mx2(torch.randn(m, k, device="cuda", dtype=torch.bfloat16))
    w = torch.randint(0, 0x70, (k, n), device="cuda", dtype=torch.uint8)
    wt = w.t().contiguous()
    s = torch.ones(1, device="cuda")
    def t(fn):
        for _ in range(3): fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): fn()
        b.record(); torch.cuda.synchronize()
        return a.elapsed_time(b) / 10
    tk = t(lambda: mx_gemm(q.codes, q.sf, s, wt, None, s))
    tm = t(lambda: mx_gemm_bkn(q.codes, q.sf, s, w, s))
    f = 2.0 * m * n * k
    print(f"{m}x{k}x{n}: K-major W^T {f / tk / 1e9:.0f} TF/s, MN-major W {f / tm / 1e9:.0f} TF/s")
PY
