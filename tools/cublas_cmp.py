"""Our tcgen05 MXFP8 GEMM vs cuBLASLt MXFP8 (torch F.scaled_mm, BlockWise1x32,
SWIZZLE_32_4_4) on the same codes and E8M0 scales, C2 shapes (M = 8192).
Both read the identical tcgen05 block-scale layout, so this is also a
cross-check of our SF layout against NVIDIA's library.  Timing: CUDA events,
L2 flushed between iterations, median of 20."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

from paper_2511_05811_b200.gemm import mx_gemm
from paper_2511_05811_b200.quantize import quantize_mx2

flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def timeit(fn, iters=20, warm=5):
    """No host sync inside the loop (the flush kernel keeps the queue ahead of
    the host), so the events bracket device time only."""
    for _ in range(warm):
        fn()
    ev = []
    for _ in range(iters):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        ev.append((s, e))
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in ev)
    return ts[len(ts) // 2]


def main():
    M = int(os.environ.get("M", 8192))
    shapes = [("qkv", 4096, 12288), ("o", 4096, 4096), ("gate_up", 4096, 22016), ("down", 11008, 4096)]
    print(f"{'shape':10s} {'M':>6s} {'N':>6s} {'K':>6s} | {'ours TF/s':>10s} {'cublas mx TF/s':>15s} {'cublas bf16':>12s} | rel diff")
    for name, K, N in shapes:
        for (m, n, k, tag) in [(M, N, K, "fwd"), (M, K, N, "dgrad"), (N, K, M, "wgrad")]:
            a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
            b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
            qa = quantize_mx2(a, row=True)
            qb = quantize_mx2(b, row=True)
            out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            one = torch.ones(1, device="cuda")
            ours = lambda: mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out=out)
            fl = 2.0 * m * n * k
            t_ours = timeit(ours)
            A8 = qa.codes.view(torch.float8_e4m3fn)
            B8 = qb.codes.view(torch.float8_e4m3fn).t()
            sa = qa.sf.view(torch.float8_e8m0fnu)
            sb = qb.sf.view(torch.float8_e8m0fnu)
            try:
                cub = lambda: F.scaled_mm(A8, B8, sa, F.ScalingType.BlockWise1x32, sb, F.ScalingType.BlockWise1x32,
                                          swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                                          output_dtype=torch.bfloat16)
                t_cub = timeit(cub)
                ref = cub().float()
                ours()
                rel = ((out.float() - ref).norm() / ref.norm()).item()
            except Exception as ex:  # noqa: BLE001
                t_cub, rel = float("nan"), str(ex)[:80]
            bt = b.t()
            t_bf = timeit(lambda: torch.mm(a, bt))
            print(f"{name + '.' + tag:14s} {m:6d} {n:6d} {k:6d} | {fl / t_ours / 1e9:10.0f} {fl / t_cub / 1e9:15.0f} "
                  f"{fl / t_bf / 1e9:12.0f} | {rel}")
            del a, b, qa, qb, out


if __name__ == "__main__":
    main()
