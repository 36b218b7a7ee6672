#!/usr/bin/env python
"""MOSS FP8 training-step benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], as a training step):
  the five Llama-7B linear shapes of one decoder layer (QKV 4096->12288,
  O 4096->4096, gate/up 4096->2x11008 fused, down 11008->4096) at M = 8192
  tokens per GPU, through the public API (MossLinear + MossAdamW):
  forward + backward with every input and gradient two-level quantized
  (row- and column-wise) and every GEMM an FP8 tcgen05 block-scaled GEMM
  (fwd, dgrad, wgrad), then the fused AdamW + autoscale + FP8 weight copy.
  N > 1: data parallel, per-rank batch fixed (weak scaling), FP32 gradients
  all-reduced over NCCL in buckets overlapped with backward.

metric/unit: BASELINE.json's metric; value = whole-job GEMM FLOPs per second
  (6 * tokens * sum(N*K) per step / step time, all ranks), TFLOP/s.
e2e: the same step with the input copied from pinned host memory and the loss
  read back to the host every step.
roofline: the dominant kernel (the GEMM), FLOPs per launch / CUDA-event
  duration per launch over the timed region, vs 2x the measured dense bf16
  peak (MEASURED_PEAKS.json; fp8 dense = 2x bf16 on B200).
  The peak is cuBLASLt MXFP8 (8192^3) measured in the same run, sustained
  (back-to-back for ~3 s, the kernel is timed inside a long step) and burst.
cpu_baseline / --impl reference: the CPU oracle port (oracle/numpy_ref, the
  reference's own numpy dataflow) timed on ONE bounded sample of the same
  workload (REF_SAMPLE below), on the host cores; the reference arm prints
  exactly this arm's ``config``.
--gpus N (N > 1) without WORLD_SIZE in the environment re-executes itself
  under torchrun with N ranks (one per GPU, NCCL); under torchrun the world
  size must equal --gpus.  Every N runs the same timing mode (CUDA-graph
  replays, the NCCL collectives captured in the graph) and reports the
  Llama-2-7B-shape step (configs[3]/[4]) tokens/s beside the layer value.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP8 GEMM TFLOP/s, quantize GB/s; 7B-shape train tokens/s at 1/2/4/8 B200"
LAYER_WORKLOAD = ("configs[1]: MOSS quantize + MXFP8 fwd/dgrad/wgrad GEMMs over the Llama-7B linear shapes "
                  "(QKV 4096->12288, O 4096->4096, gate/up 4096->2x11008, down 11008->4096) + fused "
                  "AdamW/autoscale/FP8-copy, as one training step")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--workload", choices=["layer", "llama7b"], default="layer",
                    help="layer: configs[1] (default); llama7b: configs[3]/[4] Llama-2-7B-shape decoder step")
    ap.add_argument("--layers", type=int, default=32, help="llama7b: decoder layers (truncate to fit)")
    ap.add_argument("--seq", type=int, default=4096, help="llama7b: sequence length")
    ap.add_argument("--llama-batch", type=int, default=1,
                    help="llama7b: sequences per GPU per step (configs[3]/SURVEY 8(d) C4: batch 1)")
    ap.add_argument("--no-llama-batch2", action="store_true",
                    help="skip the extra 7B measurement at 2 sequences per GPU (llama7b_batch2: 8192 tokens, "
                         "145 GB peak on 1 B200; profiles/r02_llama7b_batch_sweep.json)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-llama", action="store_true",
                    help="layer workload: skip the Llama-2-7B-shape tokens/s sub-measurement (configs[3])")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA-graph replays")
    ap.add_argument("--zero1", action="store_true",
                    help="N>1: ZeRO-1 (reduce-scatter grads, sharded K3, FP8 all-gather) instead of all-reduce DP")
    ap.add_argument("--no-fp8-roof", action="store_true", help="skip the cuBLASLt MXFP8 roof measurement")
    ap.add_argument("--llama-steps", type=int, default=8, help="default line: timed steps of the 7B sub-measure")
    ap.add_argument("--launch-probe", action="store_true",
                    help="test hook: spawn/check the ranks, print who ran, touch no GPU")
    return ap.parse_args()


_BLAS_LIMITS = None


def free_port() -> int:
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def maybe_spawn(args) -> int | None:
    """--gpus N > 1 outside torchrun: run this script under torchrun with N
    ranks (the driver's own launch line) and return its exit code."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def launch_probe(args, world: int, rank: int, local: int) -> None:
    import torch.distributed as dist
    info = {"rank": rank, "local_rank": local, "pid": os.getpid(), "world": world}
    infos = [info]
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
        infos = [None] * world
        dist.all_gather_object(infos, info)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"launch_probe": True, "n_gpus": world, "gpus_flag": args.gpus, "ranks": infos}), flush=True)


# ------------------------------------------------------------------ CPU oracle leg
def cpu_linear_step(tokens: int, d_in: int, d_out: int, seed: int = 0, ops: dict | None = None) -> float:
    """One MOSS linear fwd + dgrad + wgrad + AdamW/autoscale step through the
    CPU oracle (the reference's numpy dataflow: per-32-block float64 GEMMs,
    gemm.py:115-129; float64 AdamW, optim.py:78-106).  Returns seconds; the
    per-op seconds (quant_two_level, weight encode,
    gemm_mx_epilogue, adamw_step, auto_scale_advance) accumulate into ``ops``."""
    import numpy as np

    from oracle import numpy_ref as R

    ops = {} if ops is None else ops

    def timed(name, fn, *a):
        t = time.perf_counter()
        r = fn(*a)
        ops[name] = ops.get(name, 0.0) + time.perf_counter() - t
        return r

    rng = np.random.default_rng(seed)
    x = rng.standard_normal((tokens, d_in)).astype(np.float32)
    w = rng.standard_normal((d_out, d_in)) * 0.02
    dy = (rng.standard_normal((tokens, d_out)) * 1e-3).astype(np.float32)
    st = R.adam_init(w.shape, eta=3e-4, weight_decay=0.1)
    sched = R.Schedule(s_t=R.jit_scale(w))
    t0 = time.perf_counter()
    wc, _ = timed("weight_encode", R.encode_weight, w, sched.s_t)                  # train.py:168
    qx = timed("quant_two_level", R.quant_two_level, x)                             # train.py:171
    timed("gemm_mx_epilogue", R.gemm_mx_epilogue, wc, sched.s_t, qx)                # fwd
    qdy = timed("quant_two_level", R.quant_two_level, dy)
    timed("gemm_mx_epilogue", R.gemm_mx_epilogue, np.ascontiguousarray(wc.T), sched.s_t, qdy)   # dgrad
    qdy_t = timed("quant_two_level", R.quant_two_level, np.ascontiguousarray(dy.T))
    qx_t = timed("quant_two_level", R.quant_two_level, np.ascontiguousarray(x.T))

    def wgrad():
        a = R.dequantize_two_level(qdy_t)
        b = R.fp8_decode(qx_t.codes).astype(np.float64)
        ss = R.e8m0_decode(qx_t.micro_codes).astype(np.float64)
        dw = np.zeros((d_out, d_in))
        for blk in range(tokens // 32):                         # wgrad, same block dataflow
            sl = slice(blk * 32, (blk + 1) * 32)
            dw += (a[:, sl] @ b[:, sl].T) * ss[None, :, blk]
        return dw * qx_t.global_scale
    dw = timed("gemm_mx_epilogue", wgrad)
    w, _ = timed("adamw_step", R.adamw_step, w, dw, st)                             # optim.py:78-106
    timed("auto_scale_advance", R.advance, sched, 3e-4)                             # autoscale.py:71-79
    return time.perf_counter() - t0


# The ONE bounded CPU sample of the workload, shared by cpu_baseline (our arm)
# and the reference arm: a quarter of configs[0] (BASELINE configs[0] is
# tokens = K = N = 4096; its full size is ~36 s per step through the port,
# ~15 min for the driver's 25 steps).  tools/ref_vs_port_timing.py times the
# literal mossq against the port on this sample (profiles/r02_ref_vs_port.txt).
REF_SAMPLE = {"tokens": 1024, "d": 4096}


def ref_sample_desc() -> str:
    return (f"one MOSS linear fwd+dgrad+wgrad+AdamW/autoscale step, tokens={REF_SAMPLE['tokens']}, "
            f"{REF_SAMPLE['d']}x{REF_SAMPLE['d']} (1/4 of configs[0]), oracle/numpy_ref (the reference's numpy "
            f"dataflow: per-32-block float64 GEMMs, float64 AdamW), all host threads")


def cpu_sample(tokens: int, d: int, reps: int = 1) -> dict:
    ops: dict = {}
    secs = min(cpu_linear_step(tokens, d, d, seed=r, ops=ops) for r in range(reps))
    flops = 6.0 * tokens * d * d
    return {"value": flops / secs / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
            "sample": ref_sample_desc() + f"; {secs:.2f} s",
            "per_op_seconds": {k: round(v / reps, 4) for k, v in ops.items()},
            "seconds": secs}


def run_reference(args, world: int, rank: int) -> None:
    """Reference arm: the reference's CPU path (the oracle port) on REF_SAMPLE
    per step, rank 0 only; same metric/unit/config as this script's GPU arm."""
    if rank != 0:
        return
    tokens, d = REF_SAMPLE["tokens"], REF_SAMPLE["d"]
    for i in range(args.warmup):
        cpu_linear_step(tokens, d, d, seed=1000 + i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        cpu_linear_step(tokens, d, d, seed=i)
    secs = (time.perf_counter() - t0) / args.steps
    value = 6.0 * tokens * d * d / secs / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 (reference numpy)", "data": "synthetic",
            "config": layer_config(args, world),
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": "per step: " + ref_sample_desc()},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def layer_config(args, world: int) -> dict:
    """``config`` of the default line (configs[1] as a training step), shared by both arms."""
    from paper_2511_05811_b200.workloads import LLAMA7B_SHAPES
    T = args.tokens
    par = f"dp{world}"
    if world > 1:
        par += (" (ZeRO-1: NCCL reduce-scatter fp32 grads, sharded K3, FP8 all-gather)" if args.zero1
                else " (NCCL bucketed fp32 grad all-reduce, captured in the step graph)")
    elif args.zero1:
        par += " (ZeRO-1 driver)"
    return {"workload": LAYER_WORKLOAD, "tokens_per_gpu": T, "global_batch_tokens": T * world, "parallelism": par,
            "gemm_flops_per_step_per_gpu": 6.0 * T * sum(k * n for k, n in LLAMA7B_SHAPES.values()),
            "l2": "not flushed: per-step working set ~3 GB >> 126 MB L2"}


# ------------------------------------------------------------------ library reference for the GEMM roofline
def gemm_vs_cublas(dev, tokens: int) -> dict | None:
    """Our K2 and cuBLASLt MXFP8 (torch F.scaled_mm, BlockWise1x32) on the same
    codes/scales for the 12 GEMMs of one layer step (fwd, dgrad, wgrad of the
    Llama-7B linears); FLOP-weighted TFLOP/s of each, back-to-back launches
    timed with CUDA events (device time only).  cuBLAS is a library
    measurement of this box's attainable MXFP8 rate, not part of the product."""
    import torch
    import torch.nn.functional as F

    from paper_2511_05811_b200.gemm import mx_gemm
    from paper_2511_05811_b200.quantize import quantize_mx2
    if not hasattr(F, "scaled_mm"):
        return None
    shapes = []
    for k, n in [(4096, 12288), (4096, 4096), (4096, 22016), (11008, 4096)]:
        shapes += [(tokens, n, k), (tokens, k, n), (n, k, tokens)]
    one = torch.ones(1, device=dev)
    t_ours = t_cub = flops = 0.0
    for (m, n, k) in shapes:
        a = torch.randn(m, k, device=dev, dtype=torch.bfloat16)
        b = torch.randn(n, k, device=dev, dtype=torch.bfloat16)
        qa, qb = quantize_mx2(a), quantize_mx2(b)
        out = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
        A8, B8 = qa.codes.view(torch.float8_e4m3fn), qb.codes.view(torch.float8_e4m3fn).t()
        sa, sb = qa.sf.view(torch.float8_e8m0fnu), qb.sf.view(torch.float8_e8m0fnu)

        def ours():
            mx_gemm(qa.codes, qa.sf, one, qb.codes, qb.sf, one, out=out)

        def cub():
            F.scaled_mm(A8, B8, sa, F.ScalingType.BlockWise1x32, sb, F.ScalingType.BlockWise1x32,
                        swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                        output_dtype=torch.bfloat16)
        for fn in (ours, cub):
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        # interleaved rounds (the power-capped clock drifts within a run), CUPTI kernel spans
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(4):
                for fn in (ours, cub):
                    for _ in range(3):
                        fn()
            torch.cuda.synchronize()
        ko = sorted(ev.device_time for ev in prof.events()
                    if ev.device_type == torch.autograd.DeviceType.CUDA and "gemm_mxf8" in ev.name)
        lib: dict = {}                 # the library's GEMM kernel: the non-moss kernel with the most time
        for ev in prof.events():
            if ev.device_type == torch.autograd.DeviceType.CUDA and "moss::" not in ev.name:
                lib.setdefault(ev.name, []).append(ev.device_time)
        kc = sorted(max(lib.values(), key=sum)) if lib else [float("nan")]
        t_ours += ko[len(ko) // 2] / 1e3
        t_cub += kc[len(kc) // 2] / 1e3
        flops += 2.0 * m * n * k
        del a, b, qa, qb, out
    return {"ours_tflops": flops / (t_ours / 1e3) / 1e12, "cublas_mxfp8_tflops": flops / (t_cub / 1e3) / 1e12,
            "ours_over_cublas": t_cub / t_ours,
            "how": "12 layer GEMMs (fwd/dgrad/wgrad of QKV, O, gate_up, down) at M=%d, same codes and E8M0 scales, "
                   "4 interleaved rounds of 3 launches each, median CUPTI kernel span; cuBLASLt via torch "
                   "F.scaled_mm" % tokens}


def quantizer_rates(dev, tokens: int, hbm: float) -> dict:
    """K1 on the 8 tensors one layer step quantizes (inputs and output-gradients
    of the four linears, row + column-wise), both modes: the single launch with
    the in-kernel amax (input read twice when it exceeds smem + L2) and the
    producer-amax mode the Llama decoder runs (input read once).  GB/s of
    ALGORITHMIC bytes (4.063 B/elem), back-to-back launches."""
    import torch

    from paper_2511_05811_b200 import _lib
    from paper_2511_05811_b200.quantize import sf_buffer
    fl = _lib.FlagWord(dev)
    res = {}
    for mode in ("single_launch_amax", "producer_amax"):
        byts = ms = 0.0
        for cols in (4096, 4096, 4096, 11008, 12288, 4096, 22016, 4096):
            x = torch.randn(tokens, cols, device=dev, dtype=torch.bfloat16)
            am = x.float().abs().max().reshape(1)
            c = torch.empty(tokens, cols, dtype=torch.uint8, device=dev)
            ct = torch.empty(cols, tokens, dtype=torch.uint8, device=dev)
            sf, sft = sf_buffer(tokens, cols, dev), sf_buffer(cols, tokens, dev)
            g = torch.empty(1, device=dev)
            fn = lambda: _lib.quant_mx2_fused(x, am, fl, amax_given=mode == "producer_amax", codes=c, sf=sf,
                                               codes_t=ct, sf_t=sft, g_out=g)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            # kernel spans (CUPTI): host-issued ctypes launches of a ~25 us kernel can leave
            # the GPU idle between launches, which an event pair around the loop would count
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                for _ in range(10):
                    fn()
                torch.cuda.synchronize()
            ts = sorted(ev.device_time for ev in prof.events() if "quant_mx2" in ev.name)
            ms += ts[len(ts) // 2] / 1e3                      # median launch, us -> ms
            byts += tokens * cols * (4 + 2 / 32)
        res[mode] = {"achieved_gbs": byts / (ms / 1e3) / 1e9, "frac_of_hbm": byts / (ms / 1e3) / 1e9 / hbm,
                     "ms_per_step": ms}
    fl.raise_if_set("quantizer_rates")
    res["how"] = ("the 8 row+col quantizations of one layer step at M=%d, 10 back-to-back launches each (inputs > "
                  "L2 are re-read by the single-launch mode), median CUPTI kernel span per tensor, algorithmic "
                  "bytes 4.063 B/elem; measured at the end of the bench run (hot, power-capped GPU)" % tokens)
    return res


def fp8_roof(dev, gpu_index: int, seconds: float = 3.0) -> dict:
    """The FP8 roofline denominator, measured: cuBLASLt MXFP8 (torch
    F.scaled_mm, BlockWise1x32 E8M0 scales, bf16 out) at 8192^3.  burst = best
    single launch of 10 (a kernel timed alone); sustained = back-to-back
    launches for ``seconds`` under the power cap (a kernel timed inside a long
    step), with the SM clocks of each.  A library measurement, not the product."""
    import torch
    import torch.nn.functional as F

    from paper_2511_05811_b200.quantize import quantize_mx2
    n = 8192
    a = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    b = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    qa, qb = quantize_mx2(a), quantize_mx2(b)
    A8, B8 = qa.codes.view(torch.float8_e4m3fn), qb.codes.view(torch.float8_e4m3fn).t()
    sa, sb = qa.sf.view(torch.float8_e8m0fnu), qb.sf.view(torch.float8_e8m0fnu)

    def cub():
        return F.scaled_mm(A8, B8, sa, F.ScalingType.BlockWise1x32, sb, F.ScalingType.BlockWise1x32,
                           swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                           output_dtype=torch.bfloat16)
    flops = 2.0 * n ** 3
    for _ in range(5):
        cub()
    torch.cuda.synchronize()
    best = float("inf")
    with ClockSampler(gpu_index) as ck_b:
        for _ in range(10):
            s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            cub()
            e0.record()
            torch.cuda.synchronize()
            best = min(best, s0.elapsed_time(e0))
    reps = max(20, int(seconds * 1e3 / best))
    with ClockSampler(gpu_index) as ck_s:
        s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(reps):
            cub()
        e0.record()
        torch.cuda.synchronize()
    sus = s0.elapsed_time(e0) / reps
    return {"burst_tflops": flops / (best / 1e3) / 1e12, "sustained_tflops": flops / (sus / 1e3) / 1e12,
            "clocks_burst": ck_b.summary(), "clocks_sustained": ck_s.summary(), "sustained_launches": reps,
            "how": "cuBLASLt MXFP8 via torch F.scaled_mm (BlockWise1x32, SWIZZLE_32_4_4), 8192^3, bf16 out; burst = "
                   "best of 10 single launches, sustained = %d back-to-back launches (~%.0f s)" % (reps, seconds)}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region (NVML in a
    background thread every 20 ms; nvidia-smi is the fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.th = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                             int(get_reasons(h))))
                    except Exception:  # noqa: BLE001
                        pass
                    self._stop.wait(0.02)
            self.th = threading.Thread(target=run, daemon=True)
            self.th.start()
        except Exception:  # noqa: BLE001 - no NVML: no samples, reported as such
            self.th = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.th is not None:
            self.th.join(timeout=2)
        return False

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"], "samples": 0}
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(c for c, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "NVML, 20 ms period, timed region"}


# ------------------------------------------------------------------ GPU arm
def _max_over_ranks(v: float, dev, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def foreign_launches(step, x) -> dict | None:
    """Kernels of one eager step that are not ours (torch.profiler / CUPTI):
    name -> count.  Evidence for ``gpu_launches`` (which counts our kernels)."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step(x)
            torch.cuda.synchronize()
        out: dict = {}
        for ev in prof.events():
            if ev.device_type == torch.autograd.DeviceType.CUDA and "moss::" not in ev.name \
                    and not ev.name.startswith(("Memcpy", "Memset", "ncclDevKernel")):
                out[ev.name[:80]] = out.get(ev.name[:80], 0) + 1
        return out
    except Exception as ex:  # noqa: BLE001 - evidence only
        return {"error": str(ex)[:160]}


_KINDS = (("gemm_mxf8", "gemm"), ("quant_mx2", "quant"), ("adamw_fp8", "adamw"), ("amax_kernel", "amax"),
          ("rmsnorm", "producer"), ("swiglu", "producer"), ("rope_", "producer"), ("glue_kernel", "producer"),
          ("sumsq", "producer"))


def replay_kernel_times(runner, x, reps: int, sleep_cycles: int = 0) -> dict | None:
    """Per-kind kernel time of the TIMED mode itself (CUDA-graph replays), from
    the hardware start/end timestamps CUPTI records for every kernel (torch.profiler):
    kind -> {"ms": per step, "launches": per step}.  Unlike the event-bracketed
    eager pass, no event record or launch latency sits inside a kernel's span.
    With ``sleep_cycles`` (the eager pass) each step is preceded by a device sleep
    and followed by a synchronize, exactly as in the event-bracketed pass."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(reps):
                if sleep_cycles:
                    torch.cuda._sleep(sleep_cycles)
                runner(x)
                if sleep_cycles:
                    torch.cuda.synchronize()
            torch.cuda.synchronize()
        out: dict = {}
        seq: list = []
        for ev in prof.events():
            if ev.device_type != torch.autograd.DeviceType.CUDA:
                continue
            if "quant_mx2" in ev.name or "gemm_mxf8" in ev.name:
                seq.append(("q" if "quant" in ev.name else "g", round(ev.device_time, 1)))
            if sleep_cycles and "spin_kernel" in ev.name:
                continue                                     # the device sleep ahead of each step
            if "moss::" not in ev.name:
                kind = "memset/memcpy" if ev.name.startswith(("Memset", "Memcpy")) else "foreign"
            else:
                kind = next((k for pat, k in _KINDS if pat in ev.name), "other")
            d = out.setdefault(kind, {"ms": 0.0, "launches": 0})
            d["ms"] += ev.device_time / 1e3 / reps           # device_time: us
            d["launches"] += 1
        for d in out.values():
            d["launches"] /= reps
        per = len(seq) // reps if reps else 0
        out["last_replay_quant_gemm_us"] = seq[-per:] if per else []
        return out
    except Exception as ex:  # noqa: BLE001 - evidence only
        return {"error": str(ex)[:160]}


def measure(kind: str, args, dev, rank: int, world: int, steps: int, want_e2e: bool, batch: int | None = None) -> dict:
    """Build one workload, warm it up, time it; returns the measurements.
    kind: "layer" (configs[1] as a training step) or "llama7b" (configs[3]/[4])."""
    import torch
    import torch.distributed as dist

    from paper_2511_05811_b200 import _lib
    from paper_2511_05811_b200.dist import GradBuckets
    from paper_2511_05811_b200.nn import CudaGraphStep, MossAdamW
    from paper_2511_05811_b200.workloads import LayerStack

    torch.manual_seed(1234)          # identical initial weights on every rank (DP)
    if kind == "llama7b":
        from paper_2511_05811_b200.llama import LLAMA2_7B, LlamaConfig, LlamaModel
        from paper_2511_05811_b200.trainer import make_optimizer
        cfg = LlamaConfig(**{**LLAMA2_7B.__dict__, "n_layers": args.layers, "max_seq": args.seq})
        model = LlamaModel(cfg, device=dev)
        opt = make_optimizer(model, 3e-4, 10_000, 100)
        B = batch or args.llama_batch
        T = args.seq * B
        g = torch.Generator(device=dev).manual_seed(99 + rank)      # per-rank batch shard
        tok = torch.randint(0, cfg.vocab, (B, args.seq + 1), device=dev, generator=g)
        x, y_tok = tok[:, :-1].contiguous(), tok[:, 1:].contiguous()
        flops_step = float(cfg.gemm_flops_per_token()) * T
        fwd = lambda xin: model(xin, y_tok)
    else:
        model = LayerStack(device=dev)
        opt = MossAdamW(model, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
        T = args.tokens
        torch.manual_seed(4321 + rank)   # per-rank batch shard
        # the step's input requires grad: all 12 GEMMs (fwd, dgrad, wgrad of the 4 linears) run,
        # matching the FLOP count (the first layer's dgrad is the gradient a real model passes down)
        x = torch.randn(T, model.d, device=dev, dtype=torch.bfloat16).requires_grad_(True)
        flops_step = float(model.gemm_flops_per_token()) * T
        fwd = model
    if args.zero1:
        from paper_2511_05811_b200.zero import Zero1
        buckets = Zero1(opt, bucket_mb=64)
    else:
        buckets = GradBuckets(model, bucket_mb=64) if world > 1 else None
    if buckets is not None:
        opt.grad_scale = buckets.grad_scale

    one = torch.ones((), device=dev, dtype=torch.float32)

    def fwd_bwd(xin):
        loss = fwd(xin)
        loss.backward(one)          # a resident seed gradient: no fill kernel per step
        return loss

    def step(xin):
        if buckets is not None:
            buckets.reset()
        else:
            opt.zero_grad()
        if xin.is_floating_point():
            xin = xin.detach().requires_grad_(True)   # fresh leaf: dX of the first layer is computed, not accumulated
        loss = fwd_bwd(xin)
        if buckets is not None:
            buckets.finish()
        if hasattr(buckets, "step"):
            buckets.step()
        else:
            opt.step()
        return loss

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        step(x)
    opt.check("warmup")
    barrier()

    # ---- per-kernel timing pass (eager, every launch bracketed by CUDA events).
    # A device-side sleep ahead of each step lets the host enqueue the whole
    # step first, so the events bracket GPU time only (no host launch gaps).
    h0 = time.perf_counter()
    step(x)
    torch.cuda.synchronize()
    issue_ms = (time.perf_counter() - h0) * 1e3
    sleep_cycles = int(issue_ms * 2.5 * 2.0e6)          # ~2.5x the host issue time at ~2 GHz
    _lib.INSTR.start(timing=True)
    if hasattr(buckets, "timing"):
        buckets.timing = True
    for _ in range(steps):
        torch.cuda._sleep(sleep_cycles)
        step(x)
        torch.cuda.synchronize()
    _lib.INSTR.stop()
    comm = buckets.comm_summary() if hasattr(buckets, "comm_summary") else None
    if hasattr(buckets, "timing"):
        buckets.timing = False
    kern = _lib.INSTR.summary()
    launches = _lib.INSTR.launches // steps
    # every rank runs the profiled step (it contains the gradient collectives); rank 0 reports
    foreign = foreign_launches(step, x)
    barrier()
    # the same eager pass with CUPTI kernel timestamps instead of events (no event
    # record / launch latency inside a kernel's span: matters for ~30 us kernels)
    eager_kern = replay_kernel_times(step, x, min(steps, 10 if kind == "layer" else 2), sleep_cycles=sleep_cycles)
    barrier()

    # ---- the same timing mode at every N: CUDA-graph replays of the whole step
    # (forward, backward, the captured NCCL collectives, the optimizer kernels)
    runner, mode = step, "eager steps"
    quant_modes = None
    if not args.no_graph:
        try:
            static_x = x.detach().clone().requires_grad_(x.requires_grad)
            graphed = CudaGraphStep(fwd_bwd, opt, (static_x,), buckets=buckets)
            runner = lambda xin: graphed(xin)
            for _ in range(3):          # first call is eager + capture, then replays
                runner(x)
            mode = "CUDA-graph replays"
            quant_modes = getattr(graphed, "capture_quant_modes", None)
        except Exception as ex:  # noqa: BLE001 - record and time eagerly rather than lose the line
            runner, mode = step, f"eager steps (graph capture failed: {str(ex)[:120]})"
        barrier()

    # ---- timed region: inputs resident in HBM; working set per step >> L2
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clocks:
        s_ev.record()
        h0 = time.perf_counter()
        for _ in range(steps):
            loss = runner(x)
        host_ms = (time.perf_counter() - h0) * 1e3 / steps
        e_ev.record()
        torch.cuda.synchronize()
    barrier()
    ms = _max_over_ranks(s_ev.elapsed_time(e_ev) / steps, dev, world)
    opt.check("timed region")
    # per-kernel hardware durations inside the timed mode (after the timed region)
    with ClockSampler(dev.index) as rclocks:
        replay_kern = replay_kernel_times(runner, x, min(steps, 10))
    if isinstance(replay_kern, dict):
        replay_kern["clocks"] = rclocks.summary()
    barrier()

    # ---- e2e: input from pinned host memory, loss read back every step.
    # Input pipeline as a training loop runs it: the H2D copy of step i+1's
    # batch (pinned -> device staging buffer, copy engine, own stream) overlaps
    # step i's compute; each step's loss is copied D2H into a pinned slot
    # without stalling the host.  All copies are inside the timed region.
    e2e = None
    if want_e2e:
        x_host = x.detach().cpu().pin_memory()
        loss_host = torch.empty(steps, dtype=torch.float32).pin_memory()
        stage = [torch.empty_like(x) for _ in range(2)]
        cstream = torch.cuda.Stream(device=dev)
        ready = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        barrier()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()

        def prefetch(i):
            b = i % 2
            with torch.cuda.stream(cstream):
                cstream.wait_event(s2)
                if i >= 2:
                    cstream.wait_event(consumed[b])          # step i-2 is done reading this buffer
                with torch.no_grad():
                    stage[b].copy_(x_host, non_blocking=True)
                ready[b].record(cstream)

        prefetch(0)
        for i in range(steps):
            b = i % 2
            if i + 1 < steps:
                prefetch(i + 1)
            torch.cuda.current_stream().wait_event(ready[b])
            loss = runner(stage[b])
            consumed[b].record()
            loss_host[i].copy_(loss.detach().reshape(()), non_blocking=True)
        e2.record()
        torch.cuda.synchronize()
        assert bool(torch.isfinite(loss_host).all()), "non-finite loss in the e2e run"
        ms_e2e = _max_over_ranks(s2.elapsed_time(e2) / steps, dev, world)
        e2e = {"ms_per_step": ms_e2e, "h2d_bytes_per_step": x_host.numel() * x_host.element_size(),
               "d2h_bytes_per_step": 4,
               "pipeline": "pinned H2D of step i+1 on a copy stream overlapped with step i; per-step loss D2H async"}
    # peak device memory of the training run (weights, optimizer state, FP8 copies,
    # the stashed FP8 activation codes, graph pool), before any side measurement
    peak_gb = torch.cuda.max_memory_allocated(dev) / 1e9
    return {"ms": ms, "host_ms": host_ms, "kern": kern, "replay_kern": replay_kern, "eager_kern": eager_kern,
            "launches": launches,
            "quant_modes": quant_modes,
            "foreign": foreign, "comm": comm,
            "clocks": clocks.summary(), "e2e": e2e, "peak_gb": peak_gb, "mode": mode, "flops_step": flops_step,
            "T": T, "steps": steps}


def _free_cuda() -> None:
    import gc

    import torch
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()


def _rates(kern: dict, steps: int, hbm: float, replay: dict | None = None, eager: dict | None = None):
    """kind -> rates: the event-bracketed eager pass (achieved_gbs, frac_of_hbm),
    the CUPTI durations of the same eager pass (cupti_*: kernel start/end
    timestamps, no event/launch latency) and of the graph replays (replay_*); the
    algorithmic work per step is the same for all three."""
    def rate(kind):
        d = kern.get(kind)
        if not d or not d["launches"]:
            return None
        w = d["work"] / steps
        out = {"launches_per_step": d["launches"] // steps,
               "event_ms_per_step": d["ms"] / steps,
               "event_achieved_gbs": w / (d["ms"] / steps / 1e3) / 1e9,
               "event_frac_of_hbm": w / (d["ms"] / steps / 1e3) / 1e9 / hbm}
        for tag, src in (("cupti", eager), ("replay", replay)):
            rp = (src or {}).get(kind)
            if isinstance(rp, dict) and rp.get("ms"):
                out.update({f"{tag}_ms_per_step": rp["ms"], f"{tag}_launches_per_step": rp["launches"],
                            f"{tag}_achieved_gbs": w / (rp["ms"] / 1e3) / 1e9,
                            f"{tag}_frac_of_hbm": w / (rp["ms"] / 1e3) / 1e9 / hbm})
        # headline: the kernels' own hardware spans in the instrumented eager pass (CUPTI);
        # the event brackets add the launch latency and event processing (~2 us per launch)
        src = "cupti" if "cupti_ms_per_step" in out else "event"
        out.update({"ms_per_step": out[f"{src}_ms_per_step"], "achieved_gbs": out[f"{src}_achieved_gbs"],
                    "frac_of_hbm": out[f"{src}_frac_of_hbm"], "source": src})
        return out
    return rate


def _our_launches(r: dict) -> int:
    """Launches of our kernels per step: every moss:: kernel CUPTI saw in the eager pass
    (the Python spans miss the one-thread resets a launcher issues ahead of its kernel)."""
    ek = r.get("eager_kern")
    if isinstance(ek, dict) and "error" not in ek:
        n = sum(v["launches"] for k, v in ek.items()
                if isinstance(v, dict) and "launches" in v and k not in ("foreign", "memset/memcpy"))
        if n:
            return int(round(n))
    return r["launches"]


def replay_gaps(r: dict) -> dict | None:
    """Step time not covered by any kernel in the graph replays (launch gaps,
    dependencies waiting on the front end): step ms - sum of CUPTI kernel times."""
    rk = r.get("replay_kern")
    if not isinstance(rk, dict) or "error" in rk:
        return None
    busy = sum(d["ms"] for d in rk.values() if isinstance(d, dict) and "ms" in d)
    return {"kernel_ms_per_step": busy, "uncovered_ms_per_step": r["ms"] - busy,
            "launches_per_step": sum(d["launches"] for d in rk.values() if isinstance(d, dict) and "launches" in d)}


def llama_summary(r: dict, world: int, args, batch: int | None = None) -> dict:
    g = r["kern"].get("gemm", {"launches": 0, "ms": 1e-9, "work": 0})
    return {"tokens_per_s": world * r["T"] / (r["ms"] / 1e3), "ms_per_step": r["ms"], "steps": r["steps"],
            "n_gpus": world, "tokens_per_gpu_per_step": r["T"],
            "config": (f"configs[3]/[4]: Llama-2-7B-shape decoder training step (d 4096, ffn 11008, 32 heads, vocab "
                       f"32000, {args.layers} layers, seq {args.seq}, batch {batch or args.llama_batch}/GPU), MOSS FP8 linears, bf16 SDPA/norm/"
                       f"head, MossAdamW over all params; dp{world}" +
                       (" ZeRO-1" if args.zero1 else (" bucketed NCCL all-reduce" if world > 1 else ""))),
            "timing_mode": r["mode"],
            "gemm_tflops_in_step": g["work"] / (g["ms"] / 1e3) / 1e12 if g["launches"] else None,
            "gemm_share_of_step": (g["ms"] / r["steps"]) / r["ms"] if g["launches"] else None,
            "replay_kernel_ms_per_step": r.get("replay_kern"), "replay_gaps": replay_gaps(r),
            "captured_quant_amax_modes": r.get("quant_modes"),
            "collectives": r["comm"], "clocks": r["clocks"], "peak_allocated_gb": r["peak_gb"]}


def main() -> None:
    args = parse()
    rc = maybe_spawn(args)
    if rc is not None:
        sys.exit(rc)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"error": f"world size {world} != --gpus {args.gpus}"}), flush=True)
        sys.exit(2)
    if args.launch_probe:
        launch_probe(args, world, rank, local)
        return
    if args.impl == "reference":
        # all host threads (torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 is the only worker)
        for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[k] = str(os.cpu_count())
        try:
            from threadpoolctl import threadpool_limits
            global _BLAS_LIMITS
            _BLAS_LIMITS = threadpool_limits(os.cpu_count())
        except Exception:  # noqa: BLE001
            pass
        run_reference(args, world, rank)       # CPU only: no process group, no GPU
        return
    import torch
    import torch.distributed as dist

    # MOSS_BENCH_SHARED_GPU=1 (tests only): every rank on cuda:0 over gloo, so the N > 1
    # code path of this script runs on a one-GPU box (NCCL refuses two ranks on one GPU)
    shared = os.environ.get("MOSS_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
        args.no_graph = True          # gloo collectives cannot be captured in a CUDA graph
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo", init_method="env://")
        else:
            dist.init_process_group("nccl", device_id=dev)
    elif args.zero1:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0, world_size=1)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    llama_only = args.workload == "llama7b"
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)

    main_kind = "llama7b" if llama_only else "layer"
    r = measure(main_kind, args, dev, rank, world, args.steps, want_e2e=not args.no_e2e)
    _free_cuda()
    barrier()
    llama = None
    if not llama_only and not args.no_llama:
        try:
            rl = measure("llama7b", args, dev, rank, world, args.llama_steps, want_e2e=False)
            llama = llama_summary(rl, world, args)
        except Exception as ex:  # noqa: BLE001 - a sub-measurement must not sink the bench line
            llama = {"error": str(ex)[:300]}
        _free_cuda()
        barrier()
    llama2 = None
    if not llama_only and not args.no_llama and not args.no_llama_batch2 and args.llama_batch == 1:
        # the same step at 2 sequences per GPU: K3's fixed 29 B/param over twice the tokens
        try:
            rl = measure("llama7b", args, dev, rank, world, args.llama_steps, want_e2e=False, batch=2)
            llama2 = llama_summary(rl, world, args, batch=2)
        except Exception as ex:  # noqa: BLE001
            llama2 = {"error": str(ex)[:300]}
        _free_cuda()
        barrier()

    # communicator evidence: which GPUs the ranks drove
    comm_info = None
    if world > 1 or args.zero1:
        me = {"rank": rank, "uuid": str(getattr(torch.cuda.get_device_properties(dev), "uuid", "")),
              "pci_bus_id": getattr(torch.cuda.get_device_properties(dev), "pci_bus_id", None)}
        every = [None] * dist.get_world_size()
        dist.all_gather_object(every, me)
        comm_info = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                     "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                     "shared_gpu_test_mode": shared,
                     "ranks": every, "distinct_devices": len({e["uuid"] for e in every})}

    if rank != 0:
        barrier()
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    roof = None
    if not args.no_fp8_roof:
        try:
            roof = fp8_roof(dev, local)
        except Exception as ex:  # noqa: BLE001
            roof = {"error": str(ex)[:200]}
    have_roof = roof is not None and "burst_tflops" in roof
    # the BURST cuBLASLt MXFP8 figure: the in-step GEMM runs at the SM clock of a mixed
    # memory/tensor step (see clocks), far above the ~1 GHz a seconds-long dense GEMM loop
    # settles at under the 1 kW cap, so the sustained figure is no same-clock denominator
    # (reported beside it as frac_of_sustained)
    fp8_peak = roof["burst_tflops"] if have_roof else 2.0 * peaks.get("bf16_tflops", 1590.0)
    peak_src = ("cuBLASLt MXFP8 8192^3 burst (best single launch at max clock), measured in this run"
                if have_roof else "2 x bf16_tflops (burst) of MEASURED_PEAKS.json (no fp8 roof measured)")
    kern, ms, steps = r["kern"], r["ms"], r["steps"]
    g = kern.get("gemm", {"launches": 0, "ms": 1e-9, "work": 0})
    gemm_tflops = g["work"] / (g["ms"] / 1e3) / 1e12 if g["launches"] else 0.0
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")))
        traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass
    rate = _rates(kern, steps, hbm, r.get("replay_kern"), r.get("eager_kern"))
    rg = (r.get("replay_kern") or {}).get("gemm")
    gemm_replay_tflops = (g["work"] / steps) / (rg["ms"] / 1e3) / 1e12 if isinstance(rg, dict) and rg.get("ms") \
        else None
    total_kernel_ms = sum(d["ms"] for d in kern.values()) / steps
    T, flops_step = r["T"], r["flops_step"]
    e2e = None
    if r["e2e"] is not None:
        me2e = r["e2e"]["ms_per_step"]
        e2e = {**r["e2e"], "value": (world * T / (me2e / 1e3)) if llama_only
               else world * flops_step / (me2e / 1e3) / 1e12,
               "unit": "tokens/s" if llama_only else "TFLOP/s"}
    if llama_only:
        wl = llama_summary(r, world, args)["config"]
        config = {"workload": wl, "tokens_per_gpu": T, "global_batch_tokens": T * world,
                  "parallelism": f"dp{world}", "l2": "not flushed: per-step working set >> 126 MB L2"}
    else:
        config = layer_config(args, world)
    line = {
        "metric": METRIC,
        "value": (world * T / (ms / 1e3)) if llama_only else world * flops_step / (ms / 1e3) / 1e12,
        "unit": "tokens/s" if llama_only else "TFLOP/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "e4m3 x e4m3 -> fp32 accumulate (MXFP8, E8M0 block scales); bf16 activations; fp32 master/optimizer",
        "data": "synthetic (randn bf16 activations, N(0,0.02^2) weights, random init)",
        "config": config,
        "timing_mode": r["mode"],
        "tokens_per_s": world * T / (ms / 1e3),
        "gemm_tflops_per_s_whole_step": world * flops_step / (ms / 1e3) / 1e12,
        "gpu_launches": _our_launches(r),
        "gpu_launches_how": "moss:: kernels per step in the CUPTI profile of the instrumented eager pass "
                            "(incl. the one-thread amax/flag resets); spans of the Python API: %d" % r["launches"],
        "foreign_launches_per_step": r["foreign"],
        "clocks": r["clocks"],
        "roofline": {"bound": "tensor", "kernel": "moss::gemm_mxf8_2cta_kernel (tcgen05.mma.cta_group::2 kind::mxf8f6f4.block_scale)",
                     "achieved": gemm_tflops, "peak": fp8_peak, "unit": "TFLOP/s", "frac": gemm_tflops / fp8_peak,
                     "peak_source": peak_src,
                     "frac_of_sustained": gemm_tflops / roof["sustained_tflops"] if have_roof else None,
                     "frac_of_nominal_4500": gemm_tflops / 4500.0, "traffic": traffic,
                     "achieved_replay_cupti": gemm_replay_tflops,
                     "frac_replay_cupti": gemm_replay_tflops / fp8_peak if gemm_replay_tflops else None,
                     "share_of_step": (g["ms"] / steps) / ms if g["launches"] else None,
                     "fp8_roof": roof},
        "kernels": {"quantize": rate("quant"), "amax": rate("amax"), "adamw_fp8": rate("adamw"),
                    "producers": rate("producer"),
                    "gemm_ms_per_step": g["ms"] / steps, "all_kernels_ms_per_step": total_kernel_ms,
                    "host_issue_ms_per_step": r["host_ms"],
                    "timing_source": "quantize/adamw_fp8/producers: ms_per_step, achieved_gbs, frac_of_hbm = "
                                     "CUPTI kernel start/end timestamps (cupti_*) of an instrumented eager pass "
                                     "of the same step (device sleep ahead of each step); event_*: the same pass "
                                     "with every launch bracketed by CUDA events (adds launch latency); "
                                     "replay_*: CUPTI kernel start/end timestamps of 10 replays of the timed "
                                     "mode after the timed region (torch.profiler); "
                                     "value/ms_per_step from " + r["mode"],
                    "replay_kernel_ms_per_step": r.get("replay_kern"), "replay_gaps": replay_gaps(r),
                    "captured_quant_amax_modes": r.get("quant_modes")},
        "e2e": e2e,
        "memory": {"peak_allocated_gb": r["peak_gb"],
                   "note": "torch.cuda.max_memory_allocated over warm-up, instrumented pass and timed steps"},
    }
    if r["comm"] is not None or comm_info is not None:
        line["collectives"] = {**(r["comm"] or {}), "communicator": comm_info,
                               "note": "bucketed FP32 gradient all-reduce on the comm stream, events per "
                                       "bucket over the instrumented steps (overlaps backward)"}
    if llama is not None:
        line["llama7b"] = llama
    if llama2 is not None:
        line["llama7b_batch2"] = llama2
    if not llama_only:
        try:
            cmp = gemm_vs_cublas(dev, T)
        except Exception as ex:  # noqa: BLE001 - a library comparison must not sink the bench line
            cmp = {"error": str(ex)[:200]}
        if cmp:
            line["roofline"]["library_reference"] = cmp
        try:
            line["kernels"]["quantize_standalone"] = quantizer_rates(dev, T, hbm)
        except Exception as ex:  # noqa: BLE001
            line["kernels"]["quantize_standalone"] = {"error": str(ex)[:200]}
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_sample(REF_SAMPLE["tokens"], REF_SAMPLE["d"])
        line["cpu_baseline"].pop("seconds", None)
    print(json.dumps(line), flush=True)
    barrier()
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
