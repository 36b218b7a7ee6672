"""CPU-container timing of the LITERAL reference (mossq from /root/reference)
against the oracle port (oracle/numpy_ref) on bench.py's REF_SAMPLE — the
one-linear fwd+dgrad+wgrad+AdamW step the reference arm and cpu_baseline time
(tokens=1024, 4096x4096).  Shows the port's speed is representative of the
reference's own CPU path.  Run here (the GPU box has no /root/reference):

    python tools/ref_vs_port_timing.py > profiles/r02_ref_vs_port.txt
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from mossq import fp8 as MF  # noqa: E402
from mossq.gemm import GemmOperands, gemm_mx_epilogue  # noqa: E402
from mossq.optim import adamw_step, init_state  # noqa: E402
from mossq.quantize import PerTensorQuant, quant_two_level  # noqa: E402

import bench  # noqa: E402
from oracle import numpy_ref as R  # noqa: E402

T, D = bench.REF_SAMPLE["tokens"], bench.REF_SAMPLE["d"]
rng = np.random.default_rng(0)
x = rng.standard_normal((T, D)).astype(np.float32)
w = rng.standard_normal((D, D)) * 0.02
dy = (rng.standard_normal((T, D)) * 1e-3).astype(np.float32)
s = float(np.abs(w).max() / 448.0)


def timed(fn, *a):
    t = time.perf_counter()
    r = fn(*a)
    return r, time.perf_counter() - t


rows = []
# weight encode at the schedule scale (train.py:113-118)
ref_wc, t_ref = timed(lambda: MF.fp8_encode(np.float32(w) / np.float32(s), MF.E4M3))
(port_wc, _), t_port = timed(R.encode_weight, w, s)
assert np.array_equal(ref_wc, port_wc)
rows.append(("weight encode", t_ref, t_port))
# quant_two_level of x, dy, dy^T, x^T (quantize.py:127-173)
tr = tp = 0.0
for a in (x, dy, np.ascontiguousarray(dy.T), np.ascontiguousarray(x.T)):
    q_ref, t1 = timed(quant_two_level, a, MF.E4M3)
    q_port, t2 = timed(R.quant_two_level, a)
    assert np.array_equal(q_ref.codes, q_port.codes)
    tr += t1
    tp += t2
rows.append(("quant_two_level x4", tr, tp))
# the three GEMMs through gemm_mx_epilogue's dataflow (gemm.py:115-129)
qw = PerTensorQuant(codes=ref_wc, scale=s, fmt=MF.E4M3)
tr = tp = 0.0
for a in (x, dy, np.ascontiguousarray(x.T)):     # fwd, dgrad (same shapes), wgrad-shaped (K = tokens)
    if a.shape[1] != D:
        continue
    qx = quant_two_level(a, MF.E4M3)
    _, t1 = timed(gemm_mx_epilogue, GemmOperands(qw=qw, qx=qx))
    _, t2 = timed(R.gemm_mx_epilogue, port_wc, s, R.quant_two_level(a))
    tr += t1
    tp += t2
# wgrad: [D, T] x [D, T]^T, contraction over the T tokens
qa_t = quant_two_level(np.ascontiguousarray(dy.T), MF.E4M3)
qb_t = quant_two_level(np.ascontiguousarray(x.T), MF.E4M3)
wq = PerTensorQuant(codes=qa_t.codes, scale=float(qa_t.global_scale), fmt=MF.E4M3)
_, t1 = timed(gemm_mx_epilogue, GemmOperands(qw=wq, qx=qb_t))
tr += t1
ops = {}
t0 = time.perf_counter()
bench.cpu_linear_step(T, D, D, ops=ops)
tp = sum(v for k, v in ops.items() if k == "gemm_mx_epilogue")
rows.append(("gemm_mx_epilogue fwd+dgrad+wgrad", tr, tp))
# AdamW (optim.py:78-106)
g = rng.standard_normal(w.shape) * 1e-3
st = init_state(w.shape, eta=3e-4, weight_decay=0.1)
_, t1 = timed(adamw_step, w, g, st)
_, t2 = timed(R.adamw_step, w, g, R.adam_init(w.shape, eta=3e-4, weight_decay=0.1))
rows.append(("adamw_step", t1, t2))
print(f"# REF_SAMPLE tokens={T}, {D}x{D}; {os.cpu_count()} host cores; numpy {np.__version__}")
print(f"# {'op':36s} {'mossq (s)':>10s} {'port (s)':>10s} {'port/ref':>9s}")
tot_r = tot_p = 0.0
for name, a, b in rows:
    tot_r += a
    tot_p += b
    print(f"  {name:36s} {a:10.3f} {b:10.3f} {b / a:9.3f}")
print(f"  {'step total':36s} {tot_r:10.3f} {tot_p:10.3f} {tot_p / tot_r:9.3f}")
