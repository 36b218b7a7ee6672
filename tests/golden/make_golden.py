"""Generate golden vectors from the REFERENCE itself (mossq 0.1.0).

Run here, where /root/reference exists:
    python tests/golden/make_golden.py
It imports ``mossq`` from /root/reference/pkg/src (read-only, never copied)
and writes tests/golden/golden.npz.  The fixtures travel with the repo; the
GPU box never reads /root/reference.

Contents (all produced by reference calls, cited):
  codec_*     fp8_encode / fp8_decode / e8m0_encode on anchor, tie, saturation,
              subnormal and random vectors            (fp8.py:121-223)
  q2l_<case>_* quant_two_level on hand-built and seeded tensors, including
              FP8-midpoint vectors and outlier-injected tensors that force
              micro codes <= 118                    (quantize.py:127-173)
  qpt_<case>_* quant_per_tensor                         (quantize.py:92-98)
  wenc_*      the training-loop weight encode at a schedule scale
                                                      (train.py:113-118)
  gemm_<shape>_* gemm_mx_epilogue outputs + operands      (gemm.py:115-129)
  adam_*      adamw_step trajectories                  (optim.py:78-106)
  sched_*     auto_scale_advance / rescale sequences   (autoscale.py:71-96)
  train_*     toy train() logs (quantized + fp)          (train.py:126-204)
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from mossq.autoscale import (ScaleSchedule, auto_scale_advance, jit_scale,  # noqa: E402
                             rescale_due, rescale_interval, schedule_from_weights)
from mossq.fp8 import (E4M3, E5M2, E8m0Rounding, e8m0_encode, fp8_decode,  # noqa: E402
                       fp8_encode)
from mossq.gemm import gemm_mx_epilogue, quantize_gemm_operands  # noqa: E402
from mossq.optim import adamw_step, init_state  # noqa: E402
from mossq.quantize import quant_per_tensor, quant_two_level  # noqa: E402
from mossq.tensor import tensor_randn  # noqa: E402
from mossq.train import TrainConfig, _quantize_weight, train  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def midpoint_tensors(n_tensors: int, seed: int) -> np.ndarray:
    """1x64 tensors whose second block holds exact E4M3 midpoints times eff.

    Element 0 = 448*g with a short-mantissa g, so g = RN(448g/448) exactly;
    block 1 = g*2^-3 * m * 2^k with m an E4M3 midpoint."""
    rng = np.random.default_rng(seed)
    pos = fp8_decode(np.arange(0x7F, dtype=np.uint8), E4M3).astype(np.float64)
    mids = (pos[1:] + pos[:-1]) / 2.0
    out = np.zeros((n_tensors, 64), dtype=np.float32)
    for i in range(n_tensors):
        g = float(np.float32(rng.integers(1, 1 << 10) / 1024.0 * 2.0 ** rng.integers(-20, 20)))
        out[i, 0] = np.float32(448.0 * g)
        out[i, 1:32] = np.float32(g) * rng.standard_normal(31).astype(np.float32)
        m = rng.choice(mids, 32)
        # block max = 448*g*2^-3 so the micro exponent is exactly -3
        m[0] = 448.0
        out[i, 32:] = (np.float32(g) * np.float32(2.0 ** -3) * m).astype(np.float32)
    return out


def main() -> None:
    G: dict[str, np.ndarray] = {}

    # ---------------- codec ----------------
    codes = np.arange(256, dtype=np.uint8)
    G["codec_decode_e4m3"] = fp8_decode(codes, E4M3)
    G["codec_decode_e5m2"] = fp8_decode(codes, E5M2)
    rng = np.random.default_rng(7)
    vals = np.concatenate([
        np.array([0.0, -0.0, 1.0, -1.0, 448.0, 449.0, 464.0, 479.9, 480.0, 500.0,
                  8 * 448.0, 3e38, -3e38, 25.0, 27.0, 2.0 ** -9, 2.0 ** -10,
                  3 * 2.0 ** -11, 2.0 ** -6, 1e-40, -1e-40, 1.4e-45, 2.0 ** -126],
                 dtype=np.float32),
        rng.uniform(-448, 448, 4000).astype(np.float32),
        rng.normal(0, 1e-3, 2000).astype(np.float32),
        rng.normal(0, 150, 2000).astype(np.float32),
        (rng.standard_normal(2000) * 10.0 ** rng.uniform(-12, 6, 2000)).astype(np.float32),
    ])
    G["codec_encode_in"] = vals
    G["codec_encode_e4m3"] = fp8_encode(vals, E4M3)
    G["codec_encode_e5m2"] = fp8_encode(vals, E5M2)
    r = np.concatenate([2.0 ** np.arange(-127, 128, dtype=np.float64),
                        np.array([0.75, 0.5, 1.0, 1.5, 3.0, 0.3]),
                        10.0 ** rng.uniform(-30, 30, 500)])
    G["codec_e8m0_in"] = r
    G["codec_e8m0_ceil"] = e8m0_encode(r, E8m0Rounding.CEIL_POW2)
    G["codec_e8m0_near"] = e8m0_encode(r, E8m0Rounding.NEAREST_LOG2)

    # ---------------- two-level quantizer ----------------
    cases: dict[str, np.ndarray] = {}
    hw = np.zeros((1, 64), np.float32)
    hw[0, 0] = 448.0
    hw[0, 32] = 0.875
    cases["handworked"] = hw                       # test_quantize.py:105-113
    zb = np.zeros((1, 64), np.float32)
    zb[0, 0] = 8.0
    cases["zeroblock"] = zb                        # test_quantize.py:150-156
    cases["allzero"] = np.zeros((2, 64), np.float32)
    cases["gauss"] = tensor_randn([64, 256], seed=1)
    cases["outlier50"] = tensor_randn([64, 512], seed=2, dist="outlier_injected")
    cases["outlier2000"] = tensor_randn([32, 512], seed=3, dist="outlier_injected",
                                        outlier_magnitude=2000.0)
    cases["laplace"] = tensor_randn([16, 1024], seed=4, dist="laplace")
    cases["midpoints"] = midpoint_tensors(128, seed=5)
    sub = tensor_randn([8, 128], seed=6) * np.float32(1e-39)   # f32 subnormals
    sub[0, :32] *= np.float32(1e3)   # one block of normals next to subnormal blocks
    cases["subnormal"] = sub.astype(np.float32)
    neg0 = np.zeros((2, 64), np.float32)
    neg0[0, :32] = -0.0
    neg0[1, 5] = -2.5
    cases["negzero"] = neg0
    wide = tensor_randn([4, 256], seed=8) * np.float32(1e-30)
    wide[0, 0] = np.float32(1e6)
    cases["widerange"] = wide.astype(np.float32)
    for name, x in cases.items():
        q = quant_two_level(x, E4M3)
        G[f"q2l_{name}_x"] = x
        G[f"q2l_{name}_codes"] = q.codes
        G[f"q2l_{name}_micro"] = q.micro_codes
        G[f"q2l_{name}_g"] = np.float32(q.global_scale)
    G["q2l_cases"] = np.array(sorted(cases))

    # midpoint recipe needs one g per tensor: quantize each 1x64 row alone
    rows = midpoint_tensors(128, seed=55)
    qs = [quant_two_level(rows[i:i + 1], E4M3) for i in range(rows.shape[0])]
    G["q2l_midrows_x"] = rows
    G["q2l_midrows_codes"] = np.concatenate([q.codes for q in qs])
    G["q2l_midrows_micro"] = np.concatenate([q.micro_codes for q in qs])
    G["q2l_midrows_g"] = np.array([q.global_scale for q in qs], np.float32)

    # E8M0 range error: block max < 2.6e-36 with g >= 1
    rerr = np.zeros((1, 64), np.float32)
    rerr[0, 0] = 448.0
    rerr[0, 32] = np.float32(1e-37)
    G["q2l_rangeerr_x"] = rerr
    try:
        quant_two_level(rerr, E4M3)
        G["q2l_rangeerr_raises"] = np.array(False)
    except Exception as e:  # E8m0RangeError
        G["q2l_rangeerr_raises"] = np.array(type(e).__name__ == "E8m0RangeError")

    # ---------------- per tensor + weight copy ----------------
    pt = {"exact": np.array([-448.0, 224.0, 0.0], np.float32),
          "two": np.array([896.0, -448.0], np.float32),
          "gauss": tensor_randn([4096], seed=5),
          "w": tensor_randn([128, 256], seed=9) * np.float32(0.02)}
    for name, x in pt.items():
        q = quant_per_tensor(x, E4M3)
        G[f"qpt_{name}_x"] = x
        G[f"qpt_{name}_codes"] = q.codes
        G[f"qpt_{name}_scale"] = np.float64(q.scale)
    w = tensor_randn([64, 128], seed=10).astype(np.float64) * 0.02
    for i, s in enumerate([jit_scale(w, E4M3), jit_scale(w, E4M3) * 0.5,
                           jit_scale(w, E4M3) + 3e-4 / 448.0 * 17]):
        deq, sat = _quantize_weight(w, s, E4M3)
        G[f"wenc_{i}_w"] = w
        G[f"wenc_{i}_s"] = np.float64(s)
        G[f"wenc_{i}_deq"] = deq
        G[f"wenc_{i}_sat"] = np.int64(sat)

    # ---------------- GEMM ----------------
    for (m, n, k) in [(64, 64, 64), (16, 48, 96), (128, 128, 256), (256, 128, 512)]:
        wmat = tensor_randn([m, k], seed=m + k)
        xmat = tensor_randn([n, k], seed=n + k + 1, dist="outlier_injected")
        ops = quantize_gemm_operands(wmat, xmat)
        out, _ = gemm_mx_epilogue(ops)
        tag = f"gemm_{m}x{n}x{k}"
        G[tag + "_w"] = wmat
        G[tag + "_x"] = xmat
        G[tag + "_wcodes"] = ops.qw.codes
        G[tag + "_wscale"] = np.float64(ops.qw.scale)
        G[tag + "_xcodes"] = ops.qx.codes
        G[tag + "_xmicro"] = ops.qx.micro_codes
        G[tag + "_xg"] = np.float64(ops.qx.global_scale)
        G[tag + "_out"] = out

    # ---------------- AdamW ----------------
    for tag, kw in {"dec": dict(eta=3e-4, weight_decay=0.1, decoupled_decay=True),
                    "cpl": dict(eta=1e-3, weight_decay=0.1, decoupled_decay=False),
                    "nowd": dict(eta=1e-2, weight_decay=0.0)}.items():
        grng = np.random.default_rng(11)
        w0 = grng.standard_normal(2048) * 0.02
        st = init_state(w0.shape, **kw)
        wt = w0.copy()
        ws, ms, vs, gs, ds = [], [], [], [], []
        for step in range(20):
            g = grng.standard_normal(2048) * (10.0 ** grng.uniform(-4, 0))
            g = g.astype(np.float32).astype(np.float64)
            wt, st, d = adamw_step(wt, g, st)
            ws.append(wt.copy()); ms.append(st.m.copy()); vs.append(st.v.copy())
            gs.append(g); ds.append(d)
        G[f"adam_{tag}_w0"] = w0
        G[f"adam_{tag}_g"] = np.stack(gs)
        G[f"adam_{tag}_w"] = np.stack(ws)
        G[f"adam_{tag}_m"] = np.stack(ms)
        G[f"adam_{tag}_v"] = np.stack(vs)
        G[f"adam_{tag}_delta"] = np.stack(ds)
        G[f"adam_{tag}_hp"] = np.array([kw["eta"], kw["weight_decay"],
                                        float(kw.get("decoupled_decay", True))])

    # ---------------- autoscale ----------------
    s = ScaleSchedule(s0=0.01, s_t=0.01, t=0, interval=500, delta_max=448.0)
    for _ in range(1000):
        auto_scale_advance(s, 3e-4)
    G["sched_eq10_s"] = np.float64(s.s_t)
    etas = np.array([1e-3 * 0.5 * (1 + math.cos(math.pi * t / 300)) for t in range(300)])
    s = ScaleSchedule(s0=0.05, s_t=0.05, t=0, interval=120, delta_max=448.0)
    wsched = tensor_randn([64], seed=1)
    traj = []
    for t, e in enumerate(etas):
        auto_scale_advance(s, float(e))
        if rescale_due(s):
            rescale_interval(wsched * (1 + t / 1000.0), s, E4M3)
        traj.append(s.s_t)
    G["sched_cos_eta"] = etas
    G["sched_cos_w"] = wsched
    G["sched_cos_traj"] = np.array(traj)
    G["sched_s0_jit"] = np.float64(schedule_from_weights(wsched, E4M3).s0)

    # ---------------- toy training (train.py) ----------------
    cfg = TrainConfig(steps=300, interval=100, seed=3, quantize=True)
    log = train(cfg)
    G["train_q_fp_loss"] = log.fp_loss
    G["train_q_train_loss"] = log.train_loss
    G["train_q_s_auto"] = log.s_auto
    G["train_q_s_jit"] = log.s_jit
    G["train_q_lr"] = log.lr
    G["train_q_rescale_steps"] = np.array([e[0] for e in log.rescale_events])
    G["train_q_saturation"] = np.int64(log.saturation_events)
    logf = train(TrainConfig(steps=300, seed=3, quantize=False))
    G["train_fp_fp_loss"] = logf.fp_loss

    np.savez_compressed(OUT, **G)
    print(f"wrote {OUT}: {len(G)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
