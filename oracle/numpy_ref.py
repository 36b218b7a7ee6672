"""Numpy restatement of the reference MOSS hot path — TEST INFRASTRUCTURE ONLY.

Every function below restates one reference function (cited file:line, paths
relative to /root/reference/pkg/src/mossq/).  The algorithms are written
independently: e.g. the FP8 encoder rounds in float64 on the format's own grid
and looks the code up in the monotone positive table, instead of the
reference's integer bit manipulation (fp8.py:131-183); both are correctly
rounded, saturating, sign-preserving encoders, and the golden vectors pin that
they agree bit for bit.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# formats (fp8.py:46-72)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Fmt:
    name: str
    ebits: int
    mbits: int
    bias: int
    max_value: float
    has_inf: bool


E4M3 = Fmt("e4m3", 4, 3, 7, 448.0, False)
E5M2 = Fmt("e5m2", 5, 2, 15, 57344.0, True)


def _positive_table(fmt: Fmt) -> np.ndarray:
    """Finite non-negative values in code order (codes 0 .. max_finite_code)."""
    n_codes = (1 << (fmt.ebits + fmt.mbits))
    vals = []
    for code in range(n_codes):
        e = code >> fmt.mbits
        m = code & ((1 << fmt.mbits) - 1)
        if e == 0:
            v = m * 2.0 ** (1 - fmt.bias - fmt.mbits)
        else:
            v = (1.0 + m / (1 << fmt.mbits)) * 2.0 ** (e - fmt.bias)
        if v > fmt.max_value:
            break
        vals.append(v)
    return np.array(vals, dtype=np.float64)


_POS = {E4M3.name: _positive_table(E4M3), E5M2.name: _positive_table(E5M2)}


def decode_table(fmt: Fmt) -> np.ndarray:
    """256-entry decode table (fp8.py:87-118): NaN/Inf patterns included."""
    pos = _POS[fmt.name]
    out = np.full(256, np.nan, dtype=np.float32)
    out[: len(pos)] = pos
    out[0x80: 0x80 + len(pos)] = -pos
    if fmt.has_inf:
        inf_code = (1 << fmt.ebits) - 1 << fmt.mbits
        out[inf_code] = np.inf
        out[0x80 | inf_code] = -np.inf
    return out


def fp8_decode(codes, fmt: Fmt = E4M3) -> np.ndarray:
    """fp8.py:121-128."""
    return decode_table(fmt)[np.asarray(codes, dtype=np.uint8)]


def fp8_encode(x, fmt: Fmt = E4M3) -> np.ndarray:
    """Correctly rounded (RNE), saturating f32 -> FP8 encoder (fp8.py:131-183).

    f32 subnormal inputs encode to signed zero (fp8.py:148-149); NaN/Inf raise
    (fp8.py:138-139).  Rounding is done in float64, where y / quantum is exact
    because the quantum is a power of two.
    """
    xf = np.asarray(x, dtype=np.float32)
    if not np.all(np.isfinite(xf)):
        raise ValueError("fp8_encode requires finite input")
    bits = np.ascontiguousarray(xf).reshape(-1).view(np.uint32).reshape(xf.shape)
    sign = ((bits >> 24) & 0x80).astype(np.uint8)
    y = np.abs(xf.astype(np.float64))
    f32_subnormal = (bits & 0x7F800000) == 0
    # binade exponent floor(log2 y), clamped to the format's min normal exponent
    _, ex = np.frexp(np.where(y > 0, y, 1.0))
    e = np.maximum(ex - 1, 1 - fmt.bias)
    quantum = np.ldexp(1.0, e - fmt.mbits)
    n = np.rint(y / quantum)            # rint = round half to even
    v = np.minimum(n * quantum, fmt.max_value)
    code = np.searchsorted(_POS[fmt.name], v).astype(np.uint8)
    code = np.where(f32_subnormal, np.uint8(0), code)
    return (code | sign).astype(np.uint8)


def e8m0_decode(codes) -> np.ndarray:
    """fp8.py:186-191 (code 255 is reserved)."""
    c = np.asarray(codes, dtype=np.uint8)
    if np.any(c == 255):
        raise ValueError("e8m0 code 255 is reserved")
    return np.ldexp(np.float32(1.0), c.astype(np.int32) - 127)


def e8m0_encode_ceil(r) -> np.ndarray:
    """CEIL_POW2 branch of fp8.py:194-223: smallest 2^e >= r, e in [-127,127]."""
    rf = np.asarray(r, dtype=np.float64)
    if not np.all(np.isfinite(rf)) or np.any(rf <= 0):
        raise ValueError("e8m0_encode requires finite r > 0")
    mant, ex = np.frexp(rf)
    e = ex - (mant == 0.5)
    if np.any(e > 127) or np.any(e < -127):
        raise OverflowError("e8m0 range")
    return (e + 127).astype(np.uint8)


# --------------------------------------------------------------------------
# quantizers (quantize.py:92-98, 127-173, 176-203)
# --------------------------------------------------------------------------


@dataclass
class TwoLevel:
    codes: np.ndarray
    global_scale: float
    micro_codes: np.ndarray
    e8m0_range_error: bool = False


def quant_two_level(x, fmt: Fmt = E4M3, k2: int = 32) -> TwoLevel:
    """quantize.py:127-173 with the default CEIL_POW2 rounding and k1=None.

    s_i  = f32(blockmax / f32(max))             quantize.py:149
    g    = max_i s_i  (0 -> 1.0)                quantize.py:151-155
    e_i  = ceil_log2(f64(s_i) / f64(g))         quantize.py:164-168 (zero block -> 127)
    eff  = f32(f32(g) * 2^e_i)                  quantize.py:170
    code = encode(f32(x / eff))                 quantize.py:171
    An exponent below -127 raises E8m0RangeError in the reference; here the
    condition is reported in ``e8m0_range_error`` so that tests can assert it.
    """
    xf = np.ascontiguousarray(x, dtype=np.float32)
    if xf.ndim == 0:
        raise ValueError("needs at least one dimension")
    if not np.all(np.isfinite(xf)):
        raise ValueError("quantization requires finite input")
    if xf.shape[-1] % k2:
        raise ValueError("last dim not divisible by k2")
    blocks = xf.reshape(xf.shape[:-1] + (xf.shape[-1] // k2, k2))
    s = (np.abs(blocks).max(axis=-1) / np.float32(fmt.max_value)).astype(np.float32)
    g = float(s.max()) if s.size else 0.0
    if g == 0.0:
        g = 1.0
    ratio = s.astype(np.float64) / np.float64(np.float32(g))
    micro = np.full(s.shape, 127, dtype=np.uint8)
    nz = ratio > 0
    range_err = False
    if np.any(nz):
        mant, ex = np.frexp(ratio[nz])
        e = ex - (mant == 0.5)
        range_err = bool(np.any(e < -127) or np.any(e > 127))
        micro[nz] = np.clip(e + 127, 0, 254).astype(np.uint8)
    eff = (np.float32(g) * e8m0_decode(micro)).astype(np.float32)
    y = (blocks / eff[..., None]).astype(np.float32)
    codes = fp8_encode(y, fmt).reshape(xf.shape)
    return TwoLevel(codes=codes, global_scale=g, micro_codes=micro,
                    e8m0_range_error=range_err)


def quant_per_tensor(x, fmt: Fmt = E4M3):
    """quantize.py:92-98 -> (codes, scale)."""
    xf = np.ascontiguousarray(x, dtype=np.float32)
    amax = float(np.abs(xf).max()) if xf.size else 0.0
    scale = np.float32(amax / fmt.max_value) if amax > 0 else np.float32(1.0)
    return fp8_encode((xf / scale).astype(np.float32), fmt), float(scale)


def encode_weight(w, s_t: float, fmt: Fmt = E4M3):
    """Weight copy at the schedule scale, train.py:113-118 -> (codes, n_saturated)."""
    wf = np.asarray(w, dtype=np.float32)
    sat = int(np.sum(np.abs(wf) > np.float32(s_t * fmt.max_value)))
    return fp8_encode((wf / np.float32(s_t)).astype(np.float32), fmt), sat


def dequantize_two_level(q: TwoLevel, k2: int = 32) -> np.ndarray:
    """f64 exact dequantization, gemm.py:178-186."""
    ss = e8m0_decode(q.micro_codes).astype(np.float64)
    vals = fp8_decode(q.codes).astype(np.float64)
    shp = vals.shape
    vals = vals.reshape(shp[:-1] + (shp[-1] // k2, k2))
    return (vals * (q.global_scale * ss)[..., None]).reshape(shp)


def dequantize_per_tensor(codes, scale: float) -> np.ndarray:
    """gemm.py:168-169."""
    return fp8_decode(codes).astype(np.float64) * float(scale)


def gemm_f64(a, b_t) -> np.ndarray:
    """C = A @ B_t.T in float64 — the one-shot form of gemm_oracle (gemm.py:190-209)."""
    return np.asarray(a, np.float64) @ np.asarray(b_t, np.float64).T


def gemm_mx_epilogue(w_codes, w_scale, x: TwoLevel, k2: int = 32) -> np.ndarray:
    """Block-wise dataflow of gemm.py:115-129: per-32 partials x micro scale,
    then one epilogue multiply by s_W * s_x.  Output (M_out, N_tokens)."""
    wv = fp8_decode(w_codes).astype(np.float64)
    xv = fp8_decode(x.codes).astype(np.float64)
    ss = e8m0_decode(x.micro_codes).astype(np.float64)
    k = wv.shape[1]
    acc = np.zeros((wv.shape[0], xv.shape[0]))
    for b in range(k // k2):
        sl = slice(b * k2, (b + 1) * k2)
        acc += (wv[:, sl] @ xv[:, sl].T) * ss[None, :, b]
    return acc * (float(w_scale) * float(x.global_scale))


# --------------------------------------------------------------------------
# optimizer + automatic scaling (optim.py:52-106, autoscale.py:36-96)
# --------------------------------------------------------------------------


@dataclass
class AdamState:
    m: np.ndarray
    v: np.ndarray
    t: int = 0
    beta1: float = 0.9
    beta2: float = 0.95
    eta: float = 1e-3
    weight_decay: float = 0.1
    eps: float = 1e-8
    decoupled_decay: bool = True


def adam_init(shape, **kw) -> AdamState:
    """optim.py:65-75."""
    return AdamState(m=np.zeros(shape), v=np.zeros(shape), **kw)


def adamw_step(w, g, st: AdamState):
    """optim.py:78-106 in float64; returns (w_next, delta) and mutates st."""
    wf = np.asarray(w, np.float64)
    gf = np.asarray(g, np.float64)
    if not np.all(np.isfinite(gf)):
        raise ValueError("gradient contains NaN/Inf")
    if not st.decoupled_decay and st.weight_decay != 0.0:
        gf = gf + st.weight_decay * wf
    st.t += 1
    st.m = st.beta1 * st.m + (1.0 - st.beta1) * gf
    st.v = st.beta2 * st.v + (1.0 - st.beta2) * gf * gf
    delta = st.eta * (st.m / (1.0 - st.beta1 ** st.t)) / (
        np.sqrt(st.v / (1.0 - st.beta2 ** st.t)) + st.eps)
    w_next = wf - delta
    if st.decoupled_decay and st.weight_decay != 0.0:
        w_next = w_next - st.eta * st.weight_decay * wf
    return w_next, delta


@dataclass
class Schedule:
    s_t: float
    t: int = 0
    interval: int = 500
    delta_max: float = 448.0
    last_rescale_step: int = 0
    history: list = field(default_factory=list)


def jit_scale(w, fmt: Fmt = E4M3) -> float:
    """autoscale.py:53-59."""
    amax = float(np.max(np.abs(np.asarray(w))))
    return amax / fmt.max_value if amax > 0.0 else 1.0


def advance(s: Schedule, eta: float) -> None:
    """autoscale.py:71-79: s += eta / delta_max; t += 1 (no weight data)."""
    s.s_t += eta / s.delta_max
    s.t += 1


def rescale_due(s: Schedule) -> bool:
    """autoscale.py:82-83."""
    return s.t - s.last_rescale_step >= s.interval


def rescale(w, s: Schedule, fmt: Fmt = E4M3) -> None:
    """autoscale.py:86-96 (the returned PerTensorQuant is discarded by train.py:201)."""
    s.s_t = jit_scale(w, fmt)
    s.last_rescale_step = s.t


def lr_at(step: int, *, lr_peak: float, warmup: int, steps: int,
          floor_frac: float = 0.1) -> float:
    """train.py:75-82: linear warmup then cosine to floor_frac * peak."""
    if step < warmup:
        return lr_peak * (step + 1) / warmup
    span = max(1, steps - warmup)
    progress = min(1.0, (step - warmup) / span)
    floor = lr_peak * floor_frac
    return floor + 0.5 * (lr_peak - floor) * (1.0 + math.cos(math.pi * progress))
