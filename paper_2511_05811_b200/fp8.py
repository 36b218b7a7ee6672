"""FP8 / E8M0 formats and device codecs — same names as mossq.fp8
(reference fp8.py:32-43).  Tensors live on the GPU; the encoder is the
sm_100a kernel (cvt.rn.satfinite.e4m3x2 after an IEEE division), the decoders
are table lookups.

Only E4M3 has a device encoder (the MOSS hot path); E5M2 is
kept as a format descriptor and for decoding, and its encoder raises
InvalidArgumentError.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import torch

from . import _lib
from .errors import E8m0RangeError, InvalidArgumentError, InvalidValueError

__all__ = ["Fp8Format", "E4M3", "E5M2", "E8m0Rounding", "fp8_encode", "fp8_decode", "decode_table",
           "e8m0_encode", "e8m0_decode", "E8M0_INVALID_CODE", "FORMATS"]


@dataclass(frozen=True)
class Fp8Format:
    """Descriptor of one 8-bit float encoding (fp8.py:46-66)."""

    name: str
    exponent_bits: int
    mantissa_bits: int
    bias: int
    max_value: float
    has_infinity: bool

    @property
    def max_finite_code(self) -> int:
        e = (1 << self.exponent_bits) - (2 if self.has_infinity else 1)
        m = (1 << self.mantissa_bits) - (1 if self.has_infinity else 2)
        return (e << self.mantissa_bits) | m


E4M3 = Fp8Format("e4m3", 4, 3, 7, 448.0, False)
E5M2 = Fp8Format("e5m2", 5, 2, 15, 57344.0, True)
FORMATS = {"e4m3": E4M3, "e5m2": E5M2}
E8M0_INVALID_CODE = 255


class E8m0Rounding(str, enum.Enum):
    CEIL_POW2 = "ceil_pow2"
    NEAREST_LOG2 = "nearest_log2"


def _table_values(fmt: Fp8Format) -> list[float]:
    nan, inf = float("nan"), float("inf")
    out = []
    mmask = (1 << fmt.mantissa_bits) - 1
    emask = (1 << fmt.exponent_bits) - 1
    for code in range(256):
        sign = -1.0 if code & 0x80 else 1.0
        e = (code >> fmt.mantissa_bits) & emask
        m = code & mmask
        if e == emask and (fmt.has_infinity or m == mmask):
            out.append(nan if (not fmt.has_infinity or m) else sign * inf)
            continue
        if e == 0:
            v = m * 2.0 ** (1 - fmt.bias - fmt.mantissa_bits)
        else:
            v = (1.0 + m / (1 << fmt.mantissa_bits)) * 2.0 ** (e - fmt.bias)
        out.append(sign * v)
    return out


_TABLES: dict[tuple[str, str], torch.Tensor] = {}


def decode_table(fmt: Fp8Format, device="cuda") -> torch.Tensor:
    """All 256 decoded values (fp8.py:114-118)."""
    key = (fmt.name, str(device))
    if key not in _TABLES:
        _TABLES[key] = torch.tensor(_table_values(fmt), dtype=torch.float32, device=device)
    return _TABLES[key]


def fp8_decode(codes: torch.Tensor, fmt: Fp8Format = E4M3) -> torch.Tensor:
    """codes (uint8) -> exact float32 values (fp8.py:121-128)."""
    return decode_table(fmt, codes.device)[codes.long()]


def fp8_encode(x: torch.Tensor, fmt: Fp8Format = E4M3) -> torch.Tensor:
    """Round-to-nearest-even, saturating E4M3 encode on the GPU (fp8.py:131-183).

    Raises InvalidValueError on NaN/Inf input (checked on the device, one sync).
    """
    if fmt.name != "e4m3":
        raise InvalidArgumentError("the device encoder implements E4M3 only")
    _lib.require_cuda(x, "x")
    xf = x.float() if x.dtype not in (torch.float32, torch.bfloat16) else x
    flat = xf.reshape(-1).contiguous()
    n = flat.numel()
    pad = (-n) % 8
    if pad:
        flat = torch.cat([flat, flat.new_zeros(pad)])
    codes = torch.empty(flat.numel(), dtype=torch.uint8, device=x.device)
    flags = _lib.FlagWord(x.device)
    _lib.encode_scaled(flat.view(1, -1), flags, scale_host=1.0, codes=codes)
    flags.raise_if_set("fp8_encode")
    return codes[:n].view(x.shape)


def e8m0_decode(codes: torch.Tensor) -> torch.Tensor:
    """2^(code-127) as float32; code 255 is reserved (fp8.py:186-191)."""
    c = codes.to(torch.int32)
    if bool((c == E8M0_INVALID_CODE).any()):
        raise InvalidValueError("e8m0 code 255 is reserved")
    return torch.ldexp(torch.ones_like(c, dtype=torch.float32), c - 127)


def e8m0_encode(r: torch.Tensor, rounding: E8m0Rounding = E8m0Rounding.CEIL_POW2) -> torch.Tensor:
    """Positive values -> E8M0 codes (fp8.py:194-223), computed in float64."""
    rf = r.to(torch.float64)
    if not bool(torch.isfinite(rf).all()) or bool((rf <= 0).any()):
        raise InvalidValueError("e8m0_encode requires finite r > 0")
    mant, ex = torch.frexp(rf)
    is_pow2 = mant == 0.5
    if rounding == E8m0Rounding.CEIL_POW2:
        e = torch.where(is_pow2, ex - 1, ex)
    elif rounding == E8m0Rounding.NEAREST_LOG2:
        lo = ex - 1
        log2r = torch.log2(rf)
        d_lo, d_hi = log2r - lo, (lo + 1) - log2r
        pick_hi = (d_hi < d_lo) | ((d_hi == d_lo) & (lo % 2 != 0))
        e = torch.where(is_pow2, lo, torch.where(pick_hi, lo + 1, lo))
    else:
        raise InvalidValueError(f"unknown e8m0 rounding mode: {rounding!r}")
    if bool((e > 127).any()):
        raise E8m0RangeError("value exceeds 2^127")
    if bool((e < -127).any()):
        raise E8m0RangeError("value below 2^-127")
    return (e + 127).to(torch.uint8)
