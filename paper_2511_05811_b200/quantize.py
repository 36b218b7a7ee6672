"""MOSS quantizers on the GPU — the drop-in for mossq.quantize
(reference quantize.py:31-39 names; semantics quantize.py:92-203).

``quant_two_level`` returns the reference's dataclass fields (codes,
global_scale, micro_codes, fmt, k2, k1) as CUDA tensors, plus the operands
the GEMM consumes directly: ``sf`` (micro codes already in the tcgen05
block-scale layout) and, on request, the column-wise codes of x^T
(``codes_t``/``sf_t``/``micro_t``, what quant_two_level(x.T) returns, with the
same global scale) for the wgrad GEMM.

Differences from the reference, by design:
  * ``global_scale``/``scale`` are 0-d float32 device tensors (float(q.global_scale)
    and comparisons work as before; no host sync per call).
  * rounding=NEAREST_LOG2, k1 spans and k2 != 32 are not on the MOSS training
    path and raise InvalidArgumentError.
  * NaN/Inf input and E8M0 range errors are detected on the device; with
    check=True (default) the call syncs once and raises the reference's
    exception; with check=False the flag word is left for a later check.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .errors import InvalidArgumentError, InvalidShapeError
from .fp8 import E4M3, E8m0Rounding, Fp8Format, e8m0_decode, fp8_decode

__all__ = ["PerTensorQuant", "TwoLevelQuant", "PerGroupQuant", "quant_per_tensor", "quant_two_level",
           "quant_per_group", "dequantize", "MX2Operand", "quantize_mx2", "sf_buffer"]


@dataclass(frozen=True)
class PerTensorQuant:
    codes: torch.Tensor     # uint8, source shape
    scale: torch.Tensor     # 0-d float32 (device)
    fmt: Fp8Format
    codes_t: torch.Tensor | None = None   # transposed codes of a 2-D tensor

    @property
    def shape(self):
        return tuple(self.codes.shape)


@dataclass(frozen=True)
class TwoLevelQuant:
    codes: torch.Tensor         # uint8, source shape
    global_scale: torch.Tensor  # 0-d float32 (device)
    micro_codes: torch.Tensor   # uint8 E8M0, outer shape + (n_blocks,)
    fmt: Fp8Format
    k2: int = 32
    k1: int | None = None
    sf: torch.Tensor | None = None        # micro codes in the tcgen05 block-scale layout
    codes_t: torch.Tensor | None = None   # quant_two_level(x.T).codes  (2-D inputs only)
    sf_t: torch.Tensor | None = None
    micro_t: torch.Tensor | None = None

    @property
    def shape(self):
        return tuple(self.codes.shape)

    def micro_scales(self) -> torch.Tensor:
        return e8m0_decode(self.micro_codes)


@dataclass(frozen=True)
class PerGroupQuant:
    """quant_per_group result (quantize.py:54-62): the COAT-style comparator, not the MOSS path."""
    codes: torch.Tensor     # uint8, source shape
    scales: torch.Tensor    # float32, outer shape + (n_groups,)
    group_size: int
    fmt: Fp8Format

    @property
    def shape(self):
        return tuple(self.codes.shape)


def quant_per_group(x, fmt: Fp8Format = E4M3, group_size: int = 128) -> PerGroupQuant:
    """One f32 scale per contiguous group of ``group_size`` along the last axis
    (quantize.py:100-124) on the GPU (csrc/pergroup.cu).  The ablation
    comparator of the paper's per-group (COAT) contrast; group_size 128, the
    last dim a multiple of 128 (the reference's ragged final group is not on
    the comparator's shapes)."""
    if group_size < 1:
        raise InvalidArgumentError(f"group_size must be >= 1, got {group_size}")
    if fmt != E4M3 or group_size != 128:
        raise InvalidArgumentError("the GPU per-group comparator covers E4M3, group_size=128")
    xf = _to_device_2d(x)
    rows, cols = xf.shape
    if cols % 128:
        raise InvalidShapeError(f"last dim {cols} not a multiple of the group size 128")
    codes = torch.empty((rows, cols), dtype=torch.uint8, device=xf.device)
    scales = torch.empty((rows, cols // 128), dtype=torch.float32, device=xf.device)
    fl = _lib.FlagWord(xf.device)
    _lib.quant_per_group(xf, codes, scales, fl)
    fl.raise_if_set("quant_per_group")
    shp = tuple(x.shape) if hasattr(x, "shape") else xf.shape
    return PerGroupQuant(codes=codes.view(shp), scales=scales.view(tuple(shp[:-1]) + (cols // 128,)),
                         group_size=group_size, fmt=fmt)


def sf_buffer(rows: int, cols: int, device) -> torch.Tensor:
    """Block-scale buffer; padding bytes (rows % 128, blocks % 4) hold unit scales."""
    nbytes = _lib.sf_bytes(rows, cols)
    if rows % 128 == 0 and (cols // 32) % 4 == 0:
        return torch.empty(nbytes, dtype=torch.uint8, device=device)
    return torch.full((nbytes,), 127, dtype=torch.uint8, device=device)


@dataclass
class MX2Operand:
    """Hot-path result of the two-level quantizer on a 2-D tensor."""

    codes: torch.Tensor | None
    sf: torch.Tensor | None
    g: torch.Tensor               # [1] float32 global scale
    codes_t: torch.Tensor | None = None
    sf_t: torch.Tensor | None = None
    micro: torch.Tensor | None = None
    micro_t: torch.Tensor | None = None


FUSED = True   # K0 folded into K1 (one launch); False: the two-launch K0 + K1 path (A/B tests)


def quantize_mx2(x2d: torch.Tensor, *, row: bool = True, col: bool = False, micro: bool = False,
                 flags: _lib.FlagWord | None = None, amax_buf: torch.Tensor | None = None,
                 amax: torch.Tensor | None = None) -> MX2Operand:
    """Two-level quantization (global amax + K1) of a contiguous 2-D bf16/f32 tensor.

    One launch (moss_quant_mx2_fused) and no host synchronisation; ``amax``
    (a device f32 [1] max|x| computed by the producer kernel) skips the
    in-kernel reduction.  ``amax_buf`` receives the computed amax.
    Data-dependent errors go to ``flags``.
    """
    rows, cols = x2d.shape
    dev = x2d.device
    flags = flags or _lib.FlagWord(dev)
    given = amax is not None
    amax_t = amax if given else (amax_buf if amax_buf is not None else torch.empty(1, dtype=torch.float32, device=dev))
    g = torch.empty(1, dtype=torch.float32, device=dev)
    op = MX2Operand(codes=None, sf=None, g=g)
    if row:
        op.codes = torch.empty((rows, cols), dtype=torch.uint8, device=dev)
        op.sf = sf_buffer(rows, cols, dev)
        if micro:
            op.micro = torch.empty((rows, cols // 32), dtype=torch.uint8, device=dev)
    if col:
        op.codes_t = torch.empty((cols, rows), dtype=torch.uint8, device=dev)
        op.sf_t = sf_buffer(cols, rows, dev)
        if micro:
            op.micro_t = torch.empty((cols, rows // 32), dtype=torch.uint8, device=dev)
    outs = dict(codes=op.codes, sf=op.sf, micro=op.micro, codes_t=op.codes_t, sf_t=op.sf_t, micro_t=op.micro_t,
                g_out=g)
    if FUSED:
        _lib.quant_mx2_fused(x2d, amax_t, flags, amax_given=given, **outs)
    else:
        if not given:
            _lib.amax(x2d, amax_t, flags)
        _lib.quant_mx2(x2d, amax_t, flags, **outs)
    return op


def _to_device_2d(x) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x, dtype=torch.float32)
    if not x.is_cuda:
        x = x.to("cuda")
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.float()
    if x.dim() == 0:
        raise InvalidShapeError("quantization needs at least one dimension")
    x = x.contiguous()
    if x.data_ptr() % 16:
        x = x.clone()
    return x


def quant_two_level(x, fmt: Fp8Format = E4M3, rounding: E8m0Rounding = E8m0Rounding.CEIL_POW2,
                    k2: int = 32, k1: int | None = None, *, transpose: bool = False,
                    check: bool = True) -> TwoLevelQuant:
    """Two-level quantization (quantize.py:127-173) on the GPU.

    ``transpose=True`` also emits the column-wise quantization of a 2-D x
    (== quant_two_level(x.T) with x's global scale) in one pass.
    """
    if fmt.name != "e4m3":
        raise InvalidArgumentError("the MOSS device quantizer implements E4M3")
    if rounding != E8m0Rounding.CEIL_POW2:
        raise InvalidArgumentError("only CEIL_POW2 micro scales are on the MOSS path")
    if k2 != 32:
        raise InvalidArgumentError("k2 must be 32 (the tcgen05 MX block)")
    xf = _to_device_2d(x)
    last = xf.shape[-1]
    if last % k2 != 0:
        raise InvalidShapeError(f"last dim {last} not divisible by k2={k2}")
    if k1 is not None:
        if k1 % k2 != 0 or last % k1 != 0:
            raise InvalidShapeError(f"k1={k1} must be a multiple of k2 dividing {last}")
        raise InvalidArgumentError("k1 level-1 spans are not supported on the device path")
    if transpose and xf.dim() != 2:
        raise InvalidShapeError("transpose=True needs a 2-D tensor")
    x2d = xf.reshape(-1, last)
    if transpose and x2d.shape[0] % 32:
        raise InvalidShapeError("column-wise quantization needs rows % 32 == 0")
    flags = _lib.FlagWord(xf.device)
    op = quantize_mx2(x2d, row=True, col=transpose, micro=True, flags=flags)
    if check:
        flags.raise_if_set("quant_two_level")
    return TwoLevelQuant(codes=op.codes.view(xf.shape), global_scale=op.g.view(()),
                         micro_codes=op.micro.view(xf.shape[:-1] + (last // k2,)), fmt=fmt, k2=k2, k1=k1,
                         sf=op.sf, codes_t=op.codes_t, sf_t=op.sf_t, micro_t=op.micro_t)


def quant_per_tensor(x, fmt: Fp8Format = E4M3, *, transpose: bool = False,
                     check: bool = True) -> PerTensorQuant:
    """scale = f32(max|x|/448) (1.0 for all-zero x); codes = E4M3(x/scale) (quantize.py:92-98)."""
    if fmt.name != "e4m3":
        raise InvalidArgumentError("the device encoder implements E4M3")
    xf = _to_device_2d(x)
    flat = xf.reshape(-1)
    n = flat.numel()
    flags = _lib.FlagWord(xf.device)
    amax_t = torch.empty(1, dtype=torch.float32, device=xf.device)
    scale = torch.empty(1, dtype=torch.float32, device=xf.device)
    codes_t = None
    if transpose:
        if xf.dim() != 2 or xf.shape[0] % 32 or xf.shape[1] % 8:
            raise InvalidShapeError("transpose=True needs a 2-D tensor with rows % 32 == 0, cols % 8 == 0")
        _lib.amax(xf, amax_t, flags)
        codes = torch.empty(xf.shape, dtype=torch.uint8, device=xf.device)
        codes_t = torch.empty((xf.shape[1], xf.shape[0]), dtype=torch.uint8, device=xf.device)
        _lib.encode_scaled(xf, flags, scale_t=amax_t, from_amax=True, codes=codes, codes_t=codes_t,
                           scale_out=scale)
    else:
        pad = (-n) % 8
        src = torch.cat([flat, flat.new_zeros(pad)]) if pad else flat
        _lib.amax(src, amax_t, flags)
        codes = torch.empty(src.numel(), dtype=torch.uint8, device=xf.device)
        _lib.encode_scaled(src.view(1, -1), flags, scale_t=amax_t, from_amax=True, codes=codes, scale_out=scale)
        codes = codes[:n].view(xf.shape)
    if check:
        flags.raise_if_set("quant_per_tensor")
    return PerTensorQuant(codes=codes, scale=scale.view(()), fmt=fmt, codes_t=codes_t)


def dequantize(q) -> torch.Tensor:
    """code * scale(s) in float32 (quantize.py:186-203)."""
    if isinstance(q, PerTensorQuant):
        return fp8_decode(q.codes, q.fmt) * q.scale.float()
    if isinstance(q, TwoLevelQuant):
        eff = (q.global_scale.float() * e8m0_decode(q.micro_codes)).float()
        vals = fp8_decode(q.codes, q.fmt)
        shp = vals.shape
        vals = vals.reshape(shp[:-1] + (shp[-1] // q.k2, q.k2))
        return (vals * eff[..., None]).reshape(shp)
    raise InvalidArgumentError(f"not a quantized tensor: {type(q).__name__}")
