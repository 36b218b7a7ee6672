"""MXFP8 GEMM with epilogue dequantisation — drop-in for mossq.gemm
(reference gemm.py:36-46 names; dataflow gemm.py:115-129).

``gemm_mx_epilogue(GemmOperands(qw, qx))`` returns C[i, j] = sum_k W[i,k] X[j,k]
(out_features x tokens, float32 on the GPU) and the same closed-form
counters as the reference.  The arithmetic is one launch of the sm_100a
block-scaled tcgen05 kernel: the activation micro scales are applied by the
tensor core (E8M0 scale operands in TMEM), the two FP32 global scales once
per output in the epilogue.  Accumulation is FP32 (the reference's oracle is
float64; tests state the tolerance).

``mx_gemm`` is the hot-path entry (no host sync, any of fwd/dgrad/wgrad):
both operands K-major E4M3 codes with block-scale buffers; shapes that are
not multiples of 128 are zero-padded here (zero codes contribute nothing).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .errors import InvalidArgumentError, InvalidShapeError
from .fp8 import E4M3, E8m0Rounding, Fp8Format
from .quantize import PerTensorQuant, TwoLevelQuant, quant_per_tensor, quant_two_level

__all__ = ["GemmCounters", "GemmOperands", "quantize_gemm_operands", "gemm_mx_epilogue",
           "mx_epilogue_counters", "mx_gemm"]


@dataclass(frozen=True)
class GemmCounters:
    mainloop_dequant_multiplies: int
    epilogue_dequant_multiplies: int
    block_scale_multiplies: int
    mac_count: int


def mx_epilogue_counters(m: int, n: int, k: int, k2: int = 32) -> GemmCounters:
    """Closed-form cost counts of the epilogue dataflow (gemm.py:57-64)."""
    if k % k2 != 0:
        raise InvalidShapeError(f"K={k} not divisible by block size {k2}")
    return GemmCounters(0, m * n, m * n * (k // k2), m * n * k)


def pergroup_mainloop_counters(m: int, n: int, k: int, group_size: int = 128) -> GemmCounters:
    """Closed-form cost counts of the main-loop dataflow (gemm.py:67-74)."""
    if k % group_size != 0:
        raise InvalidShapeError(f"K={k} not divisible by group size {group_size}")
    return GemmCounters(m * n * (k // group_size), 0, 0, m * n * k)


def gemm_pergroup_mainloop(qa, qb) -> tuple[torch.Tensor, GemmCounters]:
    """C = sum_g (A_g B_g^T) * sa_g sb_g^T with every 128-deep partial product
    rescaled in the K loop (gemm.py:132-157) — the COAT-style comparator on
    tcgen05 (kind::f8f6f4, no block scale) + CUDA-core promotion
    (csrc/pergroup.cu).  Returns (C float32 [M, N] on the GPU, counters)."""
    if qa.codes.dim() != 2 or qb.codes.dim() != 2:
        raise InvalidShapeError("gemm operands must be 2-D")
    if qa.codes.shape[1] != qb.codes.shape[1]:
        raise InvalidShapeError(f"K mismatch: {tuple(qa.codes.shape)} vs {tuple(qb.codes.shape)}")
    if qa.group_size != qb.group_size:
        raise InvalidArgumentError("operands must share one group size")
    m, k = qa.codes.shape
    n = qb.codes.shape[0]
    group = qa.group_size
    if k % group != 0:
        raise InvalidShapeError(f"K={k} not divisible by group size {group}")
    if m % 128 or n % 128:
        raise InvalidShapeError("the per-group comparator covers M, N multiples of 128")
    d = torch.empty((m, n), dtype=torch.float32, device=qa.codes.device)
    _lib.gemm_pergroup(qa.codes, qa.scales.t().contiguous(), qb.codes, qb.scales.t().contiguous(), d)
    return d, pergroup_mainloop_counters(m, n, k, group)


@dataclass(frozen=True)
class GemmOperands:
    """Quantized W (M, K) per-tensor and X (N, K) two-level (gemm.py:77-105)."""

    qw: PerTensorQuant
    qx: TwoLevelQuant

    def __post_init__(self):
        if self.qw.codes.dim() != 2 or self.qx.codes.dim() != 2:
            raise InvalidShapeError("gemm operands must be 2-D")
        if self.qw.codes.shape[1] != self.qx.codes.shape[1]:
            raise InvalidShapeError(
                f"K mismatch: weights {tuple(self.qw.codes.shape)} vs activations {tuple(self.qx.codes.shape)}")
        if self.qx.codes.shape[1] % self.qx.k2 != 0:
            raise InvalidShapeError("K must be divisible by the micro block size")
        if self.qx.k1 is not None:
            raise InvalidArgumentError("gemm requires a single global activation scale")

    @property
    def m(self) -> int:
        return self.qw.codes.shape[0]

    @property
    def n(self) -> int:
        return self.qx.codes.shape[0]

    @property
    def k(self) -> int:
        return self.qw.codes.shape[1]


def quantize_gemm_operands(w, x, fmt: Fp8Format = E4M3,
                           rounding: E8m0Rounding = E8m0Rounding.CEIL_POW2) -> GemmOperands:
    """gemm.py:108-112."""
    return GemmOperands(qw=quant_per_tensor(w, fmt), qx=quant_two_level(x, fmt, rounding=rounding))


def _round_up(v: int, m: int) -> int:
    return (v + m - 1) // m * m


def _pad_codes(codes: torch.Tensor, rows: int, cols: int) -> torch.Tensor:
    r, c = codes.shape
    if r == rows and c == cols and codes.is_contiguous() and codes.data_ptr() % 16 == 0:
        return codes
    out = torch.zeros((rows, cols), dtype=torch.uint8, device=codes.device)
    out[:r, :c] = codes
    return out


def mx_gemm(a_codes: torch.Tensor, a_sf: torch.Tensor | None, s_a: torch.Tensor, b_codes: torch.Tensor,
            b_sf: torch.Tensor | None, s_b: torch.Tensor, *, out: torch.Tensor | None = None,
            out_dtype: torch.dtype = torch.bfloat16, accumulate: bool = False,
            amax_out: torch.Tensor | None = None) -> torch.Tensor:
    """D[M, N] = (A . SFA)(B . SFB)^T * s_a * s_b on tcgen05 (one launch).

    a_codes [M, K], b_codes [N, K] uint8 E4M3; a_sf / b_sf block-scale buffers
    (None = unit scales, i.e. a per-tensor operand); s_a, s_b 1-element f32
    device tensors.  Non-multiple-of-128 shapes are zero padded.  ``amax_out``
    (device f32 [1]) receives max|D| from the epilogue (not with accumulate).
    """
    m, k = a_codes.shape
    n, kb = b_codes.shape
    if k != kb:
        raise InvalidShapeError(f"K mismatch: {k} vs {kb}")
    if k % 32:
        raise InvalidShapeError(f"K={k} not divisible by 32")
    mp, np_, kp = _round_up(m, 128), _round_up(n, 128), _round_up(k, 128)
    dev = a_codes.device
    a = _pad_codes(a_codes, mp, kp)
    b = _pad_codes(b_codes, np_, kp)
    unit_a = a_sf is None
    if unit_a:
        a_sf = torch.full((_lib.sf_bytes(mp, kp),), 127, dtype=torch.uint8, device=dev)
    padded = (mp, np_) != (m, n)
    if out is not None and not padded:
        d = out
    else:
        if accumulate and out is not None:
            d = torch.zeros((mp, np_), dtype=out.dtype, device=dev)
            d[:m, :n] = out
        else:
            d = torch.empty((mp, np_), dtype=out.dtype if out is not None else out_dtype, device=dev)
    if amax_out is not None and (accumulate or not d.is_contiguous()):
        raise InvalidArgumentError("the amax epilogue needs a fresh, contiguous output")
    _lib.gemm(a, a_sf, b, b_sf, s_a, s_b, d, accumulate=accumulate, amax=amax_out)
    if d is out:
        return out
    if out is not None:
        out.copy_(d[:m, :n])
        return out
    return d[:m, :n] if padded else d


def mx_gemm_bkn(a_codes: torch.Tensor, a_sf: torch.Tensor, s_a: torch.Tensor, w_codes: torch.Tensor,
                s_w: torch.Tensor, *, out_dtype: torch.dtype = torch.bfloat16, out: torch.Tensor | None = None,
                amax_out: torch.Tensor | None = None) -> torch.Tensor:
    """D[M, N] = (A . SFA) W * s_a * s_w with W = w_codes [K, N] as stored (per-tensor
    E4M3, unit scales): the dgrad product dX = dY W without a transposed copy of W
    (MN-major tcgen05 B operand).  Shapes off the kernel's grid (M % 256, N % 256,
    K % 128) go through ``mx_gemm`` with W^T materialised.  ``amax_out`` (device
    f32 [1]) receives max|D| (the amax epilogue: D is the next output-gradient
    to be quantized)."""
    m, k = a_codes.shape
    kw, n = w_codes.shape
    if k != kw:
        raise InvalidShapeError(f"K mismatch: {k} vs {kw}")
    if m % 256 or n % 256 or k % 128 or not w_codes.is_contiguous() or not a_codes.is_contiguous():
        return mx_gemm(a_codes, a_sf, s_a, w_codes.t().contiguous(), None, s_w, out_dtype=out_dtype, out=out,
                       amax_out=amax_out)
    d = torch.empty((m, n), dtype=out_dtype, device=a_codes.device) if out is None else out
    _lib.gemm_bkn(a_codes, a_sf, w_codes, s_a, s_w, d, amax=amax_out)
    return d


def gemm_mx_epilogue(ops: GemmOperands) -> tuple[torch.Tensor, GemmCounters]:
    """C = W X^T with all FP32 dequantisation in the epilogue (gemm.py:115-129).

    Returns (C float32 [M_out, N_tokens] on the GPU, counters).  Runs the
    kernel as D = X W^T (activations as the A operand, unit-scale weights as
    B) and returns the transposed view, which is C.
    """
    m, n, k = ops.m, ops.n, ops.k
    qx = ops.qx
    sf_x = qx.sf
    if sf_x is None:
        raise InvalidArgumentError("activation operand lacks block-scale factors (quantize on the GPU)")
    d = mx_gemm(qx.codes, sf_x, qx.global_scale.reshape(1), ops.qw.codes, None, ops.qw.scale.reshape(1),
                out_dtype=torch.float32)
    return d.t(), mx_epilogue_counters(m, n, k, qx.k2)
