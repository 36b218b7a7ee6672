"""ctypes binding of the C ABI in include/moss_b200.h.

There is deliberately no CPU fallback: if the in-tree library is missing or
CUDA is unavailable, every entry point raises.  PyTorch provides device
memory and the current stream; the arithmetic is all in libmoss_b200.so.
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import errors
from .build import LIB

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_F = ctypes.c_float

MOSS_F32 = 0
MOSS_BF16 = 1


class AdamParams(ctypes.Structure):
    _fields_ = [("lr", _F), ("beta1", _F), ("beta2", _F), ("eps", _F), ("weight_decay", _F),
                ("bc1", _F), ("bc2", _F), ("decoupled", _I), ("grad_scale", _F), ("step", ctypes.c_uint32)]


_SIGS = {
    "moss_version": (_I, []),
    "moss_strerror": (ctypes.c_char_p, [_I]),
    "moss_sf_bytes": (_I64, [_I64, _I64]),
    "moss_amax": (_I, [_P, _I, _I64, _P, _P, _P]),
    "moss_quant_mx2": (_I, [_P, _I, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "moss_quant_mx2_fused": (_I, [_P, _I, _I64, _I64, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "moss_workspace_bytes": (_I64, []),
    "moss_rmsnorm_fwd": (_I, [_P, _P, _P, _P, _F, _P, _P, _P, _I64, _I64, _P]),
    "moss_rmsnorm_bwd": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _P]),
    "moss_rmsnorm_bwd_workspace_bytes": (_I64, [_I64, _I64]),
    "moss_swiglu_fwd": (_I, [_P, _P, _P, _I64, _I64, _P]),
    "moss_swiglu_bwd": (_I, [_P, _P, _P, _P, _I64, _I64, _P]),
    "moss_rope_fwd": (_I, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I, _P]),
    "moss_rope_bwd": (_I, [_P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I, _P]),
    "moss_cross_entropy_fwd": (_I, [_P, _P, _P, _P, _I64, _I64, _P]),
    "moss_glue": (_I, [_I, _P, _P, _P, _F, _P, _P, _I64, _I64, _P]),
    "moss_gemm_mxf8_bkn": (_I, [_P, _P, _P, _P, _P, _P, _I, _I64, _I64, _I64, _I64, _P, _P]),
    "moss_sumsq": (_I, [_P, _P, _I64, _F, _P, _P, _P]),
    "moss_cross_entropy_bwd": (_I, [_P, _P, _P, _P, _P, _I64, _I64, _P]),
    "moss_quant_per_group": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, _P, _P]),
    "moss_gemm_pergroup": (_I, [_P, _P, _P, _P, _P, _I, _I64, _I64, _I64, _I64, _P]),
    "moss_encode_scaled": (_I, [_P, _I, _I64, _I64, _P, _F, _I, _P, _P, _P, _P, _P, _P]),
    "moss_gemm_mxf8": (_I, [_P, _P, _P, _P, _P, _P, _P, _I, _I64, _I64, _I64, _I64, _I, _P, _P, _P]),
    "moss_check_finite": (_I, [_P, _I, _I64, ctypes.c_uint32, _P, _P]),
    "moss_adamw_fp8": (_I, [_P, _P, _I, _P, _P, _I64, _I64, ctypes.POINTER(AdamParams), _F, _P, _P, _P,
                            _P, _P, _P]),
    "moss_adamw_fp8_dev": (_I, [_P, _P, _I, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load (building first if needed) the sm_100a library; raise if impossible."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("MOSS_B200_LIB", LIB)     # override: debug builds (tools/gemm_timeline.py)
    if path != LIB:
        handle = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
        return _lib
    if not os.path.exists(LIB):
        from .build import build
        try:
            build()
        except Exception as e:  # pragma: no cover - environment failure
            raise errors.CudaError(f"libmoss_b200.so missing and build failed: {e}") from e
    handle = ctypes.CDLL(LIB)
    for name, (res, args) in _SIGS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return _lib


_STATUS_EXC = {
    1: errors.InvalidShapeError,
    2: errors.InvalidValueError,
    3: errors.InvalidArgumentError,
    4: errors.E8m0RangeError,
    5: errors.CudaError,
    6: errors.InvalidArgumentError,
}


def check(status: int, what: str) -> None:
    if status:
        msg = lib().moss_strerror(status).decode()
        raise _STATUS_EXC.get(status, errors.MossqError)(f"{what}: {msg}")


def require_cuda(t: torch.Tensor, name: str) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise errors.InvalidArgumentError(f"{name} must be a CUDA tensor")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return MOSS_BF16
    if t.dtype == torch.float32:
        return MOSS_F32
    raise errors.InvalidArgumentError(f"unsupported dtype {t.dtype} (bf16 or f32)")


def sf_bytes(rows: int, cols: int) -> int:
    return int(lib().moss_sf_bytes(rows, cols))


NO_STEP = 0xFFFFFFFF


class FlagWord:
    """Device flag words shared by a group of launches: [0] the MOSS_FLAG_*
    error bits, [1] the smallest optimizer step whose K3 update was skipped
    because an error bit was already set (0xFFFFFFFF = none)."""

    def __init__(self, device=None):
        # no host->device copy: a flag word may be created during CUDA-graph capture
        self.t = torch.zeros(2, dtype=torch.int32, device=device or "cuda")
        self.t[1:].fill_(-1)
        self._init = self.t.clone()

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def read(self) -> tuple[int, int]:
        """(error bits, first skipped step or NO_STEP) — one device sync."""
        a, b = self.t.tolist()
        return a & 0xFFFFFFFF, b & 0xFFFFFFFF

    def raise_if_set(self, where: str = "") -> None:
        errors.raise_for_flags(int(self.t[0].item()), where)

    def reset(self) -> None:
        self.t.copy_(self._init)


_WS: dict[tuple[str, int], torch.Tensor] = {}


def workspace(device) -> torch.Tensor:
    """Workspace of the fused quantizer (its grid-barrier words), one per
    (device, stream), zeroed once: launches on one stream are ordered, and two
    streams quantizing concurrently never share barrier words."""
    dev = torch.device(device)
    key = (str(dev), torch.cuda.current_stream(dev).cuda_stream)
    if key not in _WS:
        nbytes = int(lib().moss_workspace_bytes())
        _WS[key] = torch.zeros((nbytes + 15) // 16 * 4, dtype=torch.int32, device=dev)
    return _WS[key]


# ---------------------------------------------------------------- live instrumentation
class Instrument:
    """Counts our kernel launches and (optionally) brackets each with CUDA
    events on the launching stream, recording the algorithmic work of the
    launch (FLOPs for GEMMs, bytes for the HBM-bound kernels).  bench.py
    turns this into per-kernel roofline numbers over its timed region."""

    def __init__(self):
        self.active = False
        self.timing = False
        self.external = False     # events captured into a CUDA graph (timeline of replays); records only while capturing
        self.launches = 0
        self.records: list[tuple[str, float, torch.cuda.Event, torch.cuda.Event]] = []

    def start(self, timing: bool = True, external: bool = False) -> None:
        self.active, self.timing, self.launches, self.records = True, timing, 0, []
        self.external = external

    def stop(self) -> None:
        self.active = False

    def summary(self) -> dict:
        out: dict[str, dict] = {}
        for kind, work, s, e in self.records:
            d = out.setdefault(kind, {"launches": 0, "ms": 0.0, "work": 0.0})
            d["launches"] += 1
            d["ms"] += s.elapsed_time(e)
            d["work"] += work
        return out


INSTR = Instrument()


class _Span:
    __slots__ = ("kind", "work", "s")

    def __init__(self, kind: str, work: float, kernels: int = 1):
        self.kind, self.work, self.s = kind, work, None
        if INSTR.active:
            INSTR.launches += kernels
            if INSTR.timing and (not INSTR.external or torch.cuda.is_current_stream_capturing()):
                self.s = torch.cuda.Event(enable_timing=True, external=INSTR.external)
                self.s.record()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        if self.s is not None and exc[0] is None:
            e = torch.cuda.Event(enable_timing=True, external=INSTR.external)
            e.record()
            INSTR.records.append((self.kind, self.work, self.s, e))
        return False


# ---------------------------------------------------------------- thin launchers
def amax(x: torch.Tensor, out: torch.Tensor, flags: FlagWord) -> None:
    with _Span("amax", x.numel() * x.element_size()):
        check(lib().moss_amax(x.data_ptr(), dtype_code(x), x.numel(), out.data_ptr(), flags.ptr, stream()),
              "moss_amax")


def quant_mx2(x2d: torch.Tensor, amax_t: torch.Tensor, flags: FlagWord, *, codes=None, sf=None, micro=None,
              codes_t=None, sf_t=None, micro_t=None, g_out=None) -> None:
    rows, cols = x2d.shape
    n = rows * cols
    out_b = (n + n / 32) * ((codes is not None) + (codes_t is not None))
    with _Span("quant", n * x2d.element_size() + out_b):
        check(lib().moss_quant_mx2(x2d.data_ptr(), dtype_code(x2d), rows, cols, amax_t.data_ptr(), ptr(codes),
                                   ptr(sf), ptr(micro), ptr(codes_t), ptr(sf_t), ptr(micro_t), ptr(g_out), flags.ptr,
                                   stream()),
              "moss_quant_mx2")


def quant_mx2_fused(x2d: torch.Tensor, amax_t: torch.Tensor, flags: FlagWord, *, amax_given: bool = False,
                    codes=None, sf=None, micro=None, codes_t=None, sf_t=None, micro_t=None, g_out=None) -> None:
    """K0+K1 in one launch (amax computed in-kernel unless ``amax_given``)."""
    rows, cols = x2d.shape
    n = rows * cols
    out_b = (n + n / 32) * ((codes is not None) + (codes_t is not None))
    with _Span("quant", n * x2d.element_size() + out_b):
        check(lib().moss_quant_mx2_fused(x2d.data_ptr(), dtype_code(x2d), rows, cols, amax_t.data_ptr(),
                                         int(amax_given), ptr(codes), ptr(sf), ptr(micro), ptr(codes_t), ptr(sf_t),
                                         ptr(micro_t), ptr(g_out), workspace(x2d.device).data_ptr(), flags.ptr,
                                         stream()),
              "moss_quant_mx2_fused")


def encode_scaled(x2d: torch.Tensor, flags: FlagWord, *, scale_t=None, scale_host: float = 0.0,
                  from_amax: bool = False, codes=None, codes_t=None, scale_out=None, n_saturated=None) -> None:
    rows, cols = x2d.shape
    n = rows * cols
    with _Span("encode", n * x2d.element_size() + n * ((codes is not None) + (codes_t is not None))):
        check(lib().moss_encode_scaled(x2d.data_ptr(), dtype_code(x2d), rows, cols, ptr(scale_t), float(scale_host),
                                       int(from_amax), ptr(codes), ptr(codes_t), ptr(scale_out), ptr(n_saturated),
                                       flags.ptr, stream()),
              "moss_encode_scaled")


def gemm(a, sfa, b, sfb, s_a, s_b, d, *, accumulate: bool = False, amax=None, flags: "FlagWord | None" = None) -> None:
    """``amax`` (device f32 [1], optional): receives max|D| (the amax epilogue)."""
    m, k = a.shape
    n = b.shape[0]
    if amax is not None and flags is None:
        flags = FlagWord(d.device)
    with _Span("gemm", 2.0 * m * n * k):
        check(lib().moss_gemm_mxf8(a.data_ptr(), sfa.data_ptr(), b.data_ptr(), ptr(sfb), s_a.data_ptr(),
                                   s_b.data_ptr(), d.data_ptr(), dtype_code(d), d.stride(0), m, n, k,
                                   int(accumulate), ptr(amax), flags.ptr if flags is not None else None, stream()),
              "moss_gemm_mxf8")


def gemm_bkn(a, sfa, b_kn, s_a, s_b, d, *, amax=None) -> None:
    """D = A B with B = b_kn [K, N] row-major (the weight as stored), unit B scales;
    ``amax`` (device f32 [1], optional) receives max|D|."""
    m, k = a.shape
    n = b_kn.shape[1]
    with _Span("gemm", 2.0 * m * n * k):
        check(lib().moss_gemm_mxf8_bkn(a.data_ptr(), sfa.data_ptr(), b_kn.data_ptr(), s_a.data_ptr(), s_b.data_ptr(),
                                       d.data_ptr(), dtype_code(d), d.stride(0), m, n, k, ptr(amax), stream()),
              "moss_gemm_mxf8_bkn")


def adamw_fp8_dev(w, g, m, v, rows: int, cols: int, p_dev: int, enc_dev: int | None, flags: FlagWord, *,
                  scale_out=None, w_fp8=None, w_fp8_t=None, w_amax=None, n_saturated=None) -> None:
    """K3 reading its hyper-parameters / encode scale from device memory (graph-capturable)."""
    n = rows * cols
    nbytes = n * (4 + g.element_size() + 8) + n * 12 + n * ((w_fp8 is not None) + (w_fp8_t is not None))
    with _Span("adamw", nbytes):
        check(lib().moss_adamw_fp8_dev(w.data_ptr(), g.data_ptr(), dtype_code(g), m.data_ptr(), v.data_ptr(), rows,
                                       cols, p_dev, enc_dev, ptr(scale_out), ptr(w_fp8), ptr(w_fp8_t), ptr(w_amax),
                                       ptr(n_saturated), flags.ptr, stream()),
              "moss_adamw_fp8_dev")


def check_finite(x: torch.Tensor, flags: FlagWord, bit: int = 4) -> None:
    """Set ``bit`` (default MOSS_FLAG_GRAD_NONFINITE) if x has a NaN/Inf."""
    with _Span("check", x.numel() * x.element_size()):
        check(lib().moss_check_finite(x.data_ptr(), dtype_code(x), x.numel(), bit, flags.ptr, stream()),
              "moss_check_finite")


def adamw_fp8(w, g, m, v, rows: int, cols: int, params: AdamParams, enc_scale: float, flags: FlagWord, *,
              w_fp8=None, w_fp8_t=None, w_amax=None, n_saturated=None) -> None:
    n = rows * cols
    nbytes = n * (4 + g.element_size() + 8) + n * 12 + n * ((w_fp8 is not None) + (w_fp8_t is not None))
    with _Span("adamw", nbytes):
        check(lib().moss_adamw_fp8(w.data_ptr(), g.data_ptr(), dtype_code(g), m.data_ptr(), v.data_ptr(), rows,
                                   cols, ctypes.byref(params), float(enc_scale), ptr(w_fp8), ptr(w_fp8_t),
                                   ptr(w_amax), ptr(n_saturated), flags.ptr, stream()),
              "moss_adamw_fp8")


# ---------------------------------------------------------------- producer kernels (bf16)
def _bf16(t, name):
    if t is not None and t.dtype != torch.bfloat16:
        raise errors.InvalidArgumentError(f"{name} must be bfloat16")


def rmsnorm_fwd(x, delta, x_out, w, eps: float, y, rstd, amax) -> None:
    T, d = x.shape
    _bf16(x, "x"), _bf16(delta, "delta"), _bf16(y, "y")
    with _Span("producer", T * d * (2 + 2 + (4 if delta is not None else 0))):
        check(lib().moss_rmsnorm_fwd(x.data_ptr(), ptr(delta), ptr(x_out), w.data_ptr(), float(eps), y.data_ptr(),
                                     rstd.data_ptr(), ptr(amax), T, d, stream()), "moss_rmsnorm_fwd")


def rmsnorm_bwd(dy, x, w, rstd, d_res, dx, dw, amax) -> None:
    """dw (nullable) is ACCUMULATED into (fixed-order reduction of per-CTA sums)."""
    T, d = x.shape
    _bf16(dy, "dy"), _bf16(x, "x"), _bf16(d_res, "d_res")
    ws = None
    if dw is not None:
        nb = int(lib().moss_rmsnorm_bwd_workspace_bytes(T, d))
        ws = torch.empty(max(nb, 4) // 4, dtype=torch.float32, device=x.device)
    with _Span("producer", T * d * (2 + 2 + 2 + (2 if d_res is not None else 0)), kernels=2 if dw is not None else 1):
        check(lib().moss_rmsnorm_bwd(dy.data_ptr(), x.data_ptr(), w.data_ptr(), rstd.data_ptr(), ptr(d_res),
                                     dx.data_ptr(), ptr(dw), ptr(amax), ptr(ws), T, d, stream()), "moss_rmsnorm_bwd")


def swiglu_fwd(gu, h, amax) -> None:
    T, f2 = gu.shape
    _bf16(gu, "gu")
    with _Span("producer", T * f2 * 2 + T * f2):
        check(lib().moss_swiglu_fwd(gu.data_ptr(), h.data_ptr(), ptr(amax), T, f2 // 2, stream()), "moss_swiglu_fwd")


def swiglu_bwd(dh, gu, dgu, amax) -> None:
    T, f2 = gu.shape
    _bf16(dh, "dh"), _bf16(gu, "gu")
    with _Span("producer", T * f2 * 2 * 2 + T * f2):
        check(lib().moss_swiglu_bwd(dh.data_ptr(), gu.data_ptr(), dgu.data_ptr(), ptr(amax), T, f2 // 2, stream()),
              "moss_swiglu_bwd")


def rope_fwd(qkv, cos, sin, q, k, v, B: int, S: int, H: int, hd: int, bshd: bool = False) -> None:
    """q, k, v memory [B, H, S, hd] or (bshd) [B, S, H, hd]."""
    _bf16(qkv, "qkv")
    with _Span("producer", B * S * 3 * H * hd * 4):
        check(lib().moss_rope_fwd(qkv.data_ptr(), cos.data_ptr(), sin.data_ptr(), q.data_ptr(), k.data_ptr(),
                                  v.data_ptr(), B, S, H, hd, int(bshd), stream()), "moss_rope_fwd")


def rope_bwd(dq, dk, dv, cos, sin, dqkv, amax, B: int, S: int, H: int, hd: int, bshd: bool = False) -> None:
    with _Span("producer", B * S * 3 * H * hd * 4):
        check(lib().moss_rope_bwd(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), cos.data_ptr(), sin.data_ptr(),
                                  dqkv.data_ptr(), ptr(amax), B, S, H, hd, int(bshd), stream()), "moss_rope_bwd")


def quant_per_group(x2d, codes, scales, flags: FlagWord, group: int = 128) -> None:
    rows, cols = x2d.shape
    with _Span("quant_pg", rows * cols * (x2d.element_size() + 1)):
        check(lib().moss_quant_per_group(x2d.data_ptr(), dtype_code(x2d), rows, cols, group, codes.data_ptr(),
                                         scales.data_ptr(), flags.ptr, stream()), "moss_quant_per_group")


def gemm_pergroup(a, sa_t, b, sb_t, d) -> None:
    m, k = a.shape
    n = b.shape[0]
    with _Span("gemm_pg", 2.0 * m * n * k):
        check(lib().moss_gemm_pergroup(a.data_ptr(), sa_t.data_ptr(), b.data_ptr(), sb_t.data_ptr(), d.data_ptr(),
                                       dtype_code(d), d.stride(0), m, n, k, stream()), "moss_gemm_pergroup")


def cross_entropy_fwd(logits, targets, lse, loss) -> None:
    T, V = logits.shape
    with _Span("producer", T * V * 2):
        check(lib().moss_cross_entropy_fwd(logits.data_ptr(), targets.data_ptr(), lse.data_ptr(), loss.data_ptr(),
                                           T, V, stream()), "moss_cross_entropy_fwd")


def cross_entropy_bwd(logits, targets, lse, scale, dlogits) -> None:
    T, V = logits.shape
    with _Span("producer", T * V * 4):
        check(lib().moss_cross_entropy_bwd(logits.data_ptr(), targets.data_ptr(), lse.data_ptr(), scale.data_ptr(),
                                           dlogits.data_ptr(), T, V, stream()), "moss_cross_entropy_bwd")


def glue(mode: int, x, out, amax, *, y=None, scale=None, alpha: float = 1.0, T: int, d: int) -> None:
    with _Span("producer", T * d * (2 + (4 if mode in (0, 1) else 2) + (2 if mode == 2 or (mode == 3 and y is not None)
                                                                       else 0))):
        check(lib().moss_glue(mode, x.data_ptr(), ptr(y), ptr(scale), float(alpha), out.data_ptr(), ptr(amax), T, d,
                              stream()),
              "moss_glue")


SUMSQ_PARTIALS = 1024       # include/moss_b200.h MOSS_SUMSQ_PARTIALS


def sumsq(x, acc, scale: float = 1.0, offset=None) -> None:
    """acc[0] = scale * sum (x + offset)^2 (f32, fixed-order: reproducible; offset optional, same
    shape); acc must hold 1 + SUMSQ_PARTIALS floats (the tail is the kernel's scratch)."""
    with _Span("producer", x.numel() * (2 if offset is None else 4), kernels=2):
        check(lib().moss_sumsq(x.data_ptr(), ptr(offset), x.numel(), float(scale), acc.data_ptr(), acc.data_ptr() + 4,
                               stream()),
              "moss_sumsq")
