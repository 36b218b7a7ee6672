"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/moss_b200.h declares, and its host-side argument checks
map to the reference's error classes before any launch; host logic of the
Python layer (schedules, operand validation) matches the reference."""

import ctypes
import inspect
import os
import re

import pytest
import torch

from paper_2511_05811_b200 import _lib, autoscale, errors
from paper_2511_05811_b200.build import LIB

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "moss_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(moss_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 8, syms
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib._SIGS), "ctypes signatures must cover the header exactly"


def test_host_only_entry_points():
    lib = _lib.lib()
    assert lib.moss_version() >= 100
    assert lib.moss_sf_bytes(8192, 4096) == 8192 * 4096 // 32
    assert lib.moss_sf_bytes(100, 96) == 512            # padded to one 128 x 4 chunk
    assert lib.moss_sf_bytes(1, 33) == -1
    assert lib.moss_strerror(1) == b"invalid shape"


def test_argument_checks_precede_launch():
    lib = _lib.lib()
    fake = ctypes.c_void_p(16)
    # cols % 32 -> InvalidShapeError, checked before touching the device
    assert lib.moss_quant_mx2(fake, 1, 4, 33, fake, fake, None, None, None, None, None, None, fake, None) == 1
    # K % 128 -> shape error
    assert lib.moss_gemm_mxf8(fake, fake, fake, None, fake, fake, fake, 1, 128, 128, 128, 96, 0, None, None,
                              None) == 1
    # accumulate into bf16 -> argument error
    assert lib.moss_gemm_mxf8(fake, fake, fake, None, fake, fake, fake, 1, 128, 128, 128, 128, 1, None, None,
                              None) == 3
    # amax epilogue with accumulate (the stored sum is not seen) -> argument error
    assert lib.moss_gemm_mxf8(fake, fake, fake, None, fake, fake, fake, 0, 128, 128, 128, 128, 1, fake, fake,
                              None) == 3
    # amax epilogue needs a contiguous D (ldd == N)
    assert lib.moss_gemm_mxf8(fake, fake, fake, None, fake, fake, fake, 1, 256, 128, 128, 128, 0, fake, fake,
                              None) == 3
    # misaligned pointer -> alignment error
    odd = ctypes.c_void_p(17)
    assert lib.moss_amax(odd, 1, 64, fake, fake, None) == 6
    # bad dtype
    assert lib.moss_amax(fake, 7, 64, fake, fake, None) == 3
    # fused quantizer: workspace is required; cols % 32
    assert lib.moss_quant_mx2_fused(fake, 1, 128, 128, fake, 0, fake, fake, None, None, None, None, fake, None,
                                    fake, None) == 3
    assert lib.moss_quant_mx2_fused(fake, 1, 128, 100, fake, 0, fake, fake, None, None, None, None, fake, fake,
                                    fake, None) == 1
    assert lib.moss_workspace_bytes() >= 16
    # producer kernels: d % 8, d <= 8192, f % 8, hd % 8, missing outputs
    assert lib.moss_rmsnorm_fwd(fake, None, None, fake, ctypes.c_float(1e-5), fake, fake, None, 4, 100, None) == 1
    assert lib.moss_rmsnorm_fwd(fake, None, None, fake, ctypes.c_float(1e-5), fake, fake, None, 4, 16384, None) == 1
    assert lib.moss_rmsnorm_fwd(fake, fake, None, fake, ctypes.c_float(1e-5), fake, fake, None, 4, 128, None) == 3
    assert lib.moss_rmsnorm_bwd(fake, fake, fake, fake, None, None, None, None, None, 4, 128, None) == 3
    assert lib.moss_rmsnorm_bwd(fake, fake, fake, fake, None, fake, fake, None, None, 4, 128, None) == 3  # dw w/o ws
    assert lib.moss_rmsnorm_bwd_workspace_bytes(4, 100) == -1
    assert lib.moss_swiglu_fwd(fake, fake, None, 4, 12, None) == 1
    assert lib.moss_swiglu_bwd(odd, fake, fake, None, 4, 16, None) == 6
    assert lib.moss_rope_fwd(fake, fake, fake, fake, fake, fake, 1, 4, 2, 12, 1, None) == 1
    assert lib.moss_rope_bwd(fake, fake, fake, fake, fake, None, None, 1, 4, 2, 16, 1, None) == 3
    with pytest.raises(errors.InvalidShapeError):
        _lib.check(1, "x")
    with pytest.raises(errors.E8m0RangeError):
        _lib.check(4, "x")


def test_flag_bits_to_reference_exceptions():
    with pytest.raises(errors.InvalidValueError):
        errors.raise_for_flags(errors.FLAG_NONFINITE)
    with pytest.raises(errors.E8m0RangeError):
        errors.raise_for_flags(errors.FLAG_E8M0_RANGE)
    with pytest.raises(errors.InvalidValueError):
        errors.raise_for_flags(errors.FLAG_GRAD_NONFINITE)
    errors.raise_for_flags(0)
    # same ancestry as the reference hierarchy (errors.py:4-45)
    assert issubclass(errors.InvalidShapeError, ValueError) and issubclass(errors.E8m0RangeError, errors.MossqError)


def test_schedule_host_logic_matches_reference(golden):
    s = autoscale.ScaleSchedule(s0=0.01, s_t=0.01, t=0, interval=500, delta_max=448.0)
    for _ in range(1000):
        autoscale.auto_scale_advance(s, 3e-4)
    assert s.s_t == float(golden["sched_eq10_s"])       # bit-identical f64 accumulation
    assert list(inspect.signature(autoscale.auto_scale_advance).parameters) == ["sched", "current_eta"]
    s = autoscale.ScaleSchedule(s0=0.01, s_t=0.01, t=0, interval=5, delta_max=448.0, eta_schedule=lambda t: 1e-3)
    autoscale.auto_scale_advance(s)
    assert s.s_t == pytest.approx(0.01 + 1e-3 / 448.0)
    with pytest.raises(errors.InvalidArgumentError):
        autoscale.auto_scale_advance(autoscale.ScaleSchedule(0.01, 0.01, 0, 5, 448.0))
    with pytest.raises(errors.InvalidArgumentError):
        autoscale.ScaleSchedule(0.01, 0.01, 0, 0, 448.0)
    s = autoscale.ScaleSchedule(0.01, 0.01, t=1, interval=10, delta_max=448.0)
    assert not autoscale.rescale_due(s)
    with pytest.raises(errors.InvalidArgumentError):
        autoscale.rescale_interval(torch.ones(8), s, __import__("paper_2511_05811_b200").E4M3)


def test_gemm_operand_validation_cpu():
    from paper_2511_05811_b200.gemm import GemmOperands, mx_epilogue_counters
    from paper_2511_05811_b200.quantize import PerTensorQuant, TwoLevelQuant
    from paper_2511_05811_b200.fp8 import E4M3
    z = torch.zeros
    qw = PerTensorQuant(codes=z(4, 64, dtype=torch.uint8), scale=torch.tensor(1.0), fmt=E4M3)
    qx = TwoLevelQuant(codes=z(4, 32, dtype=torch.uint8), global_scale=torch.tensor(1.0),
                       micro_codes=z(4, 1, dtype=torch.uint8), fmt=E4M3)
    with pytest.raises(errors.InvalidShapeError):
        GemmOperands(qw=qw, qx=qx)
    qx2 = TwoLevelQuant(codes=z(4, 64, dtype=torch.uint8), global_scale=torch.tensor(1.0),
                        micro_codes=z(4, 2, dtype=torch.uint8), fmt=E4M3, k1=32)
    with pytest.raises(errors.InvalidArgumentError):
        GemmOperands(qw=qw, qx=qx2)
    c = mx_epilogue_counters(4, 4, 4096)
    assert (c.mainloop_dequant_multiplies, c.epilogue_dequant_multiplies, c.block_scale_multiplies,
            c.mac_count) == (0, 16, 16 * 128, 16 * 4096)          # test_gemm.py:65-73
