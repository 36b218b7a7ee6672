"""B200-native (sm_100a) MOSS FP8 training hot path.

Drop-in for the reference package ``mossq`` 0.1.0 on the path the MOSS paper
(arXiv 2511.05811) accelerates: two-level microscaled activation
quantization, MXFP8 GEMMs with epilogue dequantisation, and AdamW fused with
automatic per-tensor weight scaling.  Top-level names mirror
mossq/__init__.py:3-36 for the hot-path subset; the torch training wrappers
(MossLinear, MossAdamW) live in ``paper_2511_05811_b200.nn``.

All arithmetic runs in the in-tree CUDA library (paper_2511_05811_b200/_build/
libmoss_b200.so, C ABI in include/moss_b200.h).  There is no CPU fallback.
"""

from .errors import (E8m0RangeError, InvalidArgumentError, InvalidShapeError, InvalidValueError, MossqError,
                     TrainDivergedError)
from .fp8 import E4M3, E5M2, E8m0Rounding, Fp8Format, decode_table, e8m0_decode, e8m0_encode, fp8_decode, fp8_encode
from .quantize import PerTensorQuant, TwoLevelQuant, dequantize, quant_per_tensor, quant_two_level

__version__ = "0.1.0"

__all__ = [
    "MossqError", "InvalidShapeError", "InvalidValueError", "InvalidArgumentError", "E8m0RangeError",
    "TrainDivergedError", "E4M3", "E5M2", "E8m0Rounding", "Fp8Format", "fp8_encode", "fp8_decode",
    "decode_table", "e8m0_encode", "e8m0_decode", "PerTensorQuant", "TwoLevelQuant", "quant_per_tensor",
    "quant_two_level", "dequantize", "__version__",
]
