"""Exception contract of the drop-in boundary.

Same class names and the same ``ValueError`` ancestry as the reference's
``mossq.errors`` (reference: pkg/src/mossq/errors.py:4-45), so code written
against the reference keeps catching the right things.

Host-checkable conditions (shape, K % 32, k1, dtype, alignment) raise before
any kernel is launched.  Data-dependent conditions that the reference detects
synchronously (non-finite input, E8M0 exponent below -127) are detected on the
device: the kernels OR bits into a ``flags`` word and the host turns the bits
into these exceptions at the next check (``raise_for_flags``).  That is the one
documented deviation from the reference, which raises inside each numpy call.
"""

from __future__ import annotations


class MossqError(Exception):
    """Base class for every error raised by this package."""


class InvalidShapeError(MossqError, ValueError):
    """Empty / non-positive shape, or operand shapes that disagree."""


class InvalidValueError(MossqError, ValueError):
    """A numeric precondition failed (NaN/Inf input, r <= 0, E8M0 code 255)."""


class InvalidArgumentError(MossqError, ValueError):
    """An argument lies outside its domain (bad enum, k1 with GEMM, betas ...)."""


class E8m0RangeError(MossqError, ValueError):
    """A power-of-two scale does not fit E8M0's [2^-127, 2^127]."""


class UndefinedModelError(MossqError, ValueError):
    """Kept for name parity with the reference (SNR models are out of scope)."""


class FormatError(MossqError):
    """Base for tensor-file parsing errors (kept for name parity)."""


class BadMagicError(FormatError):
    pass


class VersionMismatchError(FormatError):
    pass


class TruncatedPayloadError(FormatError):
    pass


class TrainDivergedError(MossqError):
    """Training loss exceeded the divergence threshold (train.py:184-185)."""


class CudaError(MossqError, RuntimeError):
    """The CUDA runtime reported a failure inside the native library."""


# Device flag bits written by the kernels (include/moss_b200.h MOSS_FLAG_*).
FLAG_NONFINITE = 1
FLAG_E8M0_RANGE = 2
FLAG_GRAD_NONFINITE = 4


def raise_for_flags(flags: int, where: str = "") -> None:
    """Turn a device flag word into the reference's exception classes."""
    suffix = f" ({where})" if where else ""
    if flags & FLAG_NONFINITE:
        raise InvalidValueError("quantization requires finite input" + suffix)
    if flags & FLAG_GRAD_NONFINITE:
        raise InvalidValueError("gradient contains NaN/Inf" + suffix)
    if flags & FLAG_E8M0_RANGE:
        raise E8m0RangeError("value below 2^-127" + suffix)
