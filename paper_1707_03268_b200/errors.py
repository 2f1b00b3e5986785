"""Error taxonomy and input coercion of the drop-in scoring path.

Mirrors ``cpdetect.validation`` (reference ``pkg/src/cpdetect/validation.py:21-86``):
``CpdetectError`` is the base, ``ValidationError`` is also a ``ValueError``,
``NumericError`` an ``ArithmeticError``.  When the reference package is
importable in the caller's process, each class here additionally derives from
the reference class of the same name, so ``except cpdetect.ValidationError``
keeps working after a caller switches its scoring calls to this package.
"""

import numpy as np

try:  # pragma: no cover - depends on the caller's environment
    from cpdetect import validation as _ref_validation  # type: ignore

    _REF = (
        _ref_validation.CpdetectError,
        _ref_validation.ValidationError,
        _ref_validation.FormatError,
        _ref_validation.NumericError,
    )
except Exception:  # reference absent: plain hierarchy
    _REF = None

__all__ = [
    "CpdetectError",
    "ValidationError",
    "FormatError",
    "NumericError",
    "DeviceError",
    "check_tensor3",
    "check_feature_map",
]


if _REF is None:

    class CpdetectError(Exception):
        """Base class for all errors raised by this package."""

    class ValidationError(CpdetectError, ValueError):
        """An input violates a documented precondition (validation.py:25-26)."""

    class FormatError(CpdetectError, ValueError):
        """A serialized payload is malformed (validation.py:29-31)."""

    class NumericError(CpdetectError, ArithmeticError):
        """A numerical computation failed irrecoverably (validation.py:34-35)."""

else:  # pragma: no cover

    class CpdetectError(_REF[0]):
        """Base class for all errors raised by this package."""

    class ValidationError(CpdetectError, _REF[1]):
        """An input violates a documented precondition (validation.py:25-26)."""

    class FormatError(CpdetectError, _REF[2]):
        """A serialized payload is malformed (validation.py:29-31)."""

    class NumericError(CpdetectError, _REF[3]):
        """A numerical computation failed irrecoverably (validation.py:34-35)."""


class DeviceError(CpdetectError, RuntimeError):
    """The B200 extension is missing, or a CUDA call failed.

    There is no CPU fallback: the product path raises this instead."""


def _finite_f64(a, name):
    arr = np.asarray(a, dtype=np.float64)
    if arr.size and not np.isfinite(arr).all():
        raise ValidationError(f"{name} contains non-finite values")
    return np.ascontiguousarray(arr)


def check_tensor3(a, name="tensor"):
    """Finite order-3 array with positive extents (validation.py:65-76)."""
    arr = _finite_f64(a, name)
    if arr.ndim != 3:
        raise ValidationError(f"{name} must be 3-dimensional, got shape {arr.shape}")
    if min(arr.shape) < 1:
        raise ValidationError(f"{name} must have positive extents, got {arr.shape}")
    return arr


def check_feature_map(a, channels=None, name="feature map"):
    """(height, width, channels) feature map (validation.py:79-86)."""
    arr = check_tensor3(a, name)
    if channels is not None and arr.shape[2] != channels:
        raise ValidationError(f"{name} has {arr.shape[2]} channels, expected {channels}")
    return arr
