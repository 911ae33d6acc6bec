"""Exception types of the reference (errors.py:4-13), shared when available.

When the reference package ``tensortune`` is importable its classes are used
directly, so ``except tensortune.errors.DataValidationError`` and the CLI's
exit-code mapping (cli.py:569-577) keep working after ``install()``.
Otherwise identical stand-ins are defined.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from tensortune.errors import DataValidationError, NumericFailure, TensorTuneError
except Exception:  # noqa: BLE001

    class TensorTuneError(Exception):
        """Base class for every error raised by this package."""

    class DataValidationError(TensorTuneError):
        """Input data violates the dataset schema or a structural invariant."""

    class NumericFailure(TensorTuneError):
        """A numeric computation produced a NaN or overflowed its domain."""


__all__ = ["TensorTuneError", "DataValidationError", "NumericFailure"]
