"""Error taxonomy shared with the reference (kernelgp errors.py:4-17).

The C library returns integer codes; ``_lib.check`` raises one of these. If the
reference package is importable in this interpreter its classes are reused, so
callers that catch ``kernelgp.errors.*`` keep working after the switch.
"""

try:  # pragma: no cover - only where the reference is installed
    from kernelgp import errors as _ref_errors  # type: ignore

    KernelGpError = _ref_errors.KernelGpError
    NumericalError = _ref_errors.NumericalError
    BreakdownError = _ref_errors.BreakdownError
    ResourceLimitError = _ref_errors.ResourceLimitError
except Exception:

    class KernelGpError(Exception):
        """Root of every error this package raises on purpose."""

    class NumericalError(KernelGpError):
        """Non-finite values, a non-SPD matrix, or a non-positive Ritz value."""

    class BreakdownError(NumericalError):
        """p^T A p <= 0 inside CG/PCG, or a failed landmark factorisation."""

    class ResourceLimitError(KernelGpError):
        """Dense materialisation above the budget, or device memory exhausted."""


__all__ = ["KernelGpError", "NumericalError", "BreakdownError", "ResourceLimitError"]
