"""Exception types, mirroring the reference's ``drrtrace.errors`` hierarchy
(``pkg/src/drrtrace/errors.py:1-36``) so callers can catch the same names.

The C-ABI status codes of ``include/drr_b200.h`` map onto these classes in
:func:`paper_2208_12737_b200._lib.check`.
"""


class DrrTraceError(Exception):
    """Base class for all renderer errors (errors.py:4-5)."""


class InvalidArgumentError(DrrTraceError, ValueError):
    """An argument violates a documented precondition (errors.py:8-9)."""


class DegenerateRayError(DrrTraceError):
    """A ray has zero length: source coincides with a pixel (errors.py:27-28)."""


class MetricUndefinedError(DrrTraceError):
    """A similarity metric is undefined for the inputs (errors.py:31-32)."""


class GradientUndefinedError(DrrTraceError):
    """The pose gradient is undefined at the parameters (errors.py:35-36)."""


class KernelError(DrrTraceError, RuntimeError):
    """A CUDA launch or runtime failure inside the native library."""


class HeaderParseError(DrrTraceError):
    """A volume header could not be parsed (errors.py:12-20); ``offset`` is the
    byte offset where parsing failed."""

    def __init__(self, message, offset):
        super().__init__(f"{message} (byte offset {offset})")
        self.offset = offset


class CorruptFileError(DrrTraceError):
    """File contents disagree with the declared sizes (errors.py:23-24)."""
