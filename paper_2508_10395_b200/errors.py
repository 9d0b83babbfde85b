"""Exception hierarchy of the B200 XQuant path.

Mirrors the reference's ``xcache.errors`` one-for-one
(/root/reference/pkg/src/xcache/errors.py:4-35) so callers that catch the
reference's exceptions keep working. The C-ABI returns integer status codes
(include/xquant.h, ``XQ_E*``); :func:`raise_for_status` maps them onto these
classes.
"""


class XCacheError(Exception):
    """Base class for all package errors (errors.py:4-5)."""


class ShapeError(XCacheError):
    """Operands have incompatible dimensions (errors.py:8-9)."""


class ConfigError(XCacheError):
    """Invalid configuration value (errors.py:12-13)."""


class DataError(XCacheError):
    """Input violates a precondition, e.g. NaN/Inf (errors.py:16-17)."""


class FormatError(XCacheError):
    """Malformed binary artifact (errors.py:20-27)."""

    def __init__(self, message: str, offset: int | None = None):
        if offset is not None:
            message = f"{message} (at byte offset {offset})"
        super().__init__(message)
        self.offset = offset


class NumericalError(XCacheError):
    """An iterative method failed to converge (errors.py:30-31)."""


class UsageError(XCacheError):
    """Operation called on a state that does not support it (errors.py:34-35)."""


class CudaError(XCacheError):
    """The CUDA runtime reported an error inside the native library."""


# Status codes of the C-ABI (include/xquant.h). Keep in sync.
XQ_OK = 0
XQ_ESHAPE = 1
XQ_ECONFIG = 2
XQ_EUSAGE = 3
XQ_ENONFINITE = 4
XQ_ECUDA = 5

_STATUS = {
    XQ_ESHAPE: ShapeError,
    XQ_ECONFIG: ConfigError,
    XQ_EUSAGE: UsageError,
    XQ_ENONFINITE: DataError,
    XQ_ECUDA: CudaError,
}


def raise_for_status(status: int, what: str, detail: str = "") -> None:
    """Raise the exception class mapped to a non-zero C-ABI status."""
    if status == XQ_OK:
        return
    cls = _STATUS.get(status, XCacheError)
    msg = f"{what} failed with status {status}"
    if detail:
        msg += f": {detail}"
    raise cls(msg)
