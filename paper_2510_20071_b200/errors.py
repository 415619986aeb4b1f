"""Exception types raised at the reconstruction boundary.

Same class names and inheritance as the reference package
(`fibar/errors.py:4-41`) so callers' ``except`` clauses keep working when they
switch engines.  Native status codes from the C-ABI layer
(`include/fibar_b200.h`, ``FIBAR_E_*``) are translated into these classes by
:func:`raise_for_status`.
"""

from __future__ import annotations


class FibarError(Exception):
    """Root of every error this package raises."""


class ConfigError(FibarError):
    """A parameter or configuration value is invalid."""


class FormatError(FibarError):
    """Bytes do not form a valid event stream (magic, header)."""


class TruncationError(FormatError):
    """The stream stops in the middle of a record."""

    def __init__(self, message, byte_offset):
        self.byte_offset = byte_offset
        super().__init__(f"{message} (byte offset {byte_offset})")


class DataError(FibarError):
    """The container is well formed but a payload value is not (pixel out of range...)."""


class OrderError(FibarError):
    """Timestamps go backwards where they must not."""


class RangeError(FibarError):
    """A value does not fit the field it has to be encoded into."""


class EstimationError(FibarError):
    """Threshold estimation has no usable pixels."""


class InvariantError(FibarError):
    """Internal bookkeeping went inconsistent (e.g. a saturated counter)."""


class DeviceError(FibarError):
    """The CUDA layer reported a failure (launch error, out of memory, no device)."""


# status codes shared with include/fibar_b200.h
_STATUS = {
    1: ConfigError,
    2: DataError,
    3: OrderError,
    4: InvariantError,
    5: DeviceError,
    6: DeviceError,
}


def raise_for_status(code: int, what: str) -> None:
    """Map a non-zero C-ABI status to the matching exception."""
    if code == 0:
        return
    cls = _STATUS.get(code, DeviceError)
    raise cls(f"{what} failed (status {code})")
