"""The reference's exception taxonomy (core.hpp:14-57), raised by the host mirror."""
from __future__ import annotations


class SemsplatError(Exception):
    """Base of every error this package raises."""


class FormatError(SemsplatError):
    """Malformed file contents (core.hpp:15)."""


class DataError(SemsplatError):
    """Well-formed input carrying invalid values (core.hpp:21)."""


class ContractError(SemsplatError):
    """Caller violated an operation precondition (core.hpp:27)."""


class NumericError(SemsplatError):
    """Numerically unusable input (core.hpp:33)."""


class IoError(SemsplatError):
    """Filesystem failure (core.hpp:39)."""


class LookupError_(SemsplatError):
    """Lookup-table miss (core.hpp:45)."""


class PipelineError(SemsplatError):
    """Aggregated failure of the per-device workers; keeps per-worker status
    lines like the reference's PipelineError (core.hpp:51-57)."""

    def __init__(self, what: str, worker_status=None, caused_by_data: bool = False):
        super().__init__(what)
        self.worker_status = list(worker_status or [])
        self.caused_by_data = caused_by_data


class DeviceError(SemsplatError):
    """CUDA / driver failure (no reference analogue)."""


_KINDS = {1: ContractError, 2: DataError, 3: NumericError, 4: FormatError, 5: IoError, 6: PipelineError,
          7: DeviceError}


def raise_for(kind: int, message: str):
    raise _KINDS.get(kind, DeviceError)(message)
