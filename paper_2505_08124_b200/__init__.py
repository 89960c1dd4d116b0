"""paper_2505_08124_b200 -- B200-native (sm_100a) implementation of SLAG's
per-Gaussian language-embedding pass and cosine top-k query, behind the
reference's semsplat API (include/semsplat_b200.h)."""
from .errors import (ContractError, DataError, DeviceError, FormatError, IoError, NumericError,  # noqa: F401
                     PipelineError, SemsplatError)

__all__ = ["ContractError", "DataError", "DeviceError", "FormatError", "IoError", "NumericError", "PipelineError",
           "SemsplatError"]
