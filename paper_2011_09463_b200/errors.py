"""Error taxonomy of the reference (error.hpp:10-51) as Python exceptions.

C-ABI status codes map onto these classes: 1 ShapeError, 2 ValueError,
3 ConfigError, 4 DataError, 5 Error, 6 CheckpointError, 7 VersionError,
8 DigestError, 9 TruncatedError.  ``ValueError`` also derives from the
builtin so idiomatic ``except ValueError`` keeps working.
"""
import builtins


class Error(RuntimeError):
    """mt::Error (error.hpp:10-13): base of everything the toolkit raises."""


class ShapeError(Error):
    """mt::ShapeError (error.hpp:16-18): tensor dimension mismatches."""


class ValueError(Error, builtins.ValueError):  # noqa: A001 - mirrors mt::ValueError
    """mt::ValueError (error.hpp:21-23): bad argument values."""


class ConfigError(Error):
    """mt::ConfigError (error.hpp:26-28): invalid configuration."""


class DataError(Error):
    """mt::DataError (error.hpp:31-33): problems with input data."""


class CheckpointError(DataError):
    """mt::CheckpointError (error.hpp:34-37): checkpoint load failures."""


class VersionError(CheckpointError):
    """mt::VersionError (error.hpp:38-40): unsupported format_version."""


class DigestError(CheckpointError):
    """mt::DigestError (error.hpp:41-43): payload SHA-256 mismatch."""


class TruncatedError(CheckpointError):
    """mt::TruncatedError (error.hpp:44-46): file shorter than its header says."""


class ConsistencyError(Error):
    """dp_step's "replica divergence detected before step -> consistency
    error"; error.hpp has no dedicated class, so it derives
    from mt::Error.  Raised host-side by dp.DataParallel."""


_BY_STATUS = {1: ShapeError, 2: ValueError, 3: ConfigError, 4: DataError, 5: Error,
              6: CheckpointError, 7: VersionError, 8: DigestError, 9: TruncatedError}


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    from ._lib import lib

    msg = lib.mtk_last_error().decode(errors="replace")
    raise _BY_STATUS.get(status, Error)(f"{what}: {msg}" if what else msg)
