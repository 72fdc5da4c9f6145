"""B200-native shadow-model training / MMD / membership-attack path.

Drop-in for the reference's (arXiv 2011.09463 companion, ``minitransfer``)
data-parallel privacy-analysis path; see DESIGN.md.  The compute path is
libmtk.so (hand-written CUDA for sm_100a behind the C ABI in
include/minitransfer/mtk.h).  Importing ``api`` loads it and fails loudly if
it has not been built.
"""
from .errors import ConfigError, DataError, Error, ShapeError, ValueError  # noqa: F401

__all__ = ["Error", "ShapeError", "ValueError", "ConfigError", "DataError"]
