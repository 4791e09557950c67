"""B200-native AoS<->SoA + reduced-precision SPH hot path (arxiv 2512.05516).

The product is the sm_100a shared library ``libsoaforge_b200.so`` behind the
C ABI in include/soaforge_b200.h; ``api`` mirrors the reference operator
interface on top of it.
"""
from . import api  # noqa: F401
from ._lib import LIB_PATH, SfError, SfInvalidArg, SfParseError, lib  # noqa: F401
