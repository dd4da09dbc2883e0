"""B200-native phi-function action engine (arXiv 2211.00696 hot path).

The product is the C-ABI library libpq_b200.so (sm_100a kernels + C++ host engine, see
include/pq_b200.h); this package is its Python mirror of the reference phiquad API.
"""
from .phiquad import *  # noqa: F401,F403
from .phiquad import __all__  # noqa: F401
from ._lib import LIB_PATH  # noqa: F401
