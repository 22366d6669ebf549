"""paper_2602_11843_b200 -- B200-native truncated Neumann series by radix kernels.

Thin ctypes binding of libnseries.so (C ABI in include/nseries.h).  The binding only
marshals arguments: every arithmetic step runs in the library's sm_100a kernels.  There is
no CPU fallback -- importing works without a GPU (plan building is host code), but every
evaluation entry point fails loudly when no sm_100 device / built library is available.
"""
from ._binding import *  # noqa: F401,F403
from ._binding import __all__  # noqa: F401
