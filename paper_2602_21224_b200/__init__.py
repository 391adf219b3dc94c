"""B200-native hidden-state tree speculative decoding (arXiv 2602.21224).

The product is the C-ABI library libhsd.so (include/hsd.h, CUDA for sm_100a);
`hsd` is its thin ctypes binding. This package never imports `oracle`.
"""
from . import hsd  # noqa: F401
