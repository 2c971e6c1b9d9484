"""B200-native (sm_100a) GN-PCG field-map solver for RGP EPI correction (arXiv 2403.10706).

The product is libhysco.so (C ABI in include/hysco.h); `hysco` is its thin
ctypes binding.  Build with `python -m paper_2403_10706_b200.build`.
"""
from . import hysco  # noqa: F401
