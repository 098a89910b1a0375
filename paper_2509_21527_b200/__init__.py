"""B200-native eighth-shell DD halo exchange (arXiv 2509.21527).

The product is libhalo.so (C ABI, include/halo.h) with hand-written sm_100a
kernels; this package is its thin Python binding plus PyTorch plumbing.
"""
from ._lib import (HALO_F_ATOMIC_UNPACK, HALO_F_DETERMINISTIC, HALO_F_CE_PATH, HALO_F_GPU_FENCE, HALO_F_NO_HOME_CHECK, HALO_F_PAPER_FLAGS, HALO_F_TIMERS, LIB_PATH,
                   load as load_library)
from .halo import Halo, HaloError

__all__ = ["Halo", "HaloError", "load_library", "LIB_PATH", "HALO_F_ATOMIC_UNPACK", "HALO_F_DETERMINISTIC", "HALO_F_CE_PATH", "HALO_F_GPU_FENCE",
           "HALO_F_NO_HOME_CHECK", "HALO_F_PAPER_FLAGS", "HALO_F_TIMERS"]
