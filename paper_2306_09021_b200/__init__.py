"""B200-native hot path of Position-Based Nonlinear Gauss-Seidel (arXiv 2306.09021).

The product is the C-ABI library libpbng.so (include/pbng.h, sources in csrc/) with hand-written sm_100a
kernels; `pbng` is its thin ctypes binding.  This package never imports the test oracle.
"""
from .pbng import (  # noqa: F401
    ACCEL,
    Context,
    DTYPE,
    Group,
    EXPORTS,
    LIB_PATH,
    MODEL,
    PBNGError,
    context_from_scene,
    lib,
    nccl_unique_id,
    weak_constraints_array,
)

__version__ = "0.1.0"
