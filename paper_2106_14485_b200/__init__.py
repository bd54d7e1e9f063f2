"""B200-native (sm_100a) Sinkhorn sweep for dynamic multi-commodity flow (arXiv:2106.14485, Alg. 2).

The product is ``libmmf.so`` (C ABI in include/mmf.h).  ``_lib`` is its ctypes binding (same names);
``Solver`` strings those calls together for a ``workloads.Problem``-like object, with PyTorch
providing only device memory (the workspace) and the CUDA stream.
"""
from ._lib import MMFError, MMF_FP32, MMF_FP64, load, mmf_version  # noqa: F401
from .api import Solver  # noqa: F401
