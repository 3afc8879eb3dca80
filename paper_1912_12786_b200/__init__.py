"""paper_1912_12786_b200 — B200-native custom-intersector BVH ray tracing (arXiv 1912.12786).

The product: ``libvsr.so`` (C ABI in ``include/vsr.h``; CUDA kernels for sm_100a in
``csrc/``) and the thin ctypes binding :mod:`paper_1912_12786_b200.vsr`.
It never imports ``oracle/`` (test infrastructure) and has no CPU fallback.
"""
from . import vsr  # noqa: F401
from .vsr import (ANY, CLOSEST, COUNT, COUNT_ALPHA_TEXTURE, DEFAULT, NONE,  # noqa: F401
                  ALPHA_PROCEDURAL, ALPHA_TEXTURE, Scene, VsrError, hits_to_numpy,
                  counts_to_numpy)

__all__ = ["vsr", "Scene", "VsrError", "CLOSEST", "ANY", "NONE", "DEFAULT", "ALPHA_TEXTURE",
           "ALPHA_PROCEDURAL", "COUNT", "COUNT_ALPHA_TEXTURE", "hits_to_numpy", "counts_to_numpy"]
