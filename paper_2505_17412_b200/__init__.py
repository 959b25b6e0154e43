"""paper_2505_17412_b200 — B200-native Spatial Sparse Attention (Direct3D-S2, arXiv 2505.17412 §4.1).

The product is the C-ABI shared library libssa_b200.so (include/ssa.h) built from csrc/ for sm_100a;
`ssa` is its thin ctypes binding. There is no CPU fallback: importing works without a GPU, but every
compute call needs a CUDA device and the built library.
"""
from . import ssa  # noqa: F401
from .ssa import (AttnCfg, Plan, Saved, SSAError, SSAFunction, ssa_backward, ssa_build_blocks,  # noqa: F401
                  ssa_forward)

__all__ = ["ssa", "AttnCfg", "Plan", "Saved", "SSAError", "SSAFunction", "ssa_build_blocks", "ssa_forward",
           "ssa_backward"]
