"""B200-native fused SwiGLU-MLP decode path (DeepFusionKernel, arXiv 2602.11808).

The product is the CUDA library ``paper_2602_11808_b200/lib/libdfk.so``
(sm_100a kernels + the C ABI declared in ``include/dfk.h``).  This module is
the Python host side over that ABI (ctypes; no torch, no CPU fallback):

* :mod:`paper_2602_11808_b200.runtime` — handles: :class:`Context`,
  :class:`Weights`, :class:`DeviceArray`, :class:`Config`.
* :mod:`paper_2602_11808_b200.deepfusion` — a mirror of the reference's
  operator API (``/root/reference/proj/include/deepfusion/*.hpp``):
  ``run_fused_stage1``, ``run_fused``, ``down_projection``, ``run_stage1``,
  ``run_variant``, ``run_tp_mlp``, ``balanced_ranges``, ``make_plan``,
  ``Tuner``..., with the same argument meaning and error classes.

Importing this package loads the library; if it is missing and cannot be
built, the import fails loudly.
"""
from .runtime import (  # noqa: F401
    Config,
    Context,
    DeviceArray,
    DfkError,
    ShapeError,
    Weights,
    block_bytes,
    lib,
    library_path,
)

__all__ = ["Config", "Context", "DeviceArray", "DfkError", "ShapeError", "Weights",
           "block_bytes", "lib", "library_path"]
