"""B200-native executor for the Delite/OptiML fused-multiloop hot path (arxiv 1109.0778).

Product layers (no CPU fallback anywhere):
  * ``libdlx.so`` — hand-written sm_100a CUDA kernels behind the C ABI in ``include/dlx.h``;
  * ``_lib``      — ctypes bindings of that ABI;
  * ``multiloops``— host-side mirror of the reference's loop families (k-means, GroupBy,
                    logistic regression, GDA, map/zipWith/reduce);
  * ``programs``  — iteration drivers (device-resident loops, CUDA graphs, multi-GPU);
  * ``comm``      — sample-sharded multi-GPU partial combine (NCCL allReduce).
"""
from . import _lib  # noqa: F401
from ._lib import DlxError, GenerationFailed, TrapError  # noqa: F401

__all__ = ["DlxError", "GenerationFailed", "TrapError"]
