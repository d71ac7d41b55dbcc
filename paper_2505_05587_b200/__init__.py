"""SteepGS (arXiv 2505.05587) hot path on B200: splitting-matrix rasterizer + steepest density control.

The compute lives in libsteepgs.so (hand-written sm_100a CUDA behind the C ABI of include/steepgs.h);
this package is the thin Python binding (`_lib`), the host-side orchestration (`pipeline`) and the
multi-GPU view sharding (`parallel`).  No CPU fallback exists.
"""
from . import _lib  # noqa: F401
from .pipeline import SMOOTH, Adam, Raster, Rasterizer, Schedule, Trainer, require_cuda  # noqa: F401

__all__ = ["Rasterizer", "Raster", "SMOOTH", "Trainer", "Adam", "Schedule", "require_cuda"]
