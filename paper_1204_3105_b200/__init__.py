"""B200-native FMM for the complex log kernel of arXiv:1204.3105 (quadtree / septree /
triangle-quadtree), behind the C ABI of include/fmm_b200.h.

This module is argument marshalling only: every step of the path runs in the
CUDA kernels of libfmm_b200.so.  There is no CPU fallback; importing the
binding without the built library raises.
"""
from .native import (  # noqa: F401
    Comm,
    Config,
    FmmError,
    Tree,
    X,
    lib,
    library_path,
    QUADTREE,
    SEPTREE,
    TRIQUAD,
    UnitCosts,
    choose_depth,
    direct,
    nccl_version,
    predict_cost,
    sample_cells,
)

__all__ = ["Comm", "nccl_version", "Config", "FmmError", "Tree", "UnitCosts", "X", "choose_depth", "direct", "lib", "predict_cost", "sample_cells", "library_path", "QUADTREE", "SEPTREE", "TRIQUAD"]
