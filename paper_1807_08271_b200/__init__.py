"""B200-native RGBiD-SLAM front-end hot path (arXiv 1807.08271).

Dense inverse-depth photometric + geometric IRLS alignment and keyframe fusion
as hand-written sm_100a CUDA kernels behind a C-ABI (include/rgbid_b200.h);
``rgbid`` mirrors the reference's ``namespace rgbid`` entry points.
"""
from . import abi  # noqa: F401
from .rgbid import *  # noqa: F401,F403

__all__ = [n for n in dir() if not n.startswith("_")]
