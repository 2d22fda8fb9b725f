"""paper_2406_06911_b200 -- B200-native AsyncDiff (arXiv 2406.06911) async denoising engine.

The product is libasyncdiff_b200.so (hand-written sm_100a CUDA kernels + a C++
executor behind the C ABI in include/asyncdiff_b200.h).  This package is the
host-side mirror of the reference's pipeline API over that ABI (asyncdiff.py).
"""
from . import asyncdiff  # noqa: F401
from .asyncdiff import *  # noqa: F401,F403
from ._lib import SO_PATH, lib  # noqa: F401

__version__ = "0.1.0"
