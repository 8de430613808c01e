"""B200-native separable rectangular morphology (erosion / dilation / opening / closing /
gradient, u8 and u16) and tile / image transposes -- the hot path of arxiv 2002.09474
("Fast Implementation of Morphological Filtering Using ARM NEON Extension") re-designed for
sm_100a, behind the reference ``rectmorph`` library's own entry points.

Native pieces (built in-tree by ``paper_2002_09474_b200.build``):
  librmgpu.so            CUDA kernels + the C-ABI of include/rmgpu.h
  librectmorph_b200.so   C++ drop-in (namespace rectmorph) on that C-ABI
"""
from .api import *  # noqa: F401,F403
from .api import (BorderPolicy, DispatchConfig, Errc, Error, GpuError, OpKind, PassAlgorithm,  # noqa: F401
                  StructuringElement, VerticalStrategy, Axis, make_se)
from ._native import LIB_PATH, HOSTLIB_PATH, lib  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
