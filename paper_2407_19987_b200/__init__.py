"""B200-native HOBOTAN hot path (arXiv 2407.19987): batched HOBO tensor contraction.

The package exposes the C ABI of include/hobo.h through a thin ctypes binding
(`hobo.HoboTensor`).  The CUDA library is built in-tree by `build.py`.
"""
from .hobo import HoboError, HoboTensor, lib  # noqa: F401
