"""paper_1105_4002_b200 — libtvreg, a B200-native hot path for accelerated-gradient TV CT
reconstruction (Jorgensen et al., arXiv:1105.4002).

The product is the C-ABI shared library ``libtvreg.so`` (include/libtvreg.h) with hand-written
sm_100a CUDA kernels; :mod:`paper_1105_4002_b200.tvreg` is its thin ctypes binding.
"""
from . import tvreg  # noqa: F401
from .tvreg import Problem, TVRError, lib  # noqa: F401

__all__ = ["tvreg", "Problem", "TVRError", "lib"]
