"""ametro-b200: B200-native spatio-temporal dependency tracker of AI Metropolis
(arXiv 2411.03519) -- CUDA kernels for sm_100a behind the C ABI in include/am.h.

The package never imports ``oracle`` (the CPU oracle is test infrastructure only)
and has no CPU fallback: the ``Tracker`` and ``Replay`` classes raise if
libametro.so is not built.
"""
from ._lib import AmError, load, lib_path  # noqa: F401
from .tracker import Tracker, IDLE, RUNNING, DONE  # noqa: F401
from .driver import Replay  # noqa: F401

__all__ = ["Tracker", "Replay", "AmError", "load", "lib_path", "IDLE", "RUNNING", "DONE"]
