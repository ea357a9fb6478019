"""B200-native LLM-as-operator executor (Helium, arXiv 2603.16104 hot path).

Host C++ executor + sm_100a CUDA kernels behind the C-ABI in
include/helium_b200.h; this package holds the sources (csrc/), the in-tree
build (build.py -> libhelium_b200.so), and thin ctypes mirrors of the
reference interfaces (helios.py, engine.py).
"""
from . import _lib  # noqa: F401

__all__ = ["helios", "engine", "workloads", "models"]
