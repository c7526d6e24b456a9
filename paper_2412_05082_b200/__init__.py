"""B200-native vertex-patch Schwarz smoother for the C0IP biharmonic problem (arXiv 2412.05082).

The compute path is the C-ABI CUDA library libc0ip.so (include/c0ip.h); `api` is a thin
torch-tensor binding.  Importing `api` loads the library and raises if it is missing.
"""
from . import _lib  # noqa: F401

__all__ = ["api", "_lib"]
