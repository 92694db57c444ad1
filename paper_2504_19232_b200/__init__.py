"""B200-native zero-bubble pipeline-parallel training step (Adaptra, arXiv 2504.19232).

The compute path is libadaptra.so (csrc/, C-ABI in include/adaptra.h); this
package is the thin Python binding and the torch-side driver (device memory,
streams, process groups).
"""
from . import _lib  # noqa: F401

__all__ = ["_lib"]
