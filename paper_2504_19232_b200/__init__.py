"""B200-native zero-bubble pipeline-parallel training step (Adaptra, arXiv 2504.19232).

The compute path is libadaptra.so (csrc/, C-ABI in include/adaptra.h); this
package is the thin Python binding and the torch-side driver (device memory,
streams, process groups).
"""
import os

# Streams that block on stream memory waits must not share a hardware channel
# with the streams that release them: give every stream its own connection.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# Load all kernels when the context is created: a kernel loaded lazily while a
# flag-wait kernel spins on the device can stall behind it (must be set before
# the CUDA driver initialises; bench.py and tests/conftest.py set it first).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

from . import _lib  # noqa: E402,F401

__all__ = ["_lib"]
