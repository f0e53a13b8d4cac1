"""B200-native DARTS hot path (arXiv 2402.03106): transient volumetric path
tracing with residual-time sampling, as hand-written sm_100a CUDA behind the C
ABI of ``include/dts.h`` (``libdts.so``).  ``dts`` is the thin ctypes binding.
There is no CPU fallback: importing the binding without the built library, or
calling it without a CUDA device, raises."""
from . import dts  # noqa: F401

__all__ = ["dts"]
