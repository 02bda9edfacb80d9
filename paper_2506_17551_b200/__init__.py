"""B200-native data-parallel gradient path of arXiv 2506.17551.

compress (EF top-k / 1-bit / 8-bit) -> aggregate (NCCL over NVLink) -> apply
(fused scatter-mean + SGD), behind the reference's parsim interface.

  _lib      ctypes binding of include/psb.h (libpsb.so, sm_100a kernels)
  engine    Context: device-level API over the C ABI
  parsim    reference-shaped API (same names/semantics as namespace parsim)
  scheduler sync / bounded-staleness async step drivers (streams + events)
"""
from ._lib import PsbError, PsbInvalidArgument, PsbNonFinite, LIB_PATH, load  # noqa: F401

__all__ = ["PsbError", "PsbInvalidArgument", "PsbNonFinite", "LIB_PATH", "load"]
