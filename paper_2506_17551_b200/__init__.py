"""B200-native data-parallel gradient path of arXiv 2506.17551.

compress (EF top-k / 1-bit / 8-bit) -> aggregate (NVLink peer exchange or
NCCL) -> apply (fused scatter-mean + SGD), behind the reference's parsim
interface.  All compute is in libpsb.so (sm_100a kernels); the modules here
are host bindings:

  _lib       ctypes binding of include/psb.h (loads libpsb.so; no CPU fallback)
  engine     Context: device-level API over the C ABI, including the sync
             step, the async rounds and their stream/event pipeline
             (Context.async_pipeline / async_sync -> psb_async_pipeline)
  parsim     reference-shaped API (same names/semantics as namespace parsim)
  dist       NCCL communicator bootstrap over torch.distributed
  train      the reference trainer around the device path (BPR producer)
  costmodel  the reference's alpha-beta model and the measured B200 step model
"""
from ._lib import PsbError, PsbInvalidArgument, PsbNonFinite, LIB_PATH, load  # noqa: F401

__all__ = ["PsbError", "PsbInvalidArgument", "PsbNonFinite", "LIB_PATH", "load"]
