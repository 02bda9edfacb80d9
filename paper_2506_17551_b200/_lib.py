"""ctypes binding of the C ABI in include/psb.h (libpsb.so, built in-tree).

The library is the product: there is no CPU or Python fallback.  Importing this
module without the built library, or calling into it without a CUDA device,
raises immediately.
"""
from __future__ import annotations

import ctypes
import os

import torch  # noqa: F401  (loads the NCCL/cudart the library links against first)

_HERE = os.path.dirname(os.path.abspath(__file__))
# PSB_LIB: an alternative build of the same library (diagnostics builds such
# as libpsb_trace.so from tools/); the product path is libpsb.so
LIB_PATH = os.path.join(_HERE, os.environ.get("PSB_LIB") or "libpsb.so")

# psb_status
PSB_OK, PSB_EINVAL, PSB_ENONFINITE, PSB_ECUDA, PSB_ENCCL, PSB_ENOMEM, PSB_ESTATE = range(7)
# psb_dtype
PSB_F32, PSB_F64 = 0, 1
# psb_order
PSB_ORDER_NAIVE, PSB_ORDER_RING, PSB_ORDER_HIER = 0, 1, 2
# psb_compressor
PSB_COMP_NONE, PSB_COMP_ONEBIT, PSB_COMP_TOPK, PSB_COMP_TOPK_Q8, PSB_COMP_Q8 = range(5)
# psb_dist
PSB_DIST_UNIFORM, PSB_DIST_LLMREC, PSB_DIST_TIES = 0, 1, 2


class PsbError(RuntimeError):
    """CUDA / NCCL / state error reported by libpsb."""


class PsbInvalidArgument(ValueError):
    """Precondition failure; the reference throws std::invalid_argument here
    (parsim/numerics.hpp:20-26)."""


class PsbNonFinite(PsbInvalidArgument):
    """Non-finite residual or parameter (reference: check_finite ->
    std::invalid_argument, parsim/numerics.hpp:57-61)."""


class Topology(ctypes.Structure):
    _fields_ = [("racks", ctypes.c_uint32), ("nodes_per_rack", ctypes.c_uint32),
                ("devices_per_node", ctypes.c_uint32)]


class StepDesc(ctypes.Structure):
    _fields_ = [
        ("compressor", ctypes.c_int),
        ("dtype", ctypes.c_int),
        ("n", ctypes.c_size_t),
        ("k", ctypes.c_size_t),
        ("q8_block", ctypes.c_uint32),
        ("workers", ctypes.c_int),
        ("g", ctypes.c_void_p),
        ("r", ctypes.c_void_p),
        ("theta", ctypes.c_void_p),
        ("lr", ctypes.c_double),
        ("order", ctypes.c_int),
        ("topo", Topology),
        ("mean_out", ctypes.c_void_p),
        ("m", ctypes.c_void_p),
        ("beta", ctypes.c_double),
    ]


PSB_WIRE_DENSE, PSB_WIRE_SIGNBIT, PSB_WIRE_TOPK = 0, 1, 2

_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_i = ctypes.c_int
_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64
_d = ctypes.c_double

_SIGS = {
    "psb_abi_version": (_i, []),
    "psb_status_string": (ctypes.c_char_p, [_i]),
    "psb_ctx_create": (_i, [ctypes.POINTER(_vp), _i, _sz, _sz, _i]),
    "psb_ctx_destroy": (None, [_vp]),
    "psb_last_error": (ctypes.c_char_p, [_vp]),
    "psb_check": (_i, [_vp, _vp]),
    "psb_launch_count": (_u64, [_vp]),
    "psb_payload_bytes": (_sz, [_i, _i, _sz]),
    "psb_topk_stats": (_i, [_vp, _i, ctypes.POINTER(_u64)]),
    "psb_topk_phases": (_i, [_vp, ctypes.POINTER(_u64)]),
    "psb_profile_enable": (_i, [_vp, _i]),
    "psb_profile_read": (_i, [_vp, ctypes.POINTER(_d), ctypes.POINTER(_u64)]),
    "psb_comm_unique_id": (_i, [_vp]),
    "psb_comm_init": (_i, [_vp, _i, _i, _vp]),
    "psb_comm_rank": (_i, [_vp]),
    "psb_comm_size": (_i, [_vp]),
    "psb_allgather": (_i, [_vp, _vp, _sz, _vp]),
    "psb_peer_mode": (_i, [_vp, _i]),
    "psb_peer_active": (_i, [_vp]),
    "psb_generate": (_i, [_i, _u64, _u32, _u32, _sz, _vp, _vp]),
    "psb_ef_topk": (_i, [_vp, _i, _i, _vp, _vp, _sz, _sz, _vp, _vp, _vp]),
    "psb_ef_topk_q8": (_i, [_vp, _i, _vp, _vp, _sz, _sz, _vp, _vp, _vp, _vp]),
    "psb_ef_onebit": (_i, [_vp, _i, _vp, _vp, _sz, _vp, _vp, _vp]),
    "psb_q8_quantize": (_i, [_vp, _vp, _vp, _sz, _u32, _vp, _vp, _vp]),
    "psb_q8_dequantize": (_i, [_vp, _vp, _vp, _sz, _u32, _vp, _vp]),
    "psb_decompress_topk": (_i, [_vp, _i, _vp, _vp, _sz, _sz, _vp, _vp]),
    "psb_wire_bytes": (_sz, [_i, _u64, _sz]),
    "psb_momentum_sgd": (_i, [_vp, _i, _vp, _vp, _vp, _d, _d, _sz, _vp]),
    "psb_bpr_gradient": (_i, [_vp, _i, _vp, _u32, _u32, _u32, _vp, _vp, _vp, _u32, _vp, _vp, _vp]),
    "psb_rank_candidates": (_i, [_vp, _i, _vp, _u32, _u32, _u32, _vp, _vp, _vp, _u32, _vp, _vp]),
    "psb_wire_encode_topk": (_i, [_vp, _i, _u64, _vp, _vp, _sz, _vp, _vp]),
    "psb_wire_decode_topk": (_i, [_vp, _i, _vp, _sz, _sz, _vp, _vp, ctypes.POINTER(_u64), ctypes.POINTER(_sz),
                                  _vp]),
    "psb_wire_encode_signbit": (_i, [_vp, _u64, _vp, _vp, _vp, _vp]),
    "psb_wire_encode_dense": (_i, [_vp, _i, _vp, _u64, _vp, _vp]),
    "psb_sparse_mean_sgd": (_i, [_vp, _i, _i, _i, _vp, _sz, _i, ctypes.POINTER(Topology), _d, _vp,
                                 _sz, _vp, _vp]),
    "psb_sparse_async_apply": (_i, [_vp, _i, _i, _i, _vp, _sz, ctypes.POINTER(_d), _vp, _sz, _vp]),
    "psb_dense_mean_sgd": (_i, [_vp, _i, _i, _vp, _i, ctypes.POINTER(Topology), _d, _vp, _sz, _vp,
                                _vp]),
    "psb_onebit_mean_sgd": (_i, [_vp, _i, _i, _vp, _vp, _i, ctypes.POINTER(Topology), _d, _vp, _sz,
                                 _vp, _vp]),
    "psb_sync_step": (_i, [_vp, ctypes.POINTER(StepDesc), _vp]),
    "psb_async_round": (_i, [_vp, ctypes.POINTER(StepDesc), _u32, ctypes.POINTER(_u64), _vp]),
    "psb_profile_read_phase": (_i, [_vp, _i, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_u64)]),
    "psb_async_pipeline": (_i, [_vp, _i]),
    "psb_async_sync": (_i, [_vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load() -> ctypes.CDLL:
    """Load libpsb.so (once).  Fails loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (make -C paper_2506_17551_b200/csrc).  There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.psb_abi_version() != 1:
        raise ImportError("libpsb.so ABI version mismatch")
    _lib = lib
    return lib


def raise_for(status: int, ctx_ptr=None, where: str = "") -> None:
    if status == PSB_OK:
        return
    lib = load()
    msg = ""
    if ctx_ptr:
        raw = lib.psb_last_error(ctx_ptr)
        msg = raw.decode() if raw else ""
    if not msg:
        msg = lib.psb_status_string(status).decode()
    if where:
        msg = f"{where}: {msg}" if msg and not msg.startswith(where) else msg
    if status == PSB_ENONFINITE:
        raise PsbNonFinite(msg)
    if status == PSB_EINVAL:
        raise PsbInvalidArgument(msg)
    raise PsbError(f"[status {status}] {msg}")
