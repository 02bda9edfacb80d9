"""Device-level host API over the C ABI (include/psb.h).

`Context` owns one psb_ctx (all scratch, the NCCL communicator) bound to one
CUDA device.  Tensors are torch CUDA tensors used purely as device memory;
every computation runs in libpsb.so kernels on the tensor's current stream.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple

import torch

from . import _lib as L

_DT = {torch.float32: L.PSB_F32, torch.float64: L.PSB_F64}
ORDERS = {"naive": L.PSB_ORDER_NAIVE, "ring": L.PSB_ORDER_RING,
          "pipelined_ring": L.PSB_ORDER_RING, "hierarchical": L.PSB_ORDER_HIER}
DISTS = {"uniform": L.PSB_DIST_UNIFORM, "llmrec": L.PSB_DIST_LLMREC, "ties": L.PSB_DIST_TIES}


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise L.PsbInvalidArgument(f"unsupported dtype {t.dtype}; expected float32 or float64")


def _need_cuda(*ts: Optional[torch.Tensor]) -> None:
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise L.PsbInvalidArgument("libpsb operates on contiguous CUDA tensors")


def topology(racks: int = 0, nodes_per_rack: int = 0, devices_per_node: int = 0) -> L.Topology:
    """psb_topology; all-zero means the flat topology (devices_per_node = P)."""
    return L.Topology(racks, nodes_per_rack, devices_per_node)


def payload_bytes(compressor: int, dtype: torch.dtype, k: int) -> int:
    return int(L.load().psb_payload_bytes(compressor, _DT[dtype], k))


def generate(dist: str, seed: int, rank: int, step: int, n: int, out: torch.Tensor) -> torch.Tensor:
    """Counter-based synthetic gradient (bit-identical to orc_generate)."""
    _need_cuda(out)
    lib = L.load()
    st = torch.cuda.current_stream(out.device).cuda_stream
    L.raise_for(lib.psb_generate(DISTS[dist], seed, rank, step, n, out.data_ptr(), st), None,
                "psb_generate")
    return out


class Context:
    """One psb_ctx: scratch for gradients up to max_n, top-k up to max_k and
    max_workers payloads per step (P = local workers x ranks)."""

    def __init__(self, max_n: int, max_k: int = 1, max_workers: int = 1,
                 device: Optional[int] = None):
        self.lib = L.load()
        if not torch.cuda.is_available():
            raise L.PsbError("libpsb needs a CUDA device (no CPU fallback)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.max_n, self.max_k, self.max_workers = int(max_n), int(max(1, max_k)), int(max_workers)
        h = ctypes.c_void_p()
        st = self.lib.psb_ctx_create(ctypes.byref(h), self.device, self.max_n, self.max_k,
                                     self.max_workers)
        if st != L.PSB_OK:
            L.raise_for(st, None, "psb_ctx_create")
        self.h = h
        self.rank, self.nranks = 0, 1

    # ----------------------------------------------------------- lifecycle
    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.psb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _ck(self, status: int, where: str) -> None:
        if status != L.PSB_OK:
            L.raise_for(status, self.h, where)

    def check(self) -> None:
        """Synchronize the current stream and raise on device-side errors."""
        self._ck(self.lib.psb_check(self.h, self.stream()), "psb_check")

    @property
    def launches(self) -> int:
        return int(self.lib.psb_launch_count(self.h))

    def topk_stats(self, worker: int = 0) -> dict:
        """Diagnostics of the last K1 call (psb_topk_stats)."""
        out = (ctypes.c_uint64 * 8)()
        self._ck(self.lib.psb_topk_stats(self.h, worker, out), "psb_topk_stats")
        import struct
        return {"candidates": int(out[0]), "k": int(out[1]), "threshold_key": int(out[2]),
                "ties_taken": int(out[3]), "predicted_valid": (int(out[4]) & 0xFF) == 0,
                "first_radix_level": int(out[4]) >> 8,
                "predicted_key": int(out[5]), "calls": int(out[6]) & 0xFFFFFFFF,
                "misses": int(out[6]) >> 32,
                "margin_f": struct.unpack("<f", struct.pack("<I", int(out[7]) & 0xFFFFFFFF))[0]}

    def topk_phases_us(self) -> list:
        """Durations (us) between the candidate-phase milestones of the last K1 call."""
        out = (ctypes.c_uint64 * 16)()
        self._ck(self.lib.psb_topk_phases(self.h, out), "psb_topk_phases")
        t = [int(x) for x in out]
        return [(t[i + 1] - t[i]) / 1e3 for i in range(15) if t[i + 1] >= t[i] > 0]

    def profile_enable(self, on: bool = True) -> None:
        self._ck(self.lib.psb_profile_enable(self.h, 1 if on else 0), "psb_profile_enable")

    def profile_read(self) -> Tuple[float, int]:
        """(summed ms, launches) of the K1 streaming pass since the last read."""
        ms, cnt = ctypes.c_double(), ctypes.c_uint64()
        self._ck(self.lib.psb_profile_read(self.h, ctypes.byref(ms), ctypes.byref(cnt)),
                 "psb_profile_read")
        return float(ms.value), int(cnt.value)

    def profile_read_phase(self, phase: int) -> Tuple[float, int]:
        """(summed ms, event pairs) of phase 1 (exchange) or 2 (apply) since the last read."""
        ms, cnt = ctypes.c_double(), ctypes.c_uint64()
        self._ck(self.lib.psb_profile_read_phase(self.h, phase, ctypes.byref(ms), ctypes.byref(cnt)),
                 "psb_profile_read_phase")
        return float(ms.value), int(cnt.value)

    # --------------------------------------------------------- communicator
    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        L.raise_for(L.load().psb_comm_unique_id(buf), None, "psb_comm_unique_id")
        return buf.raw

    def comm_init(self, rank: int, nranks: int, uid: Optional[bytes]) -> None:
        buf = ctypes.create_string_buffer(uid, 128) if uid is not None else None
        self._ck(self.lib.psb_comm_init(self.h, rank, nranks, buf), "psb_comm_init")
        self.rank, self.nranks = rank, nranks

    def allgather_(self, buf: torch.Tensor, bytes_per_rank: int) -> None:
        _need_cuda(buf)
        self._ck(self.lib.psb_allgather(self.h, buf.data_ptr(), bytes_per_rank, self.stream()),
                 "psb_allgather")

    def peer_mode(self, mode) -> None:
        """Multi-rank sparse exchange (psb_peer_mode): "auto" (5, default: direct
        for top-k f32/f64, pull for top-k int8), "direct" (4: the apply reads
        the peers' NVLink arenas in place), "pull" (1), "push" (3: K1 stores
        its payload into the peers' arenas), "shard" (2), "nccl" (0)."""
        m = {"auto": 5, "full": 5, "pull": 1, "push": 3, "shard": 2, "direct": 4, "nccl": 0, True: 5,
             False: 0}.get(mode, mode)
        self._ck(self.lib.psb_peer_mode(self.h, int(m)), "psb_peer_mode")

    @property
    def peer_active(self) -> bool:
        return bool(self.lib.psb_peer_active(self.h))

    # ---------------------------------------------------------- compressors
    def ef_topk(self, g: torch.Tensor, r: Optional[torch.Tensor], k: int, worker: int = 0,
                idx_out: Optional[torch.Tensor] = None,
                val_out: Optional[torch.Tensor] = None) -> Tuple[torch.Tensor, torch.Tensor]:
        """K1: p = r + g, top-k of |p| (ties -> lower index), r := sel ? +0 : p.
        Returns (idx int32 [k] holding u32 indices, val [k])."""
        _need_cuda(g, r)
        n = g.numel()
        if idx_out is None:
            idx_out = torch.empty(max(k, 1), dtype=torch.int32, device=g.device)
        if val_out is None:
            val_out = torch.empty(max(k, 1), dtype=g.dtype, device=g.device)
        self._ck(self.lib.psb_ef_topk(self.h, _dtype_code(g), worker, g.data_ptr(), _ptr(r), n, k,
                                      idx_out.data_ptr(), val_out.data_ptr(), self.stream()),
                 "ef_compress_step")
        return idx_out[:k], val_out[:k]

    def ef_topk_q8(self, g: torch.Tensor, r: Optional[torch.Tensor], k: int, worker: int = 0):
        _need_cuda(g, r)
        idx = torch.empty(k, dtype=torch.int32, device=g.device)
        codes = torch.empty(k, dtype=torch.int8, device=g.device)
        scales = torch.empty((k + 127) // 128, dtype=torch.float32, device=g.device)
        self._ck(self.lib.psb_ef_topk_q8(self.h, worker, g.data_ptr(), _ptr(r), g.numel(), k,
                                         idx.data_ptr(), codes.data_ptr(), scales.data_ptr(),
                                         self.stream()), "ef_compress_step(topk_q8)")
        return idx, codes, scales

    def ef_onebit(self, g: torch.Tensor, r: Optional[torch.Tensor]):
        """1-bit EF: returns (sign words int32 [ceil(n/32)], scale f64 device [1])."""
        _need_cuda(g, r)
        n = g.numel()
        words = torch.empty((n + 31) // 32, dtype=torch.int32, device=g.device)
        scale = torch.empty(1, dtype=torch.float64, device=g.device)
        self._ck(self.lib.psb_ef_onebit(self.h, _dtype_code(g), g.data_ptr(), _ptr(r), n,
                                        words.data_ptr(), scale.data_ptr(), self.stream()),
                 "ef_compress_step(onebit)")
        return words, scale

    def q8_quantize(self, x: torch.Tensor, r: Optional[torch.Tensor], block: int = 256):
        _need_cuda(x, r)
        n = x.numel()
        codes = torch.empty(n, dtype=torch.int8, device=x.device)
        scales = torch.empty((n + block - 1) // block, dtype=torch.float32, device=x.device)
        self._ck(self.lib.psb_q8_quantize(self.h, x.data_ptr(), _ptr(r), n, block,
                                          codes.data_ptr(), scales.data_ptr(), self.stream()),
                 "psb_q8_quantize")
        return codes, scales

    def q8_dequantize(self, codes: torch.Tensor, scales: torch.Tensor, block: int = 256):
        out = torch.empty(codes.numel(), dtype=torch.float32, device=codes.device)
        self._ck(self.lib.psb_q8_dequantize(self.h, codes.data_ptr(), scales.data_ptr(),
                                            codes.numel(), block, out.data_ptr(), self.stream()),
                 "psb_q8_dequantize")
        return out

    def decompress_topk(self, idx: torch.Tensor, val: torch.Tensor, n: int) -> torch.Tensor:
        out = torch.zeros(n, dtype=val.dtype, device=val.device)
        self._ck(self.lib.psb_decompress_topk(self.h, _dtype_code(val), _ptr(idx), _ptr(val),
                                              val.numel(), n, out.data_ptr(), self.stream()),
                 "decompress")
        return out

    # ----------------------------------------------------- gradient producer
    def bpr_gradient(self, theta: torch.Tensor, users: int, items: int, dim: int, user: torch.Tensor,
                     pos: torch.Tensor, neg: torch.Tensor, grad: Optional[torch.Tensor] = None,
                     want_loss: bool = True):
        """bpr_batch_gradient / bpr_batch_loss (parsim/trainer.hpp:98-138) on the device."""
        _need_cuda(theta, user, pos, neg, grad)
        if grad is None:
            grad = torch.empty_like(theta)
        loss = torch.zeros(1, dtype=torch.float64, device=theta.device) if want_loss else None
        B = user.numel()
        self._ck(self.lib.psb_bpr_gradient(self.h, _dtype_code(theta), theta.data_ptr(), users, items, dim,
                                           user.data_ptr(), pos.data_ptr(), neg.data_ptr(), B, grad.data_ptr(),
                                           _ptr(loss), self.stream()), "bpr_batch_gradient")
        return grad, loss

    def rank_candidates(self, theta: torch.Tensor, users: int, dim: int, rec_user: torch.Tensor,
                        rec_item: torch.Tensor, cands: torch.Tensor) -> torch.Tensor:
        """evaluate_topk's sampled ranks (trainer.hpp:307-312); cands [R][m] int32 (-1 = padding)."""
        _need_cuda(theta, rec_user, rec_item, cands)
        R = rec_user.numel()
        rank = torch.empty(R, dtype=torch.int32, device=theta.device)
        self._ck(self.lib.psb_rank_candidates(self.h, _dtype_code(theta), theta.data_ptr(), users, dim, R,
                                              rec_user.data_ptr(), rec_item.data_ptr(), cands.data_ptr(),
                                              cands.shape[1] if cands.dim() == 2 else 0, rank.data_ptr(),
                                              self.stream()), "evaluate_topk")
        return rank

    # ---------------------------------------------------------- wire format
    def wire_encode_topk(self, dim: int, idx: torch.Tensor, val: torch.Tensor) -> torch.Tensor:
        """parsim wire_encode(TopKPayload): u64 dim | u64 count | (u64 idx, f64 val) x count."""
        k = idx.numel()
        out = torch.empty(int(self.lib.psb_wire_bytes(L.PSB_WIRE_TOPK, dim, k)), dtype=torch.uint8,
                          device=val.device)
        self._ck(self.lib.psb_wire_encode_topk(self.h, _dtype_code(val), dim, _ptr(idx), _ptr(val), k,
                                               out.data_ptr(), self.stream()), "wire_encode")
        return out

    def wire_decode_topk(self, buf: torch.Tensor, dtype: torch.dtype = torch.float32, k_cap: Optional[int] = None):
        """parsim wire_decode(topk) -> (dim, idx u32, val); ValueError on truncated input."""
        cap = k_cap if k_cap is not None else max(0, (buf.numel() - 16) // 16)
        idx = torch.empty(max(cap, 1), dtype=torch.int32, device=buf.device)
        val = torch.empty(max(cap, 1), dtype=dtype, device=buf.device)
        dim, cnt = L._u64(0), L._sz(0)
        self._ck(self.lib.psb_wire_decode_topk(self.h, _DT[dtype], buf.data_ptr(), buf.numel(), cap,
                                               idx.data_ptr(), val.data_ptr(), ctypes.byref(dim),
                                               ctypes.byref(cnt), self.stream()), "wire_decode")
        return int(dim.value), idx[:cnt.value], val[:cnt.value]

    def wire_encode_signbit(self, dim: int, words: torch.Tensor, scale: torch.Tensor) -> torch.Tensor:
        out = torch.empty(int(self.lib.psb_wire_bytes(L.PSB_WIRE_SIGNBIT, dim, 0)), dtype=torch.uint8,
                          device=words.device)
        self._ck(self.lib.psb_wire_encode_signbit(self.h, dim, words.data_ptr(), scale.data_ptr(), out.data_ptr(),
                                                  self.stream()), "wire_encode")
        return out

    def wire_encode_dense(self, x: torch.Tensor) -> torch.Tensor:
        out = torch.empty(int(self.lib.psb_wire_bytes(L.PSB_WIRE_DENSE, x.numel(), 0)), dtype=torch.uint8,
                          device=x.device)
        self._ck(self.lib.psb_wire_encode_dense(self.h, _dtype_code(x), x.data_ptr(), x.numel(), out.data_ptr(),
                                                self.stream()), "wire_encode")
        return out

    # ------------------------------------------------------ aggregate+apply
    def sparse_mean_sgd(self, payloads: torch.Tensor, P: int, k: int, dtype: torch.dtype,
                        order: str, lr: float, theta: Optional[torch.Tensor], n: int,
                        mean_out: Optional[torch.Tensor] = None,
                        topo: Optional[L.Topology] = None,
                        compressor: int = L.PSB_COMP_TOPK) -> None:
        topo = topo or topology()
        self._ck(self.lib.psb_sparse_mean_sgd(self.h, compressor, _DT[dtype], P,
                                              payloads.data_ptr(), k, ORDERS[order],
                                              ctypes.byref(topo), lr, _ptr(theta), n,
                                              _ptr(mean_out), self.stream()), "sparse_mean_sgd")

    def sparse_async_apply(self, payloads: torch.Tensor, P: int, k: int, dtype: torch.dtype,
                           scales: Sequence[float], theta: torch.Tensor,
                           compressor: int = L.PSB_COMP_TOPK) -> None:
        arr = (ctypes.c_double * P)(*scales)
        self._ck(self.lib.psb_sparse_async_apply(self.h, compressor, _DT[dtype], P,
                                                 payloads.data_ptr(), k, arr, theta.data_ptr(),
                                                 theta.numel(), self.stream()), "async_apply")

    def dense_mean_sgd(self, bufs: torch.Tensor, order: str, lr: float,
                       theta: Optional[torch.Tensor], mean_out: Optional[torch.Tensor] = None,
                       topo: Optional[L.Topology] = None) -> None:
        _need_cuda(bufs, theta, mean_out)
        P, n = bufs.shape
        topo = topo or topology()
        self._ck(self.lib.psb_dense_mean_sgd(self.h, _dtype_code(bufs), P, bufs.data_ptr(),
                                             ORDERS[order], ctypes.byref(topo), lr, _ptr(theta),
                                             n, _ptr(mean_out), self.stream()), "allreduce_mean")

    def onebit_mean_sgd(self, words: torch.Tensor, scales: torch.Tensor, n: int,
                        dtype: torch.dtype, order: str, lr: float, theta: Optional[torch.Tensor],
                        mean_out: Optional[torch.Tensor] = None,
                        topo: Optional[L.Topology] = None) -> None:
        P = scales.numel()
        topo = topo or topology()
        self._ck(self.lib.psb_onebit_mean_sgd(self.h, _DT[dtype], P, words.data_ptr(),
                                              scales.data_ptr(), ORDERS[order], ctypes.byref(topo),
                                              lr, _ptr(theta), n, _ptr(mean_out), self.stream()),
                 "onebit_mean_sgd")

    # ------------------------------------------------------------- drivers
    def step_desc(self, compressor: int, g: torch.Tensor, r: Optional[torch.Tensor],
                  theta: torch.Tensor, lr: float, k: int = 0, order: str = "naive",
                  q8_block: int = 256, topo: Optional[L.Topology] = None,
                  mean_out: Optional[torch.Tensor] = None, momentum: Optional[torch.Tensor] = None,
                  beta: float = 0.0) -> L.StepDesc:
        """psb_step_desc; momentum (a persistent [n] buffer) with factor beta
        turns the update into momentum SGD (see include/psb.h)."""
        _need_cuda(g, r, theta, mean_out, momentum)
        W = g.shape[0] if g.dim() == 2 else 1
        n = g.shape[-1]
        # the C ABI sees bare pointers: every buffer must have g's dtype and
        # the shape the step writes through (theta/mean/m: [n], r: [W][n])
        for name, t, numel in (("theta", theta, n), ("mean_out", mean_out, n), ("momentum", momentum, n),
                               ("r", r, W * n)):
            if t is None:
                continue
            if t.dtype != g.dtype:
                raise L.PsbInvalidArgument(f"step_desc: {name} dtype {t.dtype} != gradient dtype {g.dtype}")
            if t.numel() != numel:
                raise L.PsbInvalidArgument(f"step_desc: {name} has {t.numel()} elements, expected {numel}")
        if r is not None and r.dim() == 2 and tuple(r.shape) != (W, n):
            raise L.PsbInvalidArgument(f"step_desc: r shape {tuple(r.shape)} != ({W}, {n})")
        d = L.StepDesc()
        d.compressor = compressor
        d.dtype = _dtype_code(g)
        d.n, d.k, d.q8_block, d.workers = n, k, q8_block, W
        d.g, d.r, d.theta = g.data_ptr(), _ptr(r), theta.data_ptr()
        d.lr = lr
        d.order = ORDERS[order]
        d.topo = topo or topology()
        d.mean_out = _ptr(mean_out)
        d.m = _ptr(momentum)
        d.beta = beta
        return d

    def sync_step(self, desc: L.StepDesc) -> None:
        self._ck(self.lib.psb_sync_step(self.h, ctypes.byref(desc), self.stream()),
                 "sync_data_parallel_step")

    def async_pipeline(self, enable: bool = True) -> None:
        """psb_async_pipeline: round r's exchange + apply on a ctx stream,
        overlapping round r+1's compression; theta trails the current stream
        by up to one round until async_sync()."""
        self._ck(self.lib.psb_async_pipeline(self.h, 1 if enable else 0), "psb_async_pipeline")

    def async_sync(self) -> None:
        """Make the current stream wait for every pending pipelined apply."""
        self._ck(self.lib.psb_async_sync(self.h, self.stream()), "psb_async_sync")

    def async_round(self, desc: L.StepDesc, staleness_bound: int, global_updates: int) -> int:
        gu = ctypes.c_uint64(global_updates)
        self._ck(self.lib.psb_async_round(self.h, ctypes.byref(desc), staleness_bound,
                                          ctypes.byref(gu), self.stream()), "async_round")
        return int(gu.value)
