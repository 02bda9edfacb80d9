"""Reference-shaped host API: the hot-path surface of namespace parsim.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/include/parsim), so callers and the parity tests read
like the reference's own tests (proj/tests/test_compression.cpp,
test_collectives.cpp, test_strategies.cpp).  Vectors are CUDA tensors
(float64 for the reference's own precision, float32 for production); Python
sequences are accepted and become float64 CUDA tensors.  All arithmetic runs
in libpsb.so kernels; precondition failures raise ValueError subclasses, the
analogue of std::invalid_argument.

  compress_onebit          parsim/compression.hpp:67-77
  compress_topk            parsim/compression.hpp:81-99
  compress                 parsim/compression.hpp:101-111
  decompress               parsim/compression.hpp:113-142
  ef_compress_step         parsim/compression.hpp:146-157
  allreduce_mean           parsim/collectives.hpp:135-154
  sync_data_parallel_step  parsim/strategies.hpp:86-121
  async_step               parsim/strategies.hpp:125-129
  vec_axpy                 parsim/numerics.hpp:70-78
  StalenessTracker         parsim/strategies.hpp:65-77
  wire_encode/wire_decode  parsim/compression.hpp:159-239 (device codec, psb_wire.cu)
  compression_ratio(_for)  parsim/compression.hpp:243-271
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Union

import torch

from . import _lib as L
from .engine import Context, topology

Vector = Union[torch.Tensor, Sequence[float]]


class CompressorKind(enum.Enum):
    none = 0
    onebit = 1
    topk = 2


@dataclass
class CompressorConfig:
    kind: CompressorKind = CompressorKind.none
    top_k: int = 0


@dataclass
class DensePayload:
    values: torch.Tensor


@dataclass
class SignBitPayload:
    dim: int
    scale: float
    sign_bytes: torch.Tensor  # uint8 [ceil(dim/8)], bit i%8 of byte i/8, 1 = positive

    def positive_at(self, i: int) -> bool:
        return bool((int(self.sign_bytes[i // 8]) >> (i % 8)) & 1)


@dataclass
class TopKPayload:
    dim: int
    indices: torch.Tensor  # int64, strictly increasing
    values: torch.Tensor


@dataclass
class CompressedGradient:
    payload: Union[DensePayload, SignBitPayload, TopKPayload]

    def dim(self) -> int:
        p = self.payload
        return p.values.numel() if isinstance(p, DensePayload) else p.dim


@dataclass
class ErrorFeedbackState:
    residual: torch.Tensor

    @staticmethod
    def zeros(dim: int, dtype: torch.dtype = torch.float64) -> "ErrorFeedbackState":
        return ErrorFeedbackState(torch.zeros(dim, dtype=dtype, device="cuda"))


class CollectiveAlgorithm(enum.Enum):
    naive = "naive"
    ring = "ring"
    hierarchical = "hierarchical"
    pipelined_ring = "pipelined_ring"


@dataclass
class Topology:
    racks: int = 1
    nodes_per_rack: int = 1
    devices_per_node: int = 1
    intra_node_bw: float = 1.0
    inter_node_bw: float = 1.0
    inter_rack_bw: float = 1.0
    intra_node_lat: float = 0.0
    inter_node_lat: float = 0.0
    inter_rack_lat: float = 0.0

    def device_count(self) -> int:
        return self.racks * self.nodes_per_rack * self.devices_per_node


@dataclass
class WorkerGroup:
    buffers: List[Vector] = field(default_factory=list)

    def size(self) -> int:
        return len(self.buffers)

    def checked_dim(self) -> int:
        if not self.buffers:
            raise L.PsbInvalidArgument("WorkerGroup: no workers")
        dim = _numel(self.buffers[0])
        for b in self.buffers:
            if _numel(b) != dim:
                raise L.PsbInvalidArgument("WorkerGroup: dim mismatch across workers")
        return dim


class ExecutionMode(enum.Enum):
    sync = 0
    async_ = 1


@dataclass
class StrategyConfig:
    data_degree: int = 1
    tensor_degree: int = 1
    pipeline_stages: int = 1
    micro_batches: int = 1
    mode: ExecutionMode = ExecutionMode.sync
    collective: CollectiveAlgorithm = CollectiveAlgorithm.ring
    compressor: CompressorConfig = field(default_factory=CompressorConfig)
    overlap_fraction: float = 0.0


@dataclass
class HyperParams:
    learning_rate: float = 0.01
    batch_size: int = 1
    steps: int = 1

    def validate(self) -> None:
        if not self.learning_rate > 0.0:
            raise L.PsbInvalidArgument("HyperParams: learning_rate must be > 0")
        if self.batch_size < 1 or self.steps < 1:
            raise L.PsbInvalidArgument("HyperParams: counts must be >= 1")


class StalenessTracker:
    """Per-worker staleness bookkeeping (parsim/strategies.hpp:65-77)."""

    def __init__(self, workers: int):
        self._pulled = [0] * workers
        self._updates = 0

    def workers(self) -> int:
        return len(self._pulled)

    def staleness(self, p: int) -> int:
        return self._updates - self._pulled[p]

    def on_pull(self, p: int) -> None:
        self._pulled[p] = self._updates

    def on_global_update(self) -> None:
        self._updates += 1


# --------------------------------------------------------------- plumbing
_CTX: Dict[int, Context] = {}


def _ctx(n: int, k: int = 1, workers: int = 1) -> Context:
    dev = torch.cuda.current_device()
    c = _CTX.get(dev)
    if c is None or c.max_n < n or c.max_k < k or c.max_workers < workers:
        if c is not None:
            c.close()
        c = Context(max(n, 1 << 16), max(k, 1 << 12), max(workers, 16), dev)
        _CTX[dev] = c
    return c


def _numel(v: Vector) -> int:
    return v.numel() if isinstance(v, torch.Tensor) else len(v)


def as_vector(v: Vector, dtype: Optional[torch.dtype] = None) -> torch.Tensor:
    if isinstance(v, torch.Tensor):
        t = v if v.is_cuda else v.cuda()
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        return t.contiguous().view(-1)
    return torch.tensor(list(v), dtype=dtype or torch.float64, device="cuda")


def _algo(a: Union[CollectiveAlgorithm, str]) -> str:
    return a.value if isinstance(a, CollectiveAlgorithm) else str(a)


def _topo(t: Optional[Topology]):
    if t is None:
        return topology()
    if t.racks < 1 or t.nodes_per_rack < 1 or t.devices_per_node < 1:
        raise L.PsbInvalidArgument("Topology: counts must be >= 1")
    return topology(t.racks, t.nodes_per_rack, t.devices_per_node)


# ------------------------------------------------------------ compressors
def compress_onebit(g: Vector) -> CompressedGradient:
    gt = as_vector(g)
    if gt.numel() == 0:
        raise L.PsbInvalidArgument("compress_onebit: empty vector")
    c = _ctx(gt.numel())
    words, scale = c.ef_onebit(gt, None)
    c.check()
    nbytes = (gt.numel() + 7) // 8
    sign_bytes = words.view(torch.uint8)[:nbytes].clone()
    return CompressedGradient(SignBitPayload(gt.numel(), float(scale.item()), sign_bytes))


def compress_topk(g: Vector, k: int) -> CompressedGradient:
    gt = as_vector(g)
    n = gt.numel()
    if not (1 <= k <= n):
        raise L.PsbInvalidArgument(f"compress_topk: k out of range (k={k}, dim={n})")
    c = _ctx(n, k)
    idx, val = c.ef_topk(gt, None, k)
    c.check()
    return CompressedGradient(TopKPayload(n, idx.to(torch.int64) & 0xFFFFFFFF, val.clone()))


def compress(g: Vector, cfg: CompressorConfig) -> CompressedGradient:
    if cfg.kind == CompressorKind.none:
        return CompressedGradient(DensePayload(as_vector(g).clone()))
    if cfg.kind == CompressorKind.onebit:
        return compress_onebit(g)
    if cfg.kind == CompressorKind.topk:
        return compress_topk(g, cfg.top_k)
    raise L.PsbInvalidArgument("compress: unknown compressor kind")


def decompress(c: CompressedGradient) -> torch.Tensor:
    p = c.payload
    if isinstance(p, DensePayload):
        return p.values.clone()
    if isinstance(p, SignBitPayload):
        if p.sign_bytes.numel() != (p.dim + 7) // 8:
            raise L.PsbInvalidArgument("decompress: sign byte count does not match dim")
        # +-scale per sign bit on the device: the 1-bit mean kernel with one
        # worker (mean = value * (1/1), exact), as parsim_b200.hpp does
        nw = (p.dim + 31) // 32
        words = torch.zeros(nw * 4, dtype=torch.uint8, device="cuda")
        words[: p.sign_bytes.numel()] = p.sign_bytes.to(device="cuda", dtype=torch.uint8)
        scale = torch.tensor([p.scale], dtype=torch.float64, device="cuda")
        out = torch.empty(p.dim, dtype=torch.float64, device="cuda")
        ctx = _ctx(max(p.dim, 1))
        ctx.onebit_mean_sgd(words.view(torch.int32), scale, p.dim, torch.float64, "naive", 0.0, None, mean_out=out)
        ctx.check()
        return out
    if p.indices.numel() != p.values.numel():
        raise L.PsbInvalidArgument("decompress: index/value count mismatch")
    vals = as_vector(p.values)
    idx64 = p.indices.to(device="cuda", dtype=torch.int64)
    if idx64.numel() and (int(idx64.min()) < 0 or int(idx64.max()) >= p.dim):
        raise L.PsbInvalidArgument(f"decompress: index out of range for dim {p.dim}")
    ctx = _ctx(max(p.dim, 1), max(1, vals.numel()))
    out = ctx.decompress_topk(idx64.to(torch.int32), vals, p.dim)
    ctx.check()
    return out


def ef_compress_step(state: ErrorFeedbackState, g: Vector, cfg: CompressorConfig) -> CompressedGradient:
    gt = as_vector(g, state.residual.dtype)
    if state.residual.numel() != gt.numel():
        raise L.PsbInvalidArgument("ef_compress_step: residual/gradient dimension mismatch")
    n = gt.numel()
    if cfg.kind == CompressorKind.none:
        # p = r + g; msg = p; r' = p - p = +0  (compression.hpp:150-154)
        p = vec_axpy(1.0, state.residual, gt)  # 1.0*r + g == r + g exactly
        state.residual.sub_(state.residual).add_(p - p)
        return CompressedGradient(DensePayload(p))
    if cfg.kind == CompressorKind.topk:
        if not (1 <= cfg.top_k <= n):
            raise L.PsbInvalidArgument(f"compress_topk: k out of range (k={cfg.top_k}, dim={n})")
        c = _ctx(n, cfg.top_k)
        idx, val = c.ef_topk(gt, state.residual, cfg.top_k)
        c.check()
        return CompressedGradient(TopKPayload(n, idx.to(torch.int64) & 0xFFFFFFFF, val.clone()))
    if cfg.kind == CompressorKind.onebit:
        if n == 0:
            raise L.PsbInvalidArgument("compress_onebit: empty vector")
        c = _ctx(n)
        words, scale = c.ef_onebit(gt, state.residual)
        c.check()
        sign_bytes = words.view(torch.uint8)[: (n + 7) // 8].clone()
        return CompressedGradient(SignBitPayload(n, float(scale.item()), sign_bytes))
    raise L.PsbInvalidArgument("compress: unknown compressor kind")


# ------------------------------------------------------------ collectives
def allreduce_mean(group: WorkerGroup, algo: Union[CollectiveAlgorithm, str],
                   topo: Optional[Topology] = None) -> torch.Tensor:
    dim = group.checked_dim()
    bufs = torch.stack([as_vector(b) for b in group.buffers])
    P = bufs.shape[0]
    c = _ctx(max(dim, 1), 1, P)
    out = torch.empty(dim, dtype=bufs.dtype, device=bufs.device)
    t = _topo(topo) if topo is not None else topology(0, 0, 0)
    if dim:
        c.dense_mean_sgd(bufs, _algo(algo), 1.0, None, out, t)
        c.check()
    return out


def vec_axpy(a: float, x: Vector, y: Vector) -> torch.Tensor:
    xt, yt = as_vector(x), as_vector(y)
    if xt.numel() != yt.numel():
        raise L.PsbInvalidArgument(f"vec_axpy: dimension mismatch ({xt.numel()} vs {yt.numel()})")
    out = yt.to(xt.dtype).clone()
    if out.numel():
        c = _ctx(out.numel())
        c.dense_mean_sgd(xt.view(1, -1), "naive", -a, out)  # out = (-(-a)) * (x*1) + y
        c.check()
    return out


# ------------------------------------------------------------ strategies
def sync_data_parallel_step(workers: WorkerGroup, params: Vector, h: HyperParams,
                            cfg: StrategyConfig, topo: Optional[Topology] = None,
                            ef_states: Optional[List[ErrorFeedbackState]] = None) -> torch.Tensor:
    dim = workers.checked_dim()
    theta_in = as_vector(params)
    if dim != theta_in.numel():
        raise L.PsbInvalidArgument("sync_data_parallel_step: worker/param dim mismatch")
    h.validate()
    P = workers.size()
    dtype = theta_in.dtype
    g = torch.stack([as_vector(b, dtype) for b in workers.buffers])
    kind = cfg.compressor.kind
    if kind != CompressorKind.none and ef_states is not None and len(ef_states) != P:
        raise L.PsbInvalidArgument(
            "sync_data_parallel_step: one error-feedback state per worker required")
    r = None
    if kind != CompressorKind.none:
        if ef_states is None:
            r = torch.zeros_like(g)  # transient zero residuals (strategies.hpp:97-102)
        else:
            r = torch.stack([s.residual.to(dtype) for s in ef_states])
    comp = {CompressorKind.none: L.PSB_COMP_NONE, CompressorKind.onebit: L.PSB_COMP_ONEBIT,
            CompressorKind.topk: L.PSB_COMP_TOPK}[kind]
    k = cfg.compressor.top_k if kind == CompressorKind.topk else 0
    theta = theta_in.clone()
    c = _ctx(dim, max(k, 1), P)
    t = _topo(topo) if topo is not None else topology(0, 0, 0)
    desc = c.step_desc(comp, g, r, theta, h.learning_rate, k, _algo(cfg.collective), topo=t)
    c.sync_step(desc)
    c.check()
    if ef_states is not None and r is not None:
        for p, s in enumerate(ef_states):
            s.residual.copy_(r[p])
    return theta


def async_step(params: Vector, g_p: Vector, tau: int, eta: float) -> torch.Tensor:
    """params - eta/(1+tau) * g (scale computed in f64, strategies.hpp:127)."""
    scale = eta / (1.0 + float(tau))
    return vec_axpy(-scale, g_p, params)


# ------------------------------------------------------------ wire format
class WireKind(enum.Enum):
    """parsim/compression.hpp:211: the caller states which payload kind the bytes carry."""
    dense = 0
    signbit = 1
    topk = 2


def wire_encode(c: CompressedGradient) -> torch.Tensor:
    """parsim/compression.hpp:188-209: little-endian bytes (uint8 CUDA tensor), encoded on the device."""
    p = c.payload
    if isinstance(p, DensePayload):
        x = as_vector(p.values)
        return _ctx(x.numel()).wire_encode_dense(x)
    if isinstance(p, SignBitPayload):
        nw = (p.dim + 31) // 32
        words = torch.zeros(nw, dtype=torch.int32, device="cuda")
        words.view(torch.uint8)[:p.sign_bytes.numel()] = p.sign_bytes.to(device="cuda", dtype=torch.uint8)
        scale = torch.tensor([p.scale], dtype=torch.float64, device="cuda")
        return _ctx(p.dim).wire_encode_signbit(p.dim, words, scale)
    idx = p.indices.to(device="cuda", dtype=torch.int64)
    if idx.numel() and int(idx.max()) >= 1 << 32:
        raise L.PsbInvalidArgument("wire_encode: index exceeds the 32-bit range")
    vals = as_vector(p.values)
    c0 = _ctx(max(p.dim, 1), max(idx.numel(), 1))
    return c0.wire_encode_topk(p.dim, idx.to(torch.int32), vals)


def wire_decode(kind: WireKind, data: Union[torch.Tensor, bytes]) -> CompressedGradient:
    """parsim/compression.hpp:213-239; 'wire_decode: truncated input' on short data."""
    buf = data if isinstance(data, torch.Tensor) else torch.frombuffer(bytearray(data), dtype=torch.uint8)
    buf = buf.to(device="cuda", dtype=torch.uint8).contiguous()
    if kind == WireKind.topk:
        c0 = _ctx(1, max((buf.numel() - 16) // 16, 1))
        dim, idx, val = c0.wire_decode_topk(buf, torch.float64)
        return CompressedGradient(TopKPayload(dim, idx.to(torch.int64) & 0xFFFFFFFF, val))
    host = buf.cpu()
    if host.numel() < 8:
        raise L.PsbInvalidArgument("wire_decode: truncated input")
    dim = int(host[:8].view(torch.int64).item())
    if kind == WireKind.dense:
        if host.numel() < 8 + 8 * dim:
            raise L.PsbInvalidArgument("wire_decode: truncated input")
        return CompressedGradient(DensePayload(buf[8:8 + 8 * dim].view(torch.float64).clone()))
    if host.numel() < 16:
        raise L.PsbInvalidArgument("wire_decode: truncated input")
    scale = float(host[8:16].view(torch.float64).item())
    nb = (dim + 7) // 8
    if host.numel() < 16 + nb:
        raise L.PsbInvalidArgument("wire_decode: truncated sign bytes")
    return CompressedGradient(SignBitPayload(dim, scale, buf[16:16 + nb].clone()))


def compression_ratio(c: CompressedGradient) -> float:
    """parsim/compression.hpp:243-253: raw 8-byte entries over wire bytes."""
    p = c.payload
    dense = 8.0 * c.dim()
    if isinstance(p, DensePayload):
        return 1.0
    if isinstance(p, SignBitPayload):
        return dense / (8.0 + 8.0 + float((p.dim + 7) // 8))
    return dense / (8.0 + 8.0 + 16.0 * float(p.indices.numel()))


def compression_ratio_for(cfg: CompressorConfig, dim: int) -> float:
    """parsim/compression.hpp:256-271."""
    if dim < 1:
        raise L.PsbInvalidArgument("compression_ratio_for: dim must be >= 1")
    if cfg.kind == CompressorKind.none:
        return 1.0
    if cfg.kind == CompressorKind.onebit:
        return 8.0 * dim / (16.0 + float((dim + 7) // 8))
    if cfg.kind == CompressorKind.topk:
        k = min(cfg.top_k, dim)
        if k < 1:
            raise L.PsbInvalidArgument("compression_ratio_for: top_k must be >= 1")
        return 8.0 * dim / (16.0 + 16.0 * k)
    raise L.PsbInvalidArgument("compression_ratio_for: unknown compressor kind")


# The reference's alpha-beta model (collectives.hpp:156-215) lives in costmodel.py;
# forwarded here so `parsim.comm_cost` reads like the reference's namespace.
def comm_cost(algo, msg_bytes: float, P: int, topo: Topology, span_devices: int = 0) -> float:
    from .costmodel import comm_cost as f
    return f(algo, msg_bytes, P, topo, span_devices)


def slowest_link_spanning(topo: Topology, span_devices: int):
    from .costmodel import slowest_link_spanning as f
    return f(topo, span_devices)
