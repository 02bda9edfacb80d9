"""ctypes/numpy front-end of the CPU oracle.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference legs -- never by the product package.

Two libraries:
  oracle/build/libpsb_oracle.so   C restatement (psb_oracle.c), always built
  oracle/_ref/libparsim_ref.so    the unmodified reference headers behind
                                  ref_shim.cpp (built where /root/reference
                                  exists; the built .so travels to the GPU box)
Composite reference semantics (sync step, async round, q8 all-reduce) are
assembled here from the C primitives, each citing the reference lines.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libpsb_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libparsim_ref.so")

_P = ctypes.c_void_p
_SZ = ctypes.c_size_t
_D = ctypes.c_double
_U32 = ctypes.c_uint32
_U64 = ctypes.c_uint64
_I = ctypes.c_int

ORDERS = {"naive": 0, "ring": 1, "pipelined_ring": 1, "hierarchical": 2}
REF_ALGOS = {"naive": 0, "ring": 1, "hierarchical": 2, "pipelined_ring": 3}
DISTS = {"uniform": 0, "llmrec": 1, "ties": 2}

_orc = None
_ref = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def orc() -> ctypes.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = ctypes.CDLL(ORACLE_SO)
        sig = {
            "orc_mix64": (_U64, [_U64]),
            "orc_splitmix_stream": (None, [_U64, _SZ, _P]),
            "orc_generate": (None, [_I, _U64, _U32, _U32, _SZ, _P]),
            "orc_topk_f32": (_I, [_P, _SZ, _SZ, _P, _P]),
            "orc_topk_f64": (_I, [_P, _SZ, _SZ, _P, _P]),
            "orc_ef_topk_f32": (_I, [_P, _P, _SZ, _SZ, _P, _P]),
            "orc_ef_topk_f64": (_I, [_P, _P, _SZ, _SZ, _P, _P]),
            "orc_ef_onebit_f32": (_I, [_P, _P, _SZ, _P, _P]),
            "orc_ef_onebit_f64": (_I, [_P, _P, _SZ, _P, _P]),
            "orc_fold_mean_f32": (_I, [_I, _I, _SZ, _P, _U32, _U32, _P]),
            "orc_fold_mean_f64": (_I, [_I, _I, _SZ, _P, _U32, _U32, _P]),
            "orc_axpy_f32": (_I, [_D, _P, _P, _SZ]),
            "orc_axpy_f64": (_I, [_D, _P, _P, _SZ]),
            "orc_async_scale": (_D, [_D, _U64]),
            "orc_q8_quant": (_I, [_P, _P, _SZ, _U32, _P, _P]),
            "orc_q8_dequant": (None, [_P, _P, _SZ, _U32, _P]),
            "orc_momentum_f32": (None, [_P, _P, _P, _D, _D, _SZ]),
            "orc_momentum_f64": (None, [_P, _P, _P, _D, _D, _SZ]),
            "orc_wire_encode_topk": (_SZ, [_U64, _P, _P, _SZ, _P]),
            "orc_wire_decode_topk": (ctypes.c_longlong, [_P, _SZ, _P, _P, _P]),
            "orc_wire_encode_signbit": (_SZ, [_U64, _D, _P, _P]),
            "orc_wire_encode_dense": (_SZ, [_U64, _P, _P]),
        }
        for k, (res, args) in sig.items():
            f = getattr(lib, k)
            f.restype, f.argtypes = res, args
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> ctypes.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (reference headers unavailable)")
        lib = ctypes.CDLL(REF_SO)
        sig = {
            "ref_last_error": (ctypes.c_char_p, []),
            "ref_splitmix_stream": (_I, [_U64, _SZ, _P]),
            "ref_uniform_stream": (_I, [_U64, _SZ, _D, _D, _P]),
            "ref_compress_topk": (_I, [_P, _SZ, _SZ, _P, _P]),
            "ref_compress_onebit": (_I, [_P, _SZ, _P, _P]),
            "ref_ef_compress_step": (_I, [_I, _SZ, _P, _P, _SZ, _P, _P, _P, _P]),
            "ref_allreduce_mean": (_I, [_I, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _P]),
            "ref_sync_step": (_I, [_I, _SZ, _I, _SZ, _P, _P, _SZ, _D, _P, _SZ, _SZ, _SZ]),
            "ref_sync_step_threaded": (_I, [_I, _SZ, _I, _SZ, _P, _P, _SZ, _D, _P, _I]),
            "ref_async_step": (_I, [_P, _P, _SZ, _SZ, _D, _P]),
            "ref_vec_axpy": (_I, [_D, _P, _P, _SZ, _P]),
            "ref_decompress_topk": (_I, [_SZ, _P, _P, _SZ, _P]),
            "ref_wire_encode_topk": (_SZ, [_U64, _P, _P, _SZ, _P]),
            "ref_wire_decode_topk": (ctypes.c_longlong, [_P, _SZ, _P, _P, _P]),
            "ref_wire_encode_onebit": (_SZ, [_P, _SZ, _P]),
            "ref_bpr_batch_gradient": (_I, [_P, _SZ, _SZ, _SZ, _P, _P, _P, _SZ, _P, _P]),
            "ref_evaluate_topk": (_I, [_SZ, _SZ, _SZ, _P, _P, _P, _SZ, _P, _P, _SZ, _P, _P, _SZ, _SZ, _SZ, _U64, _P]),
            "ref_load_model": (_I, [ctypes.c_char_p, _P, _P, _SZ]),
            "ref_comm_cost": (_I, [_I, _D, _SZ, _P, _P, _SZ, _P]),
            "ref_synthetic_split": (_I, [_SZ, _SZ, _SZ, _U64, _P, _P, _P, _P, _P, _P, _P]),
            "ref_train": (_I, [_SZ, _SZ, _SZ, _P, _P, _SZ, _SZ, _I, _SZ, _SZ, _D, _I, _SZ, _I, _U64, _U64, _P, _P, _SZ,
                               _P]),
        }
        for k, (res, args) in sig.items():
            f = getattr(lib, k)
            f.restype, f.argtypes = res, args
        _ref = lib
    return _ref


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class RefError(ValueError):
    pass


def _ref_ck(st: int) -> None:
    if st:
        raise RefError(ref().ref_last_error().decode())


# ------------------------------------------------------------- generator
def mix64(z: int) -> int:
    return int(orc().orc_mix64(z))


def splitmix_stream(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    orc().orc_splitmix_stream(seed, n, _p(out))
    return out


def seeded_uniform(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    """SeededRng(seed).uniform(lo, hi) x n (parsim/numerics.hpp:165-167)."""
    u = splitmix_stream(seed, n)
    d = (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return lo + (hi - lo) * d


def generate(dist: str, seed: int, rank: int, step: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    orc().orc_generate(DISTS[dist], seed, rank, step, n, _p(out))
    return out


# ----------------------------------------------------------- compressors
def topk(x: np.ndarray, k: int) -> Tuple[np.ndarray, np.ndarray]:
    """compress_topk restated (compression.hpp:81-99)."""
    x = np.ascontiguousarray(x)
    idx = np.empty(k, dtype=np.uint32)
    val = np.empty(k, dtype=x.dtype)
    f = orc().orc_topk_f64 if x.dtype == np.float64 else orc().orc_topk_f32
    if f(_p(x), x.size, k, _p(idx), _p(val)):
        raise ValueError(f"compress_topk: k out of range (k={k}, dim={x.size})")
    return idx, val


def ef_topk(g: np.ndarray, r: Optional[np.ndarray], k: int) -> Tuple[np.ndarray, np.ndarray, int]:
    """ef_compress_step(topk) restated; r updated in place.  Returns (idx, val, status)."""
    idx = np.empty(k, dtype=np.uint32)
    val = np.empty(k, dtype=g.dtype)
    f = orc().orc_ef_topk_f64 if g.dtype == np.float64 else orc().orc_ef_topk_f32
    st = f(_p(g), _p(r), g.size, k, _p(idx), _p(val))
    if st == 1:
        raise ValueError(f"compress_topk: k out of range (k={k}, dim={g.size})")
    return idx, val, st


def ef_onebit(g: np.ndarray, r: Optional[np.ndarray]) -> Tuple[np.ndarray, float, int]:
    words = np.empty((g.size + 31) // 32, dtype=np.uint32)
    scale = np.empty(1, dtype=np.float64)
    f = orc().orc_ef_onebit_f64 if g.dtype == np.float64 else orc().orc_ef_onebit_f32
    st = f(_p(g), _p(r), g.size, _p(words), _p(scale))
    return words, float(scale[0]), st


def fold_mean(bufs: np.ndarray, order: str, dpn: int = 0, npr: int = 1) -> np.ndarray:
    """allreduce_mean in the reference's canonical orders (collectives.hpp:68-128).
    dpn == 0 means the flat topology (devices_per_node = P)."""
    bufs = np.ascontiguousarray(bufs)
    P, n = bufs.shape
    out = np.empty(n, dtype=bufs.dtype)
    f = orc().orc_fold_mean_f64 if bufs.dtype == np.float64 else orc().orc_fold_mean_f32
    st = f(ORDERS[order], P, n, _p(bufs), dpn or P, npr, _p(out))
    if st:
        raise ValueError("fold_mean: bad arguments")
    return out


def axpy_(a: float, x: np.ndarray, y: np.ndarray) -> int:
    """y := a*x + y (vec_axpy, numerics.hpp:70-78), in place; returns status."""
    f = orc().orc_axpy_f64 if y.dtype == np.float64 else orc().orc_axpy_f32
    return f(a, _p(np.ascontiguousarray(x)), _p(y), y.size)


def q8_quant(x: np.ndarray, r: Optional[np.ndarray], block: int):
    codes = np.empty(x.size, dtype=np.int8)
    scales = np.empty((x.size + block - 1) // block, dtype=np.float32)
    st = orc().orc_q8_quant(_p(x), _p(r), x.size, block, _p(codes), _p(scales))
    return codes, scales, st


def q8_dequant(codes: np.ndarray, scales: np.ndarray, block: int) -> np.ndarray:
    out = np.empty(codes.size, dtype=np.float32)
    orc().orc_q8_dequant(_p(codes), _p(scales), codes.size, block, _p(out))
    return out


def decompress_topk(idx: np.ndarray, val: np.ndarray, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=val.dtype)
    out[idx.astype(np.int64)] = val
    return out


def ef_topk_q8(g: np.ndarray, r: Optional[np.ndarray], k: int):
    """Top-k with int8 values (unpinned spec, psb.h psb_ef_topk_q8): select as
    ef_topk, quantize the k values in blocks of 128 with orc_q8_quant, and set
    the residual at selected indices to p - code*scale."""
    p = g.copy() if r is None else (r + g).astype(np.float32)
    idx, val = topk(p, k)
    codes, scales, _ = q8_quant(val, None, 128)
    if r is not None:
        r[:] = p
        xhat = q8_dequant(codes, scales, 128)
        r[idx.astype(np.int64)] = (val - xhat).astype(np.float32)
    return idx, codes, scales


# ------------------------------------------------------------- composites
def sync_step(grads: np.ndarray, theta: np.ndarray, lr: float, comp: str, k: int = 0,
              order: str = "naive", residuals: Optional[np.ndarray] = None, dpn: int = 0,
              npr: int = 1, q8_block: int = 256) -> np.ndarray:
    """sync_data_parallel_step (strategies.hpp:86-113) assembled from the
    restated primitives: per-worker EF compression, decompress, fold in the
    configured order, vec_axpy(-lr).  theta updated in place; returns mean."""
    P, n = grads.shape
    dt = grads.dtype
    if comp == "none":
        mean = fold_mean(grads, order, dpn, npr)
    elif comp in ("topk", "topk_q8"):
        dec = np.zeros((P, n), dtype=dt)
        for p in range(P):
            r = residuals[p] if residuals is not None else None
            if comp == "topk":
                idx, val, _ = ef_topk(grads[p], r, k)
                dec[p, idx.astype(np.int64)] = val
            else:
                idx, codes, scales = ef_topk_q8(grads[p], r, k)
                dec[p, idx.astype(np.int64)] = q8_dequant(codes, scales, 128)
        mean = fold_mean(dec, order, dpn, npr)
    elif comp == "onebit":
        dec = np.zeros((P, n), dtype=dt)
        for p in range(P):
            r = residuals[p] if residuals is not None else None
            words, scale, _ = ef_onebit(grads[p], r)
            s = dt.type(scale)
            bits = (words.view(np.uint8)[:, None] >> np.arange(8, dtype=np.uint8)) & 1
            pos = bits.reshape(-1)[:n].astype(bool)
            dec[p] = np.where(pos, s, -s)
        mean = fold_mean(dec, order, dpn, npr)
    elif comp == "q8":
        # unpinned spec (psb_q8.cu header): quantize each worker, fold the
        # dequantized values, requantize the mean per block, apply.
        dec = np.zeros((P, n), dtype=np.float32)
        for p in range(P):
            r = residuals[p] if residuals is not None else None
            codes, scales, _ = q8_quant(grads[p], r, q8_block)
            dec[p] = q8_dequant(codes, scales, q8_block)
        m = fold_mean(dec, order, dpn, npr)
        mc, ms, _ = q8_quant(m, None, q8_block)
        mean = q8_dequant(mc, ms, q8_block)
    else:
        raise ValueError(comp)
    axpy_(-lr, mean, theta)
    return mean


def async_round(grads: np.ndarray, theta: np.ndarray, lr: float, k: int, residuals: np.ndarray,
                staleness_bound: int, global_updates: int, q8: bool = False) -> int:
    """One round of the trainer's async branch (trainer.hpp:244-255) on given
    gradients: worker p's EF-compressed message is applied in order with
    scale lr/(1+tau_p), tau_p = min(updates, p mod (s+1)) (:246, s=3 in the
    reference).  Returns the new global update count."""
    P, n = grads.shape
    for p in range(P):
        tau = min(global_updates, p % (staleness_bound + 1))
        if q8:
            idx, codes, scales = ef_topk_q8(grads[p], residuals[p], k)
            val = q8_dequant(codes, scales, 128)
        else:
            idx, val, _ = ef_topk(grads[p], residuals[p], k)
        g = decompress_topk(idx, val, n)
        axpy_(-float(orc().orc_async_scale(lr, tau)), g, theta)
        global_updates += 1
    return global_updates


def momentum_(mean: np.ndarray, m: np.ndarray, theta: np.ndarray, beta: float, lr: float) -> None:
    """Momentum SGD rule of this build (north-star a24, unpinned), in place."""
    f = orc().orc_momentum_f64 if theta.dtype == np.float64 else orc().orc_momentum_f32
    f(_p(mean), _p(m), _p(theta), beta, lr, theta.size)


# ------------------------------------------------------------ wire format
def wire_encode_topk(dim: int, idx: np.ndarray, val: np.ndarray) -> np.ndarray:
    """parsim/compression.hpp:188-209 (TopK): u64 dim | u64 count | (u64 idx, f64 val) x count."""
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    out = np.empty(16 + 16 * idx.size, dtype=np.uint8)
    orc().orc_wire_encode_topk(dim, _p(idx), _p(val), idx.size, _p(out))
    return out


def wire_decode_topk(buf: np.ndarray):
    """parsim/compression.hpp:213-239 (TopK); ValueError on truncated input."""
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    dim = np.zeros(1, dtype=np.uint64)
    cnt = orc().orc_wire_decode_topk(_p(buf), buf.size, _p(dim), None, None)
    if cnt < 0:
        raise ValueError("wire_decode: truncated input")
    idx = np.empty(cnt, dtype=np.uint64)
    val = np.empty(cnt, dtype=np.float64)
    orc().orc_wire_decode_topk(_p(buf), buf.size, _p(dim), _p(idx), _p(val))
    return int(dim[0]), idx, val


def wire_encode_signbit(dim: int, scale: float, words: np.ndarray) -> np.ndarray:
    words = np.ascontiguousarray(words, dtype=np.uint32)
    out = np.empty(16 + (dim + 7) // 8, dtype=np.uint8)
    orc().orc_wire_encode_signbit(dim, scale, _p(words), _p(out))
    return out


def wire_encode_dense(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(8 + 8 * x.size, dtype=np.uint8)
    orc().orc_wire_encode_dense(x.size, _p(x), _p(out))
    return out


def ref_wire_encode_topk(dim: int, idx: np.ndarray, val: np.ndarray) -> np.ndarray:
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    val = np.ascontiguousarray(val, dtype=np.float64)
    n = ref().ref_wire_encode_topk(dim, _p(idx), _p(val), idx.size, None)
    out = np.empty(n, dtype=np.uint8)
    ref().ref_wire_encode_topk(dim, _p(idx), _p(val), idx.size, _p(out))
    return out


def ref_wire_decode_topk(buf: np.ndarray):
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    dim = np.zeros(1, dtype=np.uint64)
    cnt = ref().ref_wire_decode_topk(_p(buf), buf.size, _p(dim), None, None)
    if cnt < 0:
        raise ValueError(ref().ref_last_error().decode())
    idx = np.empty(cnt, dtype=np.uint64)
    val = np.empty(cnt, dtype=np.float64)
    ref().ref_wire_decode_topk(_p(buf), buf.size, _p(dim), _p(idx), _p(val))
    return int(dim[0]), idx, val


def ref_wire_encode_onebit(g: np.ndarray) -> np.ndarray:
    g = np.ascontiguousarray(g, dtype=np.float64)
    n = ref().ref_wire_encode_onebit(_p(g), g.size, None)
    out = np.empty(n, dtype=np.uint8)
    ref().ref_wire_encode_onebit(_p(g), g.size, _p(out))
    return out


def ref_bpr_batch_gradient(theta: np.ndarray, users: int, items: int, dim: int, u: np.ndarray, p: np.ndarray,
                           q: np.ndarray):
    """The reference's bpr_batch_gradient / bpr_batch_loss (trainer.hpp:98-138), f64."""
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    u, p, q = (np.ascontiguousarray(a, dtype=np.uint32) for a in (u, p, q))
    grad = np.empty_like(theta)
    loss = np.zeros(1, dtype=np.float64)
    _ref_ck(ref().ref_bpr_batch_gradient(_p(theta), users, items, dim, _p(u), _p(p), _p(q), u.size, _p(grad),
                                         _p(loss)))
    return grad, float(loss[0])


def ref_train(users: int, items: int, dim: int, train_u: np.ndarray, train_i: np.ndarray, P: int, mode: str,
              steps: int, batch: int, lr: float, kind: str, k: int, algo: str, seed: int, init_seed=None):
    """The reference trainer (trainer.hpp:197-261): final flat theta and loss curve."""
    tu = np.ascontiguousarray(train_u, dtype=np.uint64)
    ti = np.ascontiguousarray(train_i, dtype=np.uint64)
    theta = np.empty((users + items) * dim, dtype=np.float64)
    cap = steps // 100 + 2
    curve = np.zeros(2 * cap, dtype=np.float64)
    cn = np.zeros(1, dtype=np.uint64)
    _ref_ck(ref().ref_train(users, items, dim, _p(tu), _p(ti), tu.size, P, 0 if mode == "sync" else 1, steps, batch,
                            lr, {"none": 0, "onebit": 1, "topk": 2}[kind], k,
                            {"naive": 0, "ring": 1, "hierarchical": 2}[algo], seed,
                            seed if init_seed is None else init_seed, _p(theta), _p(curve), cap, _p(cn)))
    m = int(cn[0])
    return theta, [(int(curve[2 * j]), float(curve[2 * j + 1])) for j in range(m)]


def ref_load_model(path: str, cap: int):
    """The reference's load_model: ((users, items, dim), flat theta)."""
    dims = np.zeros(3, dtype=np.uint64)
    th = np.zeros(cap, dtype=np.float64)
    _ref_ck(ref().ref_load_model(path.encode(), _p(dims), _p(th), cap))
    u, i, d = (int(x) for x in dims)
    return (u, i, d), th[:(u + i) * d]


def ref_comm_cost(algo: int, msg_bytes: float, P: int, counts3, links6, span_devices: int = 0) -> float:
    """The reference's comm_cost (collectives.hpp:184-215); algo 0..3 = naive, ring, hierarchical, pipelined_ring;
    links6 = (intra_bw, inter_bw, rack_bw, intra_lat, inter_lat, rack_lat)."""
    c = np.ascontiguousarray(counts3, dtype=np.uint64)
    l6 = np.ascontiguousarray(links6, dtype=np.float64)
    out = np.zeros(1, dtype=np.float64)
    _ref_ck(ref().ref_comm_cost(algo, float(msg_bytes), P, _p(c), _p(l6), span_devices, _p(out)))
    return float(out[0])


def ref_synthetic_split(users: int, items: int, interactions: int, seed: int):
    """The reference's generate_synthetic + chrono_split: ((tu, ti), (vu, vi), (su, si))."""
    bufs = [np.zeros(interactions, dtype=np.uint64) for _ in range(6)]
    n3 = np.zeros(3, dtype=np.uint64)
    _ref_ck(ref().ref_synthetic_split(users, items, interactions, seed, *[_p(b) for b in bufs], _p(n3)))
    a, b, c = (int(x) for x in n3)
    return (bufs[0][:a], bufs[1][:a]), (bufs[2][:b], bufs[3][:b]), (bufs[4][:c], bufs[5][:c])


def ref_evaluate_topk(users, items, dim, theta, train, val, test, K=10, negatives=99, seed=42):
    """The reference's evaluate_topk (trainer.hpp:269-324): (hr, ndcg, evaluated, skipped)."""
    th = np.ascontiguousarray(theta, dtype=np.float64)
    arrs = [np.ascontiguousarray(a, dtype=np.uint64) for part in (train, val, test) for a in part]
    out = np.zeros(4, dtype=np.float64)
    _ref_ck(ref().ref_evaluate_topk(users, items, dim, _p(th), _p(arrs[0]), _p(arrs[1]), arrs[0].size, _p(arrs[2]),
                                    _p(arrs[3]), arrs[2].size, _p(arrs[4]), _p(arrs[5]), arrs[4].size, K, negatives,
                                    seed, _p(out)))
    return float(out[0]), float(out[1]), int(out[2]), int(out[3])


# ---------------------------------------------------------------- reference
def ref_compress_topk(g: np.ndarray, k: int) -> Tuple[np.ndarray, np.ndarray]:
    g = np.ascontiguousarray(g, dtype=np.float64)
    idx = np.empty(k, dtype=np.uint64)
    val = np.empty(k, dtype=np.float64)
    _ref_ck(ref().ref_compress_topk(_p(g), g.size, k, _p(idx), _p(val)))
    return idx, val


def ref_compress_onebit(g: np.ndarray) -> Tuple[np.ndarray, float]:
    g = np.ascontiguousarray(g, dtype=np.float64)
    sb = np.zeros((g.size + 7) // 8, dtype=np.uint8)
    sc = np.empty(1, dtype=np.float64)
    _ref_ck(ref().ref_compress_onebit(_p(g), g.size, _p(sb), _p(sc)))
    return sb, float(sc[0])


def ref_ef_step(kind: str, k: int, residual: np.ndarray, g: np.ndarray):
    kk = {"none": 0, "onebit": 1, "topk": 2}[kind]
    g = np.ascontiguousarray(g, dtype=np.float64)
    n = g.size
    idx = np.empty(max(k, 1), dtype=np.uint64)
    val = np.empty(max(k, n), dtype=np.float64)
    sb = np.zeros((n + 7) // 8, dtype=np.uint8)
    sc = np.zeros(1, dtype=np.float64)
    _ref_ck(ref().ref_ef_compress_step(kk, k, _p(residual), _p(g), n, _p(idx), _p(val), _p(sb),
                                       _p(sc)))
    if kind == "topk":
        return idx[:k], val[:k]
    if kind == "onebit":
        return sb, float(sc[0])
    return val[:n]


def ref_allreduce_mean(bufs: np.ndarray, algo: str, topo: Optional[Tuple[int, int, int]] = None):
    bufs = np.ascontiguousarray(bufs, dtype=np.float64)
    P, n = bufs.shape
    out = np.empty(n, dtype=np.float64)
    racks, npr, dpn = topo if topo else (0, 0, 0)
    _ref_ck(ref().ref_allreduce_mean(REF_ALGOS[algo], P, _p(bufs), n, racks, npr, dpn, _p(out)))
    return out


def ref_sync_step(kind: str, k: int, algo: str, grads: np.ndarray, params: np.ndarray, lr: float,
                  residuals: Optional[np.ndarray], topo: Optional[Tuple[int, int, int]] = None):
    """reference sync_data_parallel_step; params/residuals updated in place."""
    kk = {"none": 0, "onebit": 1, "topk": 2}[kind]
    grads = np.ascontiguousarray(grads, dtype=np.float64)
    P, n = grads.shape
    racks, npr, dpn = topo if topo else (0, 0, 0)
    _ref_ck(ref().ref_sync_step(kk, k, REF_ALGOS[algo], P, _p(grads), _p(params), n, lr,
                                _p(residuals), racks, npr, dpn))


def ref_sync_step_threaded(kind: str, k: int, algo: str, grads: np.ndarray, params: np.ndarray,
                           lr: float, residuals: np.ndarray, threads: int):
    kk = {"none": 0, "onebit": 1, "topk": 2}[kind]
    P, n = grads.shape
    _ref_ck(ref().ref_sync_step_threaded(kk, k, REF_ALGOS[algo], P, _p(grads), _p(params), n, lr,
                                         _p(residuals), threads))


def ref_async_step(params: np.ndarray, g: np.ndarray, tau: int, eta: float) -> np.ndarray:
    out = np.empty_like(params)
    _ref_ck(ref().ref_async_step(_p(params), _p(g), params.size, tau, eta, _p(out)))
    return out


def ref_vec_axpy(a: float, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    out = np.empty_like(y)
    _ref_ck(ref().ref_vec_axpy(a, _p(x), _p(y), y.size, _p(out)))
    return out
