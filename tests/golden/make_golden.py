"""Generate tests/golden/ref_golden.npz from the reference itself.

Runs the UNMODIFIED reference headers (oracle/_ref/libparsim_ref.so, built by
oracle/Makefile from /root/reference/proj/include) on the inputs the
reference's own tests use, and stores the outputs (or sha256 digests of
large outputs).  Committed so parity stays pinned where /root/reference is
absent (the GPU box).  Regenerate: python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from tests.refrng import SeededRng as _Rng  # noqa: E402


def h(*arrs):
    m = hashlib.sha256()
    for a in arrs:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:32]


def tie_vectors():
    """acceptance.cpp:225-247: {-1,0,1}^d for d<=8, then 2000 draws of
    {-2..2}^12 from SeededRng(5).next_below(5)."""
    vecs = []
    for d in range(1, 9):
        for code in range(3 ** d):
            v, c = [], code
            for _ in range(d):
                v.append(float(c % 3 - 1))
                c //= 3
            vecs.append(v)
    u = O.splitmix_stream(5, 2000 * 12)
    draws = (u % np.uint64(5)).astype(np.int64) - 2
    for rep in range(2000):
        vecs.append([float(x) for x in draws[rep * 12:(rep + 1) * 12]])
    return vecs


def main():
    out = {}
    # 1. tie vectors: the reference's top-k for every k, stored as the stable
    #    order (top-k for k = sorted(order[:k])) + onebit sign bytes/scale.
    vecs = tie_vectors()
    orders = np.full((len(vecs), 12), 255, dtype=np.uint8)
    dims = np.array([len(v) for v in vecs], dtype=np.uint8)
    ob_scale = np.zeros(len(vecs))
    ob_bytes = np.zeros((len(vecs), 2), dtype=np.uint8)
    for i, v in enumerate(vecs):
        g = np.array(v)
        prev = set()
        order = []
        for k in range(1, len(v) + 1):
            idx, _ = O.ref_compress_topk(g, k)
            new = set(int(x) for x in idx) - prev
            assert len(new) == 1
            order.append(new.pop())
            prev = set(int(x) for x in idx)
        orders[i, :len(v)] = order
        sb, sc = O.ref_compress_onebit(g)
        ob_scale[i] = sc
        ob_bytes[i, :sb.size] = sb
    out["tie_dims"], out["tie_orders"] = dims, orders
    out["tie_onebit_scale"], out["tie_onebit_bytes"] = ob_scale, ob_bytes

    # 2. EF sequences (test_compression.cpp:118-135 shape): 200 steps, dim 16,
    #    uniform(-5,5) from SeededRng(2024); both compressors, k=3.
    g_all = O.seeded_uniform(2024, 2 * 200 * 16, -5, 5).reshape(2, 200, 16)
    for ci, kind in enumerate(["onebit", "topk"]):
        r = np.zeros(16)
        recs = []
        for s in range(200):
            res = O.ref_ef_step(kind, 3, r, g_all[ci, s])
            if kind == "topk":
                recs.append(np.concatenate([res[0].astype(np.float64), res[1], r.copy()]))
            else:
                recs.append(np.concatenate([res[0].astype(np.float64), [res[1]], r.copy()]))
        out[f"ef_{kind}_inputs"] = g_all[ci]
        out[f"ef_{kind}_records"] = np.array(recs)

    # 3. collective equivalence (acceptance.cpp:133-170): 200 cases, seed
    #    20250808, topo racks=2 npr=2 dpn=4; digest of each algorithm's output.
    cases, digests = [], []
    gen = _Rng(20250808)
    for rep in range(200):
        P = 1 + gen.below(16)
        dim = 1 + gen.below(1000)
        bufs = np.array([[gen.uniform(-100, 100) for _ in range(dim)] for _ in range(P)])
        cases.append((P, dim))
        row = []
        for algo in ["naive", "ring", "hierarchical", "pipelined_ring"]:
            row.append(h(O.ref_allreduce_mean(bufs, algo, (2, 2, 4))))
        digests.append(row)
    out["coll_cases"] = np.array(cases)
    out["coll_digests"] = np.array(digests)

    # 4. sync step: P in {1,2,4,8}, dim 1000, 10 steps, each compressor and
    #    order, with and without EF; digest of theta (+ residuals) per step.
    sync_keys, sync_digests = [], []
    for P in (1, 2, 4, 8):
        for kind, k in (("topk", 10), ("onebit", 0), ("none", 0)):
            for algo in ("naive", "ring", "hierarchical"):
                for ef in (True, False):
                    if kind == "none" and ef:
                        continue
                    theta = np.zeros(1000)
                    res = np.zeros((P, 1000)) if ef else None
                    ds = []
                    for step in range(10):
                        grads = np.stack([O.generate("llmrec" if p % 2 else "uniform", 42, p, step, 1000)
                                          for p in range(P)]).astype(np.float64)
                        O.ref_sync_step(kind, k, algo, grads, theta, 0.05, res,
                                        (1, 2, 2) if algo == "hierarchical" and P >= 4 else None)
                        ds.append(h(theta, res) if ef else h(theta))
                    sync_keys.append(f"{P}|{kind}|{algo}|{int(ef)}")
                    sync_digests.append(ds)
    out["sync_keys"] = np.array(sync_keys)
    out["sync_digests"] = np.array(sync_digests)

    # 5. SplitMix KAT (test_numerics.cpp:66-77) as seen through the reference.
    kat = np.empty(6, dtype=np.uint64)
    s0 = np.empty(3, dtype=np.uint64)
    O.ref().ref_splitmix_stream(0, 3, O._p(s0))
    s42 = np.empty(3, dtype=np.uint64)
    O.ref().ref_splitmix_stream(42, 3, O._p(s42))
    kat[:3], kat[3:] = s0, s42
    out["splitmix_kat"] = kat

    path = os.path.join(os.path.dirname(__file__), "ref_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
