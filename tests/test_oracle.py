"""CPU: pin the oracle restatement (oracle/psb_oracle.c) against the reference.

Every check compares the restatement with (a) the golden fixtures generated
from the unmodified reference (tests/golden/make_golden.py) and, where
oracle/_ref is built, (b) the reference itself on fresh inputs.
"""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O
from tests.refrng import SeededRng

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def h(*arrs):
    m = hashlib.sha256()
    for a in arrs:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:32]


def test_splitmix_kat(golden):
    # test_numerics.cpp:66-77
    kat = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F,
           0xBDD732262FEB6E95, 0x28EFE333B266F103, 0x47526757130F9F52]
    ours = list(O.splitmix_stream(0, 3)) + list(O.splitmix_stream(42, 3))
    assert [int(x) for x in ours] == kat
    assert [int(x) for x in golden["splitmix_kat"]] == kat
    r = SeededRng(0)
    assert r.next_u64() == kat[0]
    assert O.mix64(0) == kat[0]


def test_tie_vectors_topk_and_onebit(golden):
    """acceptance.cpp criterion 5: 11,840 exhaustive tie vectors, every k."""
    dims, orders = golden["tie_dims"], golden["tie_orders"]
    assert len(dims) == 11840
    # regenerate the vectors exactly as make_golden.py / acceptance.cpp:225-247
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
    vecs += [list(map(float, draws[i * 12:(i + 1) * 12])) for i in range(2000)]
    for i, v in enumerate(vecs):
        d = int(dims[i])
        assert d == len(v)
        order = [int(x) for x in orders[i, :d]]
        for dt in (np.float64, np.float32):
            g = np.array(v, dtype=dt)
            for k in range(1, d + 1):
                idx, val = O.topk(g, k)
                assert idx.tolist() == sorted(order[:k]), (i, k)
                assert np.array_equal(val, g[idx.astype(np.int64)])
        words, scale, _ = O.ef_onebit(np.array(v), None)
        assert scale == golden["tie_onebit_scale"][i]
        nb = (d + 7) // 8
        assert words.view(np.uint8)[:nb].tolist() == golden["tie_onebit_bytes"][i, :nb].tolist()


@pytest.mark.parametrize("kind", ["onebit", "topk"])
def test_ef_sequence_bitwise(golden, kind):
    """test_compression.cpp:118-135 inputs; EF state carried 200 steps."""
    gin = golden[f"ef_{kind}_inputs"]
    rec = golden[f"ef_{kind}_records"]
    r = np.zeros(16)
    for s in range(200):
        if kind == "topk":
            idx, val, st = O.ef_topk(gin[s].copy(), r, 3)
            assert st == 0
            got = np.concatenate([idx.astype(np.float64), val, r])
        else:
            words, scale, st = O.ef_onebit(gin[s].copy(), r)
            got = np.concatenate([words.view(np.uint8)[:2].astype(np.float64), [scale], r])
        assert np.array_equal(got, rec[s]), s


def test_collective_orders_bitwise(golden):
    """acceptance.cpp:133-170: 200 cases, seed 20250808, topology 2x2x4."""
    rng = SeededRng(20250808)
    cases, dig = golden["coll_cases"], golden["coll_digests"]
    for rep in range(200):
        P = 1 + rng.below(16)
        dim = 1 + rng.below(1000)
        bufs = np.array([[rng.uniform(-100, 100) for _ in range(dim)] for _ in range(P)])
        assert (P, dim) == tuple(cases[rep])
        for j, algo in enumerate(["naive", "ring", "hierarchical", "pipelined_ring"]):
            got = O.fold_mean(bufs, algo, dpn=4, npr=2)
            assert h(got) == dig[rep, j], (rep, algo)


def test_sync_step_composite_bitwise(golden):
    """sync_data_parallel_step (strategies.hpp:86-113) == the oracle composite."""
    keys = [str(k) for k in golden["sync_keys"]]
    digs = golden["sync_digests"]
    for key, ds in zip(keys, digs):
        P, kind, algo, ef = key.split("|")
        P, ef = int(P), bool(int(ef))
        k = 10 if kind == "topk" else 0
        theta = np.zeros(1000)
        res = np.zeros((P, 1000)) if ef else None
        dpn, npr = (2, 2) if algo == "hierarchical" and P >= 4 else (0, 1)
        for step in range(10):
            grads = np.stack([O.generate("llmrec" if p % 2 else "uniform", 42, p, step, 1000)
                              for p in range(P)]).astype(np.float64)
            if res is None:
                O.sync_step(grads, theta, 0.05, kind, k, algo, None, dpn, npr)
            else:
                O.sync_step(grads, theta, 0.05, kind, k, algo, res, dpn, npr)
            got = h(theta, res) if ef else h(theta)
            assert got == ds[step], (key, step)


@needs_ref
def test_f32_inputs_widened_match_reference_topk():
    """The f32 restatement selects the same indices as the f64 reference on
    widened inputs (widening is exact and order-preserving)."""
    for dist in ("uniform", "llmrec", "ties"):
        for n, k in ((1000, 10), (4096, 400), (777, 777), (5000, 1)):
            g = O.generate(dist, 7, 1, 2, n)
            i32, v32 = O.topk(g, k)
            i64, v64 = O.ref_compress_topk(g.astype(np.float64), k)
            assert np.array_equal(i32.astype(np.uint64), i64)
            assert np.array_equal(v32.astype(np.float64), v64)


@needs_ref
def test_async_composite_matches_reference_async_step():
    """trainer.hpp:244-255 loop built from the reference's ef_compress_step,
    decompress and async_step == oracle async_round (f64, bitwise)."""
    P, n, k, lr = 8, 2000, 20, 0.1
    theta_ref = np.zeros(n)
    theta_orc = np.zeros(n)
    r_ref = np.zeros((P, n))
    r_orc = np.zeros((P, n))
    gu_ref = gu = 0
    for step in range(6):
        grads = np.stack([O.generate("llmrec", 3, p, step, n) for p in range(P)]).astype(np.float64)
        for p in range(P):
            tau = min(gu_ref, p % 4)
            idx, val = O.ref_ef_step("topk", k, r_ref[p], grads[p])
            gdec = np.zeros(n)
            gdec[idx.astype(np.int64)] = val
            theta_ref = O.ref_async_step(theta_ref, gdec, tau, lr)
            gu_ref += 1
        gu = O.async_round(grads, theta_orc, lr, k, r_orc, 3, gu)
    assert gu == gu_ref
    assert np.array_equal(theta_ref, theta_orc)
    assert np.array_equal(r_ref, r_orc)


@needs_ref
def test_reference_errors_match_contract():
    with pytest.raises(O.RefError, match="k out of range"):
        O.ref_compress_topk(np.array([1.0, 2.0]), 3)
    with pytest.raises(ValueError, match="k out of range"):
        O.topk(np.array([1.0, 2.0]), 0)


def test_generator_determinism_and_shape():
    a = O.generate("llmrec", 42, 0, 0, 1 << 16)
    b = O.generate("llmrec", 42, 0, 0, 1 << 16)
    assert np.array_equal(a, b)
    zero_frac = float(np.mean(a == 0))
    assert 0.5 < zero_frac < 0.65  # 60% embedding segment x 95% zero rows
    u = O.generate("uniform", 42, 0, 0, 1 << 16)
    assert u.min() >= -1 and u.max() < 1
    t = O.generate("ties", 42, 0, 0, 4096)
    assert set(np.unique(t).tolist()) <= {-0.5, -0.25, 0.0, 0.25, 0.5}
    assert not np.array_equal(O.generate("uniform", 42, 1, 0, 64), O.generate("uniform", 42, 0, 0, 64))


def test_q8_spec_properties():
    """Unpinned 8-bit rule: bound |p - xhat| <= scale/2, codes in [-127,127],
    EF identity r' + xhat == p (Sterbenz range) within 1 ulp."""
    g = O.generate("llmrec", 1, 0, 0, 100_000)
    r = O.generate("uniform", 1, 0, 1, 100_000) * np.float32(1e-3)
    p = (r + g).astype(np.float32)
    r2 = r.copy()
    codes, scales, st = O.q8_quant(g, r2, 256)
    assert st == 0
    assert codes.min() >= -127 and codes.max() <= 127
    xhat = O.q8_dequant(codes, scales, 256)
    sc = np.repeat(scales, 256)[: p.size]
    assert np.all(np.abs(p - xhat) <= sc * 0.5000001 + 1e-30)
    assert np.allclose(r2 + xhat, p, rtol=0, atol=np.spacing(np.abs(p)).max())


# ------------------------------------------------------------ wire format
@pytest.mark.skipif(not O.ref_available(), reason="reference headers not built (oracle/_ref)")
def test_wire_codec_matches_reference():
    """parsim wire_encode / wire_decode (compression.hpp:159-239): the C
    restatement is byte-identical to the reference on random top-k payloads,
    decodes the reference's bytes, and fails on truncation with its message."""
    rng = np.random.default_rng(7)
    for dim, k in [(1, 1), (40, 7), (1000, 50), (1 << 20, 4096)]:
        idx = np.sort(rng.choice(dim, k, replace=False)).astype(np.uint32)
        val = rng.standard_normal(k)
        ours = O.wire_encode_topk(dim, idx, val)
        theirs = O.ref_wire_encode_topk(dim, idx.astype(np.uint64), val)
        assert np.array_equal(ours, theirs)
        d, i2, v2 = O.wire_decode_topk(theirs)
        assert d == dim and np.array_equal(i2, idx.astype(np.uint64)) and np.array_equal(v2.view(np.uint64),
                                                                                         val.view(np.uint64))
        for cut in (1, 8, 15):
            with pytest.raises(ValueError, match="wire_decode: truncated input"):
                O.ref_wire_decode_topk(theirs[:-cut] if cut < theirs.size else theirs[:0])
            with pytest.raises(ValueError, match="wire_decode: truncated input"):
                O.wire_decode_topk(theirs[:-cut] if cut < theirs.size else theirs[:0])
    # sign-bit body: the oracle's sign words (u32 LE) are the reference's sign bytes
    for n in (1, 7, 8, 9, 37, 1000):
        g = rng.standard_normal(n)
        sb, sc = O.ref_compress_onebit(g)
        words = np.zeros((n + 31) // 32, dtype=np.uint32)
        words.view(np.uint8)[:sb.size] = sb
        assert np.array_equal(O.wire_encode_signbit(n, sc, words), O.ref_wire_encode_onebit(g))
    # dense layout (test_compression.cpp:215-218)
    b = O.wire_encode_dense(np.array([1.0, 2.0]))
    assert b.size == 8 + 16 and b[0] == 2
