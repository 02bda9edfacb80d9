"""GPU parity of K1 (fused EF + top-k) against the oracle and the reference.

Bar: indices, values and residuals bit-exact (SURVEY.md 8c parity statement).
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def tnp(t):
    return t.detach().cpu().numpy()


def _tie_vectors():
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
    return vecs


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_tie_vectors_every_k(ctx, golden, dtype):
    """acceptance.cpp criterion 5 (11,840 vectors x every k) on the GPU path,
    against the reference's own outputs (golden)."""
    vecs = _tie_vectors()
    orders = golden["tie_orders"]
    bad = 0
    for i, v in enumerate(vecs):
        d = len(v)
        g = torch.tensor(v, dtype=dtype, device="cuda")
        outs = []
        for k in range(1, d + 1):
            idx, val = ctx.ef_topk(g, None, k, worker=1)
            outs.append(idx.clone())
        got = tnp(torch.cat(outs)).astype(np.int64)
        order = [int(x) for x in orders[i, :d]]
        want = np.concatenate([sorted(order[:k]) for k in range(1, d + 1)])
        bad += int(not np.array_equal(got, want))
    ctx.check()
    assert bad == 0


def test_ef_sequence_f64_matches_reference(ctx, golden):
    """200-step EF top-k sequence in f64: bitwise the reference's own records
    (golden from oracle/_ref, inputs of test_compression.cpp:118-135)."""
    gin = golden["ef_topk_inputs"]
    rec = golden["ef_topk_records"]
    r = torch.zeros(16, dtype=torch.float64, device="cuda")
    for s in range(200):
        g = torch.tensor(gin[s], dtype=torch.float64, device="cuda")
        idx, val = ctx.ef_topk(g, r, 3, worker=2)
        got = np.concatenate([tnp(idx).astype(np.float64), tnp(val), tnp(r)])
        assert np.array_equal(got, rec[s]), s
    ctx.check()


@pytest.mark.parametrize("dist", ["uniform", "llmrec", "ties"])
@pytest.mark.parametrize("n,k", [(1_000_000, 10_000), (333_333, 3_333), (65_537, 6_554)])
def test_ef_topk_sequence_f32_bitwise(ctx, dist, n, k):
    """10 consecutive EF steps (residual carried, prediction path exercised)."""
    r_host = np.zeros(n, dtype=np.float32)
    r_dev = torch.zeros(n, dtype=torch.float32, device="cuda")
    for step in range(10):
        g_host = O.generate(dist, 42, 0, step, n)
        g_dev = torch.from_numpy(g_host).cuda()
        idx, val = ctx.ef_topk(g_dev, r_dev, k, worker=3)
        oi, ov, st = O.ef_topk(g_host, r_host, k)
        assert st == 0
        assert np.array_equal(tnp(idx).view(np.uint32), oi), step
        assert np.array_equal(tnp(val).view(np.uint32), ov.view(np.uint32)), step
        assert np.array_equal(tnp(r_dev).view(np.uint32), r_host.view(np.uint32)), step
    ctx.check()


def test_device_generator_matches_oracle(cuda):
    from paper_2506_17551_b200.engine import generate
    for dist in ("uniform", "llmrec", "ties"):
        for n in (1, 5, 4099, 1 << 20):
            out = torch.empty(n, dtype=torch.float32, device="cuda")
            generate(dist, 42, 3, 7, n, out)
            assert np.array_equal(tnp(out).view(np.uint32), O.generate(dist, 42, 3, 7, n).view(np.uint32))


def test_prediction_miss_falls_back_exactly(ctx):
    """Threshold collapses between calls of one worker (no EF): the predicted
    candidate set misses, the full-histogram pass must take over."""
    n, k = 200_003, 2_000
    big = O.generate("uniform", 1, 0, 0, n) * np.float32(1000)
    small = O.generate("uniform", 1, 0, 1, n) * np.float32(1e-3)
    for g in (big, small, big, small * np.float32(1e-20)):
        idx, val = ctx.ef_topk(torch.from_numpy(g).cuda(), None, k, worker=5)
        oi, ov = O.topk(g, k)
        assert np.array_equal(tnp(idx).view(np.uint32), oi)
        assert np.array_equal(tnp(val), ov)
    ctx.check()


@pytest.mark.parametrize("ef", [False, True])
def test_prediction_second_chance_exact(ctx, ef):
    """The threshold drops a few percent below the predicted margin: pass A
    misses, the second-chance compaction on G2 = 0.97 G holds (no full
    histogram pass), and the results stay bit-exact."""
    n, k = 1_000_003, 10_000
    scales = [1, 1, 1, 1, 0.93, 1, 1, 1, 0.93, 0.93, 1, 1]
    second = 0
    for wi, dt in ((7, np.float32), (8, np.float64)):
        r_host = np.zeros(n, dtype=dt)
        r_dev = torch.zeros(n, dtype=torch.float32 if dt == np.float32 else torch.float64, device="cuda")
        for s, sc in enumerate(scales):
            g = (O.generate("uniform", 3, 0, s, n) * np.float32(sc)).astype(dt)
            before = ctx.topk_stats(worker=wi)["misses"]
            idx, val = ctx.ef_topk(torch.from_numpy(g).cuda(), r_dev if ef else None, k, worker=wi)
            if ef:
                oi, ov, _ = O.ef_topk(g, r_host, k)
            else:
                oi, ov = O.topk(g, k)
            assert np.array_equal(tnp(idx).view(np.uint32), oi), (dt, s)
            assert np.array_equal(tnp(val), ov), (dt, s)
            if ef:
                assert np.array_equal(tnp(r_dev), r_host), (dt, s)
            st = ctx.topk_stats(worker=wi)
            if st["misses"] > before and st["predicted_valid"]:
                second += 1
    ctx.check()
    if not ef:
        assert second >= 1  # the second chance was taken and held at least once


@pytest.mark.parametrize("n,k", [(1, 1), (2, 2), (3, 1), (4097, 4097), (4097, 1), (12345, 12344)])
def test_edge_sizes(ctx, n, k):
    g = O.generate("ties", 9, 0, 0, n)
    for dt in (np.float32, np.float64):
        gg = g.astype(dt)
        r_host = (O.generate("uniform", 9, 1, 0, n) * 0.25).astype(dt)
        r_dev = torch.from_numpy(r_host.copy()).cuda()
        idx, val = ctx.ef_topk(torch.from_numpy(gg).cuda(), r_dev, k, worker=6)
        oi, ov, _ = O.ef_topk(gg, r_host, k)
        assert np.array_equal(tnp(idx).view(np.uint32), oi)
        assert np.array_equal(tnp(val), ov)
        assert np.array_equal(tnp(r_dev), r_host)
    ctx.check()


def test_misaligned_views_and_signed_zeros(ctx):
    n = 10_001
    base = torch.zeros(n + 3, dtype=torch.float32, device="cuda")
    g = base[1:n + 1]  # 4-byte aligned only -> scalar path
    host = np.zeros(n, dtype=np.float32)
    host[::3] = -0.0
    host[5::97] = 1.5
    host[6::97] = -1.5
    g.copy_(torch.from_numpy(host))
    for k in (1, 50, 500, 5000, n):
        idx, val = ctx.ef_topk(g, None, k, worker=7)
        oi, ov = O.topk(host, k)
        assert np.array_equal(tnp(idx).view(np.uint32), oi)
        assert np.array_equal(tnp(val).view(np.uint32), ov.view(np.uint32))
    ctx.check()


def test_nonfinite_raises(ctx):
    from paper_2506_17551_b200 import PsbNonFinite
    g = torch.ones(1000, device="cuda")
    g[17] = float("inf")
    r = torch.zeros(1000, device="cuda")
    ctx.ef_topk(g, r, 10, worker=8)
    with pytest.raises(PsbNonFinite):
        ctx.check()
    ctx.check()  # flag cleared


def test_k_out_of_range_rejected(ctx):
    from paper_2506_17551_b200 import PsbInvalidArgument
    g = torch.ones(10, device="cuda")
    with pytest.raises(PsbInvalidArgument, match="k out of range"):
        ctx.ef_topk(g, None, 0)
    with pytest.raises(PsbInvalidArgument, match="k out of range"):
        ctx.ef_topk(g, None, 11)


def test_full_size_properties_125m(cuda):
    """BASELINE cfg2 size (N = 1.25e8, k = 1%): size-independent properties
    of the exact rule, checked with torch on the device."""
    from paper_2506_17551_b200.engine import Context, generate
    n, k = 125_000_000, 1_250_000
    c = Context(n, k, 1)
    g = torch.empty(n, device="cuda")
    r = torch.zeros(n, device="cuda")
    for step in range(3):
        generate("llmrec", 42, 0, step, n, g)
        p = r + g  # torch fp32 add is IEEE RN, same as the kernel
        idx, val = c.ef_topk(g, r, k)
        c.check()
        idx64 = idx.long()
        assert idx64.numel() == k
        assert bool((idx64[1:] > idx64[:-1]).all())
        assert torch.equal(val.view(torch.int32), p[idx64].view(torch.int32))
        key = p.view(torch.int32) & 0x7FFFFFFF
        t = int((val.view(torch.int32) & 0x7FFFFFFF).min())
        n_gt = int((key > t).sum())
        n_eq = int((key == t).sum())
        assert n_gt < k <= n_gt + n_eq
        sel = torch.zeros(n, dtype=torch.bool, device="cuda")
        sel[idx64] = True
        assert bool(sel[key > t].all())
        eq_idx = torch.nonzero(key == t).view(-1)
        assert torch.equal(sel[eq_idx], torch.arange(eq_idx.numel(), device="cuda") < (k - n_gt))
        expect_r = torch.where(sel, torch.zeros_like(p), p)
        assert torch.equal(r.view(torch.int32), expect_r.view(torch.int32))
    c.close()


@pytest.mark.skipif(os.environ.get("PSB_NO_PREDICT", "0") != "0", reason="prediction disabled by PSB_NO_PREDICT")
def test_threshold_prediction_engages_and_stays_exact(cuda):
    """After the first (cold) call the worker predicts its threshold; the
    predicted candidate set must be valid in steady state and results exact."""
    from paper_2506_17551_b200.engine import Context
    n, k = 1_000_000, 10_000
    c = Context(n, k, 1)
    r_host = np.zeros(n, dtype=np.float32)
    r_dev = torch.zeros(n, dtype=torch.float32, device="cuda")
    valid = []
    for step in range(8):
        g_host = O.generate("llmrec", 11, 0, step, n)
        idx, val = c.ef_topk(torch.from_numpy(g_host).cuda(), r_dev, k)
        oi, ov, _ = O.ef_topk(g_host, r_host, k)
        assert np.array_equal(tnp(idx).view(np.uint32), oi)
        assert np.array_equal(tnp(r_dev).view(np.uint32), r_host.view(np.uint32))
        st = c.topk_stats(0)
        valid.append(st["predicted_valid"])
        assert st["candidates"] >= k
    c.check()
    assert not valid[0]          # cold call
    assert sum(valid[2:]) >= 5   # steady state predicted
    c.close()
