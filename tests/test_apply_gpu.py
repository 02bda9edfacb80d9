"""GPU parity of aggregate + apply, the other compressors and the step drivers.

Bar: bit-exact against the oracle composite whenever the reference fold order
is mirrored (all cases here); the 1-bit scale is a deterministic tree sum and
is compared at 1e-12 relative (f64) -- see DESIGN.md "Parity".
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2506_17551_b200 import _lib as L
from paper_2506_17551_b200.engine import payload_bytes, topology

pytestmark = pytest.mark.gpu


def tnp(t):
    return t.detach().cpu().numpy()


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def make_payloads(P, n, k, dtype, seed, overlap=True):
    """P top-k payloads with heavy index overlap, +-0 values and collisions."""
    rng = np.random.default_rng(seed)
    idx = np.zeros((P, k), dtype=np.uint32)
    val = np.zeros((P, k), dtype=dtype)
    pool = rng.choice(n, size=min(n, 3 * k), replace=False)
    for p in range(P):
        src = pool if overlap else np.arange(n)
        idx[p] = np.sort(rng.choice(src, size=k, replace=False))
        v = rng.standard_normal(k).astype(dtype)
        v[rng.random(k) < 0.05] = dtype(0.0)
        v[rng.random(k) < 0.05] = -dtype(0.0)
        val[p] = v
    return idx, val


def pack_payloads(idx, val, dtype_t):
    P, k = idx.shape
    blk = payload_bytes(L.PSB_COMP_TOPK, dtype_t, k)
    buf = np.zeros(P * blk, dtype=np.uint8)
    voff = (k * 4 + 15) // 16 * 16
    for p in range(P):
        buf[p * blk:p * blk + 4 * k] = idx[p].view(np.uint8)
        vb = val[p].view(np.uint8)
        buf[p * blk + voff:p * blk + voff + vb.size] = vb
    return torch.from_numpy(buf).cuda()


ORDERS = [("naive", 0, 1), ("ring", 0, 1), ("hierarchical", 2, 2), ("hierarchical", 3, 1),
          ("pipelined_ring", 0, 1)]


@pytest.mark.parametrize("dtype_t", [torch.float32, torch.float64])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8, 16])
@pytest.mark.parametrize("order,dpn,npr", ORDERS)
def test_sparse_mean_sgd_bitwise(ctx, dtype_t, P, order, dpn, npr):
    dt = np.float32 if dtype_t == torch.float32 else np.float64
    n, k = 50_021, 1_500
    idx, val = make_payloads(P, n, k, dt, seed=P * 7 + len(order))
    theta_h = (O.generate("uniform", 5, 0, 0, n)).astype(dt)
    theta_h[::11] = -0.0
    dense = np.zeros((P, n), dtype=dt)
    for p in range(P):
        dense[p, idx[p].astype(np.int64)] = val[p]
    mean_h = O.fold_mean(dense, order, dpn, npr)
    want = theta_h.copy()
    O.axpy_(-0.05, mean_h, want)
    theta = torch.from_numpy(theta_h.copy()).cuda()
    mean = torch.zeros(n, dtype=dtype_t, device="cuda")
    pl = pack_payloads(idx, val, dtype_t)
    topo = topology(1, npr, dpn) if dpn else None
    ctx.sparse_mean_sgd(pl, P, k, dtype_t, order, 0.05, theta, n, mean, topo)
    ctx.check()
    assert np.array_equal(bits(tnp(theta)), bits(want))
    touched = np.unique(idx.astype(np.int64))
    assert np.array_equal(bits(tnp(mean)[touched]), bits(mean_h[touched]))


@pytest.mark.parametrize("P", [1, 4, 8])
def test_async_apply_bitwise(ctx, P):
    n, k = 40_000, 800
    idx, val = make_payloads(P, n, k, np.float32, seed=P)
    theta_h = O.generate("llmrec", 2, 0, 0, n)
    scales = [0.1 / (1 + (p % 3)) for p in range(P)]
    want = theta_h.copy()
    for p in range(P):
        O.axpy_(-scales[p], O.decompress_topk(idx[p], val[p], n), want)
    theta = torch.from_numpy(theta_h.copy()).cuda()
    ctx.sparse_async_apply(pack_payloads(idx, val, torch.float32), P, k, torch.float32, scales, theta)
    ctx.check()
    assert np.array_equal(bits(tnp(theta)), bits(want))


@pytest.mark.parametrize("dtype_t", [torch.float32, torch.float64])
@pytest.mark.parametrize("order,dpn,npr", ORDERS)
def test_dense_mean_bitwise(ctx, dtype_t, order, dpn, npr):
    dt = np.float32 if dtype_t == torch.float32 else np.float64
    for P in (1, 3, 8):
        n = 10_007
        bufs = np.stack([O.generate("uniform", 11, p, 0, n) for p in range(P)]).astype(dt)
        theta_h = O.generate("uniform", 12, 0, 0, n).astype(dt)
        mean_h = O.fold_mean(bufs, order, dpn, npr)
        want = theta_h.copy()
        O.axpy_(-0.25, mean_h, want)
        theta = torch.from_numpy(theta_h.copy()).cuda()
        mean = torch.empty(n, dtype=dtype_t, device="cuda")
        topo = topology(1, npr, dpn) if dpn else None
        ctx.dense_mean_sgd(torch.from_numpy(bufs).cuda(), order, 0.25, theta, mean, topo)
        ctx.check()
        assert np.array_equal(bits(tnp(mean)), bits(mean_h))
        assert np.array_equal(bits(tnp(theta)), bits(want))


@pytest.mark.parametrize("dtype_t", [torch.float32, torch.float64])
def test_onebit_compress_and_mean(ctx, dtype_t):
    dt = np.float32 if dtype_t == torch.float32 else np.float64
    n = 100_003
    g_h = O.generate("llmrec", 13, 0, 0, n).astype(dt)
    r_h = (O.generate("uniform", 13, 1, 0, n) * 1e-3).astype(dt)
    r = torch.from_numpy(r_h.copy()).cuda()
    words, scale = ctx.ef_onebit(torch.from_numpy(g_h).cuda(), r)
    ctx.check()
    ow, osc, _ = O.ef_onebit(g_h, r_h)
    assert np.array_equal(tnp(words).view(np.uint32), ow)
    assert abs(float(scale.item()) - osc) <= 1e-12 * abs(osc)
    # residual: bit-exact given the scale the device computed
    s = dt(float(scale.item()))
    pp = ((O.generate("uniform", 13, 1, 0, n) * 1e-3).astype(dt) + g_h).astype(dt)
    want = (pp - np.where(pp >= 0, s, -s)).astype(dt)
    assert np.array_equal(bits(tnp(r)), bits(want))
    # 1-bit fold + SGD with the device scales
    P = 4
    ws = torch.stack([torch.from_numpy(ow.view(np.int32)).cuda()] * P)
    scales = torch.tensor([osc * (1 + p) for p in range(P)], dtype=torch.float64, device="cuda")
    theta = torch.zeros(n, dtype=dtype_t, device="cuda")
    mean = torch.empty(n, dtype=dtype_t, device="cuda")
    ctx.onebit_mean_sgd(ws, scales, n, dtype_t, "ring", 0.1, theta, mean)
    ctx.check()
    bitsv = ((ow.view(np.uint8)[:, None] >> np.arange(8, dtype=np.uint8)) & 1).reshape(-1)[:n].astype(bool)
    dense = np.stack([np.where(bitsv, dt(osc * (1 + p)), -dt(osc * (1 + p))) for p in range(P)])
    mean_h = O.fold_mean(dense, "ring")
    want_t = np.zeros(n, dtype=dt)
    O.axpy_(-0.1, mean_h, want_t)
    assert np.array_equal(bits(tnp(mean)), bits(mean_h))
    assert np.array_equal(bits(tnp(theta)), bits(want_t))


@pytest.mark.parametrize("block", [128, 256, 512, 1024])
def test_q8_quantize_bitwise(ctx, block):
    for n in (1, 1000, 262_147):
        g_h = O.generate("llmrec", 21, 0, 0, n)
        r_h = O.generate("uniform", 21, 1, 0, n) * np.float32(1e-4)
        r = torch.from_numpy(r_h.copy()).cuda()
        codes, scales = ctx.q8_quantize(torch.from_numpy(g_h).cuda(), r, block)
        oc, osc, _ = O.q8_quant(g_h, r_h, block)
        ctx.check()
        assert np.array_equal(tnp(codes), oc)
        assert np.array_equal(bits(tnp(scales)), bits(osc))
        assert np.array_equal(bits(tnp(r)), bits(r_h))
        deq = ctx.q8_dequantize(codes, scales, block)
        assert np.array_equal(bits(tnp(deq)), bits(O.q8_dequant(oc, osc, block)))


def test_q8_rounding_ties_and_near_ties(ctx):
    """Exact .5 ties (round-half-even) and values 1-3 ulp around them, where the
    reciprocal fast path must defer to the exact IEEE division."""
    base = np.array([127.0, 2.5, 3.5, -4.5, 0.5, -0.5, 126.5, 1.5], dtype=np.float32)
    vals = [base]
    for d in (1, 2, 3, 5):
        up = np.nextafter(base, np.float32(np.inf))
        dn = np.nextafter(base, np.float32(-np.inf))
        for _ in range(d - 1):
            up = np.nextafter(up, np.float32(np.inf))
            dn = np.nextafter(dn, np.float32(-np.inf))
        vals += [up.astype(np.float32), dn.astype(np.float32)]
    x = np.concatenate(vals).astype(np.float32)
    x = np.concatenate([x, np.zeros((-x.size) % 128, dtype=np.float32)])
    # scale a copy so absmax/127 is not exactly 1 as well
    for mult in (np.float32(1.0), np.float32(0.37), np.float32(3.1e-3)):
        xs = (x * mult).astype(np.float32)
        codes, scales = ctx.q8_quantize(torch.from_numpy(xs).cuda(), None, 128)
        oc, osc, _ = O.q8_quant(xs, None, 128)
        ctx.check()
        assert np.array_equal(tnp(codes), oc)
        assert np.array_equal(bits(tnp(scales)), bits(osc))


COMPS = {"topk": L.PSB_COMP_TOPK, "onebit": L.PSB_COMP_ONEBIT, "none": L.PSB_COMP_NONE,
         "q8": L.PSB_COMP_Q8, "topk_q8": L.PSB_COMP_TOPK_Q8}


@pytest.mark.parametrize("comp", ["topk", "topk_q8", "none", "q8", "onebit"])
@pytest.mark.parametrize("order", ["naive", "ring", "hierarchical"])
@pytest.mark.parametrize("W", [1, 3, 4])
def test_sync_step_virtual_workers(ctx, comp, order, W):
    """psb_sync_step with W virtual workers on one GPU (cfg1 shape) vs the
    oracle composite of sync_data_parallel_step, 10 steps, EF carried."""
    n, k, lr = 100_000, 1_000, 0.05
    # W=4: 2 nodes in one rack; W=3: a ragged node and two racks
    dpn, npr = {4: (2, 2), 3: (2, 1)}.get(W, (0, 1)) if order == "hierarchical" else (0, 1)
    topo = topology(1, npr, dpn) if dpn else None
    theta_h = np.zeros(n, dtype=np.float32)
    res_h = np.zeros((W, n), dtype=np.float32)
    theta = torch.zeros(n, device="cuda")
    res = torch.zeros(W, n, device="cuda")
    for step in range(10):
        g_h = np.stack([O.generate("llmrec", 42, w, step, n) for w in range(W)])
        g = torch.from_numpy(g_h).cuda()
        mean = torch.zeros(n, device="cuda")
        d = ctx.step_desc(COMPS[comp], g, res, theta, lr, k, order, 256, topo, mean)
        ctx.sync_step(d)
        ctx.check()
        O.sync_step(g_h, theta_h, lr, comp, k, order, res_h, dpn, npr, 256)
        if comp == "onebit":
            # scale = deterministic tree sum vs sequential fold: tolerance
            np.testing.assert_allclose(tnp(theta), theta_h, rtol=1e-5, atol=1e-7)
            theta.copy_(torch.from_numpy(theta_h))
            res.copy_(torch.from_numpy(res_h))
        else:
            assert np.array_equal(bits(tnp(theta)), bits(theta_h)), step
            assert np.array_equal(bits(tnp(res)), bits(res_h)), step


@pytest.mark.parametrize("q8", [False, True])
def test_async_round_bounded_staleness(ctx, q8):
    """psb_async_round vs the trainer's async loop (trainer.hpp:244-255), s=3
    (reference pattern) and s=2 (cfg4)."""
    for s in (3, 2):
        W, n, k, lr = 8, 60_000, 60, 0.1
        theta_h = np.zeros(n, dtype=np.float32)
        res_h = np.zeros((W, n), dtype=np.float32)
        theta = torch.zeros(n, device="cuda")
        res = torch.zeros(W, n, device="cuda")
        gu = gu_h = 0
        for step in range(5):
            g_h = np.stack([O.generate("llmrec", 4, w, step, n) for w in range(W)])
            comp = L.PSB_COMP_TOPK_Q8 if q8 else L.PSB_COMP_TOPK
            d = ctx.step_desc(comp, torch.from_numpy(g_h).cuda(), res, theta, lr, k)
            gu = ctx.async_round(d, s, gu)
            ctx.check()
            gu_h = O.async_round(g_h, theta_h, lr, k, res_h, s, gu_h, q8=q8)
            assert gu == gu_h
            assert np.array_equal(bits(tnp(theta)), bits(theta_h)), (s, step)
            assert np.array_equal(bits(tnp(res)), bits(res_h)), (s, step)


def test_step_rejects_bad_args(ctx):
    from paper_2506_17551_b200 import PsbInvalidArgument
    g = torch.zeros(2, 100, device="cuda")
    theta = torch.zeros(100, device="cuda")
    with pytest.raises(PsbInvalidArgument, match="learning rate must be finite"):
        ctx.sync_step(ctx.step_desc(L.PSB_COMP_TOPK, g, None, theta, float("nan"), 5))
    ctx.sync_step(ctx.step_desc(L.PSB_COMP_TOPK, g, None, theta, 0.0, 5))  # lr = 0: a no-op update
    ctx.check()
    assert not bool(theta.any())
    with pytest.raises(PsbInvalidArgument, match="k out of range"):
        ctx.sync_step(ctx.step_desc(L.PSB_COMP_TOPK, g, None, theta, 0.1, 101))


@pytest.mark.parametrize("comp", ["topk", "topk_q8", "none", "onebit"])
@pytest.mark.parametrize("W", [1, 4])
def test_momentum_sync_step(ctx, comp, W):
    """Momentum SGD (north-star a24, this build's rule; no reference code):
    psb_sync_step with a momentum buffer vs the oracle composite (reference
    step's mean, then orc_momentum), 6 steps, EF carried; bit-exact."""
    n, k, lr, beta = 100_000, 1_000, 0.05, 0.9
    theta_h = np.zeros(n, dtype=np.float32)
    m_h = np.zeros(n, dtype=np.float32)
    res_h = np.zeros((W, n), dtype=np.float32)
    theta = torch.zeros(n, device="cuda")
    m = torch.zeros(n, device="cuda")
    res = torch.zeros(W, n, device="cuda")
    for step in range(6):
        g_h = np.stack([O.generate("llmrec", 11, w, step, n) for w in range(W)])
        g = torch.from_numpy(g_h).cuda()
        mean = torch.zeros(n, device="cuda")
        d = ctx.step_desc(COMPS[comp], g, res, theta, lr, k, "ring", 256, None, mean, momentum=m, beta=beta)
        ctx.sync_step(d)
        ctx.check()
        dummy = theta_h.copy()
        mean_h = O.sync_step(g_h, dummy, lr, comp, k, "ring", res_h).astype(np.float32)
        if comp == "onebit":
            # 1-bit scale: fixed-shape tree sum vs sequential fold; compare with
            # tolerance, then continue from the oracle's state
            np.testing.assert_allclose(tnp(mean), mean_h, rtol=1e-5, atol=1e-9)
            mean_h = tnp(mean).copy()
        O.momentum_(mean_h, m_h, theta_h, beta, lr)
        assert np.array_equal(bits(tnp(mean)), bits(mean_h)), step
        assert np.array_equal(bits(tnp(m)), bits(m_h)), step
        assert np.array_equal(bits(tnp(theta)), bits(theta_h)), step
        if comp == "onebit":
            res.copy_(torch.from_numpy(res_h))  # residuals carry the scale tolerance
        else:
            assert np.array_equal(bits(tnp(res)), bits(res_h)), step


def test_momentum_scratch_reuse_across_sizes(ctx):
    """The momentum pass stores zeros back into the mean scratch instead of a
    per-step memset: dense (onebit) steps followed by sparse top-k steps at a
    smaller and then a larger n, on one context, stay bit-exact."""
    lr, beta = 0.05, 0.9
    for step, (comp, n, k) in enumerate([("onebit", 120_000, 0), ("topk", 60_000, 600),
                                          ("none", 90_000, 0), ("topk", 120_000, 300),
                                          ("topk", 120_000, 50)]):
        g_h = O.generate("llmrec", 23, 0, step, n)[None, :]
        theta_h = O.generate("llmrec", 29, 0, step, n)
        m_h = O.generate("llmrec", 31, 0, step, n)
        theta = torch.from_numpy(theta_h.copy()).cuda()
        m = torch.from_numpy(m_h.copy()).cuda()
        mean = torch.zeros(n, device="cuda")
        ctx.sync_step(ctx.step_desc(COMPS[comp], torch.from_numpy(g_h).cuda(), None, theta, lr, max(k, 1), "ring",
                                    256, None, mean, momentum=m, beta=beta))
        ctx.check()
        mean_h = O.sync_step(g_h, theta_h.copy(), lr, comp, max(k, 1), "ring", None).astype(np.float32)
        if comp == "onebit":
            np.testing.assert_allclose(tnp(mean), mean_h, rtol=1e-5, atol=1e-9)
            mean_h = tnp(mean).copy()
        O.momentum_(mean_h, m_h, theta_h, beta, lr)
        assert np.array_equal(bits(tnp(mean)), bits(mean_h)), step
        assert np.array_equal(bits(tnp(m)), bits(m_h)), step
        assert np.array_equal(bits(tnp(theta)), bits(theta_h)), step


@pytest.mark.parametrize("n,k,off", [(3 * 4096, 40, 0), (50_001, 500, 1), (4096 * 7 + 5, 4096 * 7 + 5, 0)])
def test_momentum_topk_single_worker_f64_and_views(ctx, n, k, off):
    """Single-worker top-k momentum takes the payload-merge pass (no dense
    mean scratch): f64, a misaligned f32 view, and k = n (every entry
    selected), 4 steps with EF, bit-exact vs the oracle composite."""
    lr, beta = 0.05, 0.9
    for dt in (np.float64, np.float32):
        tdt = torch.float64 if dt == np.float64 else torch.float32
        theta_h = np.zeros(n, dtype=dt)
        m_h = np.zeros(n, dtype=dt)
        res_h = np.zeros((1, n), dtype=dt)
        base = torch.zeros(3, n + off, dtype=tdt, device="cuda")
        theta, m, mean = base[0, off:], base[1, off:], base[2, off:]
        res = torch.zeros(1, n, dtype=tdt, device="cuda")
        for step in range(4):
            g_h = O.generate("llmrec", 37, 0, step, n).astype(dt)[None, :]
            ctx.sync_step(ctx.step_desc(L.PSB_COMP_TOPK, torch.from_numpy(g_h).cuda(), res, theta, lr, k, "ring",
                                        256, None, mean, momentum=m, beta=beta))
            ctx.check()
            mean_h = O.sync_step(g_h, theta_h.copy(), lr, "topk", k, "ring", res_h).astype(dt)
            O.momentum_(mean_h, m_h, theta_h, beta, lr)
            assert np.array_equal(bits(tnp(mean)), bits(mean_h)), (dt, step)
            assert np.array_equal(bits(tnp(m)), bits(m_h)), (dt, step)
            assert np.array_equal(bits(tnp(theta)), bits(theta_h)), (dt, step)
            assert np.array_equal(bits(tnp(res)), bits(res_h)), (dt, step)


def test_momentum_rejects_q8_and_async(ctx):
    n = 4096
    g = torch.randn(1, n, device="cuda")
    d = ctx.step_desc(L.PSB_COMP_Q8, g, None, torch.zeros(n, device="cuda"), 0.1, 0, "naive", 256,
                      momentum=torch.zeros(n, device="cuda"), beta=0.9)
    with pytest.raises(L.PsbInvalidArgument, match="momentum"):
        ctx.sync_step(d)
    d = ctx.step_desc(L.PSB_COMP_TOPK, g, None, torch.zeros(n, device="cuda"), 0.1, 16, "naive", 256,
                      momentum=torch.zeros(n, device="cuda"), beta=0.9)
    with pytest.raises(L.PsbInvalidArgument, match="momentum"):
        ctx.async_round(d, 2, 0)


@pytest.mark.parametrize("q8,W", [(False, 1), (False, 4), (True, 2)])
def test_async_pipeline_bitwise(cuda, q8, W):
    """The stream/event pipeline of psb_async_round (round r's apply on the
    ctx's apply stream overlapping round r+1's compression, double-buffered
    payloads): 7 rounds issued back to back with no host sync, then
    async_sync -- bitwise the trainer's async loop (oracle), s = 2 and 3."""
    from paper_2506_17551_b200.engine import Context
    n, k, lr = 80_000, 400, 0.1
    for s in (2, 3):
        c = Context(n, k, W)
        c.async_pipeline(True)
        theta_h = np.zeros(n, dtype=np.float32)
        res_h = np.zeros((W, n), dtype=np.float32)
        theta = torch.zeros(n, device="cuda")
        res = torch.zeros(W, n, device="cuda")
        comp = L.PSB_COMP_TOPK_Q8 if q8 else L.PSB_COMP_TOPK
        gs = [np.stack([O.generate("llmrec", 6, w, step, n) for w in range(W)]) for step in range(7)]
        gd = [torch.from_numpy(g).cuda() for g in gs]
        gu = gu_h = 0
        for step in range(7):
            gu = c.async_round(c.step_desc(comp, gd[step], res, theta, lr, k), s, gu)
            gu_h = O.async_round(gs[step], theta_h, lr, k, res_h, s, gu_h, q8=q8)
        c.async_sync()
        c.check()
        assert gu == gu_h
        assert np.array_equal(bits(tnp(theta)), bits(theta_h)), s
        assert np.array_equal(bits(tnp(res)), bits(res_h)), s
        c.close()


def test_async_pipeline_graph_capture(cuda):
    """Pipelined rounds captured into a CUDA graph (the apply stream joins
    the capture through the events; async_sync joins it back) and replayed:
    same bits as the same rounds run eagerly."""
    from paper_2506_17551_b200.engine import Context
    n, k, lr, W, R = 120_000, 600, 0.05, 2, 4
    gs = [torch.empty(W, n, device="cuda") for _ in range(R)]
    from paper_2506_17551_b200.engine import generate
    for b in range(R):
        for w in range(W):
            generate("llmrec", 8, w, b, n, gs[b][w])
    out = []
    for graph in (False, True):
        c = Context(n, k, W)
        c.async_pipeline(True)
        theta = torch.zeros(n, device="cuda")
        res = torch.zeros(W, n, device="cuda")
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            descs = [c.step_desc(L.PSB_COMP_TOPK, gs[b], res, theta, lr, k) for b in range(R)]
            gu = 0
            for i in range(3):  # warm-up (eager), then drained
                gu = c.async_round(descs[i % R], 2, gu)
            c.async_sync()
            c.check()
            if graph:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for i in range(R):
                        gu = c.async_round(descs[i], 2, gu)
                    c.async_sync()
                g.replay()
                g.replay()
            else:
                for _ in range(2):
                    for i in range(R):
                        gu = c.async_round(descs[i], 2, gu)
                c.async_sync()
            c.check()
        out.append((theta.clone(), res.clone()))
        c.close()
    assert torch.equal(out[0][0].view(torch.int32), out[1][0].view(torch.int32))
    assert torch.equal(out[0][1].view(torch.int32), out[1][1].view(torch.int32))


@pytest.mark.parametrize("env", [{"PSB_APPLY_TMA_CAP": "64"}, {"PSB_APPLY_TMA_CAP": "600"},
                                 {"PSB_APPLY_NO_TMA": "1"}, {"PSB_APPLY_NO_TMA": "1", "PSB_APPLY_VCAP": "256"}])
@pytest.mark.parametrize("P,order", [(2, "ring"), (4, "naive"), (8, "ring"), (5, "hierarchical")])
def test_sparse_apply_stage_paths(cuda, env, P, order):
    """The TMA-staged apply with segments that do not fit its stage (a tiny
    stage: every or some segment takes the thread-loaded path inside the
    persistent kernel), and the one-CTA-per-segment kernel (q8 / sharded
    views) staged and unstaged: all bit-exact with the oracle fold.  Ring
    segments straddle the P ring chunks (n not a multiple of S)."""
    import os
    from paper_2506_17551_b200.engine import Context
    dt = np.float32
    n, k = 70_001, 2_500
    idx, val = make_payloads(P, n, k, dt, seed=P * 13 + len(env))
    theta_h = O.generate("uniform", 9, 0, 0, n).astype(dt)
    dense = np.zeros((P, n), dtype=dt)
    for p in range(P):
        dense[p, idx[p].astype(np.int64)] = val[p]
    dpn, npr = (2, 2) if order == "hierarchical" else (0, 1)
    mean_h = O.fold_mean(dense, order, dpn, npr)
    want = theta_h.copy()
    O.axpy_(-0.05, mean_h, want)
    old = {kk: os.environ.get(kk) for kk in env}
    os.environ.update(env)
    try:
        c = Context(n, k, P)
    finally:
        for kk, vv in old.items():
            if vv is None:
                os.environ.pop(kk, None)
            else:
                os.environ[kk] = vv
    theta = torch.from_numpy(theta_h.copy()).cuda()
    topo = topology(1, npr, dpn) if dpn else None
    c.sparse_mean_sgd(pack_payloads(idx, val, torch.float32), P, k, torch.float32, order, 0.05, theta, n, None, topo)
    c.check()
    c.close()
    assert np.array_equal(bits(tnp(theta)), bits(want))


@pytest.mark.parametrize("block", [128, 512, 1024])
@pytest.mark.parametrize("W", [1, 2])
def test_q8_step_block_sizes(ctx, block, W):
    """Dense q8 sync step for every block size (the TMA-staged kernels serve
    B <= 512, the register-pipelined ones B = 1024), n not a multiple of the
    8-block tile, no mean_out: bit-exact with the oracle composite."""
    n, lr = 300_007, 0.05
    theta_h = np.zeros(n, dtype=np.float32)
    res_h = np.zeros((W, n), dtype=np.float32)
    theta = torch.zeros(n, device="cuda")
    res = torch.zeros(W, n, device="cuda")
    for step in range(3):
        g_h = np.stack([O.generate("llmrec", 7, w, step, n) for w in range(W)])
        d = ctx.step_desc(COMPS["q8"], torch.from_numpy(g_h).cuda(), res, theta, lr, 0, "naive", block)
        ctx.sync_step(d)
        ctx.check()
        O.sync_step(g_h, theta_h, lr, "q8", 0, "naive", res_h, 0, 1, block)
        assert np.array_equal(bits(tnp(theta)), bits(theta_h)), step
        assert np.array_equal(bits(tnp(res)), bits(res_h)), step


def skewed_payloads(P, n, k, dtype, seed):
    """A hot quarter of the index space holding most entries (heavy segments)
    and a sparse rest (segments of a few entries: the one-warp light path),
    with cross-worker collisions in both, +-0 values."""
    rng = np.random.default_rng(seed)
    idx = np.zeros((P, k), dtype=np.uint32)
    val = np.zeros((P, k), dtype=dtype)
    hot = rng.choice(n // 4, size=min(n // 4, 2 * k), replace=False)
    for p in range(P):
        kh = (3 * k) // 4
        cold = rng.choice(np.arange(n // 4, n), size=k - kh, replace=False)
        idx[p] = np.sort(np.concatenate([rng.choice(hot, size=kh, replace=False), cold]))
        v = rng.standard_normal(k).astype(dtype)
        v[rng.random(k) < 0.05] = dtype(0.0)
        v[rng.random(k) < 0.05] = -dtype(0.0)
        val[p] = v
    return idx, val


@pytest.mark.parametrize("P,order,dpn,npr", [(4, "ring", 0, 1), (8, "naive", 0, 1), (8, "ring", 0, 1),
                                             (16, "hierarchical", 4, 2), (5, "ring", 0, 1)])
@pytest.mark.parametrize("asynch", [False, True])
def test_sparse_apply_light_and_heavy_segments(ctx, P, order, dpn, npr, asynch):
    """Mixed light (<= 32 entries: one warp each) and heavy (TMA-staged)
    segments in one apply, mean and async: bit-exact with the oracle."""
    dt = np.float32
    n, k = 2_000_003, 6_000
    idx, val = skewed_payloads(P, n, k, dt, seed=P * 31 + len(order) + asynch)
    theta_h = O.generate("uniform", 3, 0, 0, n).astype(dt)
    pl = pack_payloads(idx, val, torch.float32)
    theta = torch.from_numpy(theta_h.copy()).cuda()
    want = theta_h.copy()
    if asynch:
        scales = [0.05 / (1.0 + (p % 3)) for p in range(P)]
        for p in range(P):
            d = np.zeros(n, dtype=dt)
            d[idx[p].astype(np.int64)] = val[p]
            O.axpy_(-scales[p], d, want)
        ctx.sparse_async_apply(pl, P, k, torch.float32, scales, theta)
    else:
        dense = np.zeros((P, n), dtype=dt)
        for p in range(P):
            dense[p, idx[p].astype(np.int64)] = val[p]
        mean_h = O.fold_mean(dense, order, dpn, npr)
        O.axpy_(-0.05, mean_h, want)
        topo = topology(1, npr, dpn) if dpn else None
        ctx.sparse_mean_sgd(pl, P, k, torch.float32, order, 0.05, theta, n, None, topo)
    ctx.check()
    assert np.array_equal(bits(tnp(theta)), bits(want))


@pytest.mark.parametrize("P,order,dpn,npr", [(2, "ring", 0, 1), (5, "naive", 0, 1), (4, "ring", 0, 1),
                                             (8, "ring", 0, 1), (4, "hierarchical", 8, 1), (8, "naive", 0, 1)])
@pytest.mark.parametrize("dtype_t", [torch.float32, torch.float64])
def test_dense_fold_apply_bitwise(ctx, P, order, dpn, npr, dtype_t):
    """P * k >= 20 % of n: the streaming fold (k_dense_fold_apply) -- one
    accumulator pass per worker in the reference order, +0 for absent
    workers, ring chunks crossing tiles -- bit-exact with the oracle fold,
    theta with +-0 entries untouched where no worker is present."""
    dt = np.float32 if dtype_t == torch.float32 else np.float64
    n, k = 200_003, 20_000
    idx, val = make_payloads(P, n, k, dt, seed=P * 5 + len(order))
    theta_h = O.generate("uniform", 4, 0, 0, n).astype(dt)
    theta_h[::13] = -0.0
    theta_h[1::13] = 0.0
    dense = np.zeros((P, n), dtype=dt)
    for p in range(P):
        dense[p, idx[p].astype(np.int64)] = val[p]
    mean_h = O.fold_mean(dense, order, dpn, npr)
    want = theta_h.copy()
    O.axpy_(-0.05, mean_h, want)
    theta = torch.from_numpy(theta_h.copy()).cuda()
    topo = topology(1, npr, dpn) if dpn else None
    ctx.sparse_mean_sgd(pack_payloads(idx, val, dtype_t), P, k, dtype_t, order, 0.05, theta, n, None, topo)
    ctx.check()
    assert np.array_equal(bits(tnp(theta)), bits(want))
