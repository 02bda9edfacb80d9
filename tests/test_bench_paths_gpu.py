"""GPU parity of the kernel paths the bench configs run at their real sizes.

The small-size tests (test_topk_gpu.py, test_apply_gpu.py) compare against
the oracle bit for bit; these cover what they cannot reach:

* k_cand's unstaged candidate slice (psb_cand.inl: a CTA's slice exceeds the
  shared-memory stage -- every rho >= ~2% call at 125M and the cfg5 rho = 10%
  rows), forced with PSB_NO_STAGE=1 at oracle size and reached naturally at
  32M / 125M with rho = 10%;
* cfg4 at its bench size (350M, top-k 0.1% + int8 values, async s = 2);
* the step driver's argument checks (buffers reach the C ABI as
  bare pointers, so a wrong dtype/size must be rejected on the host).

At full size the bar is the exact selection rule (reference
parsim/compression.hpp:81-99: the k largest |p|, ties to the lower index),
the EF residual (:150-154: selected ? +0 : p, or p - code*scale for int8
values) and the SGD update (numerics.hpp:70-78: RN(RN(-lr * v) + theta)),
recomputed independently here with torch on the device and compared bitwise.
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def tnp(t):
    return t.detach().cpu().numpy()


def bits(t):
    return t.view(torch.int32)


def expected_selection(p: torch.Tensor, k: int) -> torch.Tensor:
    """Boolean mask of the reference's top-k of |p| (stable_sort by |p| desc:
    every key > T, then the lowest-index keys == T)."""
    key = bits(p) & 0x7FFFFFFF
    T = int(torch.sort(key, descending=True).values[k - 1])
    sel = key > T
    n_gt = int(sel.sum())
    eq_idx = torch.nonzero(key == T).view(-1)
    sel[eq_idx[: k - n_gt]] = True
    assert int(sel.sum()) == k
    return sel


def check_payload(p, sel, idx, val):
    idx64 = idx.long()
    want = torch.nonzero(sel).view(-1)
    assert torch.equal(idx64, want)  # index set and ascending order
    assert torch.equal(bits(val), bits(p[want]))


def run_ef_sequence(ctx, n, k, steps, dist="llmrec", worker=0, fused=False, lr=0.05):
    """Bitwise vs the oracle: `steps` EF top-k calls (fused=True: through the
    P = 1 sync step, i.e. the payload write + residual fix-up + theta update
    of k_cand)."""
    from paper_2506_17551_b200 import _lib as L
    r_h = np.zeros(n, dtype=np.float32)
    r_d = torch.zeros(n, dtype=torch.float32, device="cuda")
    th_h = np.zeros(n, dtype=np.float32)
    th_d = torch.zeros(n, dtype=torch.float32, device="cuda")
    for s in range(steps):
        g_h = O.generate(dist, 17, worker, s, n)
        g_d = torch.from_numpy(g_h).cuda()
        if fused:
            ctx.sync_step(ctx.step_desc(L.PSB_COMP_TOPK, g_d.view(1, n), r_d.view(1, n), th_d, lr, k, "ring"))
            r2 = r_h.reshape(1, n)
            O.sync_step(g_h.reshape(1, n), th_h, lr, "topk", k, "ring", r2)
            assert np.array_equal(tnp(th_d).view(np.uint32), th_h.view(np.uint32)), s
        else:
            idx, val = ctx.ef_topk(g_d, r_d, k, worker=worker)
            oi, ov, st = O.ef_topk(g_h, r_h, k)
            assert st == 0
            assert np.array_equal(tnp(idx).view(np.uint32), oi), s
            assert np.array_equal(tnp(val).view(np.uint32), ov.view(np.uint32)), s
        assert np.array_equal(tnp(r_d).view(np.uint32), r_h.view(np.uint32)), s
    ctx.check()


@pytest.fixture(scope="module")
def ctx_nostage(cuda):
    """A context whose k_cand streams every slice from global memory (the
    branch taken when a slice exceeds the shared-memory stage)."""
    from paper_2506_17551_b200.engine import Context
    old = os.environ.get("PSB_NO_STAGE")
    os.environ["PSB_NO_STAGE"] = "1"
    try:
        c = Context(max_n=1 << 21, max_k=1 << 18, max_workers=2)
    finally:
        if old is None:
            del os.environ["PSB_NO_STAGE"]
        else:
            os.environ["PSB_NO_STAGE"] = old
    yield c
    c.close()


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("n,k,dist", [(1_000_000, 10_000, "llmrec"), (1_000_000, 100_000, "llmrec"),
                                      (333_333, 33_333, "ties"), (65_537, 6_554, "uniform")])
def test_unstaged_slice_bitwise(ctx_nostage, n, k, dist, fused):
    """10 EF steps through k_cand's unstaged branch, bitwise vs the oracle
    (indices, values, residuals, and theta when fused)."""
    run_ef_sequence(ctx_nostage, n, k, 10, dist, worker=1 if fused else 0, fused=fused)


@pytest.mark.parametrize("n,rho", [(32_000_000, 0.10), (125_000_000, 0.10), (125_000_000, 0.03)])
def test_unstaged_slice_full_size(cuda, n, rho):
    """cfg5 rows whose candidate slices exceed the stage (rho = 10% at 32M and
    125M, rho = 3% at 125M): 3 fused sync steps at one rank, checked against
    the selection rule, residual rule and SGD update recomputed with torch."""
    from paper_2506_17551_b200 import _lib as L
    from paper_2506_17551_b200.engine import Context, generate
    k = int(round(rho * n))
    lr = 0.05
    c = Context(n, k, 1)
    g = torch.empty(n, device="cuda")
    r = torch.zeros(n, device="cuda")
    theta = torch.zeros(n, device="cuda")
    mean = torch.zeros(n, device="cuda")
    coef = torch.tensor(-lr, dtype=torch.float32, device="cuda")
    for step in range(3):
        generate("llmrec", 42, 0, step, n, g)
        p = r + g
        th0 = theta.clone()
        mean.zero_()
        c.sync_step(c.step_desc(L.PSB_COMP_TOPK, g.view(1, n), r.view(1, n), theta, lr, k, "ring",
                                mean_out=mean))
        c.check()
        sel = expected_selection(p, k)
        assert torch.equal(bits(r), bits(torch.where(sel, torch.zeros_like(p), p))), step
        assert torch.equal(bits(mean), bits(torch.where(sel, p, torch.zeros_like(p)))), step
        upd = th0 + coef * p  # two rounded torch ops: RN(RN(-lr * v) + theta)
        assert torch.equal(bits(theta), bits(torch.where(sel, upd, th0))), step
        st = c.topk_stats(0)
        assert st["candidates"] >= k
        del p, sel, upd, th0
    c.close()


def test_cfg4_bench_size_topk_q8_async(cuda):
    """cfg4 at its bench size: 350M, top-k 0.1% with int8 values, async
    bounded staleness s = 2 (one worker: tau = 0).  Per round: the selection
    rule on p = r + g, codes/scales = the 8-bit rule over the payload values
    in blocks of 128 (oracle orc_q8_quant), residual p - code*scale at the
    selected indices and p elsewhere, theta += RN(-lr * xhat)."""
    from paper_2506_17551_b200 import _lib as L
    from paper_2506_17551_b200.engine import Context, generate
    n, k, lr = 350_000_000, 350_000, 0.05
    c = Context(n, k, 1)
    g = torch.empty(n, device="cuda")
    r = torch.zeros(n, device="cuda")
    theta = torch.zeros(n, device="cuda")
    coef = torch.tensor(-lr, dtype=torch.float32, device="cuda")
    gu = 0
    for step in range(3):
        generate("llmrec", 42, 0, step, n, g)
        p = r + g
        th0 = theta.clone()
        gu = c.async_round(c.step_desc(L.PSB_COMP_TOPK_Q8, g.view(1, n), r.view(1, n), theta, lr, k, "naive"),
                           2, gu)
        c.check()
        assert gu == step + 1
        sel = expected_selection(p, k)
        want = torch.nonzero(sel).view(-1)
        v = tnp(p[want]).astype(np.float32)
        codes, scales, st = O.q8_quant(v, None, 128)
        assert st == 0
        xhat = torch.from_numpy(O.q8_dequant(codes, scales, 128)).cuda()
        res_sel = torch.from_numpy(v).cuda() - xhat
        exp_r = p.clone()
        exp_r[want] = res_sel
        assert torch.equal(bits(r), bits(exp_r)), step
        exp_t = th0.clone()
        exp_t[want] = th0[want] + coef * xhat
        assert torch.equal(bits(theta), bits(exp_t)), step
        del p, sel, exp_r, exp_t, th0
    # the int8 payload itself through the compressor entry point, same size
    generate("llmrec", 42, 0, 9, n, g)
    r2 = r.clone()
    p = r2 + g
    idx, codes_d, scales_d = c.ef_topk_q8(g, r2, k)
    c.check()
    sel = expected_selection(p, k)
    want = torch.nonzero(sel).view(-1)
    assert torch.equal(idx.long(), want)
    codes, scales, _ = O.q8_quant(tnp(p[want]).astype(np.float32), None, 128)
    assert np.array_equal(tnp(codes_d), codes)
    assert np.array_equal(tnp(scales_d).view(np.uint32), scales.view(np.uint32))
    c.close()


def test_step_desc_rejects_mismatched_buffers(ctx):
    """Buffers reach the C ABI as bare pointers: a wrong dtype or size is a
    host-side PsbInvalidArgument, never an out-of-bounds device write."""
    from paper_2506_17551_b200 import _lib as L
    n = 4096
    g = torch.zeros(2, n, dtype=torch.float64, device="cuda")
    r = torch.zeros(2, n, dtype=torch.float64, device="cuda")
    th = torch.zeros(n, dtype=torch.float64, device="cuda")
    bad = [
        dict(theta=torch.zeros(n, device="cuda")),                                # f32 theta, f64 g
        dict(momentum=torch.zeros(n, device="cuda")),                             # f32 momentum
        dict(theta=torch.zeros(n - 1, dtype=torch.float64, device="cuda")),       # short theta
        dict(r=torch.zeros(1, n, dtype=torch.float64, device="cuda")),            # r not [W][n]
        dict(mean_out=torch.zeros(2 * n, dtype=torch.float64, device="cuda")),    # mean_out size
    ]
    for kw in bad:
        args = dict(theta=th, r=r)
        args.update(kw)
        mom = args.pop("momentum", None)
        mean = args.pop("mean_out", None)
        with pytest.raises(L.PsbInvalidArgument, match="step_desc"):
            ctx.step_desc(L.PSB_COMP_TOPK, g, args["r"], args["theta"], 0.1, 16, "naive",
                          mean_out=mean, momentum=mom, beta=0.9 if mom is not None else 0.0)
    ctx.step_desc(L.PSB_COMP_TOPK, g, r, th, 0.1, 16, "naive")  # consistent buffers pass


def test_decompress_validation(ctx):
    """decompress (compression.hpp:113-142): dense scatter, and the reference's
    errors for an index >= dim and for indices not strictly increasing
    (test_compression.cpp:62-79) through the device kernel."""
    from paper_2506_17551_b200 import _lib as L
    idx = torch.tensor([1, 3], dtype=torch.int32, device="cuda")
    val = torch.tensor([-2.0, 1.0], dtype=torch.float64, device="cuda")
    out = ctx.decompress_topk(idx, val, 4)
    ctx.check()
    assert tnp(out).tolist() == [0.0, -2.0, 0.0, 1.0]
    ctx.decompress_topk(torch.tensor([1, 7], dtype=torch.int32, device="cuda"), val, 4)
    with pytest.raises(L.PsbInvalidArgument, match="out of range"):
        ctx.check()
    ctx.decompress_topk(torch.tensor([3, 1], dtype=torch.int32, device="cuda"), val, 4)
    with pytest.raises(L.PsbInvalidArgument, match="strictly increasing"):
        ctx.check()
    ctx.decompress_topk(torch.tensor([2, 2], dtype=torch.int32, device="cuda"), val, 4)
    with pytest.raises(L.PsbInvalidArgument, match="strictly increasing"):
        ctx.check()
    ctx.check()  # flags cleared


def test_wire_decode_keeps_step_flags(ctx):
    """A failed wire_decode reports only its own error: a non-finite flag left
    by earlier async work survives for the caller's next check."""
    from paper_2506_17551_b200 import PsbNonFinite
    from paper_2506_17551_b200 import _lib as L
    g = torch.ones(1000, device="cuda")
    g[3] = float("inf")
    r = torch.zeros(1000, device="cuda")
    ctx.ef_topk(g, r, 10, worker=9)          # raises the sticky non-finite flag
    buf = torch.zeros(20, dtype=torch.uint8, device="cuda")
    buf[0] = 4
    buf[8] = 2                                # count 2 but only 4 payload bytes: truncated
    with pytest.raises(L.PsbInvalidArgument, match="truncated"):
        ctx.wire_decode_topk(buf, torch.float32, k_cap=4)
    with pytest.raises(PsbNonFinite):
        ctx.check()
    ctx.check()


@pytest.mark.parametrize("n,k", [(1_000_003, 100_000), (600_001, 30_001), (4096 * 50, 4096 * 5)])
def test_dense_payload_fused_update_bitwise(ctx, n, k):
    """rho 5-10 % at one worker through the fused P = 1 step (K1's scattered
    theta update at a dense payload) -- bitwise the oracle's sync step over
    several EF steps."""
    run_ef_sequence(ctx, n, k, 4, fused=True)


def test_dense_payload_fused_update_full_size(cuda):
    """cfg5 rho = 10 % at 125M, fused step without mean_out, theta with -0
    entries: theta = RN(RN(-lr * v) + theta) at the selected indices,
    bit-for-bit untouched elsewhere."""
    from paper_2506_17551_b200 import _lib as L
    from paper_2506_17551_b200.engine import Context, generate
    n = 125_000_000
    k = n // 10
    lr = 0.05
    c = Context(n, k, 1)
    g = torch.empty(n, device="cuda")
    r = torch.zeros(n, device="cuda")
    theta = torch.empty(n, device="cuda")
    generate("uniform", 9, 1, 0, n, theta)
    theta[::7] = -0.0
    coef = torch.tensor(-lr, dtype=torch.float32, device="cuda")
    for step in range(2):
        generate("llmrec", 42, 0, step, n, g)
        p = r + g
        th0 = theta.clone()
        c.sync_step(c.step_desc(L.PSB_COMP_TOPK, g.view(1, n), r.view(1, n), theta, lr, k, "ring"))
        c.check()
        sel = expected_selection(p, k)
        assert torch.equal(bits(r), bits(torch.where(sel, torch.zeros_like(p), p))), step
        upd = th0 + coef * p
        assert torch.equal(bits(theta), bits(torch.where(sel, upd, th0))), step
        del p, sel, upd, th0
    c.close()
