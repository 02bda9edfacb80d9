"""The gradient producer that feeds the path: device
bpr_batch_gradient / bpr_batch_loss (psb_bpr.cu) against the reference
itself (oracle/_ref, parsim/trainer.hpp:98-138), then fed into psb_sync_step.

Tolerance: the device exp() is within 1 ulp of glibc's, so the per-triple
coefficient may differ by an ulp; with exp(0) (user rows zero) the gradient is
bit-exact.  Structure (which rows are touched) is always exact."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2506_17551_b200 import _lib as L

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]


def _batch(rng, users, items, B):
    u = rng.integers(0, users, B).astype(np.uint32)
    p = rng.integers(0, items, B).astype(np.uint32)
    q = rng.integers(0, items, B).astype(np.uint32)
    q[::17] = p[::17]  # the sampler's fallback: negative == positive
    u[1::5] = u[0]     # heavy user repeats
    return u, p, q


def _dev(*arrs):
    return [torch.from_numpy(a.view(np.int32)).cuda() for a in arrs]


@pytest.mark.parametrize("users,items,dim,B,scale", [(50, 80, 16, 256, 0.01), (7, 5, 40, 64, 1.0),
                                                       (1000, 5000, 32, 4096, 0.3)])
def test_bpr_gradient_matches_reference(ctx, users, items, dim, B, scale):
    rng = np.random.default_rng(users * 7 + B)
    theta_h = rng.uniform(-scale, scale, (users + items) * dim)
    u, p, q = _batch(rng, users, items, B)
    g_ref, loss_ref = O.ref_bpr_batch_gradient(theta_h, users, items, dim, u, p, q)
    theta = torch.from_numpy(theta_h).cuda()
    grad, loss = ctx.bpr_gradient(theta, users, items, dim, *_dev(u, p, q))
    ctx.check()
    g = grad.cpu().numpy()
    assert np.array_equal(g != 0, g_ref != 0)
    np.testing.assert_allclose(g, g_ref, rtol=1e-12, atol=1e-300)
    assert float(loss.item()) == pytest.approx(loss_ref, rel=1e-13)


def test_bpr_gradient_bit_exact_when_exp_is_exact(ctx):
    """x = 0 for every triple (user rows zero): exp(0) = 1 exactly, so every
    coefficient is -0.5/B and the whole gradient must match bit for bit --
    this pins the per-row batch-order accumulation."""
    users, items, dim, B = 30, 40, 24, 512
    rng = np.random.default_rng(3)
    theta_h = rng.uniform(-1, 1, (users + items) * dim)
    theta_h[:users * dim] = 0.0
    u, p, q = _batch(rng, users, items, B)
    g_ref, _ = O.ref_bpr_batch_gradient(theta_h, users, items, dim, u, p, q)
    grad, _ = ctx.bpr_gradient(torch.from_numpy(theta_h).cuda(), users, items, dim, *_dev(u, p, q))
    ctx.check()
    assert np.array_equal(grad.cpu().numpy().view(np.uint64), g_ref.view(np.uint64))


def test_bpr_errors(ctx):
    theta = torch.zeros((4 + 4) * 8, dtype=torch.float64, device="cuda")
    u, p, q = _dev(np.array([0, 1], np.uint32), np.array([0, 4], np.uint32), np.array([1, 2], np.uint32))
    with pytest.raises(L.PsbInvalidArgument, match="out of range"):
        ctx.bpr_gradient(theta, 4, 4, 8, u, p, q)
        ctx.check()


def test_producer_feeds_the_step(ctx):
    """GPU-produced BPR gradients (f32) of 4 virtual workers through
    psb_sync_step (EF top-k, ring) for 5 steps: theta and residuals bit-exact
    against the oracle composite on the same gradients."""
    users, items, dim, B, W, k, lr = 200, 300, 16, 256, 4, 200, 0.05
    n = (users + items) * dim
    rng = np.random.default_rng(11)
    theta_h = rng.uniform(-0.01, 0.01, n).astype(np.float32)
    theta = torch.from_numpy(theta_h.copy()).cuda()
    res = torch.zeros(W, n, device="cuda")
    res_h = np.zeros((W, n), dtype=np.float32)
    for step in range(5):
        g = torch.empty(W, n, device="cuda")
        for w in range(W):
            ctx.bpr_gradient(theta, users, items, dim, *_dev(*_batch(rng, users, items, B)), grad=g[w],
                             want_loss=False)
        ctx.check()
        g_h = g.cpu().numpy()
        d = ctx.step_desc(L.PSB_COMP_TOPK, g, res, theta, lr, k, "ring")
        ctx.sync_step(d)
        ctx.check()
        O.sync_step(g_h, theta_h, lr, "topk", k, "ring", res_h)
        assert np.array_equal(theta.cpu().numpy().view(np.uint32), theta_h.view(np.uint32)), step
        assert np.array_equal(res.cpu().numpy().view(np.uint32), res_h.view(np.uint32)), step
