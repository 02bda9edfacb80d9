"""The trainer around the device path against the
reference's own train() (parsim/trainer.hpp:197-261, via oracle/_ref): same
RecModel init, same triple stream, gradients and updates on the B200.
Tolerance: the device exp() may differ from glibc's by an ulp per triple."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2506_17551_b200 import train as T

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]


def test_sampler_and_init_match_reference_stream():
    """The host draws are the reference's: RecModel::init values and the
    SplitMix64 KAT (test_numerics.cpp:66-77 seed 0)."""
    rng = T.SeededRng(0)
    ref = np.empty(4, dtype=np.uint64)
    O.ref().ref_splitmix_stream(0, 4, ref.ctypes.data)
    assert [rng.next_u64() for _ in range(4)] == [int(x) for x in ref]


@pytest.mark.parametrize("mode,kind,k,P", [("sync", "none", 0, 2), ("sync", "topk", 30, 2), ("sync", "topk", 30, 4),
                                           ("async", "topk", 30, 4), ("async", "none", 0, 2),
                                           ("sync", "onebit", 0, 2), ("async", "onebit", 0, 4)])
def test_train_matches_reference(mode, kind, k, P):
    users, items, dim, steps, batch, lr, seed = 30, 50, 8, 120, 32, 0.05, 7
    rng = np.random.default_rng(1)
    tu = rng.integers(0, users, 300)
    ti = rng.integers(0, items, 300)
    theta_ref, curve_ref = O.ref_train(users, items, dim, tu, ti, P, mode, steps, batch, lr, kind, k, "ring", seed)
    out = T.train(users, items, dim, tu, ti, P, steps, batch, lr, kind, k, "ring", mode, seed)
    got = out.theta.cpu().numpy()
    np.testing.assert_allclose(got, theta_ref, rtol=1e-9, atol=1e-13)
    assert [s for s, _ in out.loss_curve] == [s for s, _ in curve_ref]
    for (_, a), (_, b) in zip(out.loss_curve, curve_ref):
        assert a == pytest.approx(b, rel=1e-12)


@pytest.mark.parametrize("items,negatives", [(50, 20), (12, 99)])
def test_evaluate_topk_matches_reference(items, negatives):
    """Sampled HR@10 / NDCG@10 (trainer.hpp:269-324) on a trained model,
    bit-exact against the reference (incl. the small-pool fallback and
    skipped users)."""
    users, dim, seed = 30, 8, 7
    rng = np.random.default_rng(5)
    tu, ti = rng.integers(0, users, 300), rng.integers(0, items, 300)
    vu, vi = rng.integers(0, users, 40), rng.integers(0, items, 40)
    su, si = rng.integers(0, users, 60), rng.integers(0, items, 60)
    out = T.train(users, items, dim, tu, ti, 2, 60, 32, 0.05, "topk", 30, "ring", "sync", seed)
    hr, ndcg, ne, sk = O.ref_evaluate_topk(users, items, dim, out.theta.cpu().numpy(), (tu, ti), (vu, vi), (su, si),
                                           10, negatives, 42)
    r = T.evaluate_topk(out.theta, users, items, dim, (tu, ti), (vu, vi), (su, si), 10, negatives, 42)
    assert (r.num_eval_users, r.skipped) == (ne, sk)
    assert r.hr_at_10 == hr and r.ndcg_at_10 == ndcg


def test_checkpoint_resume_is_exact(tmp_path):
    """save_model (reference PSMF format, read back by the reference's
    load_model) + the error-feedback checkpoint resume a compressed sync run
    bit-exactly: 60 + 60 steps == 120 steps."""
    users, items, dim, batch, lr, seed, P, k = 30, 50, 8, 32, 0.05, 7, 2, 30
    rng = np.random.default_rng(1)
    tu, ti = rng.integers(0, users, 300), rng.integers(0, items, 300)
    full = T.train(users, items, dim, tu, ti, P, 120, batch, lr, "topk", k, "ring", "sync", seed)
    half = T.train(users, items, dim, tu, ti, P, 60, batch, lr, "topk", k, "ring", "sync", seed)
    mpath, epath = str(tmp_path / "model.bin"), str(tmp_path / "ef.bin")
    T.save_model(mpath, half.theta, users, items, dim)
    T.save_ef_state(epath, half.residuals, half.steps_done, half.sampler_state)
    (u, i, d), th_ref = O.ref_load_model(mpath, (users + items) * dim)
    assert (u, i, d) == (users, items, dim)
    assert np.array_equal(th_ref.view(np.uint64), half.theta.cpu().numpy().view(np.uint64))
    theta, u2, i2, d2 = T.load_model(mpath)
    res, done, st = T.load_ef_state(epath)
    rest = T.train(u2, i2, d2, tu, ti, P, 60, batch, lr, "topk", k, "ring", "sync", seed, resume=(theta, res, done, st))
    assert np.array_equal(rest.theta.cpu().numpy().view(np.uint64), full.theta.cpu().numpy().view(np.uint64))
    assert np.array_equal(rest.residuals.cpu().numpy().view(np.uint64), full.residuals.cpu().numpy().view(np.uint64))
    assert rest.loss_curve == [pt for pt in full.loss_curve if pt[0] >= 60]
