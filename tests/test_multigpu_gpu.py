"""GPU, >= 2 devices: the multi-rank exchange paths (one process per GPU):
payloads over NVLink peer memory (default) or NCCL all-gather, dense/q8
paths over NCCL.

Every rank owns W local workers (worker id = rank*W + w); after each step the
replicas must be bitwise identical to each other and to the oracle composite
of sync_data_parallel_step / the async loop over all P = W*R workers.
"""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _worker(rank, nranks, uid, W, comp, order, steps, q, peer="full"):
    sys.path.insert(0, ROOT)
    try:
        import torch as th

        from oracle import oracle as O
        from paper_2506_17551_b200 import _lib as L
        from paper_2506_17551_b200.engine import Context, topology

        th.cuda.set_device(rank)
        n, k, lr = 50_000, 500, 0.05
        P = W * nranks
        c = Context(n, 2 * k, P, device=rank)
        c.comm_init(rank, nranks, uid)
        c.peer_mode(peer)
        pipe = comp.endswith("_pipe")  # stream/event pipeline of the async rounds
        comp = comp[:-5] if pipe else comp
        if pipe:
            c.async_pipeline(True)
        grow = comp == "topk_grow"  # k doubles mid-run: the peer arenas are re-created
        comp = "topk" if grow else comp
        code = {"topk": L.PSB_COMP_TOPK, "topk_q8": L.PSB_COMP_TOPK_Q8, "onebit": L.PSB_COMP_ONEBIT,
                "none": L.PSB_COMP_NONE, "q8": L.PSB_COMP_Q8, "async": L.PSB_COMP_TOPK,
                "async_q8": L.PSB_COMP_TOPK_Q8}[comp]
        dpn, npr = (2, 1) if order == "hierarchical" else (0, 1)
        topo = topology(1, npr, dpn) if dpn else None
        theta = th.zeros(n, device="cuda")
        res = th.zeros(W, n, device="cuda")
        theta_h = np.zeros(n, dtype=np.float32)
        res_h = np.zeros((P, n), dtype=np.float32)
        gu = gu_h = 0
        worst = 0.0
        for step in range(steps):
            g_all = np.stack([O.generate("llmrec", 7, p, step, n) for p in range(P)])
            g = th.from_numpy(g_all[rank * W:(rank + 1) * W].copy()).cuda()
            if grow and step == steps // 2:
                k *= 2
            d = c.step_desc(code, g, res, theta, lr, k, order, 256, topo)
            if comp.startswith("async"):
                gu = c.async_round(d, 2, gu)
                if pipe:
                    c.async_sync()
                gu_h = O.async_round(g_all, theta_h, lr, k, res_h, 2, gu_h, q8=comp == "async_q8")
            else:
                c.sync_step(d)
                O.sync_step(g_all, theta_h, lr, comp, k, order, res_h, dpn, npr, 256)
            c.check()
            if comp.startswith(("topk", "async")) and c.peer_active != (peer != "nccl"):
                q.put((rank, f"peer_active={c.peer_active}, expected {peer}"))
                return
            got = theta.cpu().numpy()
            if comp == "onebit":
                worst = max(worst, float(np.max(np.abs(got - theta_h))))
                theta.copy_(th.from_numpy(theta_h))
                res.copy_(th.from_numpy(res_h[rank * W:(rank + 1) * W]))
            else:
                if not np.array_equal(got.view(np.uint32), theta_h.view(np.uint32)):
                    q.put((rank, f"theta mismatch at step {step}"))
                    return
                if not np.array_equal(res.cpu().numpy().view(np.uint32),
                                      res_h[rank * W:(rank + 1) * W].view(np.uint32)):
                    q.put((rank, f"residual mismatch at step {step}"))
                    return
        q.put((rank, "ok" if worst < 1e-6 else f"onebit deviation {worst}"))
        c.close()
    except Exception as e:  # report, never hang the parent
        q.put((rank, f"error: {type(e).__name__}: {e}"))


def _run(nranks, W, comp, order, steps=4, peer="full"):
    from paper_2506_17551_b200.engine import Context
    uid = Context.unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, nranks, uid, W, comp, order, steps, q, peer))
             for r in range(nranks)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(nranks):
        r, msg = q.get(timeout=300)
        results[r] = msg
    for p in procs:
        p.join(timeout=60)
    return results


needs2 = pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")


@needs2
@pytest.mark.parametrize("comp,order,W", [
    ("topk", "ring", 1), ("topk", "naive", 2), ("topk", "hierarchical", 2),
    ("topk_q8", "naive", 1), ("onebit", "ring", 1), ("none", "naive", 2),
    ("q8", "naive", 1), ("q8", "ring", 2), ("async", "naive", 2), ("async_q8", "naive", 1),
    ("async_pipe", "naive", 1), ("async_pipe", "naive", 2), ("async_q8_pipe", "naive", 1),
])
def test_exchange_paths_match_oracle(comp, order, W):
    nr = min(torch.cuda.device_count(), 4)
    res = _run(nr, W, comp, order)
    assert all(v == "ok" for v in res.values()), res


@needs2
@pytest.mark.parametrize("comp,order,W,peer,steps", [
    ("topk", "ring", 1, "nccl", 4), ("async", "naive", 2, "nccl", 4), ("topk_q8", "naive", 1, "nccl", 4),
    ("topk", "ring", 1, "shard", 4), ("async_q8", "naive", 2, "shard", 4), ("topk", "hierarchical", 2, "shard", 4),
    ("async", "naive", 1, "shard", 4), ("topk_q8", "ring", 2, "shard", 4),
    ("topk_grow", "ring", 1, "shard", 6), ("topk_grow", "naive", 2, "pull", 6), ("topk", "ring", 1, "pull", 12),
    ("topk", "ring", 1, "push", 4), ("async", "naive", 2, "push", 4), ("topk_grow", "ring", 2, "push", 6),
    ("topk", "ring", 1, "direct", 4), ("async_q8", "naive", 2, "direct", 4), ("topk", "hierarchical", 2, "direct", 6),
])
def test_payload_exchange_modes(comp, order, W, peer, steps):
    """NCCL all-gather fallback, the NVLink push and sharded modes, arena
    re-creation when k grows, and a long run through the device-side flags
    (the default pull mode runs in test_exchange_paths_match_oracle)."""
    nr = min(torch.cuda.device_count(), 4)
    res = _run(nr, W, comp, order, steps=steps, peer=peer)
    assert all(v == "ok" for v in res.values()), res


def _worker_full_size(rank, nranks, uid, comp, q):
    """Bench size (cfg2: 125M, top-k 1% + EF, default exchange: the apply
    reads the peers' wire16 arenas in place; cfg3:
    125M dense q8, NCCL all-to-all + all-gather): the multi-rank step must
    equal, bit for bit, the same P workers run as virtual workers on one GPU
    -- a path the oracle pins at small sizes (test_apply_gpu.py)."""
    sys.path.insert(0, ROOT)
    try:
        import torch as th

        from paper_2506_17551_b200 import _lib as L
        from paper_2506_17551_b200.engine import Context, generate

        th.cuda.set_device(rank)
        n, lr = 125_000_000, 0.05
        code, k, order = ((L.PSB_COMP_TOPK, n // 100, "ring") if comp == "topk" else (L.PSB_COMP_Q8, 0, "naive"))
        P = nranks
        c = Context(n, max(k, 1), P, device=rank)
        c.comm_init(rank, nranks, uid)
        g = th.empty(1, n, device="cuda")
        res = th.zeros(1, n, device="cuda")
        theta = th.zeros(n, device="cuda")
        steps = 3
        for s in range(steps):
            generate("llmrec", 42, rank, s, n, g[0])
            c.sync_step(c.step_desc(code, g, res, theta, lr, k, order, 256))
        c.check()
        if comp == "topk" and not c.peer_active:
            q.put((rank, "NVLink peer exchange not active"))
            return
        c2 = Context(n, max(k, 1), P, device=rank)
        g2 = th.empty(P, n, device="cuda")
        res2 = th.zeros(P, n, device="cuda")
        theta2 = th.zeros(n, device="cuda")
        for s in range(steps):
            for p in range(P):
                generate("llmrec", 42, p, s, n, g2[p])
            c2.sync_step(c2.step_desc(code, g2, res2, theta2, lr, k, order, 256))
        c2.check()
        if not th.equal(theta.view(th.int32), theta2.view(th.int32)):
            q.put((rank, "theta differs from the virtual-worker run"))
            return
        if not th.equal(res[0].view(th.int32), res2[rank].view(th.int32)):
            q.put((rank, "residual differs from the virtual-worker run"))
            return
        q.put((rank, "ok"))
        c.close()
        c2.close()
    except Exception as e:
        q.put((rank, f"error: {type(e).__name__}: {e}"))


@needs2
@pytest.mark.parametrize("comp", ["topk", "q8"])
def test_full_size_multi_rank_equals_virtual_workers(comp):
    from paper_2506_17551_b200.engine import Context
    nr = min(torch.cuda.device_count(), 4)
    uid = Context.unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_full_size, args=(r, nr, uid, comp, q)) for r in range(nr)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(nr):
        r, msg = q.get(timeout=600)
        results[r] = msg
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in results.values()), results
