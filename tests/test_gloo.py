"""CPU, world_size 2 over gloo: the multi-rank decomposition of the path.

Each rank owns W workers (worker id = rank*W + w), compresses them with the
oracle, exchanges the payloads (all_gather, the NCCL allgather's role) and
applies the rank-ordered mean: both replicas must be bitwise identical to each
other and to the single-process P-worker sync_data_parallel_step.  Also checks
the unique-id broadcast and the dense-q8 shard decomposition.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2506_17551_b200 import dist as pdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # unique-id broadcast (what bench.py uses before psb_comm_init)
        uid = pdist.broadcast_unique_id(lambda: bytes(range(128)))
        assert uid == bytes(range(128))

        W, n, k, lr = 2, 4000, 40, 0.05
        P = W * world
        theta = np.zeros(n, dtype=np.float32)
        res = np.zeros((W, n), dtype=np.float32)
        for step in range(3):
            mine = list(pdist.worker_ids(rank, W))
            idx_l, val_l = [], []
            for j, wid in enumerate(mine):
                g = O.generate("llmrec", 5, wid, step, n)
                i, v, _ = O.ef_topk(g, res[j], k)
                idx_l.append(torch.from_numpy(i.astype(np.int64)))
                val_l.append(torch.from_numpy(v))
            idx_all = [torch.empty(W * k, dtype=torch.int64) for _ in range(world)]
            val_all = [torch.empty(W * k, dtype=torch.float32) for _ in range(world)]
            dist.all_gather(idx_all, torch.cat(idx_l))
            dist.all_gather(val_all, torch.cat(val_l))
            dense = np.zeros((P, n), dtype=np.float32)
            for r_ in range(world):
                for j in range(W):
                    sl = slice(j * k, (j + 1) * k)
                    dense[r_ * W + j, idx_all[r_][sl].numpy()] = val_all[r_][sl].numpy()
            mean = O.fold_mean(dense, "ring")
            O.axpy_(-lr, mean, theta)
        # dense q8: per-rank shard reduce == full reduce
        g_all = np.stack([O.generate("uniform", 6, p, 0, 5000) for p in range(P)])
        deq = []
        for p in range(P):
            c, s, _ = O.q8_quant(g_all[p], None, 256)
            deq.append(O.q8_dequant(c, s, 256))
        full = O.fold_mean(np.stack(deq), "naive")
        lo, hi = pdist.q8_shards(5000, 256, world)[rank]
        mine_sh = full[lo * 256:min(hi * 256, 5000)]
        shards = [None] * world
        dist.all_gather_object(shards, mine_sh)
        q.put((rank, theta.tobytes(), res.tobytes(), np.array_equal(np.concatenate(shards), full)))
    except Exception as e:  # pragma: no cover
        q.put((rank, f"error {e}", None, False))
    finally:
        dist.destroy_process_group()


def test_two_rank_decomposition_matches_single_process():
    from oracle import oracle as O
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, th, rs, ok = q.get(timeout=180)
        out[r] = (th, rs, ok)
    for p in procs:
        p.join(timeout=60)
    assert isinstance(out[0][0], bytes), out
    assert out[0][0] == out[1][0], "replicas diverged"
    assert out[0][2] and out[1][2], "q8 shard decomposition differs from the full reduce"
    # single-process reference composite with all P = 4 workers
    W, n, k, lr, P = 2, 4000, 40, 0.05, 4
    theta = np.zeros(n, dtype=np.float32)
    res = np.zeros((P, n), dtype=np.float32)
    for step in range(3):
        g = np.stack([O.generate("llmrec", 5, p, step, n) for p in range(P)])
        O.sync_step(g, theta, lr, "topk", k, "ring", res)
    assert out[0][0] == theta.tobytes()
    assert out[0][1] == res[:W].tobytes() and out[1][1] == res[W:].tobytes()


def test_q8_shards_cover_blocks():
    from paper_2506_17551_b200.dist import q8_shards
    for n, b, w in ((1, 128, 8), (1000, 256, 3), (125_000_000, 256, 8), (4097, 1024, 4)):
        sh = q8_shards(n, b, w)
        nb = (n + b - 1) // b
        assert sh[0][0] == 0 and sh[-1][1] == nb
        assert all(sh[i][1] == sh[i + 1][0] or sh[i + 1][0] >= nb for i in range(w - 1))


@pytest.mark.parametrize("W,rank", [(1, 0), (3, 2)])
def test_worker_ids(W, rank):
    from paper_2506_17551_b200.dist import worker_ids
    assert list(worker_ids(rank, W)) == [rank * W + w for w in range(W)]
