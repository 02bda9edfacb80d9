"""Data-parallel trainer around the device path.

Mirrors parsim/trainer.hpp:197-261 (`train`, sync and async branches) for the
reference's BPR matrix-factorisation recommender, with every gradient and
update on the B200:

  * RecModel::init (trainer.hpp:28-38) and TripleSampler (:143-179) are the
    reference's host-side draws (SplitMix64 stream, rejection-sampled
    negatives), restated here so the triple stream is identical;
  * per step each of the P workers' contiguous batch shards gets its gradient
    from psb_bpr_gradient (device) and the step is psb_sync_step (EF
    compression + the reference fold order + SGD, all device kernels);
  * async: worker p computes its gradient on the parameters from
    tau = min(updates, p mod 4) updates ago (a device history ring of 3),
    compresses with error feedback and applies eta/(1+tau) (psb_ef_topk /
    psb_ef_onebit + the reference-order apply).

Host work per step is the sampler and launch orchestration only.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import torch

from . import _lib as L
from .engine import Context


class SeededRng:
    """SplitMix64 (parsim/numerics.hpp:152-178), bit-exact."""

    M = (1 << 64) - 1

    def __init__(self, seed: int):
        self.s = seed & self.M

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()

    def next_below(self, n: int) -> int:
        if n <= 0:
            raise L.PsbInvalidArgument("next_below: n must be positive")
        return self.next_u64() % n


def init_params(users: int, items: int, dim: int, seed: int) -> torch.Tensor:
    """RecModel::init (trainer.hpp:28-38) flattened (user rows, then item rows), f64 CUDA."""
    if users < 1 or items < 1 or dim < 1:
        raise L.PsbInvalidArgument("RecModel: sizes must be >= 1")
    rng = SeededRng(seed)
    vals = [rng.uniform(-0.01, 0.01) for _ in range((users + items) * dim)]
    return torch.tensor(vals, dtype=torch.float64, device="cuda")


class TripleSampler:
    """TripleSampler (trainer.hpp:143-179): positives uniform over the train
    records, one negative per positive rejected against the user's positives
    (up to 100 tries, else the positive itself)."""

    def __init__(self, train_users: Sequence[int], train_items: Sequence[int], num_users: int, num_items: int,
                 seed: int):
        if len(train_users) == 0:
            raise L.PsbInvalidArgument("TripleSampler: empty train split")
        self.users = list(int(u) for u in train_users)
        self.items = list(int(i) for i in train_items)
        self.num_items = num_items
        self.rng = SeededRng(seed)
        self.pos = [set() for _ in range(num_users)]
        for u, i in zip(self.users, self.items):
            self.pos[u].add(i)

    def next(self) -> Tuple[int, int, int]:
        j = self.rng.next_below(len(self.users))
        u, i = self.users[j], self.items[j]
        neg = i
        for _ in range(100):
            cand = self.rng.next_below(self.num_items)
            if cand not in self.pos[u]:
                neg = cand
                break
        return u, i, neg

    def next_batch(self, n: int) -> List[Tuple[int, int, int]]:
        return [self.next() for _ in range(n)]


@dataclass
class TrainResult:
    theta: torch.Tensor
    loss_curve: List[Tuple[int, float]] = field(default_factory=list)
    residuals: Optional[torch.Tensor] = None  # [P][n] error-feedback state at the end
    sampler_state: int = 0                    # TripleSampler SplitMix64 state at the end
    steps_done: int = 0


# ------------------------------------------------------------ checkpoints
def save_model(path: str, theta: torch.Tensor, users: int, items: int, dim: int) -> None:
    """save_model (trainer.hpp:332-349): "PSMF" | u64 users, items, dim | flat f64, little-endian
    (the reference's load_model reads it)."""
    import struct
    flat = theta.detach().to("cpu", torch.float64).contiguous()
    if flat.numel() != (users + items) * dim:
        raise L.PsbInvalidArgument("save_model: theta size mismatch")
    with open(path, "wb") as f:
        f.write(b"PSMF" + struct.pack("<QQQ", users, items, dim))
        f.write(flat.numpy().astype("<f8").tobytes())


def load_model(path: str) -> Tuple[torch.Tensor, int, int, int]:
    """load_model (trainer.hpp:351-378): (theta f64 CUDA, users, items, dim)."""
    import struct
    import numpy as np
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 4 or data[:4] != b"PSMF":
        raise RuntimeError(f"load_model: '{path}' is not a model file")
    if len(data) < 28:
        raise RuntimeError(f"load_model: corrupt header in '{path}'")
    users, items, dim = struct.unpack("<QQQ", data[4:28])
    if users == 0 or items == 0 or dim == 0:
        raise RuntimeError(f"load_model: corrupt header in '{path}'")
    n = (users + items) * dim
    if len(data) < 28 + 8 * n:
        raise RuntimeError(f"load_model: truncated '{path}'")
    theta = torch.from_numpy(np.frombuffer(data, dtype="<f8", count=n, offset=28).astype(np.float64)).cuda()
    return theta, users, items, dim


def save_ef_state(path: str, residuals: torch.Tensor, steps_done: int, sampler_state: int) -> None:
    """Error-feedback checkpoint (absent in the reference, which saves theta
    only): "PSEF" | u64 P, n, steps_done, sampler state |
    P x n f64 residuals, little-endian.  With save_model it resumes exactly."""
    import struct
    r = residuals.detach().to("cpu", torch.float64).contiguous()
    P, n = r.shape
    with open(path, "wb") as f:
        f.write(b"PSEF" + struct.pack("<QQQQ", P, n, steps_done, sampler_state & ((1 << 64) - 1)))
        f.write(r.numpy().astype("<f8").tobytes())


def load_ef_state(path: str) -> Tuple[torch.Tensor, int, int]:
    """(residuals [P][n] f64 CUDA, steps_done, sampler_state)."""
    import struct
    import numpy as np
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 36 or data[:4] != b"PSEF":
        raise RuntimeError(f"load_ef_state: '{path}' is not an error-feedback checkpoint")
    P, n, steps_done, st = struct.unpack("<QQQQ", data[4:36])
    if len(data) < 36 + 8 * P * n:
        raise RuntimeError(f"load_ef_state: truncated '{path}'")
    r = torch.from_numpy(np.frombuffer(data, dtype="<f8", count=P * n, offset=36).astype(np.float64)).cuda()
    return r.view(P, n), steps_done, st


_COMP = {"none": L.PSB_COMP_NONE, "onebit": L.PSB_COMP_ONEBIT, "topk": L.PSB_COMP_TOPK}


def train(users: int, items: int, dim: int, train_users: Sequence[int], train_items: Sequence[int], P: int,
          steps: int, batch_size: int, lr: float, compressor: str = "none", top_k: int = 0,
          algo: str = "ring", mode: str = "sync", seed: int = 42,
          ctx: Optional[Context] = None, init_seed: Optional[int] = None,
          resume: Optional[Tuple[torch.Tensor, torch.Tensor, int, int]] = None) -> TrainResult:
    """parsim train() (trainer.hpp:197-261) with the gradients and updates on the
    device (f64).  init_seed: RecModel::init seed (default: seed, as the tests
    call it; the reference CLI uses seed for init and seed + 1 for training)."""
    if lr <= 0.0:
        raise L.PsbInvalidArgument("HyperParams: learning_rate must be > 0")
    if batch_size < P:
        raise L.PsbInvalidArgument("train: batch_size must be >= data_degree")
    if mode != "sync" and resume is not None and int(resume[2]):
        raise L.PsbInvalidArgument("train: resume is supported for sync training (async history is not saved)")
    n = (users + items) * dim
    sampler = TripleSampler(train_users, train_items, users, items, seed)
    start = 0
    if resume is not None:  # (theta, residuals, steps_done, sampler_state) from the checkpoints
        theta = resume[0].to(torch.float64).clone()
        start = int(resume[2])
        sampler.rng.s = int(resume[3])
    else:
        theta = init_params(users, items, dim, seed if init_seed is None else init_seed)
    own = ctx is None
    if own:
        ctx = Context(n, max(top_k, 1), max(P, 1))
    compressed = compressor != "none"
    res = torch.zeros(P, n, dtype=torch.float64, device="cuda")
    if resume is not None:
        res.copy_(resume[1])
    grads = torch.empty(P, n, dtype=torch.float64, device="cuda")
    history: deque = deque()
    updates = 0
    out = TrainResult(theta)

    def shard(p: int) -> Tuple[int, int]:
        base, rem = batch_size // P, batch_size % P
        lo = p * base + min(p, rem)
        return lo, lo + base + (1 if p < rem else 0)

    def dev(triples):
        u = torch.tensor([t[0] for t in triples], dtype=torch.int32, device="cuda")
        ip = torch.tensor([t[1] for t in triples], dtype=torch.int32, device="cuda")
        ineg = torch.tensor([t[2] for t in triples], dtype=torch.int32, device="cuda")
        return u, ip, ineg

    try:
        for step in range(start, start + steps):
            batch = sampler.next_batch(batch_size)
            if step % 100 == 0:
                scratch = torch.empty_like(theta)
                _, loss = ctx.bpr_gradient(theta, users, items, dim, *dev(batch), grad=scratch)
                out.loss_curve.append((step, float(loss.item())))
            if mode == "sync":
                for p in range(P):
                    lo, hi = shard(p)
                    ctx.bpr_gradient(theta, users, items, dim, *dev(batch[lo:hi]), grad=grads[p], want_loss=False)
                d = ctx.step_desc(_COMP[compressor], grads, res if compressed else None, theta, lr, top_k, algo)
                ctx.sync_step(d)
            else:
                for p in range(P):
                    tau = min(updates, p % 4)
                    snap = theta if tau == 0 else history[len(history) - tau]
                    lo, hi = shard(p)
                    g = grads[p]
                    ctx.bpr_gradient(snap, users, items, dim, *dev(batch[lo:hi]), grad=g, want_loss=False)
                    onebit = None
                    if compressed:  # ef_compress_step then decompress (trainer.hpp:248)
                        if compressor == "topk":
                            idx, val = ctx.ef_topk(g, res[p], top_k)
                            g = ctx.decompress_topk(idx, val, n)
                        else:
                            onebit = ctx.ef_onebit(g, res[p])
                    history.append(theta.clone())
                    if len(history) > 3:
                        history.popleft()
                    # async_step: theta - eta/(1+tau) * g  (strategies.hpp:125-129);
                    # a 1-bit message is applied straight from its sign words
                    # (the one-worker 1-bit mean is +-scale exactly)
                    scale = lr / (1.0 + float(tau))
                    if onebit is not None:
                        ctx.onebit_mean_sgd(onebit[0], onebit[1], n, torch.float64, "naive", scale, theta)
                    else:
                        ctx.dense_mean_sgd(g.unsqueeze(0), "naive", scale, theta)
                    updates += 1
        ctx.check()
    finally:
        if own:
            ctx.close()
    out.theta = theta
    out.residuals = res
    out.sampler_state = sampler.rng.s
    out.steps_done = start + steps
    return out


def mix64(z: int) -> int:
    """parsim/numerics.hpp:181-186."""
    M = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


@dataclass
class EvalResult:
    hr_at_10: float
    ndcg_at_10: float
    num_eval_users: int
    skipped: int


def evaluate_topk(theta: torch.Tensor, users: int, items: int, dim: int, train: Tuple[Sequence[int], Sequence[int]],
                  validation: Tuple[Sequence[int], Sequence[int]], test: Tuple[Sequence[int], Sequence[int]],
                  K: int = 10, negatives: int = 99, seed: int = 42, ctx: Optional[Context] = None) -> EvalResult:
    """evaluate_topk (trainer.hpp:269-324): the per-record negatives are the
    reference's host draws (SeededRng(seed ^ mix64(rec_idx)), rejection against
    everything the user interacted with, deterministic fallback); the scores
    and ranks of all records are one device launch (psb_rank_candidates)."""
    import math
    tu, ti = test
    if len(tu) == 0:
        raise L.PsbInvalidArgument("evaluate_topk: empty test split")
    if K < 1 or negatives < 1:
        raise L.PsbInvalidArgument("evaluate_topk: K and negatives must be >= 1")
    seen = [set() for _ in range(users)]
    for us, its in (train, validation, test):
        for u, i in zip(us, its):
            seen[int(u)].add(int(i))
    rec_u, rec_i, cands, skipped = [], [], [], 0
    for rec_idx, (u, it) in enumerate(zip(tu, ti)):
        u, it = int(u), int(it)
        s = seen[u]
        available = items - len(s)
        if available == 0:
            skipped += 1
            continue
        rng = SeededRng(seed ^ mix64(rec_idx))
        want = min(negatives, available)
        negs, attempts, cap = set(), 0, 100 * (negatives + 1)
        while len(negs) < want and attempts < cap:
            attempts += 1
            c = rng.next_below(items)
            if c in s or c == it:
                continue
            negs.add(c)
        if len(negs) < want:
            for c in range(items):
                if len(negs) >= want:
                    break
                if c not in s and c != it:
                    negs.add(c)
        rec_u.append(u)
        rec_i.append(it)
        cands.append(sorted(negs) + [-1] * (negatives - len(negs)))
    if not rec_u:
        raise L.PsbInvalidArgument("evaluate_topk: all test records were skipped")
    own = ctx is None
    if own:
        ctx = Context(max(theta.numel(), 1), 1, 1)
    try:
        ranks = ctx.rank_candidates(theta, users, dim, torch.tensor(rec_u, dtype=torch.int32, device="cuda"),
                                    torch.tensor(rec_i, dtype=torch.int32, device="cuda"),
                                    torch.tensor(cands, dtype=torch.int32, device="cuda")).cpu().tolist()
        ctx.check()
    finally:
        if own:
            ctx.close()
    hits, ndcg = 0, 0.0
    for r in ranks:
        if r <= K:
            hits += 1
            ndcg += 1.0 / math.log2(float(r) + 1.0)
    n = len(ranks)
    return EvalResult(hits / n, ndcg / n, n, skipped)
