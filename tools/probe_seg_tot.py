"""Probe: distribution of the sparse apply's per-segment entry counts (tot)
for cfg2 payloads (P workers' K1 outputs), to size the TMA stage."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

n = 125_000_000
k = n // 100
c = Context(n, k, 1)
g = torch.empty(n, device="cuda")
idx = torch.empty(k, dtype=torch.int32, device="cuda")
val = torch.empty(k, device="cuda")
for P, shift in ((2, 15), (4, 14), (8, 13)):
    nseg = (n + (1 << shift) - 1) >> shift
    tot = torch.zeros(nseg, dtype=torch.int64, device="cuda")
    for p in range(P):
        generate("llmrec", 42, p, 0, n, g)
        c.ef_topk(g, None, k, 0, idx, val)
        tot += torch.bincount(idx.long() >> shift, minlength=nseg)
    t = tot.float()
    q = torch.quantile(t[: min(nseg, 1 << 24)], torch.tensor([0.5, 0.9, 0.99, 1.0], device="cuda"))
    fr = {th: float((tot > th).float().mean()) for th in (1024, 1536, 2048, 3072, 4096)}
    print(f"P={P} S=2^{shift} nseg={nseg} mean={t.mean():.0f} p50/p90/p99/max={[round(x) for x in q.tolist()]} frac>{fr}")
