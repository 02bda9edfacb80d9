"""Probe: device time of the P-payload sparse mean+SGD apply at cfg2 size on
one GPU (P payloads produced by K1 from P different gradients)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.engine import Context, generate, payload_bytes  # noqa: E402

n = 125_000_000
k = int(n * float(os.environ.get("PROBE_RHO", "0.01")))
order = sys.argv[1] if len(sys.argv) > 1 else "ring"
for P in [int(x) for x in os.environ.get("PROBE_P", "2,4,8").split(",")]:
    c = Context(n, k, P)
    blk = payload_bytes(L.PSB_COMP_TOPK, torch.float32, k)
    gath = torch.empty(P * blk, dtype=torch.uint8, device="cuda")
    voff = (k * 4 + 15) // 16 * 16
    g = torch.empty(n, device="cuda")
    for p in range(P):
        generate("llmrec", 42, p, 0, n, g)
        sl = gath[p * blk:(p + 1) * blk]
        c.ef_topk(g, None, k, 0, sl[:k * 4].view(torch.int32), sl[voff:voff + k * 4].view(torch.float32))
    th = torch.zeros(n, device="cuda")
    for _ in range(3):
        c.sparse_mean_sgd(gath, P, k, torch.float32, order, 0.05, th, n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(int(os.environ.get("PROBE_ITERS", "20"))):
        c.sparse_mean_sgd(gath, P, k, torch.float32, order, 0.05, th, n)
    e1.record()
    torch.cuda.synchronize()
    c.check()
    print(f"P={P} order={order}: apply {1e3 * e0.elapsed_time(e1) / int(os.environ.get('PROBE_ITERS', '20')):.1f} us "
          f"(payload {P * blk / 1e6:.0f} MB)", flush=True)
    c.close()
    del gath, th, g
    torch.cuda.empty_cache()
