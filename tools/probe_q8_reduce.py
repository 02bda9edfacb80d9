"""Probe: the dense q8 fold (k_q8_quant x W + k_q8_reduce) on one GPU via the
unfused single-rank path (PSB_Q8_UNFUSED=1), cfg3 size, W = 2 workers."""
import os
import sys

os.environ["PSB_Q8_UNFUSED"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

n, W = 125_000_000, 2
c = Context(n, 1, W)
g = torch.empty(W, n, device="cuda")
for w in range(W):
    generate("llmrec", 42, w, 0, n, g[w])
r = torch.zeros(W, n, device="cuda")
th = torch.zeros(n, device="cuda")
d = c.step_desc(L.PSB_COMP_Q8, g, r, th, 0.05, 0, "naive", 256)
for _ in range(3):
    c.sync_step(d)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
it = int(os.environ.get("PROBE_ITERS", "10"))
for _ in range(it):
    c.sync_step(d)
e1.record()
torch.cuda.synchronize()
c.check()
print(f"unfused q8 step W={W}: {e0.elapsed_time(e1) / it * 1e3:.1f} us", flush=True)
