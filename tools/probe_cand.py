"""Probe: steady-state K1 candidate-phase milestones (psb_topk_phases) of the
cfg2 step at one rank (sync_step, fused single-worker SGD)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 125_000_000
k = n // 100
c = Context(n, k, 1)
gs = [torch.empty(1, n, device="cuda") for _ in range(3)]
for i, g in enumerate(gs):
    generate("llmrec", 42, 0, i, n, g[0])
res = torch.zeros(1, n, device="cuda")
theta = torch.zeros(n, device="cuda")
descs = [c.step_desc(L.PSB_COMP_TOPK, g, res, theta, 0.05, k, "ring") for g in gs]
names = ["stage", "coarse", "fine", "count", "slots", "scatter"]
for step in range(40):
    c.sync_step(descs[step % 3])
    c.check()
    if step >= 34:
        ph = c.topk_phases_us()
        st = c.topk_stats(0)
        print(f"step {step} C/k={st['candidates'] / k:.3f} lvl={st['first_radix_level']} "
              + " ".join(f"{nm}={x:.1f}" for nm, x in zip(names, ph)), flush=True)
