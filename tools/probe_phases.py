"""Probe: K1 candidate-phase milestones of CTA 0 (psb_topk_phases) at
PROBE_RHO, cfg2-sized LLM-rec gradients, sync steps with the fused update."""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch  # noqa: E402

from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

n = int(os.environ.get("PROBE_N", 125_000_000))
for rho in [float(x) for x in os.environ.get("PROBE_RHO", "0.01,0.1").split(",")]:
    k = int(n * rho)
    NB = 4
    ctx = Context(n, k, 1)
    gs = [torch.empty(1, n, device="cuda") for _ in range(NB)]
    for b in range(NB):
        generate("llmrec", 42, 0, b, n, gs[b][0])
    res = torch.zeros(1, n, device="cuda")
    theta = torch.zeros(n, device="cuda")
    ds = [ctx.step_desc(2, gs[b], res, theta, 0.05, k, "ring") for b in range(NB)]
    for i in range(30):
        ctx.sync_step(ds[i % NB])
        if i >= 26:
            torch.cuda.synchronize()
            print(f"rho {rho} step {i}: phases us {[round(x, 1) for x in ctx.topk_phases_us()]} "
                  f"stats {ctx.topk_stats(0)}", flush=True)
    ctx.close()
    del gs, res, theta
    torch.cuda.empty_cache()
