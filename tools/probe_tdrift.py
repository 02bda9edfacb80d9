"""Threshold drift data for the K1 predictor (cfg2 shape).  Per step t: the
exact threshold T_t and, for y on a grid, count(|p_t| >= T_{t-1} * y) / k --
enough to replay any prediction policy offline (tools/sim_predictor.py).
PROBE_NB rotated gradient buffers (bench.py uses NB)."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch  # noqa: E402

from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

n = int(os.environ.get("PROBE_N", 125_000_000))
k = n // 100
NB = int(os.environ.get("PROBE_NB", "3"))
STEPS = int(os.environ.get("PROBE_STEPS", "40"))
dev = torch.device("cuda", 0)
ctx = Context(n, k, 1)
grads = [torch.empty(1, n, device=dev) for _ in range(NB)]
for b in range(NB):
    generate("llmrec", 42, 0, b, n, grads[b][0])
res = torch.zeros(1, n, device=dev)
theta = torch.zeros(n, device=dev)
descs = [ctx.step_desc(2, grads[b], res, theta, 0.05, k, "ring") for b in range(NB)]
ys = [round(0.80 + 0.0025 * i, 4) for i in range(161)]  # 0.80 .. 1.20
rows = []
t_prev = None
for i in range(STEPS):
    p = (res + grads[i % NB])[0].abs()
    srt, _ = torch.sort(p, descending=True)
    T_exact = float(srt[k - 1])
    cnt = None
    if t_prev is not None:
        thr = torch.tensor([t_prev * y for y in ys], device=dev, dtype=torch.float32)
        # count(p >= v) in a descending array = number of entries >= v
        cnt = (torch.searchsorted(-srt, -thr, right=True)).tolist()
        cnt = [c / k for c in cnt]
    ctx.sync_step(descs[i % NB])
    torch.cuda.synchronize()
    st = ctx.topk_stats()
    rows.append({"step": i, "T": T_exact, "C_over_k": st["candidates"] / k, "misses": st["misses"],
                 "f": st["margin_f"], "counts": cnt})
    t_prev = T_exact
    del srt, p
out = os.environ.get("PROBE_OUT", "gpurun_out/tdrift.json")
with open(out, "w") as f:
    json.dump({"n": n, "k": k, "NB": NB, "ys": ys, "rows": rows}, f)
for r in rows:
    print(r["step"], "T %.6g" % r["T"], "C/k %.3f" % r["C_over_k"], "misses", r["misses"])
