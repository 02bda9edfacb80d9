"""When does K1's threshold prediction miss?  cfg2 shape, 3 rotated gradient
buffers as in bench.py; per step: candidates/k, miss, margin f, step time."""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch  # noqa: E402

from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

n, k = 125_000_000, 1_250_000
NB = int(os.environ.get("PROBE_NB", "3"))
STEPS = int(os.environ.get("PROBE_STEPS", "300"))
dev = torch.device("cuda", 0)
ctx = Context(n, k, 1)
grads = [torch.empty(1, n, device=dev) for _ in range(NB)]
for b in range(NB):
    generate("llmrec", 42, 0, b, n, grads[b][0])
res = torch.zeros(1, n, device=dev)
theta = torch.zeros(n, device=dev)
descs = [ctx.step_desc(2, grads[b], res, theta, 0.05, k, "ring") for b in range(NB)]
prev = 0
rows = []
for i in range(STEPS):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.sync_step(descs[i % NB])
    e1.record()
    torch.cuda.synchronize()
    st = ctx.topk_stats()
    miss = st["misses"] - prev
    prev = st["misses"]
    rows.append((i, st["candidates"] / k, miss, st["margin_f"], e0.elapsed_time(e1)))
for r in rows:
    if r[2] or r[0] < 8 or r[0] % 25 == 0:
        print("step %3d ratio %.3f miss %d f %.4f ms %.3f" % r)
ms = [r[4] for r in rows[10:]]
print("misses after step 10:", sum(r[2] for r in rows[10:]), "median ms %.3f mean ms %.3f" % (sorted(ms)[len(ms) // 2], sum(ms) / len(ms)))
