"""Probe: eager vs CUDA-graph step time and host launch overhead of psb_sync_step
(cfg2 shape, one worker)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 125_000_000
k = n // 100
c = Context(n, k, 1)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    gs = [torch.empty(1, n, device="cuda") for _ in range(3)]
    for i, g in enumerate(gs):
        generate("llmrec", 42, 0, i, n, g[0])
    r = torch.zeros(1, n, device="cuda")
    th = torch.zeros(n, device="cuda")
    ds = [c.step_desc(L.PSB_COMP_TOPK, g, r, th, 0.05, k, "ring") for g in gs]
    for i in range(6):
        c.sync_step(ds[i % 3])
    c.check()
    # eager: host time per call and device time per step
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    t0 = time.perf_counter()
    K = 30
    for i in range(K):
        c.sync_step(ds[i % 3])
    t1 = time.perf_counter()
    e1.record(st)
    torch.cuda.synchronize()
    print(f"eager: host {1e6 * (t1 - t0) / K:.1f} us/call, device {1e3 * e0.elapsed_time(e1) / K:.1f} us/step")
    # graph of 3 steps
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(3):
            c.sync_step(ds[i % 3])
    torch.cuda.synchronize()
    e0.record(st)
    for i in range(10):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    c.check()
    print(f"graph: device {1e3 * e0.elapsed_time(e1) / 30:.1f} us/step")
    st_ = c.topk_stats(0)
    print(st_)
