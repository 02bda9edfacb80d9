"""Where does the K1 streaming pass lose time against the HBM roofline?
Per-CTA entry/exit timestamps of k_scan<MODE_A> (build: make
OUT=../libpsb_trace.so OBJDIR=build_trace EXTRA_NVFLAGS=-DPSB_SCAN_TRACE, run
with PSB_LIB=libpsb_trace.so)."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

for n in [int(x) for x in os.environ.get("PROBE_NS", "125000000,350000000").split(",")]:
    k = n // 100
    ctx = Context(n, k, 1)
    gs = [torch.empty(1, n, device="cuda") for _ in range(3)]
    for b in range(3):
        generate("llmrec", 42, 0, b, n, gs[b][0])
    res = torch.zeros(1, n, device="cuda")
    theta = torch.zeros(n, device="cuda")
    ds = [ctx.step_desc(2, gs[b], res, theta, 0.05, k, "ring") for b in range(3)]
    lib = L.load()
    buf = (ctypes.c_ulonglong * 8192)()
    for i in range(40):
        ctx.profile_enable(i >= 30)
        ctx.sync_step(ds[i % 3])
        torch.cuda.synchronize()
        if i >= 36:
            m = lib.psb_debug_scan_trace(buf, 4096)
            ms, cnt = ctx.profile_read()
            t = [(buf[2 * j], buf[2 * j + 1]) for j in range(m) if buf[2 * j + 1] > buf[2 * j] > 0]
            t0 = min(a for a, _ in t)
            starts = sorted((a - t0) / 1e3 for a, _ in t)
            ends = sorted((b - t0) / 1e3 for _, b in t)
            durs = sorted((b - a) / 1e3 for a, b in t)
            q = lambda v, f: v[min(len(v) - 1, int(f * len(v)))]  # noqa: E731
            print(f"n={n} step {i}: ctas={len(t)} event_ms={ms / max(cnt, 1):.4f} "
                  f"start[p0,p50,p99,max]={q(starts,0):.1f},{q(starts,.5):.1f},{q(starts,.99):.1f},{starts[-1]:.1f} "
                  f"end[min,p10,p50,p90,max]={ends[0]:.1f},{q(ends,.1):.1f},{q(ends,.5):.1f},{q(ends,.9):.1f},{ends[-1]:.1f} "
                  f"dur[min,p50,max]={durs[0]:.1f},{q(durs,.5):.1f},{durs[-1]:.1f}", flush=True)
    ctx.close()
    del gs, res, theta
    torch.cuda.empty_cache()
