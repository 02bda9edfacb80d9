"""Per-CTA view of the K1 candidate phase (which CTA ends last, and why):
needs the diagnostics build (PSB_LIB=libpsb_trace.so, see probe_scan_trace.py)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

n = int(os.environ.get("PROBE_N", 125_000_000))
rho = float(os.environ.get("PROBE_RHO", 0.01))
k = int(n * rho)
NB = 8
ctx = Context(n, k, 1)
gs = [torch.empty(1, n, device="cuda") for _ in range(NB)]
for b in range(NB):
    generate("llmrec", 42, 0, b, n, gs[b][0])
res = torch.zeros(1, n, device="cuda")
theta = torch.zeros(n, device="cuda")
ds = [ctx.step_desc(2, gs[b], res, theta, 0.05, k, "ring") for b in range(NB)]
lib = L.load()
buf = (ctypes.c_ulonglong * (16 * 1024))()
names = os.environ.get("PROBE_NAMES", "sb_scan,refine,win_copy_issue,copy_wait_prefetch,fine,scatter_count,slots,end").split(",")
for i in range(40):
    ctx.sync_step(ds[i % NB])
    torch.cuda.synchronize()
    if i >= 37:
        m = lib.psb_debug_cand_trace(buf, 1024)
        rows = []
        for c in range(m):
            w = [buf[16 * c + j] for j in range(16)]
            if w[0] == 0:
                continue
            ts = [x for x in w[:15] if x]
            rows.append((c, ts, w[15] >> 32, w[15] & 0xFFFFFFFF))
        t0 = min(r[1][0] for r in rows)
        ends = sorted(((r[1][-1] - t0) / 1e3, r[0]) for r in rows)
        print(f"step {i}: ctas={len(rows)} start spread {(max(r[1][0] for r in rows) - t0) / 1e3:.1f} us; "
              f"end min {ends[0][0]:.1f} p50 {ends[len(ends) // 2][0]:.1f} max {ends[-1][0]:.1f} (cta {ends[-1][1]})")
        for r in sorted(rows, key=lambda r: -(r[1][-1]))[:4] + rows[:2]:
            d = [(r[1][j + 1] - r[1][j]) / 1e3 for j in range(len(r[1]) - 1)]
            print(f"   cta {r[0]:3d} tiles {r[2]:6d} entries {r[3]:7d} " + " ".join(f"{nm}={x:.1f}" for nm, x in zip(names, d)))
