"""Probe (needs a build with EXTRA_NVFLAGS=-DPSB_APPLY_TRACE): per-phase CTA
time of the sparse apply, summed over segments."""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.engine import Context, generate, payload_bytes  # noqa: E402

lib = L.load()
fn = lib.psb_debug_apply_trace
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
n = 125_000_000
k = n // 100
for P in [int(x) for x in os.environ.get("PROBE_P", "2,8").split(",")]:
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
    out = (ctypes.c_ulonglong * 8)()
    c.sparse_mean_sgd(gath, P, k, torch.float32, "ring", 0.05, th, n)
    fn(out, 1)
    c.sparse_mean_sgd(gath, P, k, torch.float32, "ring", 0.05, th, n)
    fn(out, 1)
    print(f"P={P}: CTA-sum us: head {out[0] / 1e3:.0f}  phase1 {out[1] / 1e3:.0f}  phase2 {out[2] / 1e3:.0f}",
          flush=True)
    c.close()
    del gath, th, g
    torch.cuda.empty_cache()
