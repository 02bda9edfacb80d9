"""Probe: how the EF top-k threshold T moves from step to step (drives the
K1 threshold predictor design).  Prints T (magnitude), candidates and mode."""
import struct
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 125_000_000
rot = int(sys.argv[2]) if len(sys.argv) > 2 else 3
k = n // 100
c = Context(n, k, 1)
gs = [torch.empty(n, device="cuda") for _ in range(rot)]
for i, g in enumerate(gs):
    generate("llmrec", 42, 0, i, n, g)
r = torch.zeros(n, device="cuda")
prev = None
for step in range(30):
    idx, val = c.ef_topk(gs[step % rot], r, k)
    c.check()
    st = c.topk_stats(0)
    T = struct.unpack("<f", struct.pack("<I", st["threshold_key"]))[0]
    G = struct.unpack("<f", struct.pack("<I", st["predicted_key"] & 0xFFFFFFFF))[0]
    print(f"step {step:2d} T={T:.6e} ratio={T / prev if prev else 0:.5f} G/T={G / T if T else 0:.5f} "
          f"C/k={st['candidates'] / k:.3f} valid={st['predicted_valid']} lvl={st['first_radix_level']} "
          f"misses={st['misses']} f={st['margin_f']:.5f} phases_us={[round(x, 1) for x in c.topk_phases_us()]}",
          flush=True)
    prev = T
