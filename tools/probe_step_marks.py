"""Probe (torchrun, PSB_STEP_MARKS=1): per-milestone device time of the
multi-rank step, eager, per rank.  argv[1] = peer mode (shard|full|nccl).
PROBE_COMP=topk (cfg2; milestones [wait, compress, (segoff+signal |
exchange), (pull, fold, publish+scatter) | apply]) or q8 (cfg3 over NVLink;
milestones [wait_ack, quantize, flag round 1, pull codes, reduce, flag round 2,
pull mean + ack, apply])."""
import ctypes
import os
import sys

os.environ["PSB_STEP_MARKS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.dist import init_comm  # noqa: E402
from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "shard"
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
n = 125_000_000
comp = os.environ.get("PROBE_COMP", "topk")
k = n // 100 if comp == "topk" else 0
c = Context(n, max(k, 1), world, device=rank)
init_comm(c)
c.peer_mode(mode)
lib = L.load()
lib.psb_debug_marks.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.c_int]
lib.psb_debug_marks.restype = ctypes.c_int
gs = [torch.empty(1, n, device="cuda") for _ in range(3)]
for i, g in enumerate(gs):
    generate("llmrec", 42, rank, i, n, g[0])
res = torch.zeros(1, n, device="cuda")
theta = torch.zeros(n, device="cuda")
code = L.PSB_COMP_TOPK if comp == "topk" else L.PSB_COMP_Q8
descs = [c.step_desc(code, g, res, theta, 0.05, k, "ring" if comp == "topk" else "naive", 256) for g in gs]
buf = (ctypes.c_float * 32)()
acc = None
steps = 20
for s in range(30 + steps):
    c.sync_step(descs[s % 3])
    m = lib.psb_debug_marks(c.h, buf, 32)
    if s >= 30:
        v = [buf[i] for i in range(m)]
        acc = v if acc is None else [a + b for a, b in zip(acc, v)]
c.check()
t = torch.tensor([a / steps * 1e3 for a in acc], device="cuda", dtype=torch.float64)
allt = [torch.zeros_like(t) for _ in range(world)]
dist.all_gather(allt, t)
if rank == 0:
    for r, x in enumerate(allt):
        print(f"world={world} mode={mode} rank={r} us per milestone: {[round(float(v), 1) for v in x]} "
              f"sum={float(x.sum()):.1f}", flush=True)
dist.barrier()
c.close()
dist.barrier()
dist.destroy_process_group()
