"""Probe (torchrun): per-phase device time of the multi-rank top-k step
(compress / NCCL allgather / seg-offsets+apply) at cfg2 size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.dist import init_comm  # noqa: E402
from paper_2506_17551_b200.engine import Context, generate, payload_bytes  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 125_000_000
k = n // 100
c = Context(n, k, world, device=rank)
init_comm(c)
blk = payload_bytes(L.PSB_COMP_TOPK, torch.float32, k)
gath = torch.empty(world * blk, dtype=torch.uint8, device="cuda")
gs = [torch.empty(n, device="cuda") for _ in range(3)]
for i, g in enumerate(gs):
    generate("llmrec", 42, rank, i, n, g)
r = torch.zeros(n, device="cuda")
th = torch.zeros(n, device="cuda")
voff = (k * 4 + 15) // 16 * 16
mine = gath[rank * blk:(rank + 1) * blk]
idx_v = mine[:k * 4].view(torch.int32)
val_v = mine[voff:voff + k * 4].view(torch.float32)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
acc = [0.0, 0.0, 0.0]
steps = 40
for s in range(steps + 20):
    ev[0].record()
    c.ef_topk(gs[s % 3], r, k, 0, idx_v, val_v)
    ev[1].record()
    c.allgather_(gath, blk)
    ev[2].record()
    c.sparse_mean_sgd(gath, world, k, torch.float32, "ring", 0.05, th, n)
    ev[3].record()
    torch.cuda.synchronize()
    if s >= 20:
        for j in range(3):
            acc[j] += ev[j].elapsed_time(ev[j + 1])
c.check()
t = torch.tensor([a / steps for a in acc], device="cuda", dtype=torch.float64)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
if rank == 0:
    print(f"world={world} compress {1e3 * t[0]:.1f} us  allgather {1e3 * t[1]:.1f} us "
          f"({world * blk / 1e6:.1f} MB gathered)  apply {1e3 * t[2]:.1f} us", flush=True)
dist.barrier()
c.close()
dist.barrier()
dist.destroy_process_group()
