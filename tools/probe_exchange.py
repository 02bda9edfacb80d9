"""Probe (torchrun): bare NVLink payload exchange (signal + pull) per call,
max over ranks, for a few payload sizes."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.dist import init_comm  # noqa: E402
from paper_2506_17551_b200.engine import Context  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
c = Context(1 << 20, 1 << 16, world, device=rank)
init_comm(c)
lib = L.load()
lib.psb_debug_exchange.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
s = torch.cuda.current_stream()
for mb in (2.5, 10, 20):
    b = int(mb * 1e6) // 16 * 16
    assert lib.psb_debug_exchange(c.h, b, 3, s.cuda_stream) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    assert lib.psb_debug_exchange(c.h, b, 20, s.cuda_stream) == 0
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 20 * 1e3], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ingress = b * (world - 1)
        print(f"world={world} {mb} MB/rank: {float(t):.1f} us per exchange, {ingress / float(t) / 1e3:.0f} GB/s ingress",
              flush=True)
c.check()
dist.barrier()
c.close()
dist.barrier()
dist.destroy_process_group()
