"""Per-step device timeline of the multi-rank cfg2 step inside one CUDA graph
(torchrun): a timestamp kernel before every step; per rank, the step
durations and where the slow ones fall.  PROBE_STEPS, PROBE_NB."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402
from paper_2506_17551_b200.dist import init_comm  # noqa: E402
from paper_2506_17551_b200.engine import Context, generate  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
n = 125_000_000
k = n // 100
steps = int(os.environ.get("PROBE_STEPS", "40"))
NB = int(os.environ.get("PROBE_NB", "8"))
c = Context(n, k, world, device=rank)
init_comm(c)
lib = L.load()
lib.psb_debug_stamp.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
lib.psb_debug_stamps.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    gs = [torch.empty(1, n, device="cuda") for _ in range(NB)]
    for i, g in enumerate(gs):
        generate("llmrec", 42, rank, i, n, g[0])
    res = torch.zeros(1, n, device="cuda")
    theta = torch.zeros(n, device="cuda")
    descs = [c.step_desc(L.PSB_COMP_TOPK, g, res, theta, 0.05, k, "ring") for g in gs]
    for i in range(5):
        c.sync_step(descs[i % NB])
    c.check()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        for i in range(steps):
            lib.psb_debug_stamp(c.h, st.cuda_stream)
            c.sync_step(descs[(5 + i) % NB])
        lib.psb_debug_stamp(c.h, st.cuda_stream)
    graph.replay()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 4096)()
    lib.psb_debug_stamps(buf, 4096)  # drop the untimed replay's stamps
    dist.barrier()
    torch.cuda.synchronize()
    graph.replay()
    torch.cuda.synchronize()
    m = lib.psb_debug_stamps(buf, 4096)
d = [(buf[i + 1] - buf[i]) / 1e3 for i in range(m - 1)]
t = torch.tensor(d + [0.0] * (steps - len(d)), device="cuda", dtype=torch.float64)
allt = [torch.zeros_like(t) for _ in range(world)]
dist.all_gather(allt, t)
if rank == 0:
    for r, x in enumerate(allt):
        v = [round(float(a), 1) for a in x]
        print(f"rank {r}: mean {sum(v) / len(v):.1f} us  max {max(v):.1f}  steps: {v}", flush=True)
dist.barrier()
c.close()
dist.barrier()
dist.destroy_process_group()
