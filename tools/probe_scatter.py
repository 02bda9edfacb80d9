"""Probe (one process, 2 GPUs): theta[idx] = val scatter of an update list
(3.5M sorted random indices over 125M), list local vs on the peer GPU."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402

lib = L.load()
lib.psb_debug_scatter.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                  ctypes.c_void_p]
assert lib.psb_debug_enable_peer(0, 1) == 0
n = 125_000_000
cnt = int(os.environ.get("PROBE_CNT", "3500000"))
g = torch.Generator().manual_seed(0)
idx = torch.randperm(n, generator=g)[:cnt].sort().values.to(torch.int32)
val = torch.randn(cnt, generator=g)
theta = torch.zeros(n, device="cuda:0")
li0, lv0 = idx.to("cuda:0"), val.to("cuda:0")
li1, lv1 = idx.to("cuda:1"), val.to("cuda:1")
torch.cuda.set_device(0)
s = torch.cuda.current_stream(0)


def t(fn, it=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(it):
        fn()
    e1.record(s)
    torch.cuda.synchronize(0)
    return e0.elapsed_time(e1) / it * 1e3


for ctas in (592, 1184, 2368):
    loc = t(lambda: lib.psb_debug_scatter(theta.data_ptr(), li0.data_ptr(), lv0.data_ptr(), cnt, ctas, s.cuda_stream))
    rem = t(lambda: lib.psb_debug_scatter(theta.data_ptr(), li1.data_ptr(), lv1.data_ptr(), cnt, ctas, s.cuda_stream))
    print(f"cnt={cnt} ctas={ctas}: local list {loc:.1f} us, peer list {rem:.1f} us", flush=True)
