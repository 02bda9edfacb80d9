"""Probe (one process, >= 2 GPUs): NVLink bandwidth of SM-driven pulls
(remote loads), pushes (remote stores) and copy-engine peer copies."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_17551_b200 import _lib as L  # noqa: E402

lib = L.load()
lib.psb_debug_copy16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
ng = torch.cuda.device_count()
for a in range(ng):
    for b in range(ng):
        if a != b:
            assert lib.psb_debug_enable_peer(a, b) == 0
for mb in (8, 30, 100):
    nb = mb * 1_000_000 // 16 * 16
    x0 = torch.empty(nb, dtype=torch.uint8, device="cuda:0")
    y0 = torch.empty(nb, dtype=torch.uint8, device="cuda:0")
    x1 = torch.empty(nb, dtype=torch.uint8, device="cuda:1")
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
        us = e0.elapsed_time(e1) / it * 1e3
        return us, nb / us / 1e3

    for ctas in (148, 592, 1184):
        pull = t(lambda: lib.psb_debug_copy16(y0.data_ptr(), x1.data_ptr(), nb, ctas, s.cuda_stream))
        push = t(lambda: lib.psb_debug_copy16(x1.data_ptr(), y0.data_ptr(), nb, ctas, s.cuda_stream))
        loc = t(lambda: lib.psb_debug_copy16(x0.data_ptr(), y0.data_ptr(), nb, ctas, s.cuda_stream))
        print(f"{mb} MB ctas={ctas}: pull {pull[0]:.1f} us {pull[1]:.0f} GB/s | push {push[0]:.1f} us "
              f"{push[1]:.0f} GB/s | local {loc[0]:.1f} us {loc[1]:.0f} GB/s", flush=True)
    ce = t(lambda: y0.copy_(x1, non_blocking=True))
    print(f"{mb} MB copy engine peer->local: {ce[0]:.1f} us {ce[1]:.0f} GB/s", flush=True)

# --- all-peer patterns (>= 3 GPUs): GPU0 pulls from / pushes to every peer at once
if ng >= 3:
    mb = 10
    nb = mb * 1_000_000 // 16 * 16
    src = {d: torch.empty(nb, dtype=torch.uint8, device=f"cuda:{d}") for d in range(ng)}
    dst0 = [torch.empty(nb, dtype=torch.uint8, device="cuda:0") for _ in range(ng)]
    torch.cuda.set_device(0)
    streams = [torch.cuda.Stream(0) for _ in range(ng)]
    s = torch.cuda.current_stream(0)

    def multi(push):
        ev = torch.cuda.Event()
        ev.record(s)
        for d in range(1, ng):
            streams[d].wait_event(ev)
            if push:
                lib.psb_debug_copy16(src[d].data_ptr(), dst0[d].data_ptr(), nb, 148 * 4 // (ng - 1), streams[d].cuda_stream)
            else:
                lib.psb_debug_copy16(dst0[d].data_ptr(), src[d].data_ptr(), nb, 148 * 4 // (ng - 1), streams[d].cuda_stream)
        for d in range(1, ng):
            e = torch.cuda.Event()
            e.record(streams[d])
            s.wait_event(e)

    for push in (False, True):
        us, _ = t(lambda: multi(push))
        tot = nb * (ng - 1)
        print(f"{'push to' if push else 'pull from'} {ng - 1} peers x {mb} MB: {us:.1f} us, {tot / us / 1e3:.0f} GB/s "
              f"aggregate", flush=True)
