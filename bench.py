"""bench.py -- dense-equiv gradient GB/s of the compress+aggregate+apply step.

Default (no flags): N=1 GPU, BASELINE.json configs[1] shape at one rank:
125M-param LLM-rec gradient, EF top-k 1%, sparse allgather (one rank: no
exchange), sync SGD.  Under torchrun (N>1) every rank owns one worker (P = N),
compresses its own 125M gradient, the payloads are allgathered over NCCL and
every replica applies the same rank-ordered mean (weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg2|cfg3|cfg4|cfg1|cfg2m] [--n N] [--rho R]

One JSON line on rank 0 (contract in the task statement; fields explained in
DESIGN.md "Measurement").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "dense-equiv gradient GB/s per step (compress+aggregate+apply) at 1/2/4/8 B200"

CONFIGS = {
    # name: (workload text, n, rho, compressor, order, dist, mode, extra)
    "cfg2": ("cfg2: 125M-param LLM-rec gradient, top-k 1% + error feedback, sparse allgather, sync SGD",
             125_000_000, 0.01, "topk", "ring", "llmrec", "sync", {}),
    "cfg3": ("cfg3: 125M-param gradient, dense 8-bit block-quantized (B=256) hierarchical allreduce, sync SGD",
             125_000_000, 0.0, "q8", "naive", "llmrec", "sync", {"q8_block": 256}),
    "cfg4": ("cfg4: 350M-param gradient, top-k 0.1% + int8 values, async bounded staleness s=2",
             350_000_000, 0.001, "topk_q8", "naive", "llmrec", "async", {"staleness": 2}),
    "cfg1": ("cfg1: 1M-param gradient, top-k 1% + error feedback, sync SGD, 4 simulated workers",
             1_000_000, 0.01, "topk", "ring", "uniform", "sync", {"workers": 4}),
    # north-star a24 (no reference code): reported separately from the reference-semantics SGD
    "cfg2m": ("cfg2 + momentum SGD (beta 0.9, dense momentum pass; this build's rule, not the reference's)",
              125_000_000, 0.01, "topk", "ring", "llmrec", "sync", {"momentum": 0.9}),
}

CLOCK_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock + clock-event reasons sampled through NVML every ~1 ms while
    the timed region runs (the same counters nvidia-smi's clocks line reads;
    the timed region is milliseconds long, below nvidia-smi -lms granularity)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.err = None

    def __enter__(self):
        if os.environ.get("PSB_BENCH_NO_CLOCKS"):
            self.err, self.nv = "disabled", None
            return self
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception as e:  # NVML missing: report unsampled, never fake
            self.err = str(e)
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM), int(get_r(self.h))))
            except Exception as e:
                self.err = str(e)
                return
            time.sleep(0.001)

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0,
                    "note": self.err}
        reasons = set()
        for _, bits in self.samples:
            for b, name in CLOCK_REASONS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples), "source": "nvml"}


# --------------------------------------------------------------- CPU legs
def host_cpu():
    """CPU model and core count of the host the CPU leg ran on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_reference_run(n_sample: int, P: int, k: int, threads: int, budget_s: float, min_steps: int,
                      max_steps: int, dist: str, comp: str):
    """Time the reference's own sync_data_parallel_step (oracle/_ref) on a
    bounded sample; returns (GB/s dense-equiv, seconds per step, steps, kind)."""
    import numpy as np

    from oracle import oracle as O
    kind = "reference" if O.ref_available() else "port"
    grads = [np.stack([O.generate(dist, 42, p, s, n_sample) for p in range(P)]).astype(np.float64)
             for s in range(2)]
    theta = np.zeros(n_sample)
    res = np.zeros((P, n_sample))
    times = []
    t_start = time.perf_counter()
    for s in range(max_steps):
        t0 = time.perf_counter()
        if kind == "reference":
            if comp == "topk":
                O.ref_sync_step_threaded("topk", k, "ring", grads[s % 2], theta, 0.05, res, threads)
            else:
                O.ref_sync_step("none", 0, "naive", grads[s % 2], theta, 0.05, None)
        else:
            g32 = grads[s % 2].astype(np.float32)
            O.sync_step(g32, theta.astype(np.float32), 0.05, comp if comp == "topk" else "none", k,
                        "ring", res.astype(np.float32))
        times.append(time.perf_counter() - t0)
        if len(times) >= min_steps and time.perf_counter() - t_start > budget_s:
            break
    t = statistics.median(times)
    return 4.0 * n_sample * P / t / 1e9, t, len(times), kind


def reference_arm(args, cfg, world, rank):
    name, n, rho, comp, order, dist, mode, extra = cfg
    if rank != 0:
        return
    P = world * extra.get("workers", 1)
    n_sample = min(n, 2_000_000)
    k = max(1, int(round(rho * n_sample))) if comp.startswith("topk") else 0
    threads = max(1, min(P, os.cpu_count() or 1))
    ref_comp = "topk" if comp.startswith("topk") else "none"
    steps = max(1, args.steps)
    # warmup (untimed) then K timed steps, each a bounded sample of the workload
    if args.warmup:
        cpu_reference_run(n_sample, P, k, threads, 0.0, 1, 1, dist, ref_comp)
    gbs, t, done, kind = cpu_reference_run(n_sample, P, k, threads, 0.0, steps, steps, dist, ref_comp)
    sample = (f"N={n_sample} of {n} params per worker x P={P} workers, k={k} ({ref_comp}), "
              f"{done} steps of the reference sync_data_parallel_step"
              f"{' (per-worker ef_compress_step on ' + str(threads) + ' threads, serial fold)' if threads > 1 else ''}")
    line = {
        "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": done,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (same mix64 generator, widened to f64)",
        "config": {"workload": name, "n_params": n, "P": P, "sample_n": n_sample},
        "impl": "reference",
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": kind, "sample": sample,
                         "same_config": n_sample == n, "sample_n": n_sample, "full_n": n, **host_cpu()},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU arm
def ours(args, cfg, world, rank, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2506_17551_b200 import _lib as L
    from paper_2506_17551_b200.engine import Context, generate

    name, n, rho, comp, order, dist_name, mode, extra = cfg
    if args.n:
        n = args.n
    if args.rho is not None:
        rho = args.rho
    W = extra.get("workers", 1)
    P = W * world
    k = max(1, int(round(rho * n))) if comp.startswith("topk") else 0
    comp_code = {"topk": L.PSB_COMP_TOPK, "topk_q8": L.PSB_COMP_TOPK_Q8, "q8": L.PSB_COMP_Q8,
                 "onebit": L.PSB_COMP_ONEBIT, "none": L.PSB_COMP_NONE}[comp]
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(dev)
    ctx = Context(n, max(k, 1), P, device=local_rank)
    if world > 1:
        from paper_2506_17551_b200.dist import init_comm
        init_comm(ctx)  # NCCL unique id from rank 0 over the process group

    # rotated gradient buffers (each > L2: inputs larger than L2); 8 rather than
    # 3 so the sequence the threshold predictor sees is not period-3
    NB = int(os.environ.get("PSB_BENCH_NB", "8"))
    with torch.cuda.stream(stream):
        grads = [torch.empty(W, n, device=dev) for _ in range(NB)]
        for b in range(NB):
            for w in range(W):
                generate(dist_name, 42, rank * W + w, b, n, grads[b][w])
        res = torch.zeros(W, n, device=dev)
        theta = torch.zeros(n, device=dev)
        mom = torch.zeros(n, device=dev) if "momentum" in extra else None
        descs = [ctx.step_desc(comp_code, grads[b], res, theta, 0.05, k, order,
                               extra.get("q8_block", 256), momentum=mom, beta=extra.get("momentum", 0.0))
                 for b in range(NB)]
    stream.synchronize()
    gu = [0]
    pipe = mode == "async" and not os.environ.get("PSB_BENCH_NO_PIPE")
    if pipe:
        # bounded-staleness pipeline: round r's exchange + apply on the ctx's
        # apply stream overlap round r+1's compression (psb_async_pipeline)
        ctx.async_pipeline(True)

    def drain():  # join the apply stream back (before timing ends / capture closes)
        if pipe:
            ctx.async_sync()

    def step(i):
        d = descs[i % NB]
        if mode == "async":
            gu[0] = ctx.async_round(d, extra.get("staleness", 2), gu[0])
        else:
            ctx.sync_step(d)

    def barrier():
        if world > 1:
            dist.barrier()

    align = torch.zeros(1, device=dev)

    def align_start():
        # device-side rendezvous on the timing stream right before the start
        # event: the host barrier leaves ranks launching up to ~1.6 ms apart
        # (measured at N = 4), and a rank that starts early would time its
        # wait for the late one at the first exchange
        if world > 1:
            with torch.cuda.stream(stream):
                dist.all_reduce(align)

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
        drain()
        ctx.check()
        # ---- timed region: K steps, device-timed with events on our stream.
        # The K steps are captured once into a CUDA graph and replayed (the
        # step's launch sequence is fixed; all control flow is device-side),
        # with the dominant kernel bracketed by event-record nodes.
        barrier()
        torch.cuda.synchronize(dev)
        ctx.profile_enable(bool(args.eager))
        ctx.profile_read()
        l0 = ctx.launches
        graph = None
        if not args.eager:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                for i in range(args.steps):
                    step(args.warmup + i)
                drain()
        if graph is not None:
            # one untimed replay: a graph's first launch uploads it to the
            # device (measured +0.1 ms/step over a 20-step window at N = 4)
            graph.replay()
            torch.cuda.synchronize(dev)
        miss0 = ctx.topk_stats(0)["misses"] if comp.startswith("topk") else 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize(dev)
        with ClockSampler(local_rank) as clk:
            align_start()
            e0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                for i in range(args.steps):
                    step(args.warmup + i)
                drain()
            e1.record(stream)
            torch.cuda.synchronize(dev)
        barrier()
        launches = ctx.launches - l0
        ctx.check()
        # threshold-prediction misses inside the timed window (any rank's miss
        # stalls every rank at the exchange): max over ranks
        miss = torch.tensor([(ctx.topk_stats(0)["misses"] - miss0) if comp.startswith("topk") else 0],
                            device=dev, dtype=torch.int64)
        if world > 1:
            dist.all_reduce(miss, op=dist.ReduceOp.MAX)
        timed_misses = int(miss[0])
        if graph is not None:
            # dominant-kernel timing: event-record pairs around K1's streaming
            # pass need eager launches (graph event nodes are not timeable)
            ctx.profile_enable(True)
            for i in range(args.steps):
                step(args.warmup + args.steps + i)
            drain()
            torch.cuda.synchronize(dev)
        ctx.profile_enable(False)
        k1_ms, k1_count = ctx.profile_read()
        ex_ms, _ = ctx.profile_read_phase(1)  # exchange (signal + pull / NCCL), per profiled step
        ap_ms, _ = ctx.profile_read_phase(2)  # P-payload apply
        ctx.check()
        ms_local = e0.elapsed_time(e1) / args.steps
        t = torch.tensor([ms_local, k1_ms / max(k1_count, 1), ex_ms / args.steps, ap_ms / args.steps],
                         device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, k1_avg_ms, ex_step_ms, ap_step_ms = (float(x) for x in t)
        by_rank = torch.zeros(world, device=dev, dtype=torch.float64)  # each rank's own step time
        by_rank[rank] = ms_local
        if world > 1:
            dist.all_reduce(by_rank)

        # ---- e2e through the public API: pinned host gradient in, theta out
        host_g = [torch.empty(W, n, pin_memory=True) for _ in range(2)]
        for b in range(2):
            host_g[b].copy_(grads[b].cpu())
        # double-buffered: H2D of step i+1 and D2H of step i-1's theta snapshot
        # overlap step i on separate streams (PCIe is full duplex)
        host_theta = [torch.empty(n, pin_memory=True) for _ in range(2)]
        dev_g = [torch.empty(W, n, device=dev) for _ in range(2)]
        snap = [torch.empty(n, device=dev) for _ in range(2)]
        d_e2e = [ctx.step_desc(comp_code, dev_g[b], res, theta, 0.05, k, order,
                               extra.get("q8_block", 256), momentum=mom, beta=extra.get("momentum", 0.0))
                 for b in range(2)]
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = lambda: torch.cuda.Event()  # noqa: E731
        in_done = [ev(), ev()]
        comp_done = [ev(), ev()]
        out_done = [ev(), ev()]
        e_steps = max(4, min(args.steps, 24))  # 24 amortises the pipeline fill (one unoverlapped H2D)
        barrier()
        torch.cuda.synchronize(dev)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        align_start()
        f0.record(stream)
        s_in.wait_stream(stream)
        for i in range(e_steps):
            b = i % 2
            with torch.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(comp_done[b])  # step i-2 consumed dev_g[b]
                dev_g[b].copy_(host_g[b], non_blocking=True)
                in_done[b].record(s_in)
            stream.wait_event(in_done[b])
            if mode == "async":
                gu[0] = ctx.async_round(d_e2e[b], extra.get("staleness", 2), gu[0])
                drain()  # the theta snapshot below reads this round's result
            else:
                ctx.sync_step(d_e2e[b])
            if i >= 2:
                stream.wait_event(out_done[b])  # snapshot b drained to the host
            snap[b].copy_(theta)
            comp_done[b].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(comp_done[b])
                host_theta[b].copy_(snap[b], non_blocking=True)
                out_done[b].record(s_out)
        stream.wait_stream(s_out)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        ctx.check()
        te = torch.tensor([f0.elapsed_time(f1) / e_steps], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te[0])

    if rank != 0:
        return ctx
    peak, peak_src = load_peaks()
    dense_bytes = 4.0 * n * P
    value = dense_bytes / (ms_step * 1e-3) / 1e9
    e2e_value = dense_bytes / (e2e_ms * 1e-3) / 1e9
    # roofline of the dominant kernel: algorithmic bytes per launch
    if comp == "q8" and world == 1:
        # fused single-rank q8 step: per worker read g, read r, write r; theta read+write
        k1_name = "k_q8_step1 (quantize + EF + fold + requantize + SGD, one pass)"
        k1_bytes = (12.0 * W + 8.0) * n
    elif comp == "q8":
        b = extra.get("q8_block", 256)
        k1_name = "k_q8_quant (EF add + per-block int8 quantization)"
        k1_bytes = W * (13.0 + 4.0 / b) * n
    else:
        # K1 streaming pass: 12 bytes/element (read g, read r, write r) x n
        k1_name = "k_scan<float,MODE_A> (EF add + level-1 histogram)"
        k1_bytes = 12.0 * n
    k1_gbs = k1_bytes / (k1_avg_ms * 1e-3) / 1e9 if k1_avg_ms > 0 else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "k1_traffic.json")) as f:
            tr = json.load(f)
        traffic = tr.get(f"{comp}:{n}:{world}") or tr.get(f"{comp}:{n}")
    except Exception:
        pass
    # whole-step algorithmic bytes per GPU: 12N + 8k + 8Pk + 8|U| (|U| <= Pk)
    step_alg = 12.0 * n + 8.0 * k + 8.0 * P * k + 8.0 * min(P * k, n) if comp == "topk" else None
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (counter-based mix64 LLM-rec gradients generated on device before timing)",
        "config": {"workload": name, "n_params": n, "k": k, "rho": rho, "workers_per_rank": W, "P": P,
                   "launch": "eager" if args.eager else "cuda-graph of the K timed steps",
                   "compressor": comp, "order": order, "mode": mode,
                   "async_pipeline": pipe,
                   "l2": f"inputs larger than L2: {NB} rotated {4 * n * W / 1e6:.0f} MB gradient buffers"},
        "roofline": {"bound": "hbm", "kernel": k1_name,
                     "achieved": k1_gbs, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": (k1_gbs / peak) if k1_gbs else None, "traffic": traffic,
                     "alg_bytes_per_launch": k1_bytes, "avg_launch_ms": k1_avg_ms,
                     "step_alg_bytes": step_alg,
                     "step_frac": (step_alg / (ms_step * 1e-3) / 1e9 / peak) if step_alg else None},
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": 4 * n * W,
                "d2h_bytes_per_step": 4 * n, "ms_per_step": e2e_ms,
                "path": "psb_sync_step via the Python host API; per step: pinned host gradient H2D, "
                        "step, theta snapshot D2H to pinned host (copies double-buffered on side streams)"},
        "gpu_launches": launches,
    }
    if world > 1:
        # NVLink exchange: bytes this rank receives per step and their rate;
        # for an all-gather that ingress rate is the NCCL-convention busBW
        # ((P-1)/P x algBW).  The exchange window includes waiting for the
        # slowest peer.  Peak: 900 GB/s per direction (NVLink 5 spec; no
        # measured NVLink figure in MEASURED_PEAKS.json).
        a16 = lambda b: (b + 15) // 16 * 16  # noqa: E731
        if comp == "q8":
            B = extra.get("q8_block", 256)
            nb = (n + B - 1) // B
            nbs = (nb + world - 1) // world
            shard = nbs * B + 4 * nbs
            bytes_in = (world - 1) * W * shard + (world - 1) * shard  # all-to-all + all-gather
            if os.environ.get("PSB_NO_PEER") or os.environ.get("PSB_PEER_MODE", "1") == "0":
                how = "NCCL grouped send/recv all-to-all of int8 block shards + all-gather of the requantized shards"
            else:
                how = ("NVLink pulls: every remote worker's int8 codes of this rank's block shard, then every "
                       "rank's requantized shard (window: two flag rounds, both pulls and the shard reduce)")
        elif comp in ("topk", "topk_q8"):
            pm = "0" if os.environ.get("PSB_NO_PEER") else os.environ.get("PSB_PEER_MODE", "5")
            direct = comp == "topk" and pm in ("4", "5")
            if comp == "topk" and not os.environ.get("PSB_NO_WIRE16") and pm in ("1", "4", "5"):
                seg_shift = 15
                while seg_shift > 10 and (P * 8) << (seg_shift - 5) > 16 * 1024:
                    seg_shift -= 1
                nseg = (n + (1 << seg_shift) - 1) >> seg_shift
                blk = a16(2 * k) + a16(4 * k) + 4 * (nseg + 1)  # wire16 payload + offset rows
                how = "NVLink pull of wire16 payloads (u16 in-segment index | f32) + per-segment offset rows"
            else:
                from paper_2506_17551_b200.engine import payload_bytes
                blk = payload_bytes(comp_code, torch.float32, k)
                how = ("NCCL all-gather of the payloads" if pm == "0" else "NVLink pull of the payloads")
            if direct:
                # the exchange is fused into the apply: its TMA stage reads the
                # peers' arenas in place, so the window is the apply
                how = ("NVLink reads of the peers' wire16 payloads + offset rows, in place, by the TMA-staged "
                       "apply (exchange fused into the fold; window = the apply kernel)")
                ex_step_ms = ap_step_ms
            bytes_in = (P - W) * blk
        else:
            bytes_in, how = None, comp
        if bytes_in and ex_step_ms > 0:
            bw = bytes_in / (ex_step_ms * 1e-3) / 1e9
            line["exchange"] = {"bytes_in_per_rank": bytes_in, "ms_per_step": ex_step_ms, "busbw_gbs": bw,
                                "peak_gbs": 900.0, "peak_source": "NVLink 5 spec, per direction",
                                "frac": bw / 900.0, "what": how}
        if ap_step_ms > 0:
            line["apply_ms_per_step"] = ap_step_ms
        line["ms_per_step_by_rank"] = [round(float(x), 4) for x in by_rank]
    if comp.startswith("topk"):
        st = ctx.topk_stats(0)
        line["config"]["k1_last_call"] = {kk: st[kk] for kk in ("candidates", "predicted_valid", "first_radix_level",
                                                                "calls", "misses", "margin_f")}
        line["config"]["k1_misses_in_timed_window_max_over_ranks"] = timed_misses
    if world == 1 and not args.no_cpu_baseline:
        n_s = min(n, 2_000_000)
        k_s = max(1, int(round(rho * n_s))) if comp.startswith("topk") else 0
        gbs, t_s, done, kind = cpu_reference_run(n_s, P, k_s, 1, 12.0, 2, 20, dist_name,
                                                 "topk" if comp.startswith("topk") else "none")
        line["cpu_baseline"] = {
            "value": gbs, "unit": "GB/s", "cores": 1, "kind": kind,
            "sample": f"SAMPLE of the workload: {done} steps of the reference's sync_data_parallel_step at "
                      f"N={n_s} of {n} params (P={P}, k={k_s}), median {t_s:.3f} s/step, 1 thread (the reference "
                      f"is single-threaded); its per-element cost grows with N (stable_sort), so the GB/s at "
                      f"full N is lower (survey: 0.007 GB/s at 125M)",
            "same_config": n_s == n, "sample_n": n_s, "full_n": n, **host_cpu()}
    print(json.dumps(line), flush=True)
    return ctx


def _teardown_watchdog(seconds: float) -> None:
    """The JSON line is out; never let a stuck communicator teardown hang the run."""
    def _kill():
        time.sleep(seconds)
        sys.stderr.write("bench.py: teardown exceeded %.0fs, exiting\n" % seconds)
        sys.stderr.flush()
        os._exit(0)
    threading.Thread(target=_kill, daemon=True).start()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # defaults: 30 warm-up steps take the error-feedback residual (and with it
    # the top-k threshold) past its initial transient; 100 timed steps ~50 ms
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=30)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--rho", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="launch the timed steps eagerly (no CUDA graph)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "RANK" not in os.environ:
        # `python bench.py --gpus N` outside a launcher: start the N ranks
        # the way the driver does (one process per GPU, 127.0.0.1 rendezvous)
        import socket
        import subprocess
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}; measuring {world} rank(s)", file=sys.stderr)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        reference_arm(args, cfg, world, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    ctx = ours(args, cfg, world, rank, local_rank)
    _teardown_watchdog(60.0)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()          # every rank done with the communicators
        ctx.close()             # ncclCommDestroy on all ranks together
        dist.barrier()
        dist.destroy_process_group()
    else:
        ctx.close()


if __name__ == "__main__":
    main()
