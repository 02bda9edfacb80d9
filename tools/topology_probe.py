"""Calibrate the reference's alpha-beta model on this node and compare it with measured steps.

Two modes:

  torchrun --nproc-per-node N tools/topology_probe.py calibrate --out cal_N.json
      times NCCL float32 all-reduces of 1 MiB .. 256 MiB on N GPUs (CUDA
      events, max over ranks) and fits the intra-node link class
      (costmodel.calibrate_intra_node).

  python tools/topology_probe.py report --bench1 b1.json --bench b2.json cal_2.json [--bench b4.json cal_4.json]
      builds the modeled data-parallel step for each N from the calibrated
      topology (costmodel.dp_iteration: compute = the measured 1-GPU step,
      comm = comm_cost(ring, gradient_bytes / compression ratio)) and prints
      one JSON object with modeled vs measured ms per step.
"""
import argparse
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

SIZES = [1 << e for e in range(20, 29)]


def calibrate(out: str) -> None:
    import torch
    import torch.distributed as dist
    from paper_2506_17551_b200.costmodel import calibrate_intra_node, measure_allreduce

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    secs = measure_allreduce(SIZES, iters=20, warmup=5)
    t = calibrate_intra_node(world, SIZES, secs)
    if rank == 0:
        rec = {"P": world, "sizes": SIZES, "seconds": secs,
               "busbw_GBps": [2 * (world - 1) / world * m / s / 1e9 for m, s in zip(SIZES, secs)],
               "intra_node_bw": t.intra_node_bw, "intra_node_lat": t.intra_node_lat,
               "nccl_algo": os.environ.get("NCCL_ALGO", "default")}
        with open(out, "w") as f:
            json.dump(rec, f, indent=1)
        print(json.dumps({k: rec[k] for k in ("P", "intra_node_bw", "intra_node_lat")}))
    dist.destroy_process_group()


def _last_json(path: str) -> dict:
    with open(path) as f:
        lines = [l for l in f.read().splitlines() if l.startswith("{")]
    return json.loads(lines[-1])


def report(bench1: str, pairs) -> None:
    from paper_2506_17551_b200.costmodel import comm_cost, dp_iteration
    from paper_2506_17551_b200.parsim import CompressorConfig, CompressorKind, Topology

    b1 = _last_json(bench1)
    cfg = b1["config"]
    n, k = int(cfg["n_params"]), int(cfg["k"])
    compute = b1["ms_per_step"] * 1e-3
    comp = CompressorConfig(CompressorKind.topk, top_k=k)
    rows = []
    for bench, cal in pairs:
        b = _last_json(bench)
        with open(cal) as f:
            c = json.load(f)
        P = int(c["P"])
        topo = Topology(devices_per_node=P, intra_node_bw=c["intra_node_bw"], intra_node_lat=c["intra_node_lat"])
        # gradient_bytes in the reference's accounting: 8 bytes per parameter (DenseVector of doubles)
        it = dp_iteration(P, topo, 8.0 * n, comp, compute_time=compute)
        fp32_ring = comm_cost("ring", 4.0 * n, P, topo)
        rows.append({"P": P, "measured_ms": b["ms_per_step"], "modeled_ms": it.wall_time * 1e3,
                     "modeled_comm_ms": it.comm_time * 1e3, "compute_ms_from_1gpu": compute * 1e3,
                     "measured_minus_compute_ms": b["ms_per_step"] - compute * 1e3,
                     "dense_fp32_ring_allreduce_ms": fp32_ring * 1e3,
                     "topology": {"intra_node_bw": c["intra_node_bw"], "intra_node_lat": c["intra_node_lat"]},
                     "peak_busbw_GBps": max(c["busbw_GBps"])})
    print(json.dumps({"workload": cfg.get("workload"), "n": n, "k": k, "rows": rows}, indent=1))


def main() -> None:
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("calibrate")
    c.add_argument("--out", required=True)
    r = sub.add_parser("report")
    r.add_argument("--bench1", required=True)
    r.add_argument("--bench", nargs=2, action="append", metavar=("BENCH_JSON", "CAL_JSON"), required=True)
    a = ap.parse_args()
    if a.cmd == "calibrate":
        calibrate(a.out)
    else:
        report(a.bench1, a.bench)


if __name__ == "__main__":
    main()
