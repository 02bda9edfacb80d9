"""The alpha-beta communication model (costmodel.py), CPU only.

comm_cost is pinned bit-for-bit against the compiled reference
(collectives.hpp:184-215) on random topologies; the reference's own
test_collectives.cpp:101-165 and test_simulator.cpp:40-52 cases are restated;
the ring fit recovers known parameters; and a world_size-2 gloo group runs the
measure -> calibrate loop end to end.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2506_17551_b200 import _lib as L
from paper_2506_17551_b200.costmodel import (calibrate_intra_node, comm_cost, dp_iteration, fit_ring,
                                             measure_allreduce, slowest_link_spanning)
from paper_2506_17551_b200.parsim import CollectiveAlgorithm, CompressorConfig, CompressorKind, Topology
from tests.conftest import ROOT

ALGOS = list(CollectiveAlgorithm)


def _uniform(devices, bw, lat):
    # test_collectives.cpp's uniform_topo: one node of `devices`, every class equal
    return Topology(1, 1, devices, bw, bw, bw, lat, lat, lat)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_comm_cost_matches_reference_bitwise():
    rng = np.random.default_rng(7)
    for _ in range(400):
        counts = [int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 9))]
        links = [float(10 ** rng.uniform(8, 12)) for _ in range(3)] + [float(10 ** rng.uniform(-7, -4)) for _ in range(3)]
        t = Topology(*counts, *links)
        P = int(rng.integers(1, t.device_count() + 3))
        span = int(rng.integers(0, 2 * P + 1))
        msg = float(rng.choice([0.0, 1.0, 10 ** rng.uniform(0, 10)]))
        for a, algo in enumerate(ALGOS):
            assert comm_cost(algo, msg, P, t, span) == O.ref_comm_cost(a, msg, P, counts, links, span)


def test_comm_cost_basics():
    # test_collectives.cpp:101-116
    topo = _uniform(16, 12.5e9, 1e-6)
    for a in ALGOS:
        assert comm_cost(a, 1e9, 1, topo) == 0.0
    c = comm_cost("ring", 1073741824.0, 4, topo)
    assert math.isclose(c, 2 * 3 * 1e-6 + 1.5 * (1073741824.0 / 12.5e9), rel_tol=1e-12)
    assert abs(c - 0.1289) <= 2e-4
    bad = _uniform(16, 12.5e9, 1e-6)
    bad.intra_node_bw = 0.0
    with pytest.raises(L.PsbInvalidArgument):
        comm_cost("ring", 1.0, 4, bad)
    with pytest.raises(L.PsbInvalidArgument):
        comm_cost("ring", -1.0, 4, topo)
    with pytest.raises(L.PsbInvalidArgument):
        comm_cost("ring", 1.0, 0, topo)


def test_naive_grows_ring_bounded():
    # test_collectives.cpp:118-128
    topo = _uniform(16, 1e9, 0.0)
    msg = 1e8
    base = comm_cost("naive", msg, 2, topo)
    for P in (2, 4, 8, 16):
        assert math.isclose(comm_cost("naive", msg, P, topo), base * (P - 1), rel_tol=1e-12)
        assert comm_cost("ring", msg, P, topo) <= 2.0 * msg / 1e9 + 1e-12


def test_monotone_and_hierarchical():
    # test_collectives.cpp:130-165
    topo = _uniform(32, 5e9, 1e-6)
    slow = _uniform(32, 5e9, 1e-4)
    for a in ALGOS:
        prev = -1.0
        for msg in np.arange(0, 1e9 + 1, 2.5e8):
            c = comm_cost(a, float(msg), 8, topo)
            assert c >= prev
            prev = c
        assert comm_cost(a, 1e8, 8, slow) >= comm_cost(a, 1e8, 8, topo)
    h = Topology(4, 2, 8, 100e9, 50e9, 1e9, 1e-6, 2e-6, 5e-6)
    P = h.device_count()
    assert comm_cost("hierarchical", 1e9, P, h) < comm_cost("ring", 1e9, P, h)
    link = slowest_link_spanning(h, 9)
    assert (link.latency, link.bandwidth) == (2e-6, 50e9)


def test_dp_iteration_serial_and_compressed():
    # test_simulator.cpp:40-52 (serial composition) and :200-212 (compressed message)
    topo = _uniform(2, 1.0, 0.0)
    it = dp_iteration(2, topo, 1e8, CompressorConfig(CompressorKind.none), compute_time=64e-3)
    x = comm_cost("ring", 1e8, 2, topo, 2)
    assert it.comm_time == x and it.wall_time == 64e-3 + x
    t8 = _uniform(8, 100e9, 1e-6)
    cfg = CompressorConfig(CompressorKind.topk, top_k=1000)
    it = dp_iteration(8, t8, 8e8, cfg, compute_time=0.0)
    ratio = 8.0 * 1e8 / (16.0 + 16.0 * 1000)
    assert it.comm_time == comm_cost("ring", 8e8 / ratio, 8, t8, 8)
    full = dp_iteration(8, t8, 8e8, cfg, compute_time=1.0, overlap_fraction=1.0)
    assert full.wall_time == 1.0  # comm <= compute is hidden completely


def test_fit_ring_recovers_parameters():
    for P in (2, 4, 8):
        lat, bw = 7e-6, 350e9
        sizes = [2.0 ** e for e in range(16, 30)]
        times = [2 * (P - 1) * lat + 2 * (P - 1) / P * m / bw for m in sizes]
        link = fit_ring(P, sizes, times)
        assert math.isclose(link.latency, lat, rel_tol=1e-6) and math.isclose(link.bandwidth, bw, rel_tol=1e-9)
        t = calibrate_intra_node(P, sizes, times)
        assert t.devices_per_node == P and math.isclose(comm_cost("ring", 1e7, P, t),
                                                        2 * (P - 1) * lat + 2 * (P - 1) / P * 1e7 / bw, rel_tol=1e-6)
    with pytest.raises(L.PsbInvalidArgument):
        fit_ring(2, [1.0, 1.0], [1.0, 2.0])
    with pytest.raises(L.PsbInvalidArgument):
        fit_ring(1, [1.0, 2.0], [1.0, 2.0])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sizes = [1 << 16, 1 << 20, 1 << 22]
        secs = measure_allreduce(sizes, iters=4, warmup=1)
        t = calibrate_intra_node(world, sizes, secs)
        q.put((rank, secs, t.intra_node_bw, t.intra_node_lat))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


def test_gloo_measure_and_calibrate():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(60)
    assert all(isinstance(r[1], list) for r in res), res
    assert res[0][1] == res[1][1]  # max over ranks: both ranks report the same times
    assert res[0][2] > 0 and res[0][3] >= 0


def test_b200_step_model_fit_and_terms():
    """The round-2 step model: fit_line recovers a line; the fitted model
    reproduces its inputs and adds the ingress and fold terms only for P > 1."""
    from paper_2506_17551_b200.costmodel import B200StepModel, fit_line
    a, b = fit_line([1, 2, 3, 4], [3.0, 5.0, 7.0, 9.0])
    assert math.isclose(a, 1.0) and math.isclose(b, 2.0)
    k, pb = 1_250_000, 7.6e6
    m = B200StepModel.fit(compress_p1=330e-6, compress=290e-6, pack=15e-6, k=k,
                          apply_by_p={2: 90e-6, 4: 150e-6, 8: 270e-6},
                          ingress_by_p={2: 38e-6, 4: 80e-6}, payload_bytes=pb)
    assert m.step(1, k, pb) == 330e-6
    assert math.isclose(m.ingress(2, pb), 38e-6, rel_tol=1e-9) and math.isclose(m.ingress(4, pb), 80e-6, rel_tol=1e-9)
    assert abs(m.apply(4, k) - 150e-6) < 10e-6
    assert m.step(8, k, pb) > m.step(4, k, pb) > m.step(2, k, pb) > m.step(1, k, pb) * 0.9
    with pytest.raises(L.PsbInvalidArgument):
        fit_line([1, 1], [1, 2])



@pytest.mark.gpu
def test_b200_step_model_predicts_virtual_worker_step():
    """On one GPU: fit the compression and fold terms from their own
    measurements at P = 2 and 8, then predict a step the fit did not see --
    W = 4 virtual workers (4 x K1 + the 4-payload apply, no exchange) --
    within 15 %."""
    import torch
    from paper_2506_17551_b200.costmodel import B200StepModel, measure_step_parts
    from paper_2506_17551_b200.engine import Context, generate
    n, k = 16_000_000, 160_000
    c = Context(n, k, 8)
    parts = measure_step_parts(c, n, k, Ps=(2, 8))
    m = B200StepModel.fit(parts["compress_p1"], parts["compress"], 0.0, k, parts["apply_by_p"], {},
                          parts["payload_bytes"])
    W = 4
    g = torch.empty(W, n, device="cuda")
    for w in range(W):
        generate("llmrec", 42, w, 5, n, g[w])
    r = torch.zeros(W, n, device="cuda")
    th = torch.zeros(n, device="cuda")
    d = c.step_desc(L.PSB_COMP_TOPK, g, r, th, 0.05, k, "ring")
    for _ in range(5):
        c.sync_step(d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        c.sync_step(d)
    e1.record()
    torch.cuda.synchronize()
    measured = e0.elapsed_time(e1) * 1e-3 / 10
    predicted = W * parts["compress"] + m.apply(W, k)
    c.close()
    assert abs(predicted - measured) / measured < 0.15, (predicted, measured)
