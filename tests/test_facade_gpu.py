"""The C++ drop-in facade (include/parsim_b200.hpp): builds on CPU; on the GPU its
f64 results are bit-identical to the f64 oracle, which tests/test_oracle.py pins
to the reference itself."""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "build", "facade_check")


def build_facade(out=BIN):
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "facade_check.cpp"), "-o", out,
           "-L", os.path.join(ROOT, "paper_2506_17551_b200"), "-lpsb", "-L", "/usr/local/cuda/lib64",
           "-lcudart", "-Wl,-rpath," + os.path.join(ROOT, "paper_2506_17551_b200"),
           "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_facade_compiles_and_links(tmp_path):
    build_facade(str(tmp_path / "facade_check"))


@pytest.mark.gpu
def test_facade_matches_reference_f64(tmp_path):
    binary = build_facade(str(tmp_path / "facade_check"))
    P, n, k, steps, lr = 4, 20_000, 200, 3, 0.05
    g = np.stack([np.stack([O.generate("llmrec", 99, p, s, n) for p in range(P)])
                  for s in range(steps)]).astype(np.float64)
    g.tofile(tmp_path / "g.bin")
    (tmp_path / "meta.txt").write_text(f"{P} {n} {k} {steps} {lr}\n")
    out = subprocess.run([binary, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    rd = lambda name, dt=np.float64: np.fromfile(tmp_path / name, dtype=dt)  # noqa: E731

    # compress_topk
    oi, ov = O.topk(g[0, 0], k)
    assert np.array_equal(rd("topk_idx.bin", np.uint64), oi.astype(np.uint64))
    assert np.array_equal(rd("topk_val.bin"), ov)
    # ef_compress_step (topk) over the steps on worker 1
    r = np.zeros(n)
    trace = []
    for s in range(steps):
        i, v, _ = O.ef_topk(g[s, 1].copy(), r, k)
        trace += [i.astype(np.float64), v]
    trace.append(r)
    assert np.array_equal(rd("ef_res.bin"), np.concatenate(trace))
    # allreduce_mean, all algorithms
    for algo in ("naive", "ring", "hierarchical", "pipelined_ring"):
        assert np.array_equal(rd(f"mean_{algo}.bin"), O.fold_mean(g[0], algo)), algo
    # sync_data_parallel_step, top-k + EF, ring
    theta = np.zeros(n)
    res = np.zeros((P, n))
    for s in range(steps):
        O.sync_step(g[s].copy(), theta, lr, "topk", k, "ring", res)
    assert np.array_equal(rd("sync_theta.bin"), theta)
    assert np.array_equal(rd("sync_res.bin"), res.reshape(-1))
    # 1-bit EF: bits exact, scale within 1e-12 (tree vs sequential sum), residual exact given the scale
    ob = rd("onebit.bin")
    words, scale, _ = O.ef_onebit(g[0, 0].copy(), None)
    assert abs(ob[0] - scale) <= 1e-12 * abs(scale)
    assert np.array_equal(rd("onebit_bytes.bin", np.uint8), words.view(np.uint8)[: (n + 7) // 8])
    p = g[0, 0]
    assert np.array_equal(ob[1:], p - np.where(p >= 0, ob[0], -ob[0]))
    # async_step(theta = g00, g = g01, tau = 3, eta = 0.1)
    want = g[0, 0].copy()
    O.axpy_(-O.orc().orc_async_scale(0.1, 3), g[0, 1], want)
    assert np.array_equal(rd("async.bin"), want)
    errs = (tmp_path / "errors.txt").read_text().splitlines()
    assert errs[0].startswith("invalid_argument: compress_topk: k out of range")
    assert errs[1].startswith("invalid_argument: ef_compress_step: residual/gradient dimension mismatch")
