"""GPU parity of the device wire codec (psb_wire.cu) against the oracle's
restatement of parsim wire_encode / wire_decode (compression.hpp:159-239),
which tests/test_oracle.py pins byte-for-byte to the reference."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2506_17551_b200 import _lib as L
from paper_2506_17551_b200 import parsim as ps
from tests.refrng import SeededRng

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("dim,k", [(1, 1), (1000, 37), (1 << 20, 10_000), (125_000_000, 1_250_000)])
def test_topk_encode_bytes_and_round_trip(ctx, dtype, dim, k):
    if dim > ctx.max_n:
        # full cfg2 size: encode / decode through a fresh context sized for it
        from paper_2506_17551_b200.engine import Context
        c = Context(max_n=k, max_k=k, max_workers=1)
    else:
        c = ctx
    rng = np.random.default_rng(dim + k)
    idx_h = np.sort(rng.choice(dim, k, replace=False)).astype(np.uint32)
    val_h = rng.standard_normal(k).astype(np.float32 if dtype == torch.float32 else np.float64)
    idx = torch.from_numpy(idx_h.view(np.int32)).cuda()
    val = torch.from_numpy(val_h).cuda()
    wire = c.wire_encode_topk(dim, idx, val)
    ref_bytes = O.wire_encode_topk(dim, idx_h, val_h.astype(np.float64))
    assert np.array_equal(wire.cpu().numpy(), ref_bytes)
    d, i2, v2 = c.wire_decode_topk(wire, dtype)
    assert d == dim
    assert np.array_equal(i2.cpu().numpy().view(np.uint32), idx_h)
    assert torch.equal(v2, val)
    if c is not ctx:
        c.close()


def test_decode_errors(ctx):
    idx = torch.arange(0, 64, 2, dtype=torch.int32, device="cuda")
    val = torch.randn(32, device="cuda")
    wire = ctx.wire_encode_topk(100, idx, val)
    for cut in (1, 16, wire.numel() - 8):
        with pytest.raises(L.PsbInvalidArgument, match="wire_decode: truncated input"):
            ctx.wire_decode_topk(wire[:wire.numel() - cut].clone())
    with pytest.raises(L.PsbInvalidArgument, match="capacity"):
        ctx.wire_decode_topk(wire, k_cap=31)
    bad = wire.clone()
    bad[16 + 7] = 1  # index of record 0 >= 2^32
    with pytest.raises(L.PsbInvalidArgument, match="32-bit"):
        ctx.wire_decode_topk(bad)
    # the context is usable afterwards
    d, i2, _ = ctx.wire_decode_topk(wire)
    assert d == 100 and i2.numel() == 32


@pytest.mark.parametrize("n", [1, 7, 33, 1000, 1 << 20])
def test_signbit_and_dense_bytes(ctx, n):
    g = torch.from_numpy(O.generate("uniform", 3, 0, 0, n)).cuda()
    words, scale = ctx.ef_onebit(g, None)
    wire = ctx.wire_encode_signbit(n, words, scale)
    assert np.array_equal(wire.cpu().numpy(),
                          O.wire_encode_signbit(n, float(scale.item()), words.cpu().numpy().view(np.uint32)))
    dense = ctx.wire_encode_dense(g)
    assert np.array_equal(dense.cpu().numpy(), O.wire_encode_dense(g.cpu().numpy().astype(np.float64)))


def test_facade_round_trips_as_the_reference_test():
    """proj/tests/test_compression.cpp:197-219 through the reference-shaped API."""
    rng = SeededRng(4321)
    for _ in range(20):
        n = 1 + rng.below(40)
        g = torch.tensor([rng.uniform(-5, 5) for _ in range(n)], dtype=torch.float64, device="cuda")
        d = ps.CompressedGradient(ps.DensePayload(g))
        d2 = ps.wire_decode(ps.WireKind.dense, ps.wire_encode(d))
        assert torch.equal(ps.decompress(d2), ps.decompress(d))
        s = ps.compress_onebit(g)
        s2 = ps.wire_decode(ps.WireKind.signbit, ps.wire_encode(s))
        assert torch.equal(ps.decompress(s2), ps.decompress(s))
        t = ps.compress_topk(g, 1 + rng.below(n))
        t2 = ps.wire_decode(ps.WireKind.topk, ps.wire_encode(t))
        assert torch.equal(ps.decompress(t2), ps.decompress(t))
    b = ps.wire_encode(ps.CompressedGradient(ps.DensePayload(torch.tensor([1.0, 2.0], dtype=torch.float64,
                                                                         device="cuda"))))
    assert b.numel() == 8 + 16 and int(b[0]) == 2
    assert ps.compression_ratio_for(ps.CompressorConfig(ps.CompressorKind.onebit, 0), 64) == pytest.approx(512 / 24)
    assert ps.compression_ratio_for(ps.CompressorConfig(ps.CompressorKind.none, 0), 64) == 1.0
    assert ps.compression_ratio_for(ps.CompressorConfig(ps.CompressorKind.topk, 8), 8) < 1.0


@pytest.mark.parametrize("n", [1, 7, 33, 1000, 1 << 20])
def test_decompress_signbit_on_device(n):
    """decompress(SignBitPayload) (compression.hpp:118-126): +-scale per sign
    bit, ragged last byte, through the device 1-bit kernel."""
    rng = np.random.default_rng(n)
    signs = rng.integers(0, 2, n).astype(bool)
    sb = np.packbits(signs, bitorder="little")
    scale = float(rng.random()) + 0.25
    got = ps.decompress(ps.CompressedGradient(ps.SignBitPayload(n, scale, torch.from_numpy(sb))))
    want = np.where(signs, scale, -scale)
    assert got.dtype == torch.float64 and np.array_equal(got.cpu().numpy(), want)
    with pytest.raises(L.PsbInvalidArgument):
        ps.decompress(ps.CompressedGradient(ps.SignBitPayload(n + 8, scale, torch.from_numpy(sb))))
