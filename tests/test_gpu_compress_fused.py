"""One-pass GPU compress (csrc/compress.cu, hszg_compress_fused) vs the multi-kernel chain and the oracle.

The container produced by the one-pass kernel must be byte-identical to the chain's (quantize ->
decorrelate_sized -> encode_offsets -> encode_pack, itself pinned to the reference's golden containers
in test_gpu_golden.py) and to the oracle's compress (oracle/hsz_oracle.py:381, compressors.py:313-339),
including ragged last tiles, tiles crossing planes, 1-D / 2-D / 3-D boxes, non-default blocks, bit
width 0 and 31 chunks, and the EpsTooSmallError / ValueError behaviour.
"""

import zlib

import numpy as np
import pytest

from oracle import hsz_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import compressors, io, _lib

    class NS:
        pass

    ns = NS()
    ns.h, ns.comp, ns.io, ns.lib = h, compressors, io, _lib
    return ns


def _both(H, field, kind, eps, block_dims=None, monkeypatch=None):
    """(one-pass bytes, chain bytes, whether the one-pass kernel applied)."""
    import ctypes
    import torch

    K = H.h.CompressorKind(kind)
    d = torch.from_numpy(np.ascontiguousarray(field)).cuda()
    shape = H.comp.GridShape(tuple(field.shape))
    bd = H.comp.resolve_block_dims(K, shape, block_dims)
    g = H.lib.make_geom(int(K), shape.dims, bd, eps)
    applies = bool(H.lib.lib().hszg_compress_plan(ctypes.byref(g), None, None))
    ds1 = H.comp.compress_device(d, K, eps, bd)
    monkeypatch.setattr(H.comp, "_ONE_PASS", False)
    ds2 = H.comp.compress_device(d, K, eps, bd)
    monkeypatch.setattr(H.comp, "_ONE_PASS", True)
    b1 = H.io.stream_to_bytes(H.comp.CompressedStream(K, shape, bd, eps, device=ds1))
    b2 = H.io.stream_to_bytes(H.comp.CompressedStream(K, shape, bd, eps, device=ds2))
    pad = ds1.payload[ds1.payload_len: ds1.payload_len + H.lib.PAYLOAD_PAD].cpu().numpy()
    assert not pad.any(), "payload pad must be zero"
    return b1, b2, applies


CASES = [
    # (kind, dims, block_dims)
    (0, (8192 * 3 + 64,), None),           # HSZP: ragged last tile
    (0, (256, 96), None),                  # HSZP 2-D field, flat stream
    (0, (32,), None),
    (1, (5, 64, 512), None),               # HSZP_ND: 16 rows per tile, planes of 64 rows
    (1, (7, 30, 384), None),               # 21 rows per tile: tiles cross planes
    (1, (3, 5, 8192), None),               # one row per tile
    (1, (40, 96), None),                   # 2-D
    (1, (2, 1, 64), None),                 # one-row planes: every tile crosses planes
    (2, (8192 * 2 + 32 * 5,), None),       # HSZX 1-D, 32-value blocks, ragged tile
    (2, (64, 64), None),                   # HSZX on a 2-D field (flat blocks)
    (2, (4096,), (64,)),                   # 64-value blocks (2 chunks)
    (3, (16, 24, 40), None),               # HSZX_ND 8^3: 5 blocks per tile row
    (3, (8, 8, 1024), None),               # 16 blocks per tile, 8 tiles per block row
    (3, (16, 16, 16), (4, 4, 4)),          # 64-value blocks
    (3, (64, 48), None),                   # 2-D 8x8
    (3, (8, 32, 128), (8, 4, 32)),         # 1024-value blocks
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"k{c[0]}-{'x'.join(map(str, c[1]))}")
@pytest.mark.parametrize("field_kind", ["smooth", "rough"])
def test_one_pass_equals_chain_and_oracle(H, monkeypatch, case, field_kind):
    kind, dims, bd = case
    rng = np.random.default_rng(zlib.crc32(repr((kind, dims, field_kind)).encode()))
    if field_kind == "smooth":
        f = O.random_field(rng, dims).astype(np.float32)
        eps = 1e-3
    else:                                   # wide residuals: bit widths up to ~24, zero chunks too
        f = (rng.standard_normal(dims) * 10.0 ** rng.integers(-3, 5, size=dims)).astype(np.float32)
        f.reshape(-1)[: min(f.size, 96)] = 0.0
        eps = 1e-3
    b1, b2, applies = _both(H, f, kind, eps, bd, monkeypatch)
    assert applies, "the one-pass front should cover this geometry"
    assert b1 == b2
    oc = O.compress(f, kind, "abs", eps, bd)
    assert b1 == O.stream_to_bytes(oc)


def test_one_pass_bitwidth_31(H, monkeypatch):
    f = np.zeros((64, 512), np.float32)
    f[::2, ::3] = 2.0e9 * 2e-3 * 0.49      # |q| near 2^30, alternating with zero: |p| ~ 2^31 - small
    f[1::2, 1::3] = -2.0e9 * 2e-3 * 0.49
    for kind in (0, 1, 2, 3):
        b1, b2, applies = _both(H, f, kind, 1e-3, None, monkeypatch)
        assert applies and b1 == b2


def test_one_pass_not_applicable_falls_back(H, monkeypatch):
    # rows not whole chunks (HSZP_ND n2 % 32 != 0), ragged blocks, partial chunks: the chain runs
    for kind, dims in [(1, (6, 7, 50)), (3, (10, 9, 13)), (0, (1000,))]:
        f = O.random_field(np.random.default_rng(3), dims).astype(np.float32)
        b1, b2, applies = _both(H, f, kind, 1e-2, None, monkeypatch)
        assert not applies and b1 == b2
        assert b1 == O.stream_to_bytes(O.compress(f, kind, "abs", 1e-2))


def test_one_pass_errors(H):
    import torch

    big = torch.full((8192,), 3.0e38, dtype=torch.float32, device="cuda")
    for kind in (0, 1, 2, 3):
        dims = (8192,) if kind in (0, 2) else (16, 512)
        with pytest.raises(H.h.EpsTooSmallError, match="quantization index"):
            H.comp.compress_device(big.reshape(dims), H.h.CompressorKind(kind), 1e-6,
                                   H.comp.resolve_block_dims(H.h.CompressorKind(kind), H.comp.GridShape(dims), None))
    # residual overflow without an index overflow: alternating +-(2^31 - 2) * 2 eps
    alt = np.empty(8192, np.float64)
    alt[0::2], alt[1::2] = 2.0**30 + 2.0**29, -(2.0**30 + 2.0**29)
    with pytest.raises(H.h.EpsTooSmallError, match="residual"):
        H.comp.compress_device(torch.from_numpy(alt.astype(np.float32) * np.float32(2e-3 * 1.0)).cuda(),
                               H.h.CompressorKind.HSZP, 1e-3, (32,))


def test_one_pass_large_trimmed(H, monkeypatch):
    # a payload buffer wasting more than the trim threshold is copied to size; contents unchanged
    monkeypatch.setattr(H.comp, "_TRIM_BYTES", 1 << 10)
    f = O.random_field(np.random.default_rng(5), (8, 64, 512)).astype(np.float32)
    b1, b2, applies = _both(H, f, 1, 1e-3, None, monkeypatch)
    assert applies and b1 == b2
