"""GPU parity against the reference's own outputs (tests/golden, made by importing the real reference).

Everything here runs through libhszg.so on the device: compress (container
bytes), stage 2/3/4, statistics, stencils, vector operators, the chunk codec
plugin and its corruption messages.  Integers/bytes are compared bit-exact;
floats are compared bit-exact too (the kernels reproduce the reference's fp64
rounding sequence), except stage-4 statistics whose float summation order
legitimately differs (tolerance 1e-12 relative, well inside the 1e-6 target).
"""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STAGE4_STAT_RTOL = 1e-12


@pytest.fixture(scope="module")
def hsz():
    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import _kernels, codec, io
    from paper_2603_25206_b200.analytics import fields, stats

    return h, io, stats, fields, codec, _kernels


def _stream(hsz, arrays, name, key="container"):
    io = hsz[1]
    return io.stream_from_bytes(arrays[f"{name}/{key}"].tobytes())


def test_compress_container_bytes(golden, hsz):
    h, io = hsz[0], hsz[1]
    index, arrays = golden
    for case in index["cases"]:
        name = case["name"]
        field = arrays[f"{name}/field"]
        mode, req = case["bound"]
        c = h.compress(field, h.CompressorKind(case["kind"]), h.ErrorBound(mode, req), case["block_dims"])
        assert io.stream_to_bytes(c) == arrays[f"{name}/container"].tobytes(), name
        assert list(c.block_dims) == case["resolved_block_dims"]
        assert c.eps == case["eps"]


def test_stages_bit_exact(golden, hsz):
    h = hsz[0]
    index, arrays = golden
    for case in index["cases"]:
        name = case["name"]
        c = _stream(hsz, arrays, name)
        ds = h.partial_decompress(c, h.Stage.DECORRELATED)
        assert np.array_equal(ds.values, arrays[f"{name}/p"]), name
        assert np.array_equal(ds.as_grid(), arrays[f"{name}/p_grid"]), name
        q = h.partial_decompress(c, h.Stage.QUANTIZED)
        assert q.values.dtype == np.int32
        assert np.array_equal(q.values, arrays[f"{name}/q"]), name
        full = h.partial_decompress(c, h.Stage.FULL)
        assert full.dtype == np.float64
        assert np.array_equal(full, arrays[f"{name}/full"]), name
        if c.kind.is_block_mean:
            assert np.array_equal(h.partial_decompress(c, h.Stage.META), c.metadata)


def test_stats_match_reference(golden, hsz):
    h, stats = hsz[0], hsz[2]
    index, arrays = golden
    for case in index["cases"]:
        c = _stream(hsz, arrays, case["name"])
        for key, want in case["stats"].items():
            op, st = key.split("@")
            got = stats.compute_stat(c, op, h.Stage(int(st))).value
            if int(st) == 4:
                assert got == pytest.approx(want, rel=STAGE4_STAT_RTOL, abs=1e-300), (case["name"], key)
            else:
                assert got == want, (case["name"], key, got, want)   # bit-identical scalars


def test_stencils_bit_exact(golden, hsz):
    h, fields = hsz[0], hsz[3]
    index, arrays = golden
    for case in index["cases"]:
        name = case["name"]
        c = _stream(hsz, arrays, name)
        nd = len(case["dims"])
        if nd == 1:
            got = fields.compute_field_op(c, "derivative", h.Stage.QUANTIZED).components[0]
            assert np.array_equal(got, arrays[f"{name}/deriv3_0"]), name
            continue
        stages = [3, 4] + ([2] if c.kind.is_nd else [])
        for st in stages:
            d = fields.compute_field_op(c, "derivative", h.Stage(st))
            for ax, comp in enumerate(d.components):
                assert np.array_equal(comp, arrays[f"{name}/deriv{st}_{ax}"]), (name, st, ax)
            lap = fields.compute_field_op(c, "laplacian", h.Stage(st)).components[0]
            assert np.array_equal(lap, arrays[f"{name}/lap{st}"]), (name, st)
        if c.kind.is_nd:
            for ax, comp in enumerate(fields.streamed_derivative(c).components):
                assert np.array_equal(comp, arrays[f"{name}/streamed_{ax}"]), (name, ax)


def test_vector_ops_bit_exact(golden, hsz):
    h, fields = hsz[0], hsz[3]
    index, arrays = golden
    for v in index["vector"]:
        name = v["name"]
        srcs = tuple(_stream(hsz, arrays, name, f"container{j}") for j in range(len(v["dims"])))
        for st in (2, 3, 4):
            div = fields.divergence(srcs, h.Stage(st)).components[0]
            assert np.array_equal(div, arrays[f"{name}/div{st}"]), (name, st)
            for j, comp in enumerate(fields.curl(srcs, h.Stage(st)).components):
                assert np.array_equal(comp, arrays[f"{name}/curl{st}_{j}"]), (name, st, j)


def test_codec_plugin_bit_exact(golden, hsz):
    _kernels = hsz[5]
    index, arrays = golden
    for name in index["codec"]:
        vals = arrays[f"{name}/values"]
        spans = arrays[f"{name}/spans"]
        payload, offs = _kernels.encode_stream(vals, spans[:, 0], spans[:, 1])
        assert payload == arrays[f"{name}/payload"].tobytes(), name
        assert np.array_equal(offs, arrays[f"{name}/offsets"])
        back = _kernels.decode_stream(payload, spans[:, 0], spans[:, 1], offs)
        assert np.array_equal(back, vals)


def test_criterion9_codec_digest(golden, hsz):
    codec = hsz[4]
    spec = golden[0]["criterion9"]
    big = np.random.default_rng(spec["seed"])
    n = spec["n_chunks"]
    counts = big.integers(1, 33, size=n)
    widths = big.integers(0, 32, size=n)
    scales = (np.int64(1) << widths) - 1
    values = np.concatenate([big.integers(-s, s, size=k, endpoint=True) if s else np.zeros(k, np.int64)
                             for k, s in zip(counts, scales)]).astype(np.int32)
    ends = np.cumsum(counts)
    spans = np.stack([ends - counts, ends], axis=1).astype(np.int64)
    payload, offs = codec.encode_stream(values, spans)
    assert hashlib.sha256(payload).hexdigest() == spec["payload_sha256"]
    assert hashlib.sha256(offs.astype("<u8").tobytes()).hexdigest() == spec["offsets_sha256"]
    assert np.array_equal(codec.decode_stream(payload, spans, offs), values)


def test_corruption_messages(golden, hsz):
    h, _kernels = hsz[0], hsz[5]
    index, arrays = golden
    for e in index["errors"]:
        name = e["name"]
        with pytest.raises(h.CorruptStreamError) as info:
            _kernels.decode_stream(arrays[f"{name}/payload"].tobytes(), arrays[f"{name}/spans"][:, 0],
                                   arrays[f"{name}/spans"][:, 1], arrays[f"{name}/offsets"])
        assert [type(info.value).__name__, str(info.value)] == e["raises"]
