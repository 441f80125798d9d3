"""Pin the CPU oracle against fixtures produced by the real reference.

These run without a GPU.  If the oracle drifts from the reference, every GPU
parity test (which uses the oracle as its checker) would be meaningless, so
this file is the root of the parity chain.
"""

import hashlib

import numpy as np
import pytest

from oracle import hsz_oracle as O


def _stream(arrays, name, key="container"):
    return O.stream_from_bytes(arrays[f"{name}/{key}"].tobytes())


def test_worked_example_kats(golden):
    """Paper worked example (reference test_acceptance.py:129-145, test_compressors.py:39-56)."""
    index, arrays = golden
    ex = np.array([[1.2, 1.5, -2.3, -2.5], [2.5, -1.0, 2.0, 1.7]], dtype=np.float32)
    assert O.quantize(ex, 0.1).tolist() == [[6, 8, -11, -12], [13, -5, 10, 9]]
    c = O.compress(ex, O.HSZX_ND, "abs", 0.1, (2, 2))
    assert c.metadata.tolist() == [5, -1]
    p = O.stage2(c)
    assert p.tolist() == [1, 3, 8, -10, -10, -11, 11, 10]
    assert O.as_grid(p, c.kind, c.dims, c.block_dims).tolist() == [[1, 3, -10, -11], [8, -10, 11, 10]]
    assert abs(O.std_from_dp(c, p) - 2.0) <= 1e-12
    hp, _ = O.decorrelate(O.quantize(ex, 0.1), O.HSZP, (32,))
    assert hp.tolist() == [6, 2, -19, -1, 25, -18, 15, -1]
    q = O.quantize(ex, 0.1)
    assert O.std_from_dq(q, 0.1) == pytest.approx(1.99929, abs=5e-6)


def test_codec_kats():
    """test_codec.py:14-29 golden bytes and the size formula."""
    payload, offs = O.encode_stream(np.array([3, -1, 0], np.int32), np.array([[0, 3]]))
    assert payload == bytes([2, 0b10, 0b0111])
    payload, offs = O.encode_stream(np.zeros(32, np.int32), np.array([[0, 32]]))
    assert payload == b"\x00"
    for count in (1, 7, 8, 9, 31, 32):
        for bw in (1, 3, 17, 31):
            vals = np.full(count, (1 << bw) - 1, dtype=np.int32)
            payload, _ = O.encode_stream(vals, np.array([[0, count]]))
            assert len(payload) == O.chunk_byte_size(count, bw)


def test_rounding_half_up():
    """test_quant.py:22-27."""
    assert O.quantize(np.array([1.5]), 0.1)[0] == 8
    assert O.quantize(np.array([-2.3]), 0.1)[0] == -11
    assert O.quantize(np.array([0.5]), 0.25)[0] == 1
    assert O.quantize(np.array([-0.5]), 0.25)[0] == -1


def test_containers_bit_exact(golden):
    """compress + stream_to_bytes byte-identical to the reference for every case."""
    index, arrays = golden
    for case in index["cases"]:
        name = case["name"]
        field = arrays[f"{name}/field"]
        mode, req = case["bound"]
        c = O.compress(field, case["kind"], mode, req, case["block_dims"])
        assert O.stream_to_bytes(c) == arrays[f"{name}/container"].tobytes(), name
        assert list(c.block_dims) == case["resolved_block_dims"]
        assert c.eps == case["eps"]


def test_stages_bit_exact(golden):
    index, arrays = golden
    for case in index["cases"]:
        name = case["name"]
        c = _stream(arrays, name)
        p = O.stage2(c)
        assert np.array_equal(p, arrays[f"{name}/p"]), name
        q = O.stage3(c, p)
        assert np.array_equal(q, arrays[f"{name}/q"]), name
        full = O.stage4(c, q)
        assert np.array_equal(full, arrays[f"{name}/full"]), name
        assert np.array_equal(O.as_grid(p, c.kind, c.dims, c.block_dims), arrays[f"{name}/p_grid"])


def test_stats_bit_identical(golden):
    index, arrays = golden
    for case in index["cases"]:
        c = _stream(arrays, case["name"])
        for key, want in case["stats"].items():
            op, st = key.split("@")
            got = O.compute_stat(c, op, int(st))
            assert got == want, (case["name"], key, got, want)


def test_stencils_bit_identical(golden):
    index, arrays = golden
    for case in index["cases"]:
        name = case["name"]
        c = _stream(arrays, name)
        nd = len(case["dims"])
        if nd == 1:
            got = O.field_op(c, "derivative", O.QUANTIZED)[0]
            assert np.array_equal(got, arrays[f"{name}/deriv3_0"])
            continue
        stages = [O.QUANTIZED, O.FULL] + ([O.DECORRELATED] if O.is_nd(c.kind) else [])
        for st in stages:
            for ax, comp in enumerate(O.field_op(c, "derivative", st)):
                assert np.array_equal(comp, arrays[f"{name}/deriv{st}_{ax}"]), (name, st, ax)
            lap = O.field_op(c, "laplacian", st)[0]
            assert np.array_equal(lap, arrays[f"{name}/lap{st}"]), (name, st)
        if O.is_nd(c.kind):
            for ax, comp in enumerate(O.streamed_derivative(c)):
                assert np.array_equal(comp, arrays[f"{name}/streamed_{ax}"])


def test_vector_ops_bit_identical(golden):
    index, arrays = golden
    for v in index["vector"]:
        name = v["name"]
        srcs = [_stream(arrays, name, f"container{j}") for j in range(len(v["dims"]))]
        for st in (O.DECORRELATED, O.QUANTIZED, O.FULL):
            assert np.array_equal(O.divergence(srcs, st), arrays[f"{name}/div{st}"])
            for j, comp in enumerate(O.curl(srcs, st)):
                assert np.array_equal(comp, arrays[f"{name}/curl{st}_{j}"])


def test_codec_streams_bit_exact(golden):
    index, arrays = golden
    for name in index["codec"]:
        vals = arrays[f"{name}/values"]
        spans = arrays[f"{name}/spans"]
        payload, offs = O.encode_stream(vals, spans)
        assert payload == arrays[f"{name}/payload"].tobytes()
        assert np.array_equal(offs, arrays[f"{name}/offsets"])
        assert np.array_equal(O.decode_stream(payload, spans, offs), vals)


def test_criterion9_codec_digest(golden):
    """Acceptance criterion 9 stream (test_acceptance.py:311-336) reproduced byte-for-byte."""
    index, _ = golden
    spec = index["criterion9"]
    big = np.random.default_rng(spec["seed"])
    n = spec["n_chunks"]
    counts = big.integers(1, 33, size=n)
    widths = big.integers(0, 32, size=n)
    scales = (np.int64(1) << widths) - 1
    values = np.concatenate([big.integers(-s, s, size=k, endpoint=True) if s else np.zeros(k, np.int64)
                             for k, s in zip(counts, scales)]).astype(np.int32)
    ends = np.cumsum(counts)
    spans = np.stack([ends - counts, ends], axis=1).astype(np.int64)
    payload, offs = O.encode_stream(values, spans)
    assert len(payload) == spec["payload_len"]
    assert hashlib.sha256(payload).hexdigest() == spec["payload_sha256"]
    assert hashlib.sha256(offs.astype("<u8").tobytes()).hexdigest() == spec["offsets_sha256"]
    assert np.array_equal(O.decode_stream(payload, spans, offs), values)


def test_corruption_messages(golden):
    index, arrays = golden
    for e in index["errors"]:
        name = e["name"]
        with pytest.raises(O.OracleError) as info:
            O.decode_stream(arrays[f"{name}/payload"].tobytes(), arrays[f"{name}/spans"],
                            arrays[f"{name}/offsets"])
        assert [info.value.cls, info.value.msg] == e["raises"]


def test_reference_cython_codec_matches_oracle():
    """oracle/_ref (the reference's own Cython codec) agrees with the C restatement."""
    import os
    import sys

    ref_dir = os.path.join(os.path.dirname(O.__file__), "_ref")
    if not os.path.isdir(ref_dir):
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, ref_dir)
    try:
        import _bitpack
    finally:
        sys.path.remove(ref_dir)
    rng = np.random.default_rng(5)
    for _ in range(10):
        size = int(rng.integers(1, 3000))
        vals = rng.integers(-(2**20), 2**20, size=size).astype(np.int32)
        spans = O.spans_from_segments([(0, size)])
        pay_r, off_r = _bitpack.encode_stream(vals, spans[:, 0], spans[:, 1])
        pay_o, off_o = O.encode_stream(vals, spans)
        assert pay_r == pay_o and np.array_equal(off_r, off_o)
        assert np.array_equal(_bitpack.decode_stream(pay_o, spans[:, 0], spans[:, 1], off_o), vals)


def test_new_ops_definitions():
    """N1-N5 oracle definitions on a hand-checkable grid."""
    q = np.arange(24, dtype=np.int32).reshape(2, 3, 4)
    s1, s2, qmin, qmax, size = O.region_reduce(q, 2)
    assert size.shape == (1, 2, 2)
    assert int(s1[0, 0, 0]) == int(q[:2, :2, :2].sum())
    assert qmin[0, 1, 1] == q[:2, 2:, 2:].min() and qmax[0, 1, 1] == q[:2, 2:, 2:].max()
    assert O.threshold_count(q, 0.5, 2, 10.0) == 3  # regions (0,0,0),(0,0,1),(0,1,0)
    g = O.gradient_magnitude(q, 0.5)
    assert g[1, 1, 1] == pytest.approx(0.5 * np.sqrt(8**2 + 2**2))  # D0 = 0 (axis 0 has 2 layers)
    q2 = np.arange(16, dtype=np.int32).reshape(4, 4)
    g2 = O.gradient_magnitude(q2, 0.5)
    assert g2[1, 1] == pytest.approx(0.5 * np.sqrt(8**2 + 2**2))
    v = O.var_from_dq(q, 0.1)
    assert v == pytest.approx(np.var(q.astype(np.float64) * 0.2, ddof=1), rel=1e-12)
