"""GPU tests mirroring the reference's unit / acceptance tests (pkg/tests/*), checked against the oracle.

The package under test is paper_2603_25206_b200 (the drop-in for ``hsz``);
the checker is oracle/hsz_oracle.py, itself pinned to the reference by
tests/test_oracle_golden.py.
"""

import numpy as np
import pytest

from oracle import hsz_oracle as O

pytestmark = pytest.mark.gpu

ALL = [0, 1, 2, 3]
ND = [1, 3]


@pytest.fixture(scope="module")
def H():
    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import codec, compressors, grid, io, quant, stages
    from paper_2603_25206_b200.analytics import fields, regions, stats

    class NS:
        pass

    ns = NS()
    ns.h, ns.codec, ns.comp, ns.grid, ns.io, ns.quant, ns.stages = h, codec, compressors, grid, io, quant, stages
    ns.fields, ns.regions, ns.stats = fields, regions, stats
    return ns


def _oracle_of(c):
    return O.stream_from_bytes(__import__("paper_2603_25206_b200").io.stream_to_bytes(c))


# ---- quant (test_quant.py) ---------------------------------------------------------------


def test_quantize_kats(H, example_field):
    q = H.quant.quantize(example_field, 0.1)
    assert q.tolist() == [[6, 8, -11, -12], [13, -5, 10, 9]]
    assert H.quant.quantize(np.array([1.5]), 0.1)[0] == 8
    assert H.quant.quantize(np.array([-2.3]), 0.1)[0] == -11
    assert H.quant.quantize(np.array([0.5]), 0.25)[0] == 1
    assert H.quant.quantize(np.array([-0.5]), 0.25)[0] == -1
    np.testing.assert_allclose(H.quant.dequantize(np.array([6, -11, 0]), 0.1), [1.2, -2.2, 0.0])
    with pytest.raises(H.h.EpsTooSmallError):
        H.quant.quantize(np.array([1e30]), 1e-6)
    with pytest.raises(ValueError):
        H.quant.quantize_field(np.array([1.0, np.nan]), 0.1)
    with pytest.raises(H.h.ZeroValueRangeError):
        H.quant.resolve_eps(np.full(8, 3.0), H.h.ErrorBound("rel", 1e-2))
    assert H.quant.resolve_eps(np.array([-2.0, 6.0]), H.h.ErrorBound("rel", 1e-2)) == pytest.approx(0.08)


def test_quantize_matches_oracle_random(H):
    rng = np.random.default_rng(1)
    for _ in range(20):
        d = rng.normal(0, 10 ** rng.uniform(-2, 4), size=int(rng.integers(1, 5000)))
        eps = 10 ** rng.uniform(-4, 0)
        assert np.array_equal(H.quant.quantize(d, eps), O.quantize(d, eps))
        d32 = d.astype(np.float32)
        assert np.array_equal(H.quant.quantize(d32, eps), O.quantize(d32, eps))


# ---- codec (test_codec.py, test_kernels.py) ----------------------------------------------------


def test_codec_kats(H):
    ch = H.codec.encode_chunk(np.zeros(32, dtype=np.int64))
    assert ch.bitwidth == 0 and ch.to_bytes() == b"\x00" and ch.byte_size() == 1
    ch = H.codec.encode_chunk([3, -1, 0])
    assert ch.bitwidth == 2 and ch.to_bytes() == bytes([2, 0b10, 0b0111])
    back, consumed = H.codec.chunk_from_bytes(ch.to_bytes(), 3)
    assert consumed == 3 and np.array_equal(H.codec.decode_chunk(back), [3, -1, 0])
    with pytest.raises(ValueError):
        H.codec.encode_chunk([-(2**31)])
    with pytest.raises(ValueError):
        H.codec.encode_chunk(np.ones(33, dtype=np.int64))
    with pytest.raises(H.h.CorruptStreamError):
        H.codec.chunk_from_bytes(bytes([40, 0, 0]), 3)
    buf = H.codec.encode_chunk(np.arange(1, 20)).to_bytes()
    with pytest.raises(H.h.CorruptStreamError):
        H.codec.chunk_from_bytes(buf[:-1], 19)
    with pytest.raises(H.h.CorruptStreamError):
        H.codec.chunk_from_bytes(bytes([1, 0b1, 0b0]), 1)
    assert H.codec.spans_from_segments([(0, 70), (70, 75)]).tolist() == [[0, 32], [32, 64], [64, 70], [70, 75]]


def test_codec_random_streams_vs_oracle(H):
    rng = np.random.default_rng(9)
    for _ in range(30):
        size = int(rng.integers(1, 3000))
        scale = int(rng.choice([1, 7, 2**10, 2**24, 2**31 - 1]))
        vals = rng.integers(-scale, scale, size=size, endpoint=True).astype(np.int32)
        cut = int(rng.integers(0, size + 1))
        segs = [(0, cut), (cut, size)] if 0 < cut < size else [(0, size)]
        spans = H.codec.spans_from_segments(segs)
        pay, off = H.codec.encode_stream(vals, spans)
        pay_o, off_o = O.encode_stream(vals, spans)
        assert pay == pay_o and np.array_equal(off, off_o)
        assert np.array_equal(H.codec.decode_stream(pay, spans, off), vals)
    vals = rng.integers(-9, 9, size=400).astype(np.int32)
    spans = H.codec.spans_from_segments([(0, 100), (100, 400)])
    pay, off = H.codec.encode_stream(vals, spans)
    assert np.array_equal(H.codec.decode_chunk_range(pay, spans, off, 4, 8), vals[100:228])
    assert np.array_equal(H.codec.decode_chunk_range(pay, spans, off, 8, len(spans)), vals[228:])


def test_bitwidth_32_chunks(H):
    vals = np.array([2**31 - 1, -(2**31 - 1), 0, 5] * 8, dtype=np.int32)
    spans = H.codec.spans_from_segments([(0, 32)])
    pay, off = H.codec.encode_stream(vals, spans)
    assert pay[0] == 31
    assert np.array_equal(H.codec.decode_stream(pay, spans, off), vals)
    # a hand-made b=32 chunk whose magnitudes fit int32 decodes; one with the top bit set is corrupt
    mags = np.array([7, 2**31 - 1], dtype=np.uint64)
    body = bytes([32, 0b01]) + b"".join(int(m).to_bytes(4, "little") for m in mags)
    assert H.codec.decode_stream(body, np.array([[0, 2]]), np.array([0], np.uint64)).tolist() == [-7, 2**31 - 1]
    bad = bytes([32, 0]) + (2**31).to_bytes(4, "little") + (1).to_bytes(4, "little")
    with pytest.raises(H.h.CorruptStreamError, match="magnitude"):
        H.codec.decode_stream(bad, np.array([[0, 2]]), np.array([0], np.uint64))


# ---- compressors / stages (test_compressors.py, test_stages.py) ----------------------------


@pytest.mark.parametrize("kind", ALL)
@pytest.mark.parametrize("dims", [(40,), (7, 9), (5, 6, 7), (33, 17), (9, 10, 70)])
def test_decorrelate_recorrelate_identity(H, rng, kind, dims):
    if kind in ND and len(dims) < 2:
        pytest.skip("nd compressor needs 2D+")
    K = H.comp.CompressorKind(kind)
    q = rng.integers(-1000, 1000, size=dims).astype(np.int32)
    qf = H.quant.QuantizedField(q, 0.05)
    shape = H.grid.GridShape(dims)
    bd = H.comp.resolve_block_dims(K, shape, None)
    geo = H.comp.effective_geometry(K, shape, bd)
    ds = H.comp.decorrelate(qf, K, geo)
    p_o, m_o = O.decorrelate(q, kind, bd)
    assert np.array_equal(ds.values, p_o)
    if m_o is not None:
        assert np.array_equal(ds.metadata, m_o)
    assert np.array_equal(H.comp.recorrelate(ds).values, q)


def test_residual_overflow_raises(H):
    qf = H.quant.QuantizedField(np.array([-(2**30), 2**30], dtype=np.int32), 0.5)
    with pytest.raises(H.h.EpsTooSmallError):
        H.comp.decorrelate_hszp(qf)


def test_compress_rejects_nan(H):
    with pytest.raises(ValueError):
        H.h.compress(np.array([1.0, np.nan, 2.0], np.float32), H.h.CompressorKind.HSZP, H.h.ErrorBound("abs", 0.1))


@pytest.mark.parametrize("kind", ALL)
@pytest.mark.parametrize("dims", [(64,), (12, 10), (6, 7, 8), (37, 3, 41), (5, 9, 64), (3, 17, 256), (3, 17, 96), (4, 25, 384), (300, 3, 64)])
def test_stage_composition_and_error_bound(H, rng, kind, dims):
    if kind in ND and len(dims) < 2:
        pytest.skip("nd compressor needs 2D+")
    field = O.random_field(rng, dims)
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("abs", 0.01))
    ds = H.h.partial_decompress(c, H.h.Stage.DECORRELATED)
    qf = H.h.partial_decompress(c, H.h.Stage.QUANTIZED)
    full = H.h.partial_decompress(c, H.h.Stage.FULL)
    assert np.array_equal(H.comp.recorrelate(ds).values, qf.values)
    assert np.array_equal(full, H.quant.dequantize(qf.values, c.eps))
    assert full.shape == dims
    assert np.abs(full - field).max() <= c.eps * (1 + 1e-12)
    oc = _oracle_of(c)
    assert np.array_equal(qf.values, O.stage3(oc))


@pytest.mark.parametrize("kind", ALL)
def test_slab_iteration(H, rng, kind):
    dims = (20, 9) if kind in ND else (150,)
    field = O.random_field(rng, dims)
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("abs", 0.01))
    for stage in (H.h.Stage.QUANTIZED, H.h.Stage.FULL):
        whole = H.h.partial_decompress(c, stage)
        whole = whole.values if stage == H.h.Stage.QUANTIZED else whole
        slabs = list(H.h.slab_iter(c, stage))
        joined = np.concatenate([np.atleast_1d(s) for s in slabs], axis=0)
        assert np.array_equal(joined.reshape(whole.shape), whole)
    joined = np.concatenate(list(H.h.slab_iter(c, H.h.Stage.DECORRELATED)))
    assert np.array_equal(joined, H.h.partial_decompress(c, H.h.Stage.DECORRELATED).values)


def test_sliding_window_and_bounds(H, rng):
    c = H.h.compress(O.random_field(rng, (20, 9)), H.h.CompressorKind.HSZX_ND, H.h.ErrorBound("abs", 0.01))
    assert H.stages.slab_bounds(c) == [(0, 8), (8, 16), (16, 20)]
    cp = H.h.compress(O.random_field(rng, (24, 8)), H.h.CompressorKind.HSZP_ND, H.h.ErrorBound("abs", 0.01))
    H.stages.slab_tracker.reset()
    seen = sum(1 for _ in H.stages.sliding_window(cp, H.h.Stage.QUANTIZED))
    assert seen == 24 and H.stages.slab_tracker.high_water <= 3


def test_metadata_stage_rules(H, rng):
    c = H.h.compress(O.random_field(rng, (12, 10)), H.h.CompressorKind.HSZP_ND, H.h.ErrorBound("abs", 0.01))
    with pytest.raises(H.h.UnsupportedStageError):
        H.h.partial_decompress(c, H.h.Stage.META)
    cx = H.h.compress(O.random_field(rng, (12, 10)), H.h.CompressorKind.HSZX_ND, H.h.ErrorBound("abs", 0.01))
    meta = H.h.partial_decompress(cx, H.h.Stage.META)
    assert meta.dtype == np.int32 and len(meta) == cx.geometry.block_count


def test_corrupt_payload_detected(H, rng):
    c = H.h.compress(O.random_field(rng, (12, 9)), H.h.CompressorKind.HSZX_ND, H.h.ErrorBound("abs", 0.01))
    buf = H.io.stream_to_bytes(c)
    clipped = H.io.stream_from_bytes(buf[:-3])
    with pytest.raises(H.h.CorruptStreamError):
        H.h.partial_decompress(clipped, H.h.Stage.FULL)
    for bad in (b"XSZ1" + buf[4:], buf[:20]):
        with pytest.raises(H.h.CorruptStreamError):
            H.io.stream_from_bytes(bad)


def test_decode_work_ordering(H, rng):
    from paper_2603_25206_b200.counters import decode_counters

    c = H.h.compress(O.random_field(rng, (64, 64)), H.h.CompressorKind.HSZX_ND, H.h.ErrorBound("abs", 0.01))
    work, chunks = {}, {}
    for stage in H.h.Stage:
        decode_counters.reset()
        H.h.partial_decompress(c, stage)
        work[stage] = decode_counters.total_work
        chunks[stage] = decode_counters.chunks_decoded
    assert chunks[H.h.Stage.META] == 0
    assert work[H.h.Stage.META] < work[H.h.Stage.DECORRELATED] <= work[H.h.Stage.QUANTIZED] <= work[H.h.Stage.FULL]


# ---- stats (test_stats.py) ---------------------------------------------------------------


def test_exact_helpers(H, example_field):
    v = np.full(64, 2**30, dtype=np.int64)
    assert H.stats._exact_sum(v) == 64 * 2**30
    assert H.stats._exact_dot(v, v) == 64 * 2**60
    assert H.stats._exact_sum(np.zeros(0, dtype=np.int64)) == 0
    with pytest.raises(ValueError):
        H.stats._std_from_sums(3, 9, 1, 0.1)
    c = H.h.compress(example_field, H.h.CompressorKind.HSZX_ND, H.h.ErrorBound("abs", 0.1), (2, 2))
    ds = H.h.partial_decompress(c, H.h.Stage.DECORRELATED)
    assert H.stats.std_from_dp(ds) == pytest.approx(2.0, abs=1e-12)
    c = H.h.compress(example_field, H.h.CompressorKind.HSZP, H.h.ErrorBound("abs", 0.1))
    qf = H.h.partial_decompress(c, H.h.Stage.QUANTIZED)
    assert H.stats.std_from_dq(qf) == pytest.approx(np.sqrt((740 * 8 - 18 * 18) / 56) * 0.2, rel=1e-15)
    rng = np.random.default_rng(4)
    p = rng.integers(-(2**30), 2**30, size=(5, 4)).astype(np.int64)
    q = np.cumsum(np.cumsum(p, axis=0), axis=1)
    p32 = p.astype(np.int32)   # residual domain of the test is int32
    assert H.stats._lorenzo_weighted_sum(p32.ravel(), (5, 4)) == O.lorenzo_weighted_sum(p32.ravel(), (5, 4))
    small = rng.integers(-50, 50, size=(3, 4, 5)).astype(np.int64)
    q3 = small
    for ax in range(3):
        q3 = np.cumsum(q3, axis=ax)
    assert H.stats._lorenzo_weighted_sum(small.ravel(), (3, 4, 5)) == int(q3.sum())
    del q


@pytest.mark.parametrize("kind", ALL)
@pytest.mark.parametrize("dims", [(97,), (17, 13), (7, 6, 11), (64, 40, 30), (4, 9, 128), (3, 21, 160), (16, 24, 64), (4096,)])
def test_stats_vs_oracle(H, rng, kind, dims):
    if kind in ND and len(dims) < 2:
        pytest.skip("nd compressor needs 2D+")
    field = O.random_field(rng, dims)
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("abs", 0.01))
    oc = _oracle_of(c)
    stages = [2, 3, 4] + ([1] if kind in (2, 3) else [])
    for st in stages:
        for op in ("mean", "std", "var"):
            if st == 1 and op != "mean":
                continue
            got = H.stats.compute_stat(c, op, H.h.Stage(st)).value
            want = O.compute_stat(oc, op, st)
            if st == 4:
                assert got == pytest.approx(want, rel=1e-12), (st, op)
            else:
                assert got == want, (st, op, got, want)


@pytest.mark.parametrize("kind", [2, 3])
@pytest.mark.parametrize("dims", [(16, 24, 64), (8192,)])
def test_stats_wide_residuals(H, rng, kind, dims):
    """Residuals of 28-31 bits (the block-mean reduction's 128-bit path) and small ones in one
    stream: var / mean at stages 2 and 3 vs the oracle."""
    if kind == 3 and len(dims) < 2:
        pytest.skip("nd compressor needs 2D+")
    field = (rng.standard_normal(dims) * 1e9).astype(np.float32)
    field.reshape(-1)[: field.size // 2] *= 1e-6            # half the chunks narrow, half wide
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("abs", 1.0))
    oc = _oracle_of(c)
    assert max(oc.payload[int(o)] for o in oc.offsets) >= 28
    for st in (2, 3):
        for op in ("mean", "var"):
            assert H.stats.compute_stat(c, op, H.h.Stage(st)).value == O.compute_stat(oc, op, st), (st, op)


def test_std_at_meta_rejected(H, rng):
    c = H.h.compress(O.random_field(rng, (16, 16)), H.h.CompressorKind.HSZX_ND, H.h.ErrorBound("abs", 0.1))
    with pytest.raises(H.h.UnsupportedStageError):
        H.stats.compute_stat(c, "std", H.h.Stage.META)


# ---- fields (test_fields.py) -----------------------------------------------------------------


@pytest.mark.parametrize("dims", [(15, 11), (6, 7, 8), (30, 41, 19), (6, 9, 64)])
@pytest.mark.parametrize("kind", ALL)
def test_stencils_vs_oracle(H, rng, kind, dims):
    field = O.random_field(rng, dims)
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("abs", 0.01))
    oc = _oracle_of(c)
    stages = [3, 4] + ([2] if kind in ND else [])
    for st in stages:
        for op in ("derivative", "laplacian"):
            got = H.fields.compute_field_op(c, op, H.h.Stage(st)).components
            want = O.field_op(oc, op, st)
            for a, b in zip(got, want):
                assert np.array_equal(a, b), (st, op)
    f32 = H.fields.compute_field_op(c, "derivative", H.h.Stage.QUANTIZED, out_dtype=np.float32).components
    for a, b in zip(f32, O.field_op(oc, "derivative", 3)):
        assert a.dtype == np.float32 and np.array_equal(a, b.astype(np.float32))


def test_stencil_rules(H, rng):
    c = H.h.compress(O.random_field(rng, (10, 10)), H.h.CompressorKind.HSZX, H.h.ErrorBound("abs", 0.01))
    with pytest.raises(H.h.UnsupportedStageError):
        H.fields.compute_field_op(c, "derivative", H.h.Stage.DECORRELATED)
    with pytest.raises(H.h.UnsupportedStageError):
        H.fields.compute_field_op(c, "derivative", H.h.Stage.META)
    c1 = H.h.compress(O.random_field(rng, (50,)), H.h.CompressorKind.HSZP, H.h.ErrorBound("abs", 0.01))
    with pytest.raises(ValueError):
        H.fields.compute_field_op(c1, "laplacian", H.h.Stage.QUANTIZED)
    a = H.h.compress(O.random_field(rng, (8, 8)), H.h.CompressorKind.HSZP_ND, H.h.ErrorBound("abs", 0.01))
    b = H.h.compress(O.random_field(rng, (8, 9)), H.h.CompressorKind.HSZP_ND, H.h.ErrorBound("abs", 0.01))
    with pytest.raises(ValueError):
        H.fields.divergence((a, b), H.h.Stage.QUANTIZED)
    with pytest.raises(ValueError):
        H.fields.curl((a,), H.h.Stage.QUANTIZED)
    m = H.h.compress(O.random_field(rng, (8, 8)), H.h.CompressorKind.HSZX_ND, H.h.ErrorBound("abs", 0.01))
    with pytest.raises(ValueError):
        H.fields.divergence((a, m), H.h.Stage.QUANTIZED)
    d = H.fields.compute_field_op(a, "derivative", H.h.Stage.DECORRELATED).components
    assert np.all(d[0][0] == 0) and np.all(d[0][-1] == 0) and np.all(d[1][:, 0] == 0)


def test_curl_rigid_rotation(H):
    n = 16
    i = np.arange(n, dtype=np.float32)
    u = np.tile(-i, (n, 1))
    v = np.tile(i[:, None], (1, n))
    cu = H.h.compress(u, H.h.CompressorKind.HSZP_ND, H.h.ErrorBound("abs", 0.01))
    cv = H.h.compress(v, H.h.CompressorKind.HSZP_ND, H.h.ErrorBound("abs", 0.01))
    curl = H.fields.curl((cu, cv), H.h.Stage.QUANTIZED).components[0]
    np.testing.assert_allclose(curl[1:-1, 1:-1], -2.0, atol=0.05)


# ---- N2-N5 (regions) ----------------------------------------------------------------------


# row-streaming kernel (R2 in 4..128, a power of two, n2 % 4 == 0): 40x50x60/16, 33x17x20/8, 9x13x516,
# 6x40x64, 70x92; the others take the one-CTA-per-region kernel
@pytest.mark.parametrize("dims,region", [((40, 50, 60), 16), ((33, 17, 20), 8), ((70, 90), (16, 16)),
                                         ((50, 21, 9), (5, 7, 3)), ((9, 13, 516), (3, 5, 128)),
                                         ((6, 40, 64), (4, 3, 4)), ((70, 92), (16, 32))])
@pytest.mark.parametrize("kind", [1, 3])
def test_regions_vs_oracle(H, rng, kind, dims, region):
    field = O.random_field(rng, dims, "smooth")
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("rel", 1e-3))
    oc = _oracle_of(c)
    q = O.stage3(oc)
    rs = H.regions.region_stats(c, region, tau=float(np.median(field)))
    s1, s2, qmin, qmax, size = O.region_reduce(q, region)
    assert np.array_equal(rs.s1, s1.astype(np.int64)) and np.array_equal(rs.size, size)
    assert all(int(a) == int(b) for a, b in zip(rs.s2.ravel(), s2.ravel()))
    assert np.array_equal(rs.qmin, qmin) and np.array_equal(rs.qmax, qmax)
    mean, var = O.region_stats(q, c.eps, region)
    np.testing.assert_allclose(rs.mean, mean, rtol=1e-15, atol=0)
    np.testing.assert_allclose(rs.var, var, rtol=1e-12, atol=0)
    _, _, fmin, fmax = O.region_minmax(q, c.eps, region)
    assert np.array_equal(rs.vmin, fmin) and np.array_equal(rs.vmax, fmax)
    assert rs.crossing_count == O.threshold_count(q, c.eps, region, float(np.median(field)))
    g = H.regions.gradient_magnitude(c)
    np.testing.assert_array_equal(g, O.gradient_magnitude(q, c.eps))


@pytest.mark.parametrize("case", ["smooth", "noise"])
@pytest.mark.parametrize("dims", [(12, 20, 64), (40, 16, 32)])
def test_hszp_nd_narrow_prefix_and_fallback(H, rng, case, dims):
    """3-D HSZP_ND stage 3 / 4 and variance run the band scan with int16 band-local prefixes (P2 = q[z] - q[z-1])
    and fall back to int32 when one does not fit (the noisy field at a tight bound: |P2| >> 2^15); both equal the
    oracle bit for bit."""
    field = O.random_field(rng, dims, case) * (np.float32(1.0) if case == "smooth" else np.float32(1e4))
    bound = H.h.ErrorBound("rel", 1e-3 if case == "smooth" else 1e-7)
    c = H.h.compress(field, H.h.CompressorKind.HSZP_ND, bound)
    oc = _oracle_of(c)
    q = O.stage3(oc)
    if case == "noise":
        assert np.abs(np.diff(q.astype(np.int64), axis=0)).max() > 2**15       # the int32 fallback runs
    got = H.h.partial_decompress(c, H.h.Stage.QUANTIZED).values
    assert np.array_equal(got, q)
    f4 = H.h.partial_decompress(c, H.h.Stage.FULL)
    assert np.array_equal(getattr(f4, "values", f4), O.stage4(oc, q))
    assert H.stats.compute_stat(c, "var", H.h.Stage.QUANTIZED).value == O.compute_stat(oc, "var", 3)


@pytest.mark.parametrize("case", ["nd8", "nd4", "nd2x4x8", "x1d"])
def test_regions_equal_blocks_vs_oracle(H, rng, monkeypatch, case):
    """Regions that are exactly the stream's blocks (HSZX_ND 8^3: 16 chunks per block; 4^3: 2; 2x4x8: 2; HSZX 1-D
    blocks of 128: 4) take the one-writer k_region_blocks path (no accumulator); results equal the oracle's,
    including a wide-residual field (int128 S2 per block) and the min / max."""
    from paper_2603_25206_b200 import _lib

    dims, kind, bd, region = {"nd8": ((16, 24, 40), 3, (8, 8, 8), 8), "nd4": ((8, 12, 16), 3, (4, 4, 4), 4),
                              "nd2x4x8": ((6, 8, 32), 3, (2, 4, 8), (2, 4, 8)),
                              "x1d": ((64 * 128,), 2, (128,), 128)}[case]
    field = O.random_field(rng, dims, "mixed") * np.float32(50.0)
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("rel", 1e-6), block_dims=bd)
    oc = _oracle_of(c)
    q = O.stage3(oc)
    rs = H.regions.region_stats(c, region, tau=float(np.median(field)))
    s1, s2, qmin, qmax, size = O.region_reduce(q, region)
    assert np.array_equal(rs.s1, s1.astype(np.int64)) and np.array_equal(rs.size, size)
    assert all(int(a) == int(b) for a, b in zip(rs.s2.ravel(), s2.ravel()))
    assert np.array_equal(rs.qmin, qmin) and np.array_equal(rs.qmax, qmax)
    assert rs.crossing_count == O.threshold_count(q, c.eps, region, float(np.median(field)))


@pytest.mark.parametrize("dims,region", [((6, 10, 256), (3, 4, 128)), ((5, 9, 20), 8), ((7, 9, 11), 4)])
def test_region_reduce_extreme_values(H, rng, dims, region):
    """|q| near 2^31: per-region S2 beyond 2^64 (int128 path) in both K-REG kernels."""
    import torch

    q = rng.integers(-2**31, 2**31, size=dims, dtype=np.int64)
    q[0, 0, :4] = -2**31
    q = q.astype(np.int32)
    r = H.regions.region_reduce_device(torch.from_numpy(q).cuda(), 1e-3, region)
    s1, s2, qmin, qmax, size = O.region_reduce(q, region)
    g = r["grid"]
    assert np.array_equal(r["s1"].cpu().numpy().reshape(g), s1.astype(np.int64))
    lo = r["s2lo"].cpu().numpy().view(np.uint64).ravel()
    hi = r["s2hi"].cpu().numpy().ravel()
    assert [(int(h) << 64) | int(l) for h, l in zip(hi, lo)] == [int(v) for v in s2.ravel()]
    assert np.array_equal(r["qmin"].cpu().numpy().reshape(g), qmin)
    assert np.array_equal(r["qmax"].cpu().numpy().reshape(g), qmax)
    assert np.array_equal(r["size"].cpu().numpy().reshape(g), size)


# ---- a configuration-1-sized field (1800x3600, BASELINE configs[0]) ---------------------------


@pytest.mark.parametrize("kind", ALL)
def test_config1_parity(H, kind):
    from paper_2603_25206_b200 import synthetic

    field = synthetic.config1_field()
    eps = 1e-4 * (float(field.max()) - float(field.min()))
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("abs", eps))
    ref = O.compress(field, kind, "abs", eps)
    assert H.io.stream_to_bytes(c) == O.stream_to_bytes(ref)
    p = H.h.partial_decompress(c, H.h.Stage.DECORRELATED).values
    assert np.array_equal(p, O.stage2(ref))
    q = H.h.partial_decompress(c, H.h.Stage.QUANTIZED).values
    assert np.array_equal(q, O.stage3(ref))
    for op in ("mean", "var"):
        for st in (2, 3):
            assert H.stats.compute_stat(c, op, H.h.Stage(st)).value == O.compute_stat(ref, op, st)
    d = H.fields.compute_field_op(c, "derivative", H.h.Stage.QUANTIZED).components
    for a, b in zip(d, O.derivative_q(q, ref.eps)):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ALL)
def test_stats_wide_bitwidths(H, kind):
    """Bit widths ~13 put the tile kernels' shared memory just above the 48 KB default minus their
    static shared memory (a launch failure once): config-4-like log-normal field, 64^3."""
    from paper_2603_25206_b200 import synthetic

    f = synthetic.config4_field(dims=(64, 64, 64))
    c = H.h.compress(f, H.h.CompressorKind(kind), H.h.ErrorBound("rel", 1e-4))
    oc = _oracle_of(c)
    d = c.device().validate()
    assert d.desc.max_bitwidth >= 12
    for st in (H.h.Stage.DECORRELATED, H.h.Stage.QUANTIZED):
        got = H.stats.compute_stat(c, "var", st).value
        want = O.var_from_dq(O.stage3(oc), c.eps) if st == H.h.Stage.QUANTIZED or not c.kind.is_block_mean else None
        if want is not None:
            assert got == want, (kind, st)


# fused K-REG from the bytes (hszg_region_stream): HSZX* regions aligned with the blocks, every chunk full
@pytest.mark.parametrize("dims,region,bd", [((48, 40, 64), 8, (8, 8, 8)), ((48, 40, 64), (16, 8, 32), (8, 8, 8)),
                                            ((40, 50, 60), 16, (8, 8, 8)), ((64, 64), 16, (8, 8)),
                                            ((24, 32, 96), (8, 16, 48), (4, 8, 8)), ((4096,), 256, (32,)),
                                            ((48, 40, 64), 1000, (8, 8, 8))])
@pytest.mark.parametrize("scale", ["smooth", "wide"])
def test_regions_fused_from_bytes(H, rng, dims, region, bd, scale):
    kind = 2 if len(dims) == 1 else 3
    field = O.random_field(rng, dims, "smooth")
    eps = 1e-3 * float(field.max() - field.min()) if scale == "smooth" else 1e-8 * float(np.abs(field).max())
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("abs", eps), bd if kind == 3 else bd[0])
    oc = _oracle_of(c)
    q = O.stage3(oc)
    for stage in (H.h.Stage.DECORRELATED, H.h.Stage.QUANTIZED):
        rs = H.regions.region_stats(c, region, stage, tau=float(np.median(field)))
        s1, s2, qmin, qmax, size = O.region_reduce(q, region)
        assert np.array_equal(rs.s1, s1.astype(np.int64)) and np.array_equal(rs.size, size)
        assert all(int(a) == int(b) for a, b in zip(rs.s2.ravel(), s2.ravel()))
        assert np.array_equal(rs.qmin, qmin) and np.array_equal(rs.qmax, qmax)
        mean, var = O.region_stats(q, c.eps, region)
        np.testing.assert_allclose(rs.mean, mean, rtol=1e-15, atol=0)
        np.testing.assert_allclose(rs.var, var, rtol=1e-12, atol=0)
        assert rs.crossing_count == O.threshold_count(q, c.eps, region, float(np.median(field)))
        assert H.regions.threshold_count(c, region, 0.0, stage) == O.threshold_count(q, c.eps, region, 0.0)


@pytest.mark.parametrize("kind", ALL)
@pytest.mark.parametrize("scale", ["smooth", "wide", "zero"])
def test_stats_lean_decode_vs_oracle(H, rng, kind, scale):
    """K-STAT lean moments (moments.cuh): bit widths 0 (constant), <= 8, 9..16 and > 16 (exact 128-bit
    path) in one stream; mean / var / std at stages 2 and 3 bit-identical to the oracle."""
    dims = (24, 32, 64)
    f = _wide_bitwidth_field(rng, dims) if scale == "wide" else O.random_field(rng, dims, "smooth")
    if scale == "zero":
        f = np.full(dims, 0.25, dtype=np.float32)
        f[3, 4, 5] = 1.0
    eps = 1e-3 if scale != "smooth" else 1e-4 * float(f.max() - f.min())
    c = H.h.compress(f, H.h.CompressorKind(kind), H.h.ErrorBound("abs", eps))
    oc = _oracle_of(c)
    for st in (2, 3):
        for op in ("mean", "var", "std"):
            assert H.stats.compute_stat(c, op, H.h.Stage(st)).value == O.compute_stat(oc, op, st), (kind, st, op)


def _wide_bitwidth_field(rng, dims):
    """Noise whose amplitude changes every 8 x-values (bit widths 0 .. ~22), plus a constant region."""
    n2 = dims[2]
    scale = 10.0 ** rng.uniform(-4, 3, size=n2 // 8).repeat(8)
    f = rng.normal(size=dims) * scale[None, None, :]
    f[:, :, :16] = 0.5
    return f.astype(np.float32)


# ---- HSZP_ND int16 band-local prefixes with the exact redo of overflowing planes (recon.cu) -------


def _hszpnd_overflow_field(rng, dims, case):
    f = O.random_field(rng, dims, "smooth").astype(np.float64)
    if case == "first_plane":        # q ~ 5e5 everywhere: plane 0's prefix (= q itself) overflows int16
        return (f + 100.0).astype(np.float32), 1e-4
    if case == "all_planes":         # z differences of q ~ 1e5: every plane overflows
        return O.random_field(rng, dims, "noise"), 1e-5
    return f.astype(np.float32), 1e-2  # fits int16 everywhere


@pytest.mark.parametrize("case", ["fits", "first_plane", "all_planes"])
@pytest.mark.parametrize("dims", [(300, 16, 64), (40, 33, 96)], ids=["one-band", "bands"])
def test_hszpnd_l16_redo(H, rng, dims, case):
    """Stage 3 / 4 and the stage-3 variance of HSZP_ND through the int16 band scan: planes whose
    band-local prefixes do not fit int16 are redone at int32 — results identical to the oracle."""
    import torch

    field, eps = _hszpnd_overflow_field(rng, dims, case)
    c = H.h.compress(field, H.h.CompressorKind.HSZP_ND, H.h.ErrorBound("abs", eps))
    ref = _oracle_of(c)
    q = O.stage3(ref)
    if case == "all_planes":
        assert np.abs(np.diff(q.astype(np.int64), axis=0)).max() > 2**15
    if case == "first_plane":
        assert np.abs(q[0].astype(np.int64)).max() > 2**15
    assert np.array_equal(H.h.partial_decompress(c, H.h.Stage.QUANTIZED).values, q)
    full = H.h.partial_decompress(c, H.h.Stage.FULL)
    assert np.array_equal(full, O.dequantize(q, c.eps))
    f32 = H.h.partial_decompress(c, H.h.Stage.FULL, dtype=torch.float32)
    assert np.array_equal(np.asarray(f32), O.dequantize(q, c.eps).astype(np.float32))
    for op in ("mean", "var"):
        assert H.stats.compute_stat(c, op, H.h.Stage.QUANTIZED).value == O.compute_stat(ref, op, 3), op
