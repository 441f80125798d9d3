"""Out-of-core slab streaming: a container kept in host memory, decoded slab by slab
with H2D copies of fetch units (streaming.HostSlabSource), must give exactly the slabs of the
device-resident path (and of the oracle) without ever uploading the whole container."""

import numpy as np
import pytest

from oracle import hsz_oracle as O

pytestmark = pytest.mark.gpu


def _host_only(c):
    from paper_2603_25206_b200 import io

    h = io.stream_from_bytes(io.stream_to_bytes(c))
    assert h._device is None
    return h


CASES = [(0, (2000,)), (1, (12, 10, 64)), (1, (9, 40, 36)), (2, (3000,)), (3, (17, 12, 24)), (3, (16, 9, 40)),
         (1, (30, 50)), (3, (20, 24))]


@pytest.mark.parametrize("kind,dims", CASES, ids=lambda v: str(v))
@pytest.mark.parametrize("budget", [64, 4096, 1 << 30])
def test_streamed_slabs_match_resident(kind, dims, budget):
    import paper_2603_25206_b200 as h

    rng = np.random.default_rng(kind * 100 + len(dims))
    f = O.random_field(rng, dims, "smooth")
    c = h.compress(f, h.CompressorKind(kind), h.ErrorBound("rel", 1e-3))
    hc = _host_only(c)
    from paper_2603_25206_b200.counters import decode_counters

    for st in (h.Stage.DECORRELATED, h.Stage.QUANTIZED, h.Stage.FULL):
        decode_counters.reset()
        want = list(h.slab_iter(c, st))                 # resident: batched decode, per-slab views
        cw = (decode_counters.chunks_decoded, decode_counters.bytes_read, decode_counters.recorrelated_elements,
              decode_counters.dequantized_elements)
        decode_counters.reset()
        got = list(h.slab_iter(hc, st, from_host=True, budget=budget))
        cg = (decode_counters.chunks_decoded, decode_counters.bytes_read, decode_counters.recorrelated_elements,
              decode_counters.dequantized_elements)
        assert cw == cg, (st, cw, cg)                   # the reference's per-slab work counters
        assert len(got) == len(want)
        for a, b in zip(got, want):
            assert a.shape == b.shape and np.array_equal(a, b), (st, budget)
    assert hc._device is None                      # nothing uploaded whole


@pytest.mark.parametrize("kind,dims", [(1, (14, 20, 32)), (3, (24, 16, 40)), (1, (25, 33))])
def test_streamed_derivative_from_host(kind, dims):
    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200.analytics import fields

    rng = np.random.default_rng(7)
    f = O.random_field(rng, dims, "smooth")
    c = h.compress(f, h.CompressorKind(kind), h.ErrorBound("rel", 1e-3))
    hc = _host_only(c)
    got = fields.streamed_derivative(hc, from_host=True, out_dtype=np.float32).components
    want = fields.compute_field_op(c, "derivative", h.Stage.QUANTIZED, out_dtype=np.float32).components
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    assert hc._device is None
    from paper_2603_25206_b200 import io

    oc = O.stream_from_bytes(io.stream_to_bytes(c))
    for a, b in zip(fields.streamed_derivative(hc, from_host=True).components, O.derivative_q(O.stage3(oc), c.eps)):
        assert np.array_equal(a, b)


def test_streamed_corruption_is_detected_in_its_unit():
    """A chunk whose bit width byte is corrupted in a late slab raises CorruptStreamError when the
    streaming reaches its fetch unit (every unit is validated on the device)."""
    import paper_2603_25206_b200 as h

    rng = np.random.default_rng(3)
    f = O.random_field(rng, (16, 8, 64), "smooth")
    c = h.compress(f, h.CompressorKind.HSZP_ND, h.ErrorBound("rel", 1e-3))
    hc = _host_only(c)
    offs = np.asarray(hc.chunk_offsets, dtype=np.uint64)
    bad = bytearray(hc.payload)
    bad[int(offs[len(offs) - 3])] = 40                 # bit width 40 > 32
    hc._payload = bytes(bad)
    it = h.slab_iter(hc, h.Stage.QUANTIZED, from_host=True, budget=2048)
    seen = 0
    with pytest.raises(h.CorruptStreamError):
        for _ in it:
            seen += 1
    assert seen >= 1                                   # earlier units decoded before the bad one


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_pinned_file_io_roundtrip(tmp_path, kind):
    """read_compressed reads into pinned memory and keeps the payload a view of it; the device
    upload, the streamed slabs and write_compressed (from a device-resident stream) all agree
    byte for byte with the bytes path."""
    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import io

    rng = np.random.default_rng(kind)
    dims = (12, 16, 64) if kind in (1, 3) else (6000,)
    f = O.random_field(rng, dims, "smooth")
    c = h.compress(f, h.CompressorKind(kind), h.ErrorBound("rel", 1e-3))
    path = tmp_path / "c.hsz"
    io.write_compressed(c, path)                       # device-resident payload -> pinned -> file
    raw = path.read_bytes()
    assert raw == io.stream_to_bytes(c)
    pc = io.read_compressed(path)
    assert pc.pinned_payload() is not None and isinstance(pc.payload, memoryview)
    assert io.stream_to_bytes(pc) == raw
    q = h.partial_decompress(pc, h.Stage.QUANTIZED).values
    assert np.array_equal(q, h.partial_decompress(c, h.Stage.QUANTIZED).values)
    pc2 = io.read_compressed(path)
    for a, b in zip(h.slab_iter(pc2, h.Stage.QUANTIZED, from_host=True, budget=4096),
                    h.slab_iter(c, h.Stage.QUANTIZED)):
        assert np.array_equal(a, b)
    assert pc2._device is None
    bc = io.read_compressed(path, pinned=False)
    assert isinstance(bc.payload, bytes) and bc.pinned_payload() is None


@pytest.mark.parametrize("stage", [3, 4])
def test_slab_batches_fold_the_carry(monkeypatch, stage):
    """3-D HSZP_ND slab iteration in several launch groups: every group after the first reconstructs with the
    previous group's last plane folded into its z prefix (hszg_reconstruct_carry); the slabs equal the oracle's."""
    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import _lib, io as hio, stages

    rng = np.random.default_rng(31)
    dims = (21, 12, 64)
    f = O.random_field(rng, dims, "smooth")
    c = h.compress(f, h.CompressorKind.HSZP_ND, h.ErrorBound("rel", 1e-3))
    monkeypatch.setattr(stages, "SLAB_BATCH_BYTES", 4 * 12 * 64 * 3)       # three planes per launch group
    calls = []
    real = _lib.call

    def spy(name, *a, **k):
        calls.append(name)
        return real(name, *a, **k)

    monkeypatch.setattr(_lib, "call", spy)
    oc = O.stream_from_bytes(hio.stream_to_bytes(c))
    q = O.stage3(oc)
    want = q if stage == 3 else O.stage4(oc, q)
    got = np.concatenate([np.asarray(s) for s in h.slab_iter(c, h.Stage(stage))])
    assert calls.count("hszg_reconstruct_carry") >= 6
    if stage == 3:
        assert np.array_equal(got.reshape(dims), want)
    else:
        assert np.array_equal(got.reshape(dims), want.astype(got.dtype))
