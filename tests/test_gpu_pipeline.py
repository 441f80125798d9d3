"""GPU tests of the windowed / z-slab-sharded pipeline (pipeline.py) against the oracle.

* a rank's shard container is byte-identical to the global stream's chunk range (SURVEY §8(c) slab technique);
* the windowed gradient + Laplacian equals the whole-field reference stencils: bit for bit in the exact
  mode (fp32 outputs = the reference float64 values rounded to float32), within FAST_RTOL relative in the
  default fast-fp32 mode; the exact global mean/variance is bit-identical in both;
* a multi-rank run, emulated rank by rank in one process (halo planes, HSZP_ND Lorenzo carry from the
  slab totals), reproduces the same outputs.

Shapes: (64, 40, 36) has rows that are not whole chunks (general window loop for HSZP_ND);
(48, 23, 64) and (40, 17, 128) take the band-scan / z-sweep kernels; (48, 24, 64) and (48, 40, 136)
(8^3 blocks dividing the box: partial x and y strips) also take the one-pass HSZX_ND kernel.
"""

import numpy as np
import pytest

from oracle import hsz_oracle as O

pytestmark = pytest.mark.gpu

ALL_DIMS = [(64, 40, 36), (48, 23, 64), (40, 17, 128), (48, 24, 64), (48, 40, 136), (48, 30, 96)]

# fast mode: fl32(fl32(D) * fl32(eps)) vs fl32(D * eps): at most 4 roundings of 2^-24 apart (< 1e-6 target)
FAST_RTOL = 4 * 2.0**-24


def _check_fp32(got, want, exact, msg):
    if exact:
        assert np.array_equal(got, want), msg
    else:
        err = np.abs(got.astype(np.float64) - want.astype(np.float64))
        assert np.all(err <= FAST_RTOL * np.abs(want.astype(np.float64))), (msg, float(err.max()))


@pytest.fixture(scope="module", params=ALL_DIMS, ids=lambda d: "x".join(map(str, d)))
def setup(request):
    import torch

    from paper_2603_25206_b200 import pipeline
    from paper_2603_25206_b200.compressors import compress_device

    dims = request.param
    rng = np.random.default_rng(77)
    field = O.random_field(rng, dims, "smooth")
    eps = 1e-3 * float(field.max() - field.min())
    return torch, pipeline, compress_device, field, eps, dims


def _host_stream(ds, eps):
    meta = None if ds.metadata is None else ds.metadata.cpu().numpy()
    return O.Stream(ds.kind, ds.dims, ds.block_dims, eps, meta, ds.offsets.cpu().numpy().view(np.uint64),
                    ds.payload[:ds.payload_len].cpu().numpy().tobytes())


@pytest.mark.parametrize("kind", [1, 3])
@pytest.mark.parametrize("world", [2, 3])
def test_shard_containers_are_global_chunk_ranges(setup, kind, world):
    torch, pipeline, compress_device, field, eps, dims = setup
    fd = torch.from_numpy(field).cuda()
    g = compress_device(fd, kind, eps, (8, 8, 8))
    gh = _host_stream(g, eps)
    ref = O.compress(field, kind, "abs", eps, (8, 8, 8))
    assert gh.payload == ref.payload
    for r in range(world):
        z0, z1 = pipeline.shard_planes(dims[0], world, r, 16)
        lead = 1 if (kind == 1 and z0 > 0) else 0
        sf = pipeline.compress_shard(fd[z0 - lead:z1].contiguous(), kind, eps, (8, 8, 8), z0, z1, dims)
        view = g.plane_view(z0, z1)
        vo = view.offsets.cpu().numpy().view(np.uint64)
        lo = int(vo[0])
        so = sf.ds.offsets.cpu().numpy().view(np.uint64)
        assert np.array_equal(so, vo - np.uint64(lo))
        first = int(np.searchsorted(np.asarray(gh.offsets, dtype=np.uint64), np.uint64(lo)))
        last = first + view.n_chunks
        hi = int(gh.offsets[last]) if last < len(gh.offsets) else len(gh.payload)
        assert sf.ds.payload[:sf.ds.payload_len].cpu().numpy().tobytes() == gh.payload[lo:hi]
        if kind == 3:
            assert np.array_equal(sf.ds.metadata.cpu().numpy(), view.metadata.cpu().numpy())


def _oracle_outputs(field, kind, eps):
    c = O.compress(field, kind, "abs", eps, (8, 8, 8))
    q = O.stage3(c)
    outs = O.derivative_q(q, eps) + O.laplacian_q(q, eps)
    v = q.ravel()
    s1, s2 = O.exact_sum(v), O.exact_dot(v, v)
    return [o.astype(np.float32) for o in outs], s1, s2, O.mean_from_dq(q, eps), O.var_from_dq(q, eps)


@pytest.mark.parametrize("kind", [1, 3])
@pytest.mark.parametrize("window", [8, 16, 64])
@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
@pytest.mark.parametrize("one_pass", [True, False], ids=["onepass", "windows"])
def test_window_pipeline_single_rank(setup, kind, window, exact, one_pass):
    torch, pipeline, compress_device, field, eps, dims = setup
    fd = torch.from_numpy(field).cuda()
    sf = pipeline.compress_shard(fd, kind, eps, (8, 8, 8), 0, dims[0], dims)
    pipe = pipeline.WindowPipeline(sf, pipeline.Comm(), window)
    pipe.exact_fp32 = exact
    pipe.one_pass = one_pass
    pipe.lorenzo_one_pass = one_pass
    if kind == 1 and window == 16:
        pipe.band_rows_req = 5          # several bands, partial tiles and a short last band (column z-sweep)
    if kind == 1 and window == 8:
        pipe.band_rows_req = 16         # ring z-sweep with several bands
        pipe.overlap = True             # band scans on the side stream
    if kind == 3 and window == 16:
        pipe.fused_layers = 2           # several z segments of the one-pass kernel
    outs = [torch.empty(dims, dtype=torch.float32, device="cuda") for _ in range(4)]
    res = pipe.run(outs)
    want, s1, s2, mean, var = _oracle_outputs(field, kind, eps)
    if one_pass and kind == 1 and dims[2] % 64 == 0:
        assert hasattr(pipe, "lz_bands")        # took lorenzo.cu, not a silent fallback
    for k, (got, w) in enumerate(zip(outs, want)):
        _check_fp32(got.cpu().numpy(), w, exact, (kind, window, k))
    assert res["s1"] == s1 and res["s2"] == s2
    assert res["mean"] == mean and res["var"] == var
    res2 = pipe.run(outs)                 # the pipeline is re-runnable (bench steps)
    assert res2["mean"] == mean and res2["var"] == var


@pytest.mark.parametrize("kind", [1, 3])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("one_pass", [True, False], ids=["onepass", "windows"])
def test_window_pipeline_emulated_ranks(setup, kind, world, one_pass):
    torch, pipeline, compress_device, field, eps, dims = setup
    fd = torch.from_numpy(field).cuda()
    ranks = []
    for r in range(world):
        z0, z1 = pipeline.shard_planes(dims[0], world, r, 16)
        lead = 1 if (kind == 1 and z0 > 0) else 0
        sf = pipeline.compress_shard(fd[z0 - lead:z1].contiguous(), kind, eps, (8, 8, 8), z0, z1, dims)
        ranks.append(pipeline.WindowPipeline(sf, pipeline.Comm(), 8))
        ranks[-1].exact_fp32 = True
        ranks[-1].one_pass = one_pass
        ranks[-1].lorenzo_one_pass = one_pass
        ranks[-1].band_rows_req = (3 + r) if world == 2 else 16 * (r + 1)
    mine = [p.local_boundary(need_total=True) for p in ranks]
    Ts = [m["T"] for m in mine] if kind == 1 else None
    carries = [p.carry_from(Ts, r) for r, p in enumerate(ranks)]
    firsts = [p.finish_first(m, c) for p, m, c in zip(ranks, mine, carries)]
    to_lower = [f if f is not None else m["head"] for f, m in zip(firsts, mine)]
    to_upper = [m["tail"] for m in mine]
    want, s1, s2, mean, var = _oracle_outputs(field, kind, eps)
    tot1 = tot2 = 0
    for r, p in enumerate(ranks):
        lo = to_upper[r - 1] if r > 0 else None
        hi = to_lower[r + 1] if r < world - 1 else None
        p.apply_boundary(carries[r], lo, hi)
        nz = p.sf.nz
        outs = [torch.empty((nz,) + dims[1:], dtype=torch.float32, device="cuda") for _ in range(4)]
        part = p.run_prepared(outs)
        tot1 += part["s1"]
        tot2 += part["s2"]
        for got, w in zip(outs, want):
            assert np.array_equal(got.cpu().numpy(), w[p.sf.z0:p.sf.z1]), (kind, world, r)
    assert tot1 == s1 and tot2 == s2
    n = int(np.prod(dims))
    assert pipeline.finalize_mean_var(tot1, tot2, n, eps) == (mean, var)


def _wide_bitwidth_field(rng, dims):
    """Noise whose amplitude changes every 8 x-values (bit widths 0 .. ~22), plus a constant region."""
    n2 = dims[2]
    scale = 10.0 ** rng.uniform(-4, 3, size=n2 // 8).repeat(8)
    f = rng.normal(size=dims) * scale[None, None, :]
    f[:, :, :16] = 0.5                          # all-zero residual chunks (bw 0)
    return f.astype(np.float32)


@pytest.mark.parametrize("dims", [(16, 16, 256), (24, 8, 64)], ids=lambda d: "x".join(map(str, d)))
def test_fast_decode_bitwidths_hszx_nd(dims):
    """k_tile_blocks_fast (full 8^3 blocks) across bit widths 0..~22 vs the oracle's stage 3."""
    import paper_2603_25206_b200 as h

    rng = np.random.default_rng(123)
    f = _wide_bitwidth_field(rng, dims)
    c = h.compress(f, h.CompressorKind(3), h.ErrorBound("abs", 1e-3), (8, 8, 8))
    ref = O.compress(f, 3, "abs", 1e-3, (8, 8, 8))
    bws = {ref.payload[int(o)] for o in ref.offsets}
    assert 0 in bws and max(bws) > 16 and any(8 < b <= 16 for b in bws)
    q = h.partial_decompress(c, h.Stage.QUANTIZED).values
    assert np.array_equal(np.asarray(q), O.stage3(ref))


# n2 = 96 / 160 / 384: 3 / 5 / 12 chunks per row, which do not divide a 256-chunk tile (partial tiles)
# (16, 64, 256) with band_rows 1: 512 (band, plane) items per window, several per persistent CTA
@pytest.mark.parametrize("dims", [(16, 16, 256), (24, 40, 64), (12, 30, 96), (5, 44, 160), (6, 50, 384),
                                  (16, 64, 256)],
                         ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("band_rows", [None, 1, 7, 16, 32])
@pytest.mark.parametrize("overlap", [False, True], ids=["one-stream", "side-stream"])
def test_fast_decode_bitwidths_band_scan(dims, band_rows, overlap):
    """hszg_band_scan (decode32 + row prefix + banded column prefix) across bit widths, through the
    HSZP_ND window pipeline (exact mode), vs the oracle.  side-stream: the scans run as the
    persistent grid (one CTA per SM striding over (band, plane) items) on the side stream."""
    import torch

    if overlap and band_rows is None:
        pytest.skip("the one-pass kernel has no band-scan windows")

    from paper_2603_25206_b200 import pipeline

    rng = np.random.default_rng(321)
    f = _wide_bitwidth_field(rng, dims)
    eps = 1e-3
    fd = torch.from_numpy(f).cuda()
    sf = pipeline.compress_shard(fd, 1, eps, (8, 8, 8), 0, dims[0], dims)
    pipe = pipeline.WindowPipeline(sf, pipeline.Comm(), 8)
    pipe.exact_fp32 = True
    pipe.band_rows_req = band_rows
    pipe.one_pass = pipe.lorenzo_one_pass = band_rows is None   # None: the one-pass kernel; else two passes
    pipe.overlap = overlap
    outs = [torch.empty(dims, dtype=torch.float32, device="cuda") for _ in range(4)]
    res = pipe.run(outs)
    want, s1, s2, mean, var = _oracle_outputs(f, 1, eps)
    for k, (got, w) in enumerate(zip(outs, want)):
        assert np.array_equal(got.cpu().numpy(), w), k
    assert res["s1"] == s1 and res["s2"] == s2


@pytest.mark.parametrize("kind", [1, 3])
def test_fast_mode_falls_back_on_large_q(kind):
    """|q| >= 2^27 breaks the fast emitter's int32 Laplacian: the pipeline must detect it from the exact
    min / max and redo the pass exactly (outputs then bit-identical to the oracle)."""
    import torch

    from paper_2603_25206_b200 import pipeline

    dims = (48, 24, 64)
    rng = np.random.default_rng(9)
    f = O.random_field(rng, dims, "smooth")
    eps = 2e-9 * float(np.abs(f).max())            # |q| up to ~2.5e8 > 2^27
    fd = torch.from_numpy(f).cuda()
    sf = pipeline.compress_shard(fd, kind, eps, (8, 8, 8), 0, dims[0], dims)
    pipe = pipeline.WindowPipeline(sf, pipeline.Comm(), 16)
    outs = [torch.empty(dims, dtype=torch.float32, device="cuda") for _ in range(4)]
    res = pipe.run(outs)
    want, s1, s2, mean, var = _oracle_outputs(f, kind, eps)
    assert max(-res["vmin"], res["vmax"]) >= pipeline.FAST_QLIM
    for k, (got, w) in enumerate(zip(outs, want)):
        assert np.array_equal(got.cpu().numpy(), w), k
    assert res["s1"] == s1 and res["s2"] == s2 and not pipe.exact_fp32
    if kind == 1:
        assert not pipe.l16            # the int16 band-local prefixes overflowed: redone with int32


@pytest.mark.parametrize("case", ["smooth", "noise"])
@pytest.mark.parametrize("overlap", [False, True], ids=["one-stream", "side-stream"])
def test_narrow_band_prefix_widths(case, overlap):
    """HSZP_ND two-pass with int8 band-local prefixes (int16 in the window holding the field's first
    plane): a field whose z-differences are smooth keeps int8; white noise overflows int8 (flag bit 1),
    the pass is redone with int16 everywhere — bit-exact against the oracle either way."""
    import torch

    from paper_2603_25206_b200 import pipeline

    dims = (48, 32, 64)
    z, y, x = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in dims], indexing="ij")
    if case == "smooth":
        f = (np.sin(2 * np.pi * z / 48) + 0.5 * np.sin(2 * np.pi * x / 64) + 0.25 * np.cos(2 * np.pi * y / 32))
    else:
        f = np.random.default_rng(5).uniform(-1, 1, dims)
    f = f.astype(np.float32)
    eps = 1e-3 * float(f.max() - f.min())
    fd = torch.from_numpy(f).cuda()
    sf = pipeline.compress_shard(fd, 1, eps, (8, 8, 8), 0, dims[0], dims)
    pipe = pipeline.WindowPipeline(sf, pipeline.Comm(), 16)
    pipe.one_pass = pipe.lorenzo_one_pass = False
    pipe.band_rows_req = 16
    pipe.exact_fp32 = True
    pipe.overlap = overlap              # side-stream: the bench's persistent scan grid, overflow redone too
    outs = [torch.empty(dims, dtype=torch.float32, device="cuda") for _ in range(4)]
    res = pipe.run(outs)
    want, s1, s2, mean, var = _oracle_outputs(f, 1, eps)
    for k, (got, w) in enumerate(zip(outs, want)):
        assert np.array_equal(got.cpu().numpy(), w), (case, k)
    assert res["s1"] == s1 and res["s2"] == s2
    assert pipe.l16
    assert pipe.l8 == (case == "smooth")
    res2 = pipe.run(outs)                              # the chosen width is kept for later passes
    assert res2["s1"] == s1 and pipe.l8 == (case == "smooth")
